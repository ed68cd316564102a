#!/usr/bin/env bash
# ncu --set full of the row-block kernel on the C4-shape proxy (source-level SASS for
# per-instruction stall attribution), plus the matrix-free parity tests of this build
set -u
mkdir -p gpurun_out
python -c "from paper_1612_09335_b200 import _build; _build.needs_build() and _build.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q -k "matrixfree" > gpurun_out/pytest_mf.log 2>&1
echo "pytest mf exit $?"; tail -3 gpurun_out/pytest_mf.log
for c in C2 C3 C5; do
  echo "mf $c: $(timeout 600 python tools/c4_iter.py --config $c --kernel matrixfree --reps 5 2>&1 | tail -1 | cut -c1-200)"
done
timeout 600 python tools/c4_iter.py --reps 3 > gpurun_out/proxy_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k "regex:k_rowblk" -s 3 -c 1 \
    -o gpurun_out/prof_C4proxy -f python tools/c4_iter.py --reps 3 > gpurun_out/ncu_proxy.log 2>&1
echo "ncu exit $?"; tail -2 gpurun_out/ncu_proxy.log

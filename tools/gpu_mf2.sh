#!/usr/bin/env bash
# matrix-free kernel: parity tests + timings on the BASELINE configs (tools only)
set -u
mkdir -p gpurun_out
python -c "from paper_1612_09335_b200 import _build; _build.needs_build() and _build.build()" > gpurun_out/build.log 2>&1 || { echo build failed; exit 1; }
timeout 900 python -m pytest tests -m gpu -x -q -k "matrixfree or ${TESTS:-matrixfree}" > gpurun_out/pytest_mf.log 2>&1
echo "pytest exit $?"; tail -15 gpurun_out/pytest_mf.log
for c in ${CFGS:-C2 C3 C5}; do
  echo "$c: $(timeout 900 python tools/c4_iter.py --config $c --kernel matrixfree --reps ${REPS:-10} 2>&1 | tail -1 | cut -c1-400)"
done

#!/usr/bin/env bash
# matrix-free v3 (tensor-core basis transform, shared-memory Cholesky, fast rsqrt) and
# the staged-block face-trace kernel: parity tests of the default build, smoke, then
# timings of the default and the variants (tools only)
set -u
mkdir -p gpurun_out
python -c "from paper_1612_09335_b200 import _build; _build.needs_build() and _build.build()" > gpurun_out/build.log 2>&1 || { echo build failed; exit 1; }
timeout 1500 python -m pytest tests -m gpu -x -q -k "matrixfree or face_traces" > gpurun_out/pytest_mf_tr.log 2>&1
echo "pytest exit $?"; tail -4 gpurun_out/pytest_mf_tr.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke_o.log 2>&1; echo "smoke exit $?"
echo "traces default: $(timeout 900 python tools/traces_bench.py C2 C3 C5 2>&1 | cut -c1-230)"
echo "traces v1: $(CWRECO_LIBRARY=$PWD/variants/lib_tr_v1.so timeout 900 python tools/traces_bench.py C2 C3 C5 2>&1 | cut -c1-230)"
for c in ${CFGS:-C5 C3 C2}; do
  echo "$c default: $(timeout 600 python tools/c4_iter.py --config $c --kernel matrixfree --reps 10 2>&1 | tail -1 | cut -c1-300)"
  for f in variants/lib_mf_*.so; do
    echo "$c $f: $(CWRECO_LIBRARY=$PWD/$f timeout 600 python tools/c4_iter.py --config $c --kernel matrixfree --reps 10 2>&1 | tail -1 | cut -c1-300)"
  done
done

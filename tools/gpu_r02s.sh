#!/usr/bin/env bash
# matrix-free: prefetch of the next cell's stencil vertices / averages (CWR_MF_PF = 1: L1,
# 2: L2) — parity of each variant, then timings against the default
set -u
mkdir -p gpurun_out
python -c "from paper_1612_09335_b200 import _build; _build.needs_build() and _build.build()" > gpurun_out/build.log 2>&1 || { echo build failed; exit 1; }
for f in variants/lib_mf_*.so; do
  CWRECO_LIBRARY=$PWD/$f timeout 900 python -m pytest tests -m gpu -x -q -k "matrixfree" > gpurun_out/pytest_$(basename $f .so).log 2>&1
  echo "pytest $f exit $?"; tail -1 gpurun_out/pytest_$(basename $f .so).log
done
for c in ${CFGS:-C5 C3 C2}; do
  echo "$c default: $(timeout 600 python tools/c4_iter.py --config $c --kernel matrixfree --reps 10 2>&1 | tail -1 | cut -c1-300)" | tee -a gpurun_out/mf_variants.log
  for f in variants/lib_mf_*.so; do
    echo "$c $f: $(CWRECO_LIBRARY=$PWD/$f timeout 600 python tools/c4_iter.py --config $c --kernel matrixfree --reps 10 2>&1 | tail -1 | cut -c1-300)" | tee -a gpurun_out/mf_variants.log
  done
done

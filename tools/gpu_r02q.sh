#!/usr/bin/env bash
# face-trace kernel k_traces2: conflict-free point ownership (SWZ) and two thread groups
# per CTA (NG): parity of the default build and of every variant, then timings
set -u
mkdir -p gpurun_out
python -c "from paper_1612_09335_b200 import _build; _build.needs_build() and _build.build()" > gpurun_out/build.log 2>&1 || { echo build failed; exit 1; }
timeout 900 python -m pytest tests -m gpu -x -q -k "face_traces" > gpurun_out/pytest_tr.log 2>&1
echo "pytest default exit $?"; tail -3 gpurun_out/pytest_tr.log
for f in variants/lib_tr_*.so; do
  CWRECO_LIBRARY=$PWD/$f timeout 900 python -m pytest tests -m gpu -x -q -k "face_traces" > gpurun_out/pytest_tr_$(basename $f .so).log 2>&1
  echo "pytest $f exit $?"; tail -1 gpurun_out/pytest_tr_$(basename $f .so).log
done
CF=${CFGS:-C5 C3 C2}
echo "traces default: $(timeout 900 python tools/traces_bench.py $CF 2>&1 | cut -c1-230)" | tee gpurun_out/traces_variants.log
for f in variants/lib_tr_*.so; do
  echo "traces $f: $(CWRECO_LIBRARY=$PWD/$f timeout 900 python tools/traces_bench.py $CF 2>&1 | cut -c1-230)" | tee -a gpurun_out/traces_variants.log
done

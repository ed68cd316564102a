#!/usr/bin/env bash
# predictor, 3-D M = 3: 16 cells per CTA (two CTAs per SM) against 32 (one) — parity of the
# variant, timings, ncu --set full of the default on C5
set -u
mkdir -p gpurun_out
python -c "from paper_1612_09335_b200 import _build; _build.needs_build() and _build.build()" > gpurun_out/build.log 2>&1 || { echo build failed; exit 1; }
timeout 900 python -m pytest tests -m gpu -x -q -k "predict" > gpurun_out/pytest_pred.log 2>&1; echo "pytest default exit $?"; tail -1 gpurun_out/pytest_pred.log
for f in variants/lib_pred_*.so; do
  CWRECO_LIBRARY=$PWD/$f timeout 900 python -m pytest tests -m gpu -x -q -k "predict" > gpurun_out/pytest_$(basename $f .so).log 2>&1
  echo "pytest $f exit $?"; tail -1 gpurun_out/pytest_$(basename $f .so).log
done
echo "C5 default: $(timeout 600 python tools/predictor_bench.py --config C5 2>&1 | tail -1 | cut -c1-330)" | tee gpurun_out/pred_variants.log
for f in variants/lib_pred_*.so; do
  echo "C5 $f: $(CWRECO_LIBRARY=$PWD/$f timeout 600 python tools/predictor_bench.py --config C5 2>&1 | tail -1 | cut -c1-330)" | tee -a gpurun_out/pred_variants.log
done
ncu --set full --clock-control none --import-source on -k "regex:k_predictor" -s 2 -c 1 \
    -o gpurun_out/prof_pred_C5 -f python tools/predictor_bench.py --config C5 > gpurun_out/ncu_full_pred_C5.log 2>&1
echo "ncu predictor C5 exit $?"
CWRECO_LIBRARY=$PWD/variants/lib_pred_cb16.so ncu --set full --clock-control none --import-source on -k "regex:k_predictor" -s 2 -c 1 \
    -o gpurun_out/prof_pred_C5_cb16 -f python tools/predictor_bench.py --config C5 > gpurun_out/ncu_full_pred_C5_cb16.log 2>&1
echo "ncu predictor C5 cb16 exit $?"

#!/usr/bin/env bash
# predictor, 3-D M = 3: the update GEMM's column tiles over 2·(d+2) warps (CWR_PRED_WM3=2)
set -u
mkdir -p gpurun_out
python -c "from paper_1612_09335_b200 import _build; _build.needs_build() and _build.build()" > gpurun_out/build.log 2>&1 || { echo build failed; exit 1; }
timeout 900 python -m pytest tests -m gpu -x -q -k "predict" > gpurun_out/pytest_pred.log 2>&1; echo "pytest default exit $?"; tail -1 gpurun_out/pytest_pred.log
for f in variants/lib_pred_*.so; do
  CWRECO_LIBRARY=$PWD/$f timeout 900 python -m pytest tests -m gpu -x -q -k "predict" > gpurun_out/pytest_$(basename $f .so).log 2>&1
  echo "pytest $f exit $?"; tail -1 gpurun_out/pytest_$(basename $f .so).log
done
echo "C5 default: $(timeout 600 python tools/predictor_bench.py --config C5 2>&1 | tail -1 | cut -c1-330)" | tee gpurun_out/pred_variants2.log
for f in variants/lib_pred_*.so; do
  echo "C5 $f: $(CWRECO_LIBRARY=$PWD/$f timeout 600 python tools/predictor_bench.py --config C5 2>&1 | tail -1 | cut -c1-330)" | tee -a gpurun_out/pred_variants2.log
done

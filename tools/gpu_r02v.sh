#!/usr/bin/env bash
# predictor timings after the binding stopped rebuilding the host matrices per call
set -u
mkdir -p gpurun_out
python -c "from paper_1612_09335_b200 import _build; _build.needs_build() and _build.build()" > gpurun_out/build.log 2>&1 || { echo build failed; exit 1; }
timeout 900 python -m pytest tests -m gpu -x -q -k "predict" > gpurun_out/pytest_pred.log 2>&1; echo "pytest exit $?"; tail -1 gpurun_out/pytest_pred.log
for c in C2 C3 C5; do timeout 600 python tools/predictor_bench.py --config $c 2>&1 | tail -1 > gpurun_out/pred_$c.json; echo "pred $c: $(cut -c1-330 gpurun_out/pred_$c.json)"; done

#!/usr/bin/env bash
# closing tree: ncu --set full of the 10-warp predictor on C5, then all GPU tests
set -u
mkdir -p gpurun_out
python -c "from paper_1612_09335_b200 import _build; _build.needs_build() and _build.build()" > gpurun_out/build.log 2>&1 || { echo build failed; exit 1; }
ncu --set full --clock-control none --import-source on -k "regex:k_predictor" -s 2 -c 1 \
    -o gpurun_out/prof_pred_C5_wm2 -f python tools/predictor_bench.py --config C5 > gpurun_out/ncu_full_pred_C5_wm2.log 2>&1
echo "ncu predictor C5 exit $?"
bash tools/gpu_round.sh tests

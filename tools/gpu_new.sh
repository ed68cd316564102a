#!/usr/bin/env bash
# new-feature GPU checks: predictor + boundary ghosts + loopback; predictor throughput
set -u
mkdir -p gpurun_out
python -c "from paper_1612_09335_b200 import _build; _build.needs_build() and _build.build()" > gpurun_out/build.log 2>&1 || { echo build failed; tail gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests -m gpu -x -q -k "${TESTS:-predictor or boundary or loopback}" > gpurun_out/pytest_new.log 2>&1
echo "pytest exit $?"; tail -15 gpurun_out/pytest_new.log
for c in ${PRED_CFGS:-C3 C5}; do timeout 600 python tools/predictor_bench.py --config $c 2>&1 | tail -2; done

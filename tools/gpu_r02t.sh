#!/usr/bin/env bash
# closing check of the final tree: all GPU tests, smoke, the default bench line
set -u
mkdir -p gpurun_out
bash tools/gpu_round.sh tests
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print(\"smoke ok\")" > gpurun_out/smoke.log 2>&1; echo "smoke exit $?"; tail -2 gpurun_out/smoke.log
bash tools/gpu_round.sh bench
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_reference.json 2> gpurun_out/bench_reference.err; echo "reference exit $?"; cut -c1-400 gpurun_out/bench_reference.json

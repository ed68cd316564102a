#!/usr/bin/env bash
# Round-end measurement: GPU tests, bench lines C2-C5, matrix-free C5, face traces,
# launch list of the default bench and full ncu captures of C2 and C4.
set -u
mkdir -p gpurun_out
bash tools/gpu_round.sh tests
bash tools/gpu_round.sh bench
timeout 900 python bench.py --config C5 --kernel matrixfree --steps 10 --warmup 3 --no-cpu-baseline \
    > gpurun_out/bench_mf_C5.json 2> gpurun_out/bench_mf_C5.err; echo "mf C5 $?"
timeout 900 python tools/traces_bench.py C2 C5 > gpurun_out/traces_bench.json 2> gpurun_out/traces_bench.err
cmd="python bench.py --config C2 --steps 3 --warmup 3 --no-cpu-baseline"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_C2.csv $cmd \
    > gpurun_out/ncu_launch_C2.log 2>&1; echo "launch list exit $?"
bash tools/gpu_round.sh ncufull "C2 C4"

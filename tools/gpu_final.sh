set -u
mkdir -p gpurun_out
bash tools/gpu_round.sh tests
bash tools/gpu_round.sh bench
# launch list + full capture of the default bench (C2), then full capture of C4 (row-block)
cmd="python bench.py --config C2 --steps 3 --warmup 3 --no-cpu-baseline"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_C2.csv $cmd > gpurun_out/ncu_launch_C2.log 2>&1; echo "launch list exit $?"
bash tools/gpu_round.sh ncufull "C2 C4"

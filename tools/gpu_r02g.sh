#!/usr/bin/env bash
# round-2 measurement after the static stage loop: GPU tests, bench C4 (default) + C2/C3/C5,
# launch list of the default bench, full ncu captures of C4, C3, C5 (traffic keys)
set -u
mkdir -p gpurun_out
bash tools/gpu_round.sh tests
bash tools/gpu_round.sh benchall
cmd="python bench.py --steps 3 --warmup 3 --no-cpu-baseline"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_C4.csv $cmd \
    > gpurun_out/ncu_launch_C4.log 2>&1; echo "launch list exit $?"
for c in C4 C5 C3; do
  ncu --set full --clock-control none --import-source on -k "regex:k_pipelined|k_rowblk" -s 3 -c 1 \
      -o gpurun_out/prof_$c -f python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_full_$c.log 2>&1
  echo "ncu $c exit $?"
done

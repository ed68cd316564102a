#!/usr/bin/env bash
# One GPU session: GPU tests, bench lines, launch list and one full ncu capture of
# the reconstruction kernel.  Usage (from the repo root, under gpurun):
#   bash tools/gpu_round.sh [tests|bench|benchall|ncu|all] [config for ncu]
set -u
mkdir -p gpurun_out
what=${1:-all}
ncfg=${2:-C4}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/gpu.txt 2>&1
python -c "from paper_1612_09335_b200 import _build; _build.needs_build() and _build.build()" \
    > gpurun_out/build.log 2>&1 || { echo "build failed"; tail -30 gpurun_out/build.log; exit 1; }

if [[ $what == tests || $what == all ]]; then
  timeout 2400 python -m pytest tests -m gpu -x -q --durations=15 -s > gpurun_out/pytest_gpu.log 2>&1
  echo "pytest -m gpu exit $?"; tail -25 gpurun_out/pytest_gpu.log
fi
if [[ $what == bench || $what == benchall || $what == all ]]; then
  timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
  echo "bench default exit $?"; cat gpurun_out/bench_default.json; tail -3 gpurun_out/bench_default.err
fi
if [[ $what == benchall ]]; then
  for c in C2 C3 C5; do
    timeout 1200 python bench.py --config $c --steps 100 --warmup 5 --no-cpu-baseline \
        > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
    echo "bench $c exit $?"; cat gpurun_out/bench_$c.json
  done
fi
if [[ $what == ncu || $what == all ]]; then
  cmd="python bench.py --config $ncfg --steps 3 --warmup 3 --no-cpu-baseline"
  $cmd > gpurun_out/ncu_plain_$ncfg.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file gpurun_out/launches_$ncfg.csv $cmd > gpurun_out/ncu_launch_$ncfg.log 2>&1
  echo "ncu launches exit $?"
  ncu --set full --clock-control none --import-source on -k "regex:k_pipelined|k_rowblk" -s 3 -c 1 \
      -o gpurun_out/prof_$ncfg -f $cmd > gpurun_out/ncu_full_$ncfg.log 2>&1
  echo "ncu full exit $?"; tail -5 gpurun_out/ncu_full_$ncfg.log
fi

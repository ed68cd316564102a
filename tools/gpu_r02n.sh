#!/usr/bin/env bash
# round-2 final measurement: GPU tests, bench C4 (default) + C2/C3/C5, matrix-free C5,
# predictor C2/C3/C5, face traces C2/C5, launch list of the default bench, ncu of C3
set -u
mkdir -p gpurun_out
bash tools/gpu_round.sh tests
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print(\"smoke ok\")" > gpurun_out/smoke.log 2>&1; echo "smoke exit $?"; tail -2 gpurun_out/smoke.log
bash tools/gpu_round.sh benchall
timeout 900 python bench.py --config C5 --kernel matrixfree --steps 10 --warmup 3 --no-cpu-baseline \
    > gpurun_out/bench_mf_C5.json 2> gpurun_out/bench_mf_C5.err; echo "mf C5 $?"; cut -c1-300 gpurun_out/bench_mf_C5.json
for c in C2 C3 C5; do timeout 600 python tools/predictor_bench.py --config $c 2>&1 | tail -1 > gpurun_out/pred_$c.json; echo "pred $c: $(cut -c1-300 gpurun_out/pred_$c.json)"; done
timeout 900 python tools/traces_bench.py C2 C5 > gpurun_out/traces_bench.json 2> gpurun_out/traces_bench.err; cut -c1-200 gpurun_out/traces_bench.json
cmd="python bench.py --steps 3 --warmup 3 --no-cpu-baseline"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_C4.csv $cmd \
    > gpurun_out/ncu_launch_C4.log 2>&1; echo "launch list exit $?"
ncu --set full --clock-control none --import-source on -k "regex:k_pipelined|k_rowblk" -s 3 -c 1 \
    -o gpurun_out/prof_C3 -f python bench.py --config C3 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_full_C3.log 2>&1
echo "ncu C3 exit $?"

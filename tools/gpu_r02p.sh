#!/usr/bin/env bash
# round-2 closing measurement at HEAD: all GPU tests, smoke, bench C4 (default) +
# C2/C3/C5, matrix-free C5/C3, predictor, face traces, launch list of the default
# bench, ncu --set full of the C4 row-block kernel, the matrix-free kernel and k_traces2
set -u
mkdir -p gpurun_out
bash tools/gpu_round.sh tests
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print(\"smoke ok\")" > gpurun_out/smoke.log 2>&1; echo "smoke exit $?"; tail -2 gpurun_out/smoke.log
bash tools/gpu_round.sh benchall
for c in C5 C3; do
timeout 900 python bench.py --config $c --kernel matrixfree --steps 10 --warmup 3 --no-cpu-baseline \
    > gpurun_out/bench_mf_$c.json 2> gpurun_out/bench_mf_$c.err; echo "mf $c $?"; cut -c1-300 gpurun_out/bench_mf_$c.json
done
for c in C2 C3 C5; do timeout 600 python tools/predictor_bench.py --config $c 2>&1 | tail -1 > gpurun_out/pred_$c.json; echo "pred $c: $(cut -c1-300 gpurun_out/pred_$c.json)"; done
timeout 900 python tools/traces_bench.py C2 C3 C5 > gpurun_out/traces_bench.json 2> gpurun_out/traces_bench.err; cut -c1-400 gpurun_out/traces_bench.json
cmd="python bench.py --steps 3 --warmup 3 --no-cpu-baseline"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_C4.csv $cmd \
    > gpurun_out/ncu_launch_C4.log 2>&1; echo "launch list exit $?"
ncu --set full --clock-control none --import-source on -k "regex:k_pipelined|k_rowblk" -s 3 -c 1 \
    -o gpurun_out/prof_C4 -f $cmd > gpurun_out/ncu_full_C4.log 2>&1
echo "ncu C4 exit $?"
ncu --set full --clock-control none --import-source on -k "regex:k_matfree" -s 2 -c 1 \
    -o gpurun_out/prof_mf_C3 -f python bench.py --config C3 --kernel matrixfree --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_full_mf_C3.log 2>&1
echo "ncu mf C3 exit $?"
ncu --set full --clock-control none --import-source on -k "regex:k_traces" -s 2 -c 1 \
    -o gpurun_out/prof_tr_C3 -f python tools/traces_bench.py C3 > gpurun_out/ncu_full_tr_C3.log 2>&1
echo "ncu traces C3 exit $?"
ls -la gpurun_out/*.ncu-rep

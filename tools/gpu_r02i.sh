set -u
mkdir -p gpurun_out
python -c "from paper_1612_09335_b200 import _build; _build.needs_build() and _build.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q -k "traces or smaller_tile" > gpurun_out/pytest_tr.log 2>&1; echo "pytest exit $?"; tail -2 gpurun_out/pytest_tr.log
echo "--- traces wide (default)"; timeout 900 python tools/traces_bench.py C2 C3 C5 2>&1 | cut -c1-260
echo "--- traces old"; CWRECO_LIBRARY=$PWD/variants/lib_trold.so timeout 900 python tools/traces_bench.py C2 C5 2>&1 | cut -c1-260
for qb in 1 4; do echo "--- wide QB=$qb"; CWRECO_TRACE_QB=$qb CWRECO_LIBRARY=$PWD/variants/exp_tr.so timeout 900 python tools/traces_bench.py C3 C5 2>&1 | cut -c1-260; done
echo "--- rowblk gcell"
bash tools/gpu_variants.sh 2>&1 | grep -v exp_tr | grep -v trold | cut -c1-300
echo "C4 default: $(timeout 600 python tools/c4_iter.py --config C4 --reps 10 2>&1 | tail -1 | cut -c1-300)"
echo "C4 gcell: $(CWRECO_LIBRARY=$PWD/variants/lib_gcell.so timeout 600 python tools/c4_iter.py --config C4 --reps 10 2>&1 | tail -1 | cut -c1-300)"

set -u
mkdir -p gpurun_out
python -c "from paper_1612_09335_b200 import _build; _build.needs_build() and _build.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q tests/test_gpu_predictor.py > gpurun_out/pytest_pred.log 2>&1; echo "pytest pred exit $?"; tail -3 gpurun_out/pytest_pred.log
timeout 900 python -m pytest tests -m gpu -x -q -k "matrixfree_parity" > gpurun_out/pytest_mf2.log 2>&1; echo "pytest mf exit $?"; tail -1 gpurun_out/pytest_mf2.log
for c in C2 C3 C5; do
  echo "mma $c: $(timeout 600 python tools/predictor_bench.py --config $c 2>&1 | tail -1 | cut -c1-330)"
  echo "old $c: $(CWRECO_LIBRARY=$PWD/variants/lib_pred0.so timeout 600 python tools/predictor_bench.py --config $c 2>&1 | tail -1 | cut -c1-330)"
done
ITER_ARGS="--config C3" bash tools/gpu_variants.sh 2>&1 | grep -v pred0 | cut -c1-250
echo "C2 family1: $(timeout 600 python tools/c4_iter.py --config C2 --family 1 --reps 20 2>&1 | tail -1 | cut -c1-250)"
echo "C2 family0: $(timeout 600 python tools/c4_iter.py --config C2 --family 0 --reps 20 2>&1 | tail -1 | cut -c1-250)"
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest -m gpu exit $?"; tail -2 gpurun_out/pytest_gpu.log

set -u
mkdir -p gpurun_out
python -c "from paper_1612_09335_b200 import _build; _build.needs_build() and _build.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q tests/test_gpu_predictor.py > gpurun_out/pytest_pred.log 2>&1; echo "pytest pred exit $?"; tail -3 gpurun_out/pytest_pred.log
for c in C2 C3 C5; do
  echo "mma $c: $(timeout 600 python tools/predictor_bench.py --config $c 2>&1 | tail -1 | cut -c1-400)"
  echo "old $c: $(CWRECO_LIBRARY=$PWD/variants/lib_pred0.so timeout 600 python tools/predictor_bench.py --config $c 2>&1 | tail -1 | cut -c1-400)"
done

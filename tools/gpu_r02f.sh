set -u
mkdir -p gpurun_out
python -c "from paper_1612_09335_b200 import _build; _build.needs_build() and _build.build()" > gpurun_out/build.log 2>&1
bash tools/gpu_variants.sh > gpurun_out/var_c4proxy.log 2>&1; cat gpurun_out/var_c4proxy.log
ITER_ARGS="--V 5" bash tools/gpu_variants.sh > gpurun_out/var_c5shape.log 2>&1; cat gpurun_out/var_c5shape.log
ITER_ARGS="--config C3" bash tools/gpu_variants.sh > gpurun_out/var_c3.log 2>&1; cat gpurun_out/var_c3.log
timeout 2400 python -m pytest tests -m gpu -x -q --durations=10 -s > gpurun_out/pytest_gpu.log 2>&1
echo "pytest -m gpu exit $?"; grep -E "passed|failed|Error|max floored" gpurun_out/pytest_gpu.log | tail -12

set -u
mkdir -p gpurun_out
python -c "from paper_1612_09335_b200 import _build; _build.needs_build() and _build.build()" > gpurun_out/build.log 2>&1
bash tools/gpu_variants.sh > gpurun_out/var_c4proxy.log 2>&1; cat gpurun_out/var_c4proxy.log
ITER_ARGS="--V 5" bash tools/gpu_variants.sh > gpurun_out/var_c5shape.log 2>&1; cat gpurun_out/var_c5shape.log
ITER_ARGS="--config C3" bash tools/gpu_variants.sh > gpurun_out/var_c3.log 2>&1; cat gpurun_out/var_c3.log
timeout 1800 python tools/rank_projection.py --config C4 --nranks 2 8 > gpurun_out/proj2_C4.json 2> gpurun_out/proj2_C4.err
echo "proj exit $?"; grep -v "^P=. r=" gpurun_out/proj2_C4.err | tail; grep "r=0" gpurun_out/proj2_C4.err

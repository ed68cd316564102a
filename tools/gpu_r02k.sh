set -u
mkdir -p gpurun_out
python -c "from paper_1612_09335_b200 import _build; _build.needs_build() and _build.build()" > gpurun_out/build.log 2>&1
ITER_ARGS="--config C3" bash tools/gpu_variants.sh 2>&1 | cut -c1-300
timeout 2400 python tools/rank_projection.py --config C5 --weak --nranks 2 4 8 --ranks 0 > gpurun_out/proj_C5.json 2> gpurun_out/proj_C5.err
echo "proj exit $?"; tail -8 gpurun_out/proj_C5.err | cut -c1-400

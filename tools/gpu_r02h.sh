set -u
mkdir -p gpurun_out
python -c "from paper_1612_09335_b200 import _build; _build.needs_build() and _build.build()" > gpurun_out/build.log 2>&1
bash tools/gpu_variants.sh > gpurun_out/var_c4proxy.log 2>&1; cat gpurun_out/var_c4proxy.log | cut -c1-330
ITER_ARGS="--V 5" bash tools/gpu_variants.sh > gpurun_out/var_c5shape.log 2>&1; grep -v "^ \|tile" gpurun_out/var_c5shape.log | cut -c1-250
echo "C4 default: $(timeout 600 python tools/c4_iter.py --config C4 --reps 10 2>&1 | tail -1 | cut -c1-300)"
for v in l2pf8 l2pf16; do
  echo "C4 $v: $(CWRECO_LIBRARY=$PWD/variants/lib_$v.so timeout 600 python tools/c4_iter.py --config C4 --reps 10 2>&1 | tail -1 | cut -c1-300)"
done

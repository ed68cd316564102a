set -u
mkdir -p gpurun_out
python -c "from paper_1612_09335_b200 import _build; _build.needs_build() and _build.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q -s -k "matrixfree" > gpurun_out/pytest_mf.log 2>&1; echo "pytest mf exit $?"; grep -E "passed|failed|matrix-free" gpurun_out/pytest_mf.log | tail -4
for c in C2 C3 C5; do
  echo "v2 $c: $(timeout 600 python tools/c4_iter.py --config $c --kernel matrixfree --reps 5 2>&1 | tail -1 | cut -c1-200)"
  echo "v1 $c: $(CWRECO_LIBRARY=$PWD/variants/lib_mfv1.so timeout 600 python tools/c4_iter.py --config $c --kernel matrixfree --reps 5 2>&1 | tail -1 | cut -c1-200)"
done

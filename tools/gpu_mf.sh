#!/usr/bin/env bash
set -u
python -c "from paper_1612_09335_b200 import _build; _build.needs_build() and _build.build()" > /dev/null 2>&1
timeout 600 python -m pytest tests -m gpu -x -q -k "matrixfree" 2>&1 | tail -2
for n in ${MFN:-40}; do echo "mf d3 M3 V5 n$n: $(timeout 300 python tools/c4_iter.py --kernel matrixfree --d 3 --M 3 --V 5 --n $n --reps 5 2>&1 | tail -1)"; done
if [[ ${NCU:-0} == 1 ]]; then
  timeout 300 python tools/c4_iter.py --kernel matrixfree --d 3 --M 3 --V 5 --n 32 --reps 2 > /dev/null 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k "regex:k_matfree" -s 2 -c 1 -o gpurun_out/prof_mf -f \
    python tools/c4_iter.py --kernel matrixfree --d 3 --M 3 --V 5 --n 32 --reps 2 > gpurun_out/ncu_mf.log 2>&1
  echo "ncu exit $?"
fi

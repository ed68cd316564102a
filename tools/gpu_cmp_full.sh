#!/usr/bin/env bash
# Full-config comparison of the default library against variants/lib_*.so (tools only):
#   CFGS="C4 C5" bash tools/gpu_cmp_full.sh
set -u
mkdir -p gpurun_out
python -c "from paper_1612_09335_b200 import _build; _build.needs_build() and _build.build()" > gpurun_out/build.log 2>&1 || { echo build failed; exit 1; }
if [[ -n "${TESTS:-}" ]]; then
  timeout 900 python -m pytest tests -m gpu -x -q -k "$TESTS" > gpurun_out/pytest_cmp.log 2>&1
  echo "pytest exit $?"; tail -3 gpurun_out/pytest_cmp.log
fi
for c in ${CFGS:-C4}; do
  echo "$c default: $(timeout 600 python tools/c4_iter.py --config $c --reps ${REPS:-40} 2>&1 | tail -1 | cut -c1-300)"
  for f in variants/lib_*.so; do
    [[ -e $f ]] || continue
    echo "$c $f: $(CWRECO_LIBRARY=$PWD/$f timeout 600 python tools/c4_iter.py --config $c --reps ${REPS:-40} 2>&1 | tail -1 | cut -c1-300)"
  done
done

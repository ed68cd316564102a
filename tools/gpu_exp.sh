#!/usr/bin/env bash
# phase-removal experiments on the C4-shape proxy (experiments build: timing only, results wrong)
set -u
for f in 0 16 1 17 2 18; do
  echo "flags=$f: $(CWRECO_EXP_FLAGS=$f CWRECO_LIBRARY=$PWD/variants/lib_exp.so timeout 300 python tools/c4_iter.py ${ITER_ARGS:-} 2>&1 | tail -1)"
done

#!/usr/bin/env bash
set -u
python -c "from paper_1612_09335_b200 import _build; _build.needs_build() and _build.build()" > /dev/null 2>&1
timeout 600 python -m pytest tests -m gpu -x -q -k predictor 2>&1 | tail -1
for c in ${PRED_CFGS:-C5}; do
  echo "default $c: $(timeout 600 python tools/predictor_bench.py --config $c 2>&1 | tail -1 | cut -c1-260)"
  for f in variants/lib_*.so; do echo "$f $c: $(CWRECO_LIBRARY=$PWD/$f timeout 600 python tools/predictor_bench.py --config $c 2>&1 | tail -1 | cut -c1-260)"; done
done

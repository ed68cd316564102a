#!/usr/bin/env bash
# time the C4-shape kernel for the default library and every variants/lib_*.so (tools only);
# trace_* variants print CTA 0's timeline instead
set -u
python -c "from paper_1612_09335_b200 import _build; _build.needs_build() and _build.build()" > /dev/null 2>&1
echo "default: $(timeout 300 python tools/c4_iter.py --check ${ITER_ARGS:-} 2>&1 | tail -1 | cut -c1-260)"
for f in variants/lib_*.so; do
  case $f in
    *trace*) echo "$f:"; CWRECO_LIBRARY=$PWD/$f timeout 300 python tools/c4_iter.py --trace ${ITER_ARGS:-} 2>&1 | tail -6 ;;
    *) echo "$f: $(CWRECO_LIBRARY=$PWD/$f timeout 300 python tools/c4_iter.py --check ${ITER_ARGS:-} 2>&1 | tail -1 | cut -c1-260)" ;;
  esac
done

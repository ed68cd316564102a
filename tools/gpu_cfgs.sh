#!/usr/bin/env bash
set -u
python -c "from paper_1612_09335_b200 import _build; _build.needs_build() and _build.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests -m gpu -x -q -k "${TESTS:-small_mesh or many_tiles or strides or boundary or loopback or multirank}" 2>&1 | tail -2
for c in ${CFGS:-C3 C5 C2}; do echo "$c: $(timeout 300 python tools/c4_iter.py --config $c --check 2>&1 | tail -1 | cut -c1-230)"; done

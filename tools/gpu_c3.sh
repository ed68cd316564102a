#!/usr/bin/env bash
set -u
python -c "from paper_1612_09335_b200 import _build; _build.needs_build() and _build.build()" > /dev/null 2>&1
for fam in 0 1; do echo "C3 fam=$fam: $(timeout 300 python tools/c4_iter.py --config C3 --family $fam --check 2>&1 | tail -1 | cut -c1-230)"; done
for f in variants/lib_*.so; do echo "C3 $f: $(CWRECO_LIBRARY=$PWD/$f timeout 300 python tools/c4_iter.py --config C3 --family 1 --check 2>&1 | tail -1 | cut -c1-230)"; done

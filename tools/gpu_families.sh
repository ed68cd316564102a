#!/usr/bin/env bash
# kernel-family / variant comparison on the config shapes (tools only)
set -u
python -c "from paper_1612_09335_b200 import _build; _build.needs_build() and _build.build()" > /dev/null 2>&1
run() { echo "$1 $2: $(timeout 300 python tools/c4_iter.py $1 $2 --check 2>&1 | tail -1 | cut -c1-260)"; }
for shape in "--d 3 --M 2 --V 5 --n 64" "--d 2 --M 3 --V 4 --n 512"; do
  run "$shape" "--family 0"
  run "$shape" "--family 1"
  for f in variants/lib_*.so; do echo "$shape $f: $(CWRECO_LIBRARY=$PWD/$f timeout 300 python tools/c4_iter.py $shape --family 1 --check 2>&1 | tail -1 | cut -c1-260)"; done
done

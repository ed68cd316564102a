#!/usr/bin/env bash
# quick GPU iteration: small-mesh parity of the row-block family + the C4-shape timing
set -u
mkdir -p gpurun_out
python -c "from paper_1612_09335_b200 import _build; _build.needs_build() and _build.build()" > gpurun_out/build.log 2>&1 || { echo build failed; tail -20 gpurun_out/build.log; exit 1; }
timeout 600 python -m pytest tests -m gpu -x -q -k "${TESTS:-rowblk or many_tiles or loopback}" > gpurun_out/pytest_iter.log 2>&1
echo "pytest exit $?"; tail -4 gpurun_out/pytest_iter.log
timeout 600 python tools/c4_iter.py --check ${ITER_ARGS:-} 2>&1 | tail -3

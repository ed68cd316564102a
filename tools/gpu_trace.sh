#!/usr/bin/env bash
# C4-shape proxy timing (default library) + CTA-0 timeline from the trace variant
set -u
python -c "from paper_1612_09335_b200 import _build; _build.needs_build() and _build.build()" > /dev/null 2>&1
timeout 600 python -m pytest tests -m gpu -x -q -k "${TESTS:-rowblk or many_tiles or loopback}" 2>&1 | tail -2
timeout 300 python tools/c4_iter.py --check ${ITER_ARGS:-} 2>&1 | tail -1
CWRECO_LIBRARY=$PWD/variants/lib_trace.so timeout 300 python tools/c4_iter.py --trace ${ITER_ARGS:-} 2>&1 | tail -${TRACE_LINES:-16}

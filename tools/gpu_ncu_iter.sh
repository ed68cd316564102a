#!/usr/bin/env bash
# ncu --set full of the row-block kernel on the C4-shape proxy mesh (tools/c4_iter.py)
set -u
mkdir -p gpurun_out
python -c "from paper_1612_09335_b200 import _build; _build.needs_build() and _build.build()" > gpurun_out/build.log 2>&1 || { echo build failed; exit 1; }
tag=${TAG:-it}
timeout 300 python tools/c4_iter.py --reps 2 ${ITER_ARGS:-} > gpurun_out/ncu_plain_$tag.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:${KREGEX:-k_rowblk}" -s 3 -c 1 \
    -o gpurun_out/prof_$tag -f python tools/c4_iter.py --reps 2 ${ITER_ARGS:-} > gpurun_out/ncu_full_$tag.log 2>&1
echo "ncu exit $?"; tail -3 gpurun_out/ncu_full_$tag.log

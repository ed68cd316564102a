#!/usr/bin/env bash
# matrix-free full-mesh parity, one-GPU rank projection (C4 strong 2/4/8), matrix-free ncu
set -u
mkdir -p gpurun_out
python -c "from paper_1612_09335_b200 import _build; _build.needs_build() and _build.build()" > gpurun_out/build.log 2>&1 || { echo build failed; exit 1; }
timeout 900 python -m pytest tests -m gpu -x -q -s -k matrixfree_full > gpurun_out/pytest_mffull.log 2>&1
echo "pytest mf full exit $?"; grep -E "matrix-free|passed|failed|Error" gpurun_out/pytest_mffull.log | tail -5
timeout 2400 python tools/rank_projection.py --config ${PCFG:-C4} --nranks ${PN:-2 4 8} > gpurun_out/proj_${PCFG:-C4}.json 2> gpurun_out/proj_${PCFG:-C4}.err
echo "proj exit $?"; tail -20 gpurun_out/proj_${PCFG:-C4}.err
if [[ ${MFNCU:-1} == 1 ]]; then
  cmd="python bench.py --config C5 --kernel matrixfree --steps 2 --warmup 3 --no-cpu-baseline"
  ncu --set full --clock-control none --import-source on -k "regex:k_matfree" -s 2 -c 1 \
      -o gpurun_out/prof_mf_C5 -f $cmd > gpurun_out/ncu_mf_C5.log 2>&1
  echo "ncu mf exit $?"; tail -3 gpurun_out/ncu_mf_C5.log
fi

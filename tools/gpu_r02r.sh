#!/usr/bin/env bash
# k_traces2 round 2q final: parity (face traces + smoke), timings, ncu --set full on C5
set -u
mkdir -p gpurun_out
python -c "from paper_1612_09335_b200 import _build; _build.needs_build() and _build.build()" > gpurun_out/build.log 2>&1 || { echo build failed; exit 1; }
timeout 900 python -m pytest tests -m gpu -x -q -k "face_traces or c_client" > gpurun_out/pytest_tr.log 2>&1
echo "pytest default exit $?"; tail -3 gpurun_out/pytest_tr.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1; echo "smoke exit $?"
timeout 900 python tools/traces_bench.py C5 C3 C2 > gpurun_out/traces_bench.json 2> gpurun_out/traces_bench.err; cut -c1-260 gpurun_out/traces_bench.json
for f in variants/lib_tr_*.so; do
  [ -f $f ] || continue
  echo "traces $f: $(CWRECO_LIBRARY=$PWD/$f timeout 900 python tools/traces_bench.py C5 C3 2>&1 | cut -c1-230)" | tee -a gpurun_out/traces_variants2.log
done
ncu --set full --clock-control none --import-source on -k "regex:k_traces" -s 2 -c 1 \
    -o gpurun_out/prof_tr_C5 -f python tools/traces_bench.py C5 > gpurun_out/ncu_full_tr_C5.log 2>&1
echo "ncu traces C5 exit $?"

set -u
mkdir -p gpurun_out
python -c "from paper_1612_09335_b200 import _build; _build.needs_build() and _build.build()" > gpurun_out/build.log 2>&1 || { echo build failed; tail -20 gpurun_out/build.log; exit 1; }
timeout 120 python - <<'PY' > gpurun_out/nvml.log 2>&1
import torch, sys
sys.path.insert(0, ".")
import bench
torch.cuda.init()
with bench.ClockSampler(0) as c:
    x = torch.randn(4096, 4096, device="cuda")
    for _ in range(200): x = x @ x * 1e-3
    torch.cuda.synchronize()
print(c.summary())
PY
echo "nvml exit $?"; cat gpurun_out/nvml.log | tail -3
timeout 900 python -m pytest tests -m gpu -x -q -k "loopback or many_tiles or small_mesh or strides" > gpurun_out/pytest_new.log 2>&1
echo "pytest new exit $?"; tail -5 gpurun_out/pytest_new.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
echo "bench exit $?"; cat gpurun_out/bench_default.json; tail -3 gpurun_out/bench_default.err

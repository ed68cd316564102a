#!/usr/bin/env python
"""Benchmark of the CWENO reconstruction pass (arXiv 1612.09335 §2.1) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C4] [--impl ours|reference]

One "step" = one full reconstruction pass (gather → B⁺ΔQ → sectors → P0 → σ → ω →
blend → store, all rows of SURVEY §8(a)) over every cell of the workload.  The
default workload is C4 (BASELINE.json configs[3]: 12.6 M jittered tetrahedra,
M=3, 9 MHD variables, 138.6 GB of algorithmic traffic per pass) — the largest
configuration that fits one GPU, the one the north_star 60 %-of-HBM gate and
the 8-GPU efficiency gate are about.  N>1 (torchrun, one rank per GPU, NCCL):
C4 is STRONG scaling (the same mesh partitioned into N Morton ranges, halo
exchange overlapped with the interior tiles); --config C5 runs the weak ladder
n = 100/126/159/200 (R26); C2/C3 scale their box with N (weak).

Timing: W untimed warm-up steps, then K steps bracketed by a barrier and a
device synchronize; each step is timed with CUDA events on the stream the
kernel is launched on, and the L2 is flushed (a 512 MiB write) between steps,
outside the events, so every step starts cold.  Max over ranks.  SM clocks and
throttle reasons are sampled in-process (NVML, every 20 ms) during the timed
region.

Prints ONE JSON line (rank 0).  --impl reference times the CPU oracle (oracle/,
precomputed per-cell matrices, pass only, all host cores) on a bounded sample of
the same workload; so does this arm's cpu_baseline (N=1).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "CWENO reconstructed cells/sec (fp64) and % of HBM roofline at 1/2/4/8 B200"
WORKLOAD_TEXT = {
    "C1": "2D 16x16x2 periodic, M=2, Euler 4 vars, isentropic vortex (BASELINE configs[0])",
    "C2": "2D 512x512x2 periodic triangles jittered +-0.2h, M=3, Euler 4 vars, vortex + ratio-10 jump (BASELINE configs[1])",
    "C3": "3D 64^3x6 tets, M=2, Euler 5 vars, spherical explosion (BASELINE configs[2])",
    "C4": "3D 128^3x6 tets jittered +-0.1h, M=3, MHD 9 vars, Orszag-Tang-type (BASELINE configs[3])",
    "C5": "3D n^3x6 tets (n=100 per GPU weak ladder), M=3, Euler 5 vars, explosion (BASELINE configs[4])",
}


def env_rank():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


STRONG = {"C4"}   # configs partitioned as one fixed mesh across N GPUs (R26: C4 strong 1→8)


def workload_n(cfg, N):
    import gen
    base = gen.CONFIGS[cfg]["n"]
    if N == 1 or cfg in STRONG:
        return base
    if cfg == "C5":
        return gen.C5_WEAK_N.get(N, round(100 * N ** (1 / 3)))
    d = gen.CONFIGS[cfg]["d"]
    return int(round(base * N ** (1.0 / d)))


# fp64 FMA peak of B200 (derived): 148 SMs × 64 DFMA/clk × 2 flop × 1.965 GHz
FP64_PEAK_TF = 148 * 64 * 2 * 1.965e9 / 1e12
FP64_PEAK_SRC = "derived: 148 SM x 64 fp64 FMA/clk x 2 x 1.965 GHz (no measured fp64 peak in MEASURED_PEAKS.json)"


def matfree_flops_per_cell(d, M, V):
    """Algorithmic fp64 flops of one matrix-free cell (K3; FMA = 2): per row of
    A (K = n_e−1 rows) the stencil cell's vertices in the owner's reference coordinates,
    the power sums and closed-form simplex moments of the monomials of degree ≤ M, the
    basis over the monomials of degree ≤ deg(ψ_l) and ΔQ; the Gram matrix [AᵀA | AᵀΔQ]
    (upper triangle); Cholesky with the forward substitution of the V right-hand sides;
    back substitution; d+1 sector solves; the epilogue."""
    nm = (M + 1) * (M + 2) // 2 if d == 2 else (M + 1) * (M + 2) * (M + 3) // 6
    R, K = nm - 1, d * nm - 1
    cnt = (lambda n: (n + 1) * (n + 2) // 2) if d == 2 else (lambda n: (n + 1) * (n + 2) * (n + 3) // 6)
    deg = lambda l: next(n for n in range(M + 1) if l < cnt(n))
    c2, c3 = d * (d + 1) // 2, d * (d + 1) * (d + 2) // 6
    row = ((d + 1) * (2 * d * d + d)                       # vertices
           + (d + 1) * d + (2 * (d + 1) * c2 if M >= 2 else 0) + (2 * (d + 1) * c3 if M >= 3 else 0)  # power sums
           + d + (3 * c2 if M >= 2 else 0) + (12 * c3 if M >= 3 else 0)                                  # moments
           + 2 * sum(cnt(deg(l)) for l in range(1, nm))   # basis
           + V)
    gram = 2 * K * (R * (R + 1) // 2 + R * V)
    chol = R ** 3 // 3 + R * R * V
    backsub = R * R * V
    sectors = (d + 1) * (2 * d ** 3 + 2 * d * d * V)
    epilogue = V * (2 * R * (R + 1) // 2 * 2 + 40 * (d + 2))
    return K * row + gram + chol + backsub + sectors + epilogue


def measured_peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            j = json.load(f)
        return float(j["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def profiled_traffic(cfg, kernel_symbol):
    """Per-launch dram__bytes_read.sum + dram__bytes_write.sum of the kernel actually
    launched (e.g. "C4:k_rowblk"), from the committed ncu --set full capture
    (profiles/ncu_traffic.json, written by tools/ncu_summary.py); None if absent."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(p) as f:
            j = json.load(f)
        return j.get(f"{cfg}:{kernel_symbol}")
    except Exception:
        return None


class ClockSampler:
    """SM clocks + throttle reasons of one GPU sampled in-process with NVML every
    20 ms while the timed region runs (B200_PROFILING.md clocks line)."""

    REASONS = {"hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40, "sw_thermal_slowdown": 0x20,
               "sw_power_cap": 0x4, "hw_power_brake_slowdown": 0x80}

    def __init__(self, index, period_s=0.02):
        self.index, self.period = index, period_s
        self.samples, self.reasons = [], set()
        self.max_mhz = None
        self._stop = threading.Event()

    def __enter__(self):
        try:
            import pynvml as N
            N.nvmlInit()
            # torch's device index → NVML handle through the device UUID
            import torch
            h = None
            try:
                want = str(torch.cuda.get_device_properties(self.index).uuid).lower().replace("gpu-", "")
                for k in range(N.nvmlDeviceGetCount()):
                    hk = N.nvmlDeviceGetHandleByIndex(k)
                    u = N.nvmlDeviceGetUUID(hk)
                    u = (u.decode() if isinstance(u, bytes) else str(u)).lower().replace("gpu-", "")
                    if u == want:
                        h = hk
                        break
            except Exception:
                h = None
            if h is None:
                vis = os.environ.get("CUDA_VISIBLE_DEVICES", "")
                first = vis.split(",")[self.index] if vis else ""
                idx = int(first) if first.isdigit() else self.index
                h = N.nvmlDeviceGetHandleByIndex(idx)
            self.N, self.h = N, h
            self.max_mhz = float(N.nvmlDeviceGetMaxClockInfo(h, N.NVML_CLOCK_SM))
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        except Exception as e:  # no NVML: report no samples
            self.err = str(e)
            self.N = None
        return self

    def _run(self):
        N, h = self.N, self.h
        while not self._stop.is_set():
            try:
                self.samples.append(float(N.nvmlDeviceGetClockInfo(h, N.NVML_CLOCK_SM)))
                r = N.nvmlDeviceGetCurrentClocksEventReasons(h)
                for name, bit in self.REASONS.items():
                    if r & bit:
                        self.reasons.add(name)
            except Exception:
                pass
            self._stop.wait(self.period)

    def __exit__(self, *a):
        self._stop.set()
        if self.N is not None:
            self.t.join(timeout=2)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons), "samples": 0,
                    "source": "nvml"}
        return {"sm_mhz": float(np.median(self.samples)), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples), "source": "nvml, 20 ms"}


# ----------------------------------------------------------------------------- oracle arm
def _one_thread():
    """Limit numpy's BLAS/LAPACK pools to one thread per worker process."""
    try:
        from threadpoolctl import threadpool_limits
        return threadpool_limits(limits=1)
    except Exception:  # threadpoolctl missing: numpy's tiny solves stay single-threaded anyway
        import contextlib
        return contextlib.nullcontext()


_ORC = {}   # fork-inherited state of the oracle workers (mesh, averages, degree)


def _oracle_worker(conn, cells, pre_budget_s):
    """One host core: precompute the matrices of its sample cells (setup, not
    timed), then on each request run the pass (oracle.reconstruct.apply_cell) over
    them and report (cells, seconds)."""
    from oracle import reconstruct as R
    m, Q, M = _ORC["m"], _ORC["Q"], _ORC["M"]
    with _one_thread():
        t0 = time.perf_counter()
        pre = []
        for i in cells:
            if pre and time.perf_counter() - t0 > pre_budget_s:
                break
            pre.append(R.precompute_cell(m, int(i), M))
        conn.send(("ready", len(pre), time.perf_counter() - t0))
        while True:
            msg = conn.recv()
            if msg[0] == "stop":
                break
            t = time.perf_counter()
            for _ in range(msg[1]):
                for p in pre:
                    R.apply_cell(p, Q)
            conn.send((msg[1] * len(pre), time.perf_counter() - t))


class OraclePool:
    """The CPU oracle on every host core: one forked process per core,
    each with a random sample of the workload's cells and their precomputed matrices;
    a step = every worker runs the reconstruction pass over its sample once."""

    def __init__(self, w, pre_budget_s=8.0, max_workers=None, seed=0):
        import multiprocessing as mp
        from oracle.mesh import OracleMesh
        t = time.perf_counter()
        m = OracleMesh(w["nodes"], w["cells"], w["period"], w["M"])
        _ORC.update(m=m, Q=w["avgs"][m.perm], M=w["M"])
        self.mesh_s = time.perf_counter() - t
        cores = len(os.sched_getaffinity(0))
        self.cores = max(1, min(cores, max_workers or 128))
        order = np.random.default_rng(seed).permutation(m.N)
        per = max(1, min(4096, m.N // self.cores))
        ctx = mp.get_context("fork")
        self.conns, self.procs = [], []
        for k in range(self.cores):
            a, b = ctx.Pipe()
            pr = ctx.Process(target=_oracle_worker, args=(b, order[k * per:(k + 1) * per], pre_budget_s), daemon=True)
            pr.start()
            self.conns.append(a)
            self.procs.append(pr)
        rd = [c.recv() for c in self.conns]
        self.sample = sum(r[1] for r in rd)
        self.pre_s = max(r[2] for r in rd)
        self.N = m.N

    def step(self, reps=1):
        """One pass over every worker's sample; returns (cells, wall seconds)."""
        t = time.perf_counter()
        for c in self.conns:
            c.send(("run", reps))
        n = sum(c.recv()[0] for c in self.conns)
        return n, time.perf_counter() - t

    def close(self):
        for c in self.conns:
            try:
                c.send(("stop",))
            except Exception:
                pass
        for p in self.procs:
            p.join(timeout=5)

    def describe(self, cfg):
        return (f"{self.sample} random cells of {cfg} ({self.N} cells) over {self.cores} host cores "
                f"(one process each), oracle per-cell matrices precomputed first "
                f"({self.pre_s:.1f} s, not timed), pass only (oracle.reconstruct.apply_cell)")


def oracle_baseline(w, cfg, seconds):
    """cpu_baseline of our arm: the pooled oracle pass for about `seconds` of work."""
    pool = OraclePool(w)
    try:
        pool.step()                    # warm-up sweeps (the first builds each worker's Σ tables)
        n, dt = pool.step()
        reps = max(1, int(seconds / max(dt, 1e-4)))
        n, dt = pool.step(reps)
        return {"value": n / dt, "unit": "cells/s", "cores": pool.cores, "kind": "oracle",
                "sample": pool.describe(cfg) + f"; {reps} sweeps in {dt:.1f} s"}
    finally:
        pool.close()


def run_reference(args):
    rank, world, _ = env_rank()
    if rank != 0:
        return 0
    import gen
    w = gen.make(args.config, workload_n(args.config, 1))
    pool = OraclePool(w, pre_budget_s=min(8.0, 60.0 / max(1, args.steps + args.warmup) + 2.0))
    try:
        for _ in range(args.warmup):
            pool.step()
        cells, t = 0, 0.0
        for _ in range(args.steps):
            n, dt = pool.step()
            cells += n
            t += dt
    finally:
        pool.close()
    value = cells / t
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "cells/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": t / args.steps * 1e3,
            "higher_is_better": True, "scaling": "strong" if args.config in STRONG else "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"{args.config}: {WORKLOAD_TEXT[args.config]}", "n_cells": int(pool.N)},
            "cpu_baseline": {"value": value, "unit": "cells/s", "cores": pool.cores, "kind": "oracle",
                             "sample": pool.describe(args.config) + "; a step = one pass over the sample"},
            "e2e": {"value": value, "unit": "cells/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ----------------------------------------------------------------------------- our arm
def run_ours(args):
    import torch
    import torch.distributed as dist

    import gen
    import paper_1612_09335_b200 as P

    rank, world, local = env_rank()
    if world != args.gpus:
        if rank == 0:
            print(f"warning: WORLD_SIZE={world} but --gpus {args.gpus}; using WORLD_SIZE", file=sys.stderr)
    version = P.lib.cwreco_version().decode()
    if "experiments" in version:
        print(f"refusing to time {version}: rebuild without CWRECO_BUILD_EXPERIMENTS", file=sys.stderr)
        return 2
    n = workload_n(args.config, world)
    w = gen.make(args.config, n)
    # the oracle baseline forks host workers: run it before this process initialises CUDA
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = oracle_baseline(w, args.config, args.cpu_seconds)

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    t_setup = time.perf_counter()
    ctx = P.Context(w["d"], w["M"], w["V"], device=local)
    ctx.set_mesh(w["nodes"], w["cells"], w["period"])
    if world > 1:
        from paper_1612_09335_b200 import dist as pdist
        pdist.init_transport(ctx)      # NCCL communicator inside the library (id broadcast here)
    ctx.build_stencils()               # collective at N>1: the library installs its send lists
    if args.kernel == "matrixfree":
        ctx.prepare_matrixfree()        # geometry + stencils only, no matrices (NEXT-1)
    else:
        ctx.precompute()
    ctx.set_kernel(args.kernel)
    t_setup = time.perf_counter() - t_setup
    inf = ctx.info()
    perm = ctx.permutation()
    loc = ctx.local_cells()                       # local -> SFC id
    avgs_local = np.ascontiguousarray(w["avgs"][perm[loc]])  # [n_local, V] in local order
    n_owned = inf["n_owned"]
    V, nm = w["V"], ctx.nm
    A = torch.tensor(avgs_local, device=dev)
    out = torch.empty((n_owned, V, nm), dtype=torch.float64, device=dev)
    stream = torch.cuda.current_stream()
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)

    if world > 1:
        # one overlapped pass: the library's NCCL halo exchange on its comm stream,
        # interior tiles concurrently, boundary tiles after the exchange event; the
        # ghost rows of A are rewritten by the exchange every step
        def step():
            ctx.reconstruct_overlap(A, out, stream=stream)
    else:
        def step():
            ctx.reconstruct(A, out, stream=stream)

    for _ in range(max(3, args.warmup)):
        step()
    torch.cuda.synchronize()

    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        for k in range(args.steps):
            flush.fill_(k & 0xFF)          # evict L2 between steps (outside the events)
            evs[k][0].record(stream)
            step()
            evs[k][1].record(stream)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    times = np.array([a.elapsed_time(b) for a, b in evs])  # ms
    t_total = float(times.sum()) / 1e3
    if world > 1:
        tt = torch.tensor([t_total], device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_total = float(tt.item())
        cells_all = torch.tensor([float(n_owned)], device=dev)
        dist.all_reduce(cells_all)
        cells_total = float(cells_all.item())
    else:
        cells_total = float(n_owned)
    value = cells_total * args.steps / t_total
    ms_step = t_total / args.steps * 1e3

    # roofline of the dominant kernel (the reconstruction kernel is the only kernel of the pass at N=1)
    bpc = inf["algorithmic_bytes_per_cell"]
    mf_flops = matfree_flops_per_cell(w["d"], w["M"], V) if args.kernel == "matrixfree" else None
    kern_s = float(np.mean(times)) / 1e3
    achieved = bpc * n_owned / kern_s / 1e9
    peak, peak_src = measured_peak()

    # end to end through the public API with HOST buffers: at N=1 the C-ABI call
    # cwreco_reconstruct_host (pinned host avgs -> device -> reconstruct, tile ranges
    # overlapped with their device->host copies -> host coeffs); at N>1 the same
    # copies around the halo-exchange step (ghost rows come from the peers)
    h_in = torch.from_numpy(avgs_local).pin_memory()
    h_out = torch.empty((n_owned, V, nm), dtype=torch.float64).pin_memory()
    e2e_steps = max(3, min(args.steps, 50))
    if world == 1:
        def e2e_step():
            ctx.reconstruct_host(h_in, h_out, stream=stream)
        e2e_api = "cwreco_reconstruct_host (C-ABI, pinned host buffers)"
    else:
        def e2e_step():
            A.copy_(h_in, non_blocking=True)
            step()
            h_out.copy_(out, non_blocking=True)
        e2e_api = "H2D + cwreco_reconstruct_overlap (NCCL halo inside the library) + D2H"
    for _ in range(2):
        e2e_step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(e2e_steps):
        e2e_step()
    e1.record(stream)
    torch.cuda.synchronize()
    t_e2e = e0.elapsed_time(e1) / 1e3
    if world > 1:
        tt = torch.tensor([t_e2e], device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_e2e = float(tt.item())
    e2e_value = cells_total * e2e_steps / t_e2e

    clocks = clk.summary()
    if rank == 0:
        ksym = ("k_rowblk" if inf.get("kernel_family") == 1 else "k_pipelined") if args.kernel == "pipelined" \
            else ("k_simple" if args.kernel == "simple" else "k_matfree")
        line = {
            "metric": METRIC, "value": value, "unit": "cells/s", "n_gpus": world, "steps": args.steps,
            "warmup": max(3, args.warmup), "ms_per_step": ms_step, "higher_is_better": True,
            "scaling": "strong" if args.config in STRONG else "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": {"workload": f"{args.config}: {WORKLOAD_TEXT[args.config]}", "n_cells_total": int(cells_total),
                       "n_cells_per_gpu": int(n_owned), "d": w["d"], "M": w["M"], "V": V, "box_n": n,
                       "kernel": "cwr::" + ksym, "kernel_mode": args.kernel, "l2": "flushed (512 MiB write) between timed steps",
                       "parallelism": f"cell partition x{world}" + (" + library NCCL halo, overlapped" if world > 1 else ""),
                       "setup_s": round(t_setup, 3), "library": version},
            "roofline": ({"bound": "alu", "achieved": mf_flops * n_owned / kern_s / 1e12, "peak": FP64_PEAK_TF,
                          "unit": "TFLOP/s", "frac": mf_flops * n_owned / kern_s / 1e12 / FP64_PEAK_TF,
                          "traffic": None, "peak_source": FP64_PEAK_SRC, "flops_per_cell": mf_flops,
                          "kernel": "cwr::k_matfree"} if mf_flops else
                         {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "frac_vs_8tbs": achieved / 8000.0,
                         "traffic": profiled_traffic(args.config, ksym) if world == 1 else None,
                         "peak_source": peak_src, "algorithmic_bytes_per_cell": bpc,
                         "kernel": "cwr::" + ksym}),
            "cpu_baseline": cpu,
            "e2e": {"value": e2e_value, "unit": "cells/s", "h2d_bytes_per_step": int(avgs_local.nbytes),
                    "d2h_bytes_per_step": int(n_owned * V * nm * 8), "api": e2e_api},
            "gpu_launches": args.steps * (1 if world == 1 else 3),
            "clocks": clocks,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--config", default="C4", choices=["C1", "C2", "C3", "C4", "C5"])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--kernel", default="pipelined", choices=["pipelined", "simple", "matrixfree"])
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())

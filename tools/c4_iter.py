#!/usr/bin/env python
"""Fast iteration on the C4 kernel shape (d=3, M=3, V=9) on a smaller mesh: n^3x6
jittered tetrahedra (default n=64: 1.57 M cells, 17 GB of packed matrices, setup
~15 s instead of ~90 s for C4).  Prints one JSON line: ms per pass (CUDA events,
L2 flushed between passes), algorithmic GB/s and the fraction of the measured
copy peak, and whether the pipelined kernel equals k_simple bitwise."""
import argparse
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import gen  # noqa: E402
import paper_1612_09335_b200 as P  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=64)
ap.add_argument("--d", type=int, default=3)
ap.add_argument("--M", type=int, default=3)
ap.add_argument("--V", type=int, default=9)
ap.add_argument("--family", type=int, default=-1)
ap.add_argument("--reps", type=int, default=20)
ap.add_argument("--check", action="store_true")
ap.add_argument("--config", default=None, help="use a BASELINE config's mesh and data instead (C1..C5)")
ap.add_argument("--kernel", default="pipelined", choices=["pipelined", "matrixfree"])
ap.add_argument("--max-ctas", type=int, default=0)
ap.add_argument("--trace", action="store_true", help="print CTA 0's timeline (library built with -DCWR_TRACE)")
a = ap.parse_args()

t = time.time()
if a.config:
    w = gen.make(a.config)
    nodes, cells, period, Q = w["nodes"], w["cells"], w["period"], w["avgs"]
    a.d, a.M, a.V, a.n = w["d"], w["M"], w["V"], w["n"]
else:
    nodes, cells, period = gen.box_mesh(a.d, a.n, True, 0.1, 4)
    Q = np.random.default_rng(0).standard_normal((cells.shape[0], a.V)) + 2.0
if a.kernel == "matrixfree":
    ctx = P.Context(a.d, a.M, a.V, device=0)
    ctx.set_mesh(nodes, cells, period)
    ctx.build_stencils()
    ctx.prepare_matrixfree()
    ctx.set_kernel("matrixfree")
else:
    ctx = P.setup_context(nodes, cells, period, a.M, a.V, device=0, family=a.family, max_ctas=a.max_ctas)
setup = time.time() - t
inf = ctx.info()
Qd = torch.tensor(Q[ctx.permutation()], device="cuda")
out = torch.empty((inf["n_owned"], a.V, ctx.nm), dtype=torch.float64, device="cuda")
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
st = torch.cuda.current_stream()
for _ in range(3):
    ctx.reconstruct(Qd, out, stream=st)
torch.cuda.synchronize()
import bench  # noqa: E402  (NVML clock sampler)
ts = []
cs = bench.ClockSampler(0).__enter__()
for k in range(a.reps):
    flush.fill_(k & 255)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    ctx.reconstruct(Qd, out, stream=st)
    e1.record(st)
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
cs.__exit__()
clk = cs.summary()
ms = float(np.median(ts))
gbs = inf["algorithmic_bytes_per_cell"] * inf["n_owned"] / (ms * 1e-3) / 1e9
res = {"n": a.n, "cells": inf["n_owned"], "family": inf["kernel_family"], "T": inf["tile_cells"],
       "union_max": inf["union_max"], "ms": ms, "ms_min": float(np.min(ts)), "gbs": gbs, "frac": gbs / 6533.5,
       "setup_s": round(setup, 1), "sm_mhz": clk["sm_mhz"], "reasons": clk["reasons"]}
if a.kernel == "matrixfree":
    fl = bench.matfree_flops_per_cell(a.d, a.M, a.V)
    res["tflops"] = fl * inf["n_owned"] / (ms * 1e-3) / 1e12
    res["frac_fp64"] = res["tflops"] / bench.FP64_PEAK_TF
if a.check and a.kernel != "matrixfree":
    ref = out.clone()
    ctx.set_kernel("simple")
    ctx.reconstruct(Qd, out, stream=st)
    torch.cuda.synchronize()
    res["bitwise_vs_simple"] = bool(torch.equal(out, ref))
    res["maxdiff"] = float((out - ref).abs().max())
print(json.dumps(res), flush=True)
if a.trace:
    import ctypes
    buf = (ctypes.c_longlong * (64 * 16))()
    P.lib.cwreco_debug_rb_trace.argtypes = [ctypes.c_void_p]
    P.lib.cwreco_debug_rb_trace(buf)
    tr = np.array(buf[:], dtype=np.int64).reshape(64, 16)
    base = tr[0, 9]
    names = ["mw_start", "mw_q_ready", "mw_main_done", "mw_ofree", "ew_ofull", "ew_sfull", "ew_items_done",
             "ew_gather_issued", "ew_stored", "pr_start", "pr_chunks_issued", "pr_union", "pr_sector"]
    print("tile " + " ".join(f"{n:>16}" for n in names))
    for k in range(2, 40):
        print(f"{k:4d} " + " ".join(f"{(tr[k, j] - base) / 1.965e3:16.2f}" for j in range(len(names))))

#!/usr/bin/env python
"""Throughput of the space-time predictor (cwreco_predict, NEXT-2) on a BASELINE
Euler workload: the config's mesh and initial data, the GPU reconstruction as
input, CFL-sized Δt.  fp64-ALU roofline: algorithmic flops per cell (below) ÷ the
CUDA-event time, against the derived B200 fp64 peak (bench.FP64_PEAK_TF).

    python tools/predictor_bench.py [--config C5] [--reps 10]

flops per cell = 2·L·ℳ·V + 2·NU·ℳ·V (initial guess, C0 q̂⁰) + iters × (2·d·NU·L·V
(update) + L·(2·d²·V + 4·d·V + 12) (flux, contravariant flux))."""
import argparse
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import gen  # noqa: E402
import paper_1612_09335_b200 as P  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C5", choices=["C1", "C2", "C3", "C5"])
ap.add_argument("--n", type=int, default=0)
ap.add_argument("--reps", type=int, default=10)
a = ap.parse_args()
w = gen.make(a.config, a.n) if a.n else gen.make(a.config)
d, M, V = w["d"], w["M"], w["V"]
t = time.time()
ctx = P.setup_context(w["nodes"], w["cells"], w["period"], M, V, device=0)
ctx.predictor_setup(1.4)
setup = time.time() - t
perm = ctx.permutation()
A = torch.tensor(w["avgs"][perm], device="cuda")
coeffs = ctx.reconstruct(A)
n_owned = ctx.info()["n_owned"]
nodes, nk = ctx.predictor_nodes()
L, NU = nodes.shape[0], nodes.shape[0] - nk
h = 1.0 / w["n"]
qv = A.cpu().numpy()
rho = qv[:, 0]
u = qv[:, 1:1 + d] / rho[:, None]
p = 0.4 * (qv[:, d + 1] - 0.5 * rho * (u * u).sum(1))
smax = float((np.sqrt((u * u).sum(1)) + np.sqrt(1.4 * p / rho)).max())
dt = 0.3 * h / smax / d                      # CFL 0.3/d (Eq. timestep, CFL ≤ 1/d)
iters = torch.empty(n_owned, dtype=torch.int32, device="cuda")
out = torch.empty((n_owned, L, V), dtype=torch.float64, device="cuda")
st = torch.cuda.current_stream()
for _ in range(2):
    ctx.predict(coeffs, dt, out, iters, stream=st)
torch.cuda.synchronize()
ts = []
for _ in range(a.reps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    ctx.predict(coeffs, dt, out, iters, stream=st)
    e1.record(st)
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
ms = float(np.median(ts))
it = iters.cpu().numpy()
mean_it = float(np.abs(it).mean())
flops = 2 * L * nk * V + 2 * NU * nk * V + mean_it * (2 * d * NU * L * V + L * (2 * d * d * V + 4 * d * V + 12))
tf = flops * n_owned / (ms * 1e-3) / 1e12
print(json.dumps({"config": a.config, "cells": n_owned, "d": d, "M": M, "V": V, "L": L, "dt": dt,
                  "ms": ms, "cells_per_s": n_owned / (ms * 1e-3), "mean_iters": mean_it,
                  "not_converged": int((it < 0).sum()), "flops_per_cell": flops, "tflops": tf,
                  "frac_fp64_peak": tf / bench.FP64_PEAK_TF, "peak_source": bench.FP64_PEAK_SRC,
                  "setup_s": round(setup, 1)}))

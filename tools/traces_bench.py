#!/usr/bin/env python
"""Throughput of cwreco_face_traces (NEXT-3, K4) on a BASELINE workload: CUDA events
on the stream, L2 flushed between passes, algorithmic bytes = the coefficients read
(ℳ·V doubles per cell) + the traces written ((d+1)·nq·V doubles per cell).

    python tools/traces_bench.py C2 [C5 ...]   -> one JSON line per config
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import gen
import paper_1612_09335_b200 as P

peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                   "MEASURED_PEAKS.json")))["hbm_gbs"]
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
for cfg in sys.argv[1:]:
    w = gen.make(cfg)
    ctx = P.setup_context(w["nodes"], w["cells"], w["period"], w["M"], w["V"], device=0)
    A = torch.tensor(w["avgs"][ctx.permutation()], device="cuda")
    coeffs = ctx.reconstruct(A)
    tr = ctx.face_traces(coeffs)
    torch.cuda.synchronize()
    n, d, V, nm = coeffs.shape[0], w["d"], w["V"], ctx.nm
    nq = tr.shape[2]
    ts = []
    for k in range(20):
        flush.fill_(k & 0xFF)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        ctx.face_traces(coeffs, tr)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ts.sort()
    ms = ts[len(ts) // 2]
    bpc = 8 * (nm * V + (d + 1) * nq * V)
    gbs = bpc * n / ms / 1e6
    print(json.dumps({"config": cfg, "kernel": "cwr::k_traces", "cells": n, "ms": ms, "cells_per_s": n / ms * 1e3,
                      "bytes_per_cell": bpc, "GBps": gbs, "frac_of_measured_peak": gbs / peak,
                      "points_per_face": nq}), flush=True)
    del ctx, A, coeffs, tr
    torch.cuda.empty_cache()

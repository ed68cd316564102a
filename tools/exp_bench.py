#!/usr/bin/env python
"""Bottleneck experiments on the pipelined kernel (results are WRONG with flags != 0;
timing only).  CWRECO_EXP_FLAGS: 1 = no Q gather, 2 = no B⁺ FMAs, 16 = no epilogue.

    python tools/exp_bench.py C2 [C3 ...]
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import gen
import paper_1612_09335_b200 as P


def time_pass(ctx, A, out, flush, n=20):
    for _ in range(3):
        ctx.reconstruct(A, out)
    torch.cuda.synchronize()
    ts = []
    for _ in range(n):
        flush.fill_(1)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        ctx.reconstruct(A, out)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ts.sort()
    return ts[len(ts) // 2]


def main():
    for cfg in sys.argv[1:]:
        w = gen.make(cfg)
        t = time.time()
        ctx = P.setup_context(w["nodes"], w["cells"], w["period"], w["M"], w["V"], device=0)
        inf = ctx.info()
        A = torch.tensor(w["avgs"][ctx.permutation()], device="cuda")
        out = torch.empty((inf["n_owned"], w["V"], ctx.nm), dtype=torch.float64, device="cuda")
        flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
        res = {}
        for flags in [int(f) for f in os.environ.get("EXP_FLAGS_LIST", "0,1,2,16,19").split(",")]:
            os.environ["CWRECO_EXP_FLAGS"] = str(flags)
            ms = time_pass(ctx, A, out, flush)
            res[flags] = ms
        os.environ["CWRECO_EXP_FLAGS"] = "0"
        ctx.set_kernel("simple")
        res["simple"] = time_pass(ctx, A, out, flush)
        ctx.set_kernel("pipelined")
        B = inf["algorithmic_bytes_per_cell"] * inf["n_owned"]
        print(json.dumps({"config": cfg, "info": {k: inf[k] for k in ("tile_cells", "chunk_k", "tile_bytes", "n_tiles")},
                          "ms": res, "GBps_alg": {k: B / v / 1e6 for k, v in res.items()}}), flush=True)
        del ctx, A, out
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()

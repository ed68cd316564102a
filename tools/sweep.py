#!/usr/bin/env python
"""Tuning sweep of the pipelined kernel: chunk size KC (layout, needs a new
precompute) x stage cap (shared memory given to the stage ring vs L1).

    python tools/sweep.py C3 4,8 4,6,8,16
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import gen
import paper_1612_09335_b200 as P
from exp_bench import time_pass  # noqa: E402

cfg, kcs, caps = sys.argv[1], sys.argv[2].split(","), sys.argv[3].split(",")
w = gen.make(cfg)
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
for kc in kcs:
    os.environ["CWRECO_KC"] = kc
    ctx = P.setup_context(w["nodes"], w["cells"], w["period"], w["M"], w["V"], device=0)
    inf = ctx.info()
    A = torch.tensor(w["avgs"][ctx.permutation()], device="cuda")
    out = torch.empty((inf["n_owned"], w["V"], ctx.nm), dtype=torch.float64, device="cuda")
    B = inf["algorithmic_bytes_per_cell"] * inf["n_owned"]
    for cap in caps:
        os.environ["CWRECO_MAX_STAGES"] = cap
        ms = time_pass(ctx, A, out, flush)
        print(json.dumps({"config": cfg, "KC": inf["chunk_k"], "max_stages": int(cap), "ms": ms,
                          "GBps_alg": B / ms / 1e6}), flush=True)
    del ctx, A, out
    torch.cuda.empty_cache()
os.environ.pop("CWRECO_KC", None)
os.environ.pop("CWRECO_MAX_STAGES", None)

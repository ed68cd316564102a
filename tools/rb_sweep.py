#!/usr/bin/env python
"""A/B sweep: kernel family (CWRECO_FAMILY 0 = cell-variable, 1 = row-block) x stage
cap (CWRECO_MAX_STAGES) x CTAs/SM cap (CWRECO_CTAS), ms per pass (L2 flushed).

    python tools/rb_sweep.py C5 [C4 ...]      (env: STAGES=8,12,16,32 CTAS=1,2)
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import gen
import paper_1612_09335_b200 as P
from exp_bench import time_pass  # noqa: E402

stages = os.environ.get("STAGES", "8,12,16,32").split(",")
ctas = os.environ.get("CTAS", "2").split(",")
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
for cfg in sys.argv[1:]:
    w = gen.make(cfg)
    for fam in os.environ.get("FAMILIES", "1,0").split(","):
        os.environ["CWRECO_FAMILY"] = fam
        ctx = P.setup_context(w["nodes"], w["cells"], w["period"], w["M"], w["V"], device=0)
        inf = ctx.info()
        A = torch.tensor(w["avgs"][ctx.permutation()], device="cuda")
        out = torch.empty((inf["n_owned"], w["V"], ctx.nm), dtype=torch.float64, device="cuda")
        B = inf["algorithmic_bytes_per_cell"] * inf["n_owned"]
        for st in (stages if fam == "1" else ["8"]):
            for k in (ctas if fam == "1" else ["2"]):
                os.environ["CWRECO_MAX_STAGES"] = st
                os.environ["CWRECO_CTAS"] = k
                ms = time_pass(ctx, A, out, flush)
                print(json.dumps({"config": cfg, "family": int(fam), "T": inf["tile_cells"], "max_stages": int(st),
                                  "ctas_cap": int(k), "ms": round(ms, 4), "frac": round(B / ms / 1e6 / 6533.5, 3)}),
                      flush=True)
        os.environ.pop("CWRECO_MAX_STAGES")
        os.environ.pop("CWRECO_CTAS")
        del ctx, A, out
        torch.cuda.empty_cache()

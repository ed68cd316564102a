"""Multi-GPU projection measured on ONE GPU (tools only; no rank waits on another).

For a BASELINE config and a rank count P, every rank's partition (SFC range + its
stencil-closure ghosts) is set up in turn with no transport
(cwreco_set_partition(r, P, NULL)), its ghost rows are filled with the global
averages (what the exchange would deliver), and its pass is timed alone on the GPU
with CUDA events (L2 flushed between passes): PART_ALL, PART_INTERIOR and
PART_BOUNDARY.  Reported per rank: owned / ghost / interior cells, the three times,
and the bytes the halo exchange moves (ghost rows in, send rows out).

Projection (printed as such, NOT a multi-GPU measurement): a P-GPU step costs
max_r max(t_all_r, t_int_r + t_xchg_r + t_bnd_r) with t_xchg_r = (bytes in + out) /
link bandwidth (--link-gbs, default 900 GB/s: NVLink 5 per direction); strong
efficiency = t_1 / (P · that).  The single-rank time t_1 is measured in the same run
(--t1 skips it).

    python tools/rank_projection.py --config C4 --nranks 2 4 8 [--ranks 0 7]
    python tools/rank_projection.py --config C5 --weak --nranks 2 4 8 --ranks 0

--weak: the mesh grows with P as bench.py's weak ladder does (bench.workload_n: C5
n = 100/126/159/200, ≈ 6 M cells per rank); efficiency = t_1 / that step.
"""
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


def time_parts(ctx, A, out, reps, parts):
    stream = torch.cuda.current_stream()
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    res = {}
    for name, part in parts:
        for _ in range(2):
            ctx.reconstruct(A, out, part=part, stream=stream)
        ts = []
        for _ in range(reps):
            flush.fill_(1)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            ctx.reconstruct(A, out, part=part, stream=stream)
            e1.record(stream)
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        res[name] = float(np.median(ts))
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C4")
    ap.add_argument("--nranks", type=int, nargs="+", default=[2, 4, 8])
    ap.add_argument("--ranks", type=int, nargs="*", default=None, help="subset of ranks (default all)")
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--link-gbs", type=float, default=900.0)
    ap.add_argument("--t1", type=float, default=None, help="single-rank ms (skip measuring it)")
    ap.add_argument("--weak", action="store_true", help="weak ladder: the mesh grows with P (bench.workload_n)")
    args = ap.parse_args()
    import bench
    w = gen.make(args.config)
    d, M, V = w["d"], w["M"], w["V"]
    perm = None
    report = {"config": args.config, "n_cells": int(w["cells"].shape[0]), "link_gbs": args.link_gbs,
              "scaling": "weak" if args.weak else "strong",
              "library": P.lib.cwreco_version().decode(), "ranks": {}}
    all_parts = [("all", P.PART_ALL), ("interior", P.PART_INTERIOR), ("boundary", P.PART_BOUNDARY)]
    if args.t1 is None:
        t0 = time.time()
        ctx = P.setup_context(w["nodes"], w["cells"], w["period"], M, V, device=0)
        perm = ctx.permutation()
        A = torch.tensor(np.ascontiguousarray(w["avgs"][perm]), device="cuda")
        out = torch.empty((A.shape[0], V, ctx.nm), dtype=torch.float64, device="cuda")
        t1 = time_parts(ctx, A, out, args.reps, all_parts[:1])["all"]
        print(f"P=1: {t1:.3f} ms (setup {time.time() - t0:.0f} s)", file=sys.stderr, flush=True)
        del A, out
        ctx.close()
        torch.cuda.empty_cache()
    else:
        t1 = args.t1
    report["t1_ms"] = t1
    for Pn in args.nranks:
        ranks = args.ranks if args.ranks else list(range(Pn))
        rows = {}
        if args.weak:
            del w
            w = gen.make(args.config, bench.workload_n(args.config, Pn))
            perm = None
        for r in ranks:
            t0 = time.time()
            ctx = P.setup_context(w["nodes"], w["cells"], w["period"], M, V, device=0, rank=r, nranks=Pn)
            if perm is None:
                perm = ctx.permutation()
            inf = ctx.info()
            loc = ctx.local_cells()
            A = torch.tensor(np.ascontiguousarray(w["avgs"][perm[loc]]), device="cuda")
            out = torch.empty((inf["n_owned"], V, ctx.nm), dtype=torch.float64, device="cuda")
            tm = time_parts(ctx, A, out, args.reps, all_parts)
            rc, _ = ctx.halo_plan()
            rows[r] = dict(n_owned=int(inf["n_owned"]), n_ghost=int(inf["n_ghost"]),
                           n_interior=int(inf["n_interior"]), n_tiles=int(inf["n_tiles"]),
                           n_interior_tiles=int(inf["n_interior_tiles"]),
                           recv_rows=[int(x) for x in rc], **{f"t_{k}_ms": v for k, v in tm.items()})
            print(f"P={Pn} r={r}: {rows[r]} (setup {time.time() - t0:.0f} s)", file=sys.stderr, flush=True)
            del A, out
            ctx.close()
            torch.cuda.empty_cache()
        # send rows of r = what every other rank receives from r (known when all ranks ran)
        full = len(rows) == Pn
        worst = 0.0
        for r, row in rows.items():
            recv_b = row["n_ghost"] * V * 8
            send_b = sum(rows[q]["recv_rows"][r] for q in rows if q != r) * V * 8 if full else recv_b
            t_x = (recv_b + send_b) / (args.link_gbs * 1e9) * 1e3
            row["halo_bytes_in"], row["halo_bytes_out"], row["t_exchange_est_ms"] = recv_b, send_b, t_x
            row["t_overlapped_est_ms"] = max(row["t_all_ms"], row["t_interior_ms"] + t_x + row["t_boundary_ms"])
            worst = max(worst, row["t_overlapped_est_ms"])
        eff = (t1 if args.weak else t1 / Pn) / worst if worst > 0 else None
        report["ranks"][str(Pn)] = dict(per_rank=rows, step_est_ms=worst, n_cells=int(w["cells"].shape[0]),
                                        **{("weak" if args.weak else "strong") + "_eff_est": eff},
                                        all_ranks_measured=full)
        print(f"P={Pn}: projected step {worst:.3f} ms, {'weak' if args.weak else 'strong'} efficiency {eff:.3f}",
              file=sys.stderr, flush=True)
    print(json.dumps(report))


if __name__ == "__main__":
    main()

#!/usr/bin/env python
"""Small end-to-end run of every kernel for compute-sanitizer (memcheck /
racecheck / synccheck / initcheck), e.g.

    compute-sanitizer --tool racecheck python tools/sanitize_case.py

2D M=3 (periodic, jittered) and 3D M=2 / M=3 (open: invalid sectors, extras),
pipelined + simple + debug tap, dense and strided outputs, halo pack."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import gen
import paper_1612_09335_b200 as P

for (d, n, M, per, jit, V) in [(2, 10, 3, True, 0.2, 4), (3, 4, 2, False, 0.1, 5), (3, 4, 3, True, 0.1, 3)]:
    nodes, cells, period = gen.box_mesh(d, n, per, jit, 7)
    Q = np.random.default_rng(0).standard_normal((cells.shape[0], V))
    ctx = P.setup_context(nodes, cells, period, M, V, device=0)
    Qd = torch.tensor(Q[ctx.permutation()], device="cuda")
    ref = ctx.reconstruct(Qd)
    ctx.set_kernel("simple")
    b = ctx.reconstruct(Qd)
    ctx.set_kernel("pipelined")
    wide = torch.zeros((Q.shape[0], V + 1), dtype=torch.float64, device="cuda")
    wide[:, 1:] = Qd
    c = ctx.reconstruct(wide[:, 1:])
    dbg = ctx.reconstruct_debug(Qd, np.arange(0, Q.shape[0], 5))
    torch.cuda.synchronize()
    assert torch.equal(ref, b) and torch.equal(ref, c)
    print(f"d={d} M={M}: ok", flush=True)
# halo pack on a 2-rank partition (rank 0's context)
nodes, cells, period = gen.box_mesh(2, 12, True, 0.1, 3)
c0 = P.Context(2, 2, 3, device=0)
c0.set_mesh(nodes, cells, period)
c0.set_partition(0, 2)
c0.build_stencils()
c0.precompute()
cnt, ids = c0.halo_plan()
c0.set_send_lists(np.array([0, len(ids)]), np.sort(np.random.default_rng(1).choice(
    c0.local_cells()[: c0.info()["n_owned"]], len(ids), replace=False)))
A = torch.randn((c0.info()["n_owned"] + c0.info()["n_ghost"], 3), dtype=torch.float64, device="cuda")
buf = torch.empty((c0.send_total(), 3), dtype=torch.float64, device="cuda")
c0.halo_pack(A, buf)
out = torch.empty((c0.info()["n_owned"], 3, c0.nm), dtype=torch.float64, device="cuda")
c0.reconstruct(A, out, part=P.PART_INTERIOR)
c0.reconstruct(A, out, part=P.PART_BOUNDARY)
torch.cuda.synchronize()
print("sanitize case done")

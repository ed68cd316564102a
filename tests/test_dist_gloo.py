"""N>1 host path on CPU: world_size 2 over gloo.

Each rank owns a contiguous Morton range, exchanges its ghost requests with
paper_1612_09335_b200.dist.exchange_plan, installs the send lists in the
library, and moves the ghost averages with dist.exchange (all-to-all-v into
avgs[n_owned:]).  Checks: the ghost rows equal the global averages bit for
bit, and every owned cell's reconstruction (oracle, on a copy of the data in
which only the rank's local rows are defined, the rest NaN) equals the global
one — i.e. the exchange delivers everything the stencils need.  The pack is
done here with a numpy gather (the library's pack is a CUDA kernel, covered by
the GPU tests)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        import gen
        import paper_1612_09335_b200 as P
        from oracle import reconstruct as R
        from oracle.mesh import OracleMesh
        from paper_1612_09335_b200 import dist as pdist

        d, n, M, V = 2, 14, 2, 3
        nodes, cells, period = gen.box_mesh(d, n, True, 0.2, 11)
        Qin = np.random.default_rng(5).standard_normal((cells.shape[0], V))
        ctx = P.Context(d, M, V, device=None)
        ctx.set_mesh(nodes, cells, period)
        ctx.set_partition(rank, world)
        ctx.build_stencils()
        send_counts, recv_counts = pdist.setup_halo(ctx)
        perm = ctx.permutation()
        Qg = Qin[perm]                                   # global, SFC order
        loc = ctx.local_cells()
        inf = ctx.info()
        n_owned = inf["n_owned"]
        A = np.full((len(loc), V), np.nan)
        A[:n_owned] = Qg[loc[:n_owned]]
        # pack: the owned rows each peer asked for (what cwreco_halo_pack does on the GPU)
        _, recv_ids = ctx.halo_plan()
        send_ids = pdist.exchange_plan(*ctx.halo_plan())[1]
        g2l = {int(g): i for i, g in enumerate(loc)}
        sendbuf = torch.tensor(A[[g2l[int(g)] for g in send_ids]].reshape(-1, V))
        At = torch.tensor(A)
        pdist.exchange(At, sendbuf, send_counts, recv_counts, n_owned, V)
        A = At.numpy()
        ok_ghost = bool(np.array_equal(A[n_owned:], Qg[loc[n_owned:]]))
        # reconstruction of owned cells from local data only == global reconstruction
        m = OracleMesh(nodes, cells, period, M)
        Qloc = np.full_like(Qg, np.nan)
        Qloc[loc] = A
        rng = np.random.default_rng(rank)
        owned = loc[:n_owned]
        picks = list(owned[inf["n_interior"]:][:6]) + list(rng.choice(owned, 4, replace=False))
        max_diff = 0.0
        for g in picks:
            a = R.reconstruct_cell(m, int(g), Qloc, M)["w"]
            b = R.reconstruct_cell(m, int(g), Qg, M)["w"]
            max_diff = max(max_diff, float(np.nan_to_num(np.abs(a - b), nan=np.inf).max()))
        # second exchange: polynomials of the ghost cells, rows of V·ℳ
        # doubles over the same send lists; owned rows from the oracle (the library
        # has no CPU compute path), ghost rows must arrive equal to their owners'
        nm = R.n_modes(M, d)
        W = np.full((len(loc), V, nm), np.nan)
        need = set(int(g) for g in send_ids)
        for li in range(n_owned):
            if int(loc[li]) in need:
                W[li] = R.reconstruct_cell(m, int(loc[li]), Qg, M)["w"]
        Wt = torch.tensor(W.reshape(len(loc), V * nm))
        sendw = torch.tensor(W.reshape(len(loc), V * nm)[[g2l[int(g)] for g in send_ids]])
        pdist.exchange(Wt, sendw, send_counts, recv_counts, n_owned, V * nm)
        Wg = Wt.numpy().reshape(len(loc), V, nm)[n_owned:]
        ok_poly = True
        for k, g in enumerate(loc[n_owned:][:12]):
            ok_poly &= bool(np.array_equal(Wg[k], R.reconstruct_cell(m, int(g), Qg, M)["w"]))
        q.put((rank, ok_ghost and ok_poly, max_diff, int(inf["n_ghost"]), int(inf["n_owned"] - inf["n_interior"])))
        dist.destroy_process_group()
    except Exception as e:  # pragma: no cover - reported to the parent
        q.put((rank, repr(e)))


def test_two_rank_halo_exchange_gloo():
    ctxm = mp.get_context("fork")
    q = ctxm.Queue()
    port = _free_port()
    procs = [ctxm.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    for r in res:
        assert len(r) == 5, r
        rank, ok_ghost, max_diff, n_ghost, n_bnd = r
        assert ok_ghost and n_ghost > 0 and n_bnd > 0
        assert max_diff == 0.0

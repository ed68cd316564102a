"""Multi-rank plumbing: halo plan exchange and the ghost-average exchange.

The mesh is partitioned into contiguous Morton ranges (cwreco_set_partition);
each rank reconstructs only its owned cells and needs the averages of the ghost
cells its stencils reach (the paper's "exchange of cell averages before the
reconstruction").  This module moves bytes with torch.distributed
(NCCL on GPUs, gloo in the CPU tests); every index computation is in the
library (cwreco_halo_plan / cwreco_set_send_lists) and the pack is the
library's CUDA kernel (cwreco_halo_pack).

Ghost rows of the local average array are ordered by (owner rank, SFC id), so
the receive side of the all-to-all-v lands directly in avgs[n_owned:]; no
unpack step exists.
"""
from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist


def exchange_plan(recv_counts, recv_ids, group=None, device="cpu"):
    """All-to-all the ghost requests.  recv_counts[r] / recv_ids: what this rank
    needs from each rank r (cwreco_halo_plan).  Returns (send_counts, send_ids):
    what each peer needs from this rank (input of cwreco_set_send_lists)."""
    world = dist.get_world_size(group)
    rc = torch.as_tensor(np.asarray(recv_counts, dtype=np.int64), device=device)
    sc = torch.empty(world, dtype=torch.int64, device=device)
    dist.all_to_all_single(sc, rc, group=group)
    send_counts = sc.cpu().numpy()
    rid = torch.as_tensor(np.asarray(recv_ids, dtype=np.int64), device=device)
    sid = torch.empty(int(send_counts.sum()), dtype=torch.int64, device=device)
    dist.all_to_all_single(sid, rid, output_split_sizes=send_counts.tolist(),
                           input_split_sizes=np.asarray(recv_counts).tolist(), group=group)
    return send_counts, sid.cpu().numpy()


def setup_halo(ctx, group=None, device="cpu"):
    """Install the send lists on a context after cwreco_build_stencils."""
    recv_counts, recv_ids = ctx.halo_plan()
    send_counts, send_ids = exchange_plan(recv_counts, recv_ids, group, device)
    ctx.set_send_lists(send_counts, send_ids)
    ctx.recv_counts = np.asarray(recv_counts)
    return send_counts, recv_counts


def exchange(avgs, sendbuf, send_counts, recv_counts, n_owned, V, group=None):
    """Move the packed owned rows (sendbuf [Σ send, V]) into the ghost rows
    avgs[n_owned:] of every peer (avgs must be row-contiguous [n_local, V])."""
    out = avgs[n_owned:]
    dist.all_to_all_single(out.view(-1), sendbuf.view(-1),
                           output_split_sizes=[int(c) * V for c in recv_counts],
                           input_split_sizes=[int(c) * V for c in send_counts], group=group)


def exchange_polynomials(ctx, coeffs_local, send_counts, recv_counts, group=None, sendbuf=None):
    """The second communication step: after the pass, the
    reconstruction polynomials of the ghost cells.  coeffs_local: [n_local, V, ℳ]
    (owned rows written by cwreco_reconstruct, ghost rows filled here); the pack is
    the library's cwreco_halo_pack_rows with width V·ℳ, the transfer the same
    all-to-all-v as the averages."""
    n_local = coeffs_local.shape[0]
    W = coeffs_local.shape[1] * coeffs_local.shape[2]
    rows = coeffs_local.view(n_local, W)
    n_send = int(np.sum(send_counts))
    if sendbuf is None:
        sendbuf = torch.empty((max(1, n_send), W), dtype=torch.float64, device=coeffs_local.device)
    ctx.halo_pack_rows(rows, sendbuf)
    n_owned = n_local - int(np.sum(recv_counts))
    exchange(rows, sendbuf[:n_send], send_counts, recv_counts, n_owned, W, group)
    return coeffs_local


class HaloStepper:
    """One overlapped reconstruction pass on a GPU rank:
    comm stream: cwreco_halo_pack → NCCL all-to-all-v into the ghost rows;
    compute stream: interior tiles (need no ghosts) concurrently, then the
    boundary tiles after the exchange event."""

    def __init__(self, ctx, avgs, out, send_counts, recv_counts, group=None):
        self.ctx, self.avgs, self.out = ctx, avgs, out
        self.send_counts, self.recv_counts = send_counts, recv_counts
        self.group = group
        inf = ctx.info()
        self.n_owned, self.V = inf["n_owned"], ctx.V
        self.n_send = ctx.send_total()
        self.sendbuf = torch.empty((max(1, self.n_send), ctx.V), dtype=torch.float64, device=avgs.device)
        self.comm = torch.cuda.Stream(device=avgs.device)
        self.ready = torch.cuda.Event()

    def step(self):
        from . import PART_BOUNDARY, PART_INTERIOR
        comp = torch.cuda.current_stream()
        self.comm.wait_stream(comp)
        with torch.cuda.stream(self.comm):
            self.ctx.halo_pack(self.avgs, self.sendbuf, stream=self.comm)
            exchange(self.avgs, self.sendbuf[: self.n_send], self.send_counts, self.recv_counts, self.n_owned, self.V, self.group)
            self.ready.record(self.comm)
        self.ctx.reconstruct(self.avgs, self.out, part=PART_INTERIOR, stream=comp)
        comp.wait_event(self.ready)
        self.ctx.reconstruct(self.avgs, self.out, part=PART_BOUNDARY, stream=comp)

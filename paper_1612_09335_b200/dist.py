"""Multi-rank plumbing around libcwreco's own transport.

The mesh is partitioned into contiguous Morton ranges (cwreco_set_partition);
each rank reconstructs only its owned cells and needs the averages of the ghost
cells its stencils reach (the paper's "exchange of cell averages before the
reconstruction").  The exchange itself lives in the library
(cwreco_halo_exchange / cwreco_reconstruct_overlap: pack kernel → NCCL
send/recv per peer on the library's comm stream → ghost rows); this module only
bootstraps it: rank 0 makes the NCCL unique id and torch.distributed
broadcasts the 128 bytes.

For callers that move the bytes themselves (no transport id), exchange_plan /
setup_halo / exchange implement the same plan and all-to-all-v with
torch.distributed (used by the CPU gloo tests).
"""
from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist


def init_transport(ctx, group=None):
    """cwreco_set_partition(rank, world, NCCL id) on every rank of the process group:
    rank 0 creates the id, the group broadcasts it (collective)."""
    from . import nccl_unique_id
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    obj = [nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0, group=group)
    ctx.set_partition(rank, world, obj[0])
    return obj[0]


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
    """Install the send lists on a context without a transport (after the stencils)."""
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

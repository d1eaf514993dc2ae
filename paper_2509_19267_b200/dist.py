"""Row sharding helpers for the multi-GPU path (host-side plumbing only).

The method's arithmetic runs in librgdbek.so; this module decides which rows
each rank owns and bootstraps the NCCL communicator the library uses.

Partition (reading R16): A is split row-wise into contiguous blocks
"until the number of non-zero entries is almost equally divided" — a greedy
prefix on the CSR row pointer (equal rows for dense A).
"""
import numpy as np

from . import _native as N


def partition_rows(row_ptr_or_m, nparts):
    """Contiguous row ranges [(b0, e0), ...] with nnz as equal as possible.

    `row_ptr_or_m` is a CSR row pointer (length m+1) or an int m (dense rows).
    Boundary p is the first row whose nnz prefix reaches p * nnz / nparts.
    Every part is non-empty when m >= nparts.
    """
    if isinstance(row_ptr_or_m, (int, np.integer)):
        m = int(row_ptr_or_m)
        rp = np.arange(m + 1, dtype=np.int64)
    else:
        rp = np.asarray(row_ptr_or_m, dtype=np.int64)
        m = len(rp) - 1
    if nparts < 1 or m < nparts:
        raise ValueError(f"cannot split {m} rows into {nparts} non-empty parts")
    nnz = int(rp[-1])
    bounds = [0]
    for p in range(1, nparts):
        target = p * nnz / nparts
        b = int(np.searchsorted(rp, target, side="left"))
        b = min(max(b, bounds[-1] + 1), m - (nparts - p))   # keep every part non-empty
        bounds.append(b)
    bounds.append(m)
    return [(bounds[i], bounds[i + 1]) for i in range(nparts)]


def shard_csr(row_ptr, col_idx, val, begin, end):
    """Local CSR of rows [begin, end): rebased row pointer, global column ids."""
    rp = np.asarray(row_ptr, dtype=np.int64)
    p0, p1 = int(rp[begin]), int(rp[end])
    return (rp[begin:end + 1] - p0, np.asarray(col_idx[p0:p1], dtype=np.int32),
            np.asarray(val[p0:p1], dtype=np.float64))


def init_nccl_comm(device, group=None):
    """NCCL communicator for librgdbek over the torch.distributed group.

    Rank 0 draws the unique id (rgdbek_nccl_unique_id); torch.distributed
    broadcasts it; every rank calls rgdbek_nccl_comm_init.
    """
    import torch.distributed as dist
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    obj = [N.rgdbek_nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0, group=group)
    return N.rgdbek_nccl_comm_init(world, rank, obj[0], device)


def destroy_nccl_comm(comm):
    N.rgdbek_nccl_comm_destroy(comm)


def connect_peers(solver, group=None):
    """Join this process's peer-sharded rank (a Solver created with row_range and no
    nccl_comm) to the other ranks of the torch.distributed group: every rank exports its
    exchange block (CUDA IPC handle) and window, the group allgathers them, and every rank
    maps its peers (rgdbek_peer_connect).  Afterwards solver.step / solver.solve are
    collectives over the group (one persistent kernel per GPU, peer-memory exchanges)."""
    import torch.distributed as dist
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    mine = (N.rgdbek_peer_export(solver._h), tuple(solver.peer_window()[:2]))
    allv = [None] * world
    dist.all_gather_object(allv, mine, group=group)
    N.rgdbek_peer_connect(solver._h, world, rank, [a[0] for a in allv], [a[1] for a in allv])
    dist.barrier(group=group)

"""The real multi-GPU plumbing of the peer-sharded engine (CUDA IPC), on one GPU without
running the cross-waiting kernel (B200_PROFILING.md: ranks that wait on one another must
not be separate launches on one GPU): two processes create their ranks, export their
exchange arenas, allgather handles and windows over gloo and map each other
(rgdbek_peer_connect, dist.connect_peers).  Checked: the connect succeeds and the peer
mappings are right — get_x gathers every rank's OWNED columns through the IPC pointers
(each rank wrote x = its rank + 1 everywhere)."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rank(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2509_19267_b200 import Solver, _native as N
        from paper_2509_19267_b200.dist import connect_peers, partition_rows, shard_csr
        from workloads import by_name
        w = by_name("C5t")
        m, n = w.shape
        r0, r1 = partition_rows(w.A.indptr, world)[rank]
        rp, ci, val = shard_csr(*w.csr_arrays(), r0, r1)
        s = Solver.from_csr(m, n, rp, ci, val, w.b[r0:r1], eta=w.eta, row_range=(r0, r1))
        s.set_state(np.full(n, rank + 1.0), np.zeros(r1 - r0), 0)
        dist.barrier()
        connect_peers(s)
        wins = [None] * world
        dist.all_gather_object(wins, tuple(s.peer_window()[:2]))
        own = N.rgdbek_plan_ownership(wins, n)
        x = s.x()
        expect = np.concatenate([np.full(own[q + 1] - own[q], q + 1.0) for q in range(world)])
        out[rank] = (bool(np.array_equal(x, expect)), own, wins)
        dist.barrier()
        s.close()
    finally:
        dist.destroy_process_group()


def test_two_process_ipc_connect_and_owned_gather():
    from paper_2509_19267_b200 import _build
    _build.build()
    ctx = mp.get_context("spawn")
    mgr = ctx.Manager()
    out = mgr.dict()
    port = _port()
    ps = [ctx.Process(target=_rank, args=(r, 2, port, out)) for r in range(2)]
    for p in ps:
        p.start()
    for p in ps:
        p.join(300)
        assert p.exitcode == 0
    for r in range(2):
        ok, own, wins = out[r]
        assert ok, (r, own, wins)
        assert 0 < own[1] < own[2]

"""Multi-GPU plan, checked on the CPU with torch.distributed (gloo, world_size 2).

The CUDA library shards A by contiguous nnz-balanced row blocks (P:443,
reading R16) and exchanges, per iteration, exactly:
  (1) allreduce [A_p^T z_p | A_p^T xi_p | X_p]      (2n + 1 doubles)
  (2) allreduce [W_p, ||b_p - A_p x||^2]             (2 doubles)
  (3) the global row selection J (histogram allreduces + survivor allgather)
  (4) allreduce [|J_p|, hash(J_p)]                  (2 uint64)
with the column selection U replicated on every rank.  This test runs that
decomposition with gloo collectives (the row selection as an allgather of the
keys, which is what (3) computes exactly) and checks that it reproduces the
single-process oracle's trajectory: same blocks every iteration, same x, and
z equal to the concatenated shards.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2509_19267_b200.dist import partition_rows, shard_csr


def test_partition_rows_balances_nnz():
    rng = np.random.default_rng(0)
    lens = rng.integers(0, 40, size=1000)
    rp = np.concatenate([[0], np.cumsum(lens)])
    for P in (1, 2, 3, 8):
        parts = partition_rows(rp, P)
        assert parts[0][0] == 0 and parts[-1][1] == 1000
        assert all(b < e for b, e in parts)
        assert all(parts[i][1] == parts[i + 1][0] for i in range(P - 1))
        nnz = [rp[e] - rp[b] for b, e in parts]
        assert max(nnz) - min(nnz) <= 2 * lens.max()
    assert sorted(e - b for b, e in partition_rows(10, 3)) == [3, 3, 4]
    with pytest.raises(ValueError):
        partition_rows(2, 3)


def test_shard_csr_rebases():
    import scipy.sparse as sp
    A = sp.random(50, 20, density=0.2, format="csr", random_state=1)
    rp, ci, val = shard_csr(A.indptr, A.indices, A.data, 10, 30)
    B = sp.csr_matrix((val, ci, rp), shape=(20, 20))
    assert (abs(B - A[10:30]).sum()) == 0


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _sharded_run(rank, world, port, name, iters, seed, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import Oracle, block_hash, sample_keys, scores, select_block
        from workloads import by_name
        w = by_name(name)
        A = w.A
        m, n = A.shape
        parts = partition_rows(m if w.dense else A.indptr, world)
        b0, b1 = parts[rank]
        A_p = A[b0:b1]
        b_p = w.b[b0:b1]
        orc = Oracle(A, w.b, w.eta)                 # reference (every rank runs it)
        # norm caches: rho local; gamma = allreduce of local column sums (create time)
        rho_p = np.asarray((A_p.multiply(A_p)).sum(axis=1)).ravel() if not w.dense \
            else np.einsum("ij,ij->i", A_p, A_p)
        gam = torch.from_numpy(np.asarray((A_p.multiply(A_p)).sum(axis=0)).ravel() if not w.dense
                               else np.einsum("ij,ij->j", A_p, A_p)).clone()
        dist.all_reduce(gam)
        gamma = gam.numpy()
        x = np.zeros(n)
        z_p = b_p.copy()
        xi_p = np.zeros(b1 - b0)
        X_p = 0.0
        ok = True
        for k in range(iters):
            rec = orc.iterate(seed)
            # (1) [s | v | X]
            buf = torch.from_numpy(np.concatenate([A_p.T @ z_p, A_p.T @ xi_p, [X_p]]))
            dist.all_reduce(buf)
            s, v, X = buf[:n].numpy(), buf[n:2 * n].numpy(), float(buf[2 * n])
            if k > 0:
                V = float(v @ v)
                if V > 0:
                    x = x + (X / V) * v
            # replicated column selection (identical on every rank)
            eps = scores(s, gamma)
            kp = min(orc.kc, int(np.count_nonzero(eps > 0)))
            U = select_block(sample_keys(eps, seed, k, 0), kp, eps > 0)
            zeta = np.zeros(n)
            zeta[U] = s[U]
            Z = float(s[U] @ s[U])
            # (2) [W, Y]
            w_p = A_p @ zeta
            ax_p = A_p @ x
            wy = torch.tensor([float(w_p @ w_p), float((b_p - ax_p) @ (b_p - ax_p))],
                              dtype=torch.float64)
            dist.all_reduce(wy)
            W = float(wy[0])
            if kp > 0 and W > 0:
                z_p = z_p - (Z / W) * w_p
            r_p = b_p - z_p - ax_p
            eps_r = scores(r_p, rho_p)
            # (3) global row selection over GLOBAL indices (keys of all ranks)
            u_keys = np.full(b1 - b0, np.inf)
            from oracle.philox import uniforms
            uu = uniforms(np.arange(b0, b1), k, 1, seed)
            pos = eps_r > 0
            u_keys[pos] = -np.log(uu[pos]) / eps_r[pos]
            gathered = [None] * world
            dist.all_gather_object(gathered, (u_keys, pos))
            keys_all = np.concatenate([g[0] for g in gathered])
            pos_all = np.concatenate([g[1] for g in gathered])
            kpp = min(orc.kr, int(pos_all.sum()))
            J = select_block(keys_all, kpp, pos_all)
            J_p = J[(J >= b0) & (J < b1)] - b0
            xi_p = np.zeros(b1 - b0)
            xi_p[J_p] = r_p[J_p]
            X_p = float(r_p[J_p] @ r_p[J_p])
            # (4) [|J|, hash(J)]
            kpp_sum = torch.tensor([len(J_p)], dtype=torch.int64)
            dist.all_reduce(kpp_sum)
            ok &= (kp, block_hash(U)) == (rec.kp, rec.hash_u)
            ok &= (int(kpp_sum), block_hash(J)) == (rec.kpp, rec.hash_j)
        # final x update of the last iteration, as the library's next pass T does
        buf = torch.from_numpy(np.concatenate([A_p.T @ z_p, A_p.T @ xi_p, [X_p]]))
        dist.all_reduce(buf)
        v, X = buf[n:2 * n].numpy(), float(buf[2 * n])
        V = float(v @ v)
        if V > 0:
            x = x + (X / V) * v
        zs = [None] * world
        dist.all_gather_object(zs, z_p)
        z = np.concatenate(zs)
        out[rank] = (bool(ok), float(np.linalg.norm(x - orc.x) / np.linalg.norm(orc.x)),
                     float(np.linalg.norm(z - orc.z) / np.linalg.norm(w.b)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("name", ["C2si", "C5t"])
def test_world2_sharded_plan_matches_oracle(name):
    ctx = mp.get_context("spawn")
    mgr = ctx.Manager()
    out = mgr.dict()
    port = _free_port()
    procs = [ctx.Process(target=_sharded_run, args=(r, 2, port, name, 15, 3, out)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(300)
        assert p.exitcode == 0
    for r in range(2):
        ok, dx, dz = out[r]
        assert ok, f"rank {r}: blocks differ from the single-process oracle"
        assert dx <= 1e-12 and dz <= 1e-12, (dx, dz)


# ---------------------------------------------------------------------------------------
# The peer-memory sharded engine's decomposition (sharded.cuh), driven by the LIBRARY's
# ownership plan (rgdbek_plan_ownership: a host-only call of librgdbek.so, no device):
# window partials of A^T z / A^T xi, summed by the owner of each column over the ranks
# whose window holds it; keys and the selection of U on owned columns; zeta, x owned and
# copied to the neighbours' halos; rows local.  Gloo collectives stand in for the peer
# reads (all_gather of what a peer would read), and the test counts what crosses ranks.
# ---------------------------------------------------------------------------------------
def _peer_plan_run(rank, world, port, name, iters, seed, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import scipy.sparse as sp
        from oracle import Oracle, block_hash, sample_keys, scores, select_block
        from oracle.philox import uniforms
        from paper_2509_19267_b200 import _native as N
        from workloads import by_name
        w = by_name(name)
        A = w.A if not w.dense else sp.csr_matrix(w.A)
        m, n = A.shape
        parts = partition_rows(m if w.dense else A.indptr, world)
        b0, b1 = parts[rank]
        A_p = A[b0:b1]
        b_p = w.b[b0:b1]
        cols = A_p.indices
        win = (int(cols.min()), int(cols.max()) + 1) if len(cols) else (0, 0)
        if w.dense:
            win = (0, n)
        wins = [None] * world
        dist.all_gather_object(wins, win)
        own = N.rgdbek_plan_ownership(wins, n)          # the library's decomposition
        o0, o1 = own[rank], own[rank + 1]
        orc = Oracle(w.A, w.b, w.eta)
        rho_p = np.asarray(A_p.multiply(A_p).sum(axis=1)).ravel()
        gam_p = np.asarray(A_p.multiply(A_p).sum(axis=0)).ravel()

        def owner_sum(part):                             # what the owner reads from peers
            allp = [None] * world
            dist.all_gather_object(allp, part)
            tot = np.zeros(o1 - o0)
            moved = 0
            for q in range(world):
                lo, hi = max(o0, wins[q][0]), min(o1, wins[q][1])
                if hi > lo:
                    tot[lo - o0:hi - o0] += allp[q][lo:hi]
                    if q != rank:
                        moved += hi - lo
            return tot, moved

        gamma_own, _ = owner_sum(gam_p)
        x = np.zeros(n)
        z_p = b_p.copy()
        xi_p = np.zeros(b1 - b0)
        X = 0.0
        ok = True
        moved_total = 0
        for k in range(iters):
            rec = orc.iterate(seed)
            s_own, mv1 = owner_sum(A_p.T @ z_p)
            v_own, mv2 = owner_sum(A_p.T @ xi_p)
            moved_total += mv1 + mv2
            if k > 0:
                V = torch.tensor([float(v_own @ v_own)], dtype=torch.float64)
                dist.all_reduce(V)
                if float(V) > 0:
                    x[o0:o1] += (X / float(V)) * v_own
            eps = scores(s_own, gamma_own)
            kap = np.full(o1 - o0, np.inf)
            u = uniforms(np.arange(o0, o1), k, 0, seed)
            pos = eps > 0
            kap[pos] = -np.log(u[pos]) / eps[pos]
            g = [None] * world
            dist.all_gather_object(g, (kap, pos))        # = the histogram radix search
            kap_all = np.concatenate([t[0] for t in g])
            pos_all = np.concatenate([t[1] for t in g])
            kp = min(orc.kc, int(pos_all.sum()))
            U = select_block(kap_all, kp, pos_all)
            zeta = np.zeros(n)
            Uo = U[(U >= o0) & (U < o1)]
            zeta[Uo] = s_own[Uo - o0]
            Zp = torch.tensor([float(zeta[o0:o1] @ zeta[o0:o1])], dtype=torch.float64)
            dist.all_reduce(Zp)
            Z = float(Zp)
            # halo: zeta, x of the window's columns owned elsewhere
            gz = [None] * world
            dist.all_gather_object(gz, (zeta[o0:o1], x[o0:o1]))
            for q in range(world):
                if q == rank:
                    continue
                lo, hi = max(win[0], own[q]), min(win[1], own[q + 1])
                if hi > lo:
                    zeta[lo:hi] = gz[q][0][lo - own[q]:hi - own[q]]
                    x[lo:hi] = gz[q][1][lo - own[q]:hi - own[q]]
                    moved_total += 2 * (hi - lo)
            w_p = A_p @ zeta
            ax_p = A_p @ x
            Wt = torch.tensor([float(w_p @ w_p)], dtype=torch.float64)
            dist.all_reduce(Wt)
            if kp > 0 and float(Wt) > 0:
                z_p = z_p - (Z / float(Wt)) * w_p
            r_p = b_p - z_p - ax_p
            eps_r = scores(r_p, rho_p)
            kr = np.full(b1 - b0, np.inf)
            uu = uniforms(np.arange(b0, b1), k, 1, seed)
            pr = eps_r > 0
            kr[pr] = -np.log(uu[pr]) / eps_r[pr]
            gr = [None] * world
            dist.all_gather_object(gr, (kr, pr))
            kpp = min(orc.kr, int(np.concatenate([t[1] for t in gr]).sum()))
            J = select_block(np.concatenate([t[0] for t in gr]), kpp, np.concatenate([t[1] for t in gr]))
            J_p = J[(J >= b0) & (J < b1)] - b0
            xi_p = np.zeros(b1 - b0)
            xi_p[J_p] = r_p[J_p]
            Xt = torch.tensor([float(r_p[J_p] @ r_p[J_p])], dtype=torch.float64)
            dist.all_reduce(Xt)
            X = float(Xt)
            ok &= (kp, block_hash(U), kpp, block_hash(J)) == (rec.kp, rec.hash_u, rec.kpp, rec.hash_j)
        v_own, _ = owner_sum(A_p.T @ xi_p)
        V = torch.tensor([float(v_own @ v_own)], dtype=torch.float64)
        dist.all_reduce(V)
        if float(V) > 0:
            x[o0:o1] += (X / float(V)) * v_own
        gx = [None] * world
        dist.all_gather_object(gx, x[o0:o1])
        xf = np.concatenate(gx)
        zs = [None] * world
        dist.all_gather_object(zs, z_p)
        z = np.concatenate(zs)
        out[rank] = (bool(ok), float(np.linalg.norm(xf - orc.x) / np.linalg.norm(orc.x)),
                     float(np.linalg.norm(z - orc.z) / np.linalg.norm(w.b)), moved_total / iters,
                     own, wins)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("name", ["C5t", "C3s", "C2si"])
def test_world2_peer_sharded_plan_matches_oracle(name):
    ctx = mp.get_context("spawn")
    mgr = ctx.Manager()
    out = mgr.dict()
    port = _free_port()
    procs = [ctx.Process(target=_peer_plan_run, args=(r, 2, port, name, 12, 3, out)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(300)
        assert p.exitcode == 0
    from workloads import by_name
    n = by_name(name).shape[1]
    for r in range(2):
        ok, dx, dz, moved, own, wins = out[r]
        assert ok, f"rank {r}: blocks differ from the single-process oracle"
        assert dx <= 1e-12 and dz <= 1e-12, (dx, dz)
        assert own[0] == 0 and own[-1] == n
        if name != "C2si":
            # banded: only the overlap of the two windows crosses ranks (O(halo), not O(n))
            overlap = max(0, min(wins[0][1], wins[1][1]) - max(wins[0][0], wins[1][0]))
            assert 0 < moved <= 4 * overlap + 1, (moved, overlap, n)
            assert moved < 0.25 * n

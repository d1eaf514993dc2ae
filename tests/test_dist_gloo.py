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

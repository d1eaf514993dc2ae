"""Plain CPU oracle of the paper's PARALLEL RGDBEK (Algorithm 2) — TEST INFRASTRUCTURE.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU legs may
import this module; the product path never does (same rules as oracle/rgdbek.py).

Algorithm 2 (alg:rgdbek_bsas; described at P:443-449) runs on P
processes, each owning a contiguous block of rows A^(p):

* s = sum_p (A^(p))^T z^(p) = A^T z_k by an allreduce; the column
  scores eps^z_j = s_j^2 / ||A_(j)||^2 and ONE global column set U_k of n*eta
  columns, exactly as in Algorithm 1.
* Each process solves its own small least-squares problem
  z_sol^(p) = argmin_y ||A^(p)_U y - z_k^(p)|| and updates z^(p) locally
  (P:469-473).
* Each process forms its residual r^(p) = b^(p) - z^(p)_{k+1} - A^(p) x_k
  (P:475), scores its rows and samples d_p*eta of ITS OWN rows J_k^(p)
  (P:476-477), and solves x_update^(p) = argmin_y ||A^(p)_J y - r^(p)_J||
  (P:478-480).
* x_{k+1} = x_k + (1/P) sum_p x_update^(p): the lazily averaged update by an
  allreduce.

Readings (R28): the two local least-squares solves are replaced by
their first Krylov iterates, the same pseudoinverse-free substitution as
Algorithm 1's (reading R1): z^(p) -= (Z_p / W_p) A^(p) zeta_p with
zeta_p = g_p on U, g_p = (A^(p))^T z^(p), Z_p = ||zeta_p||^2, W_p =
||A^(p) zeta_p||^2 (first CGLS iterate of the local problem); x_update^(p) =
(X_p / V_p) (A^(p))^T xi_p with xi_p = r^(p) on J^(p), X_p = ||xi_p||^2,
V_p = ||(A^(p))^T xi_p||^2 (first Craig iterate).  Rows are split as
[floor(m p / P), floor(m (p+1) / P)); d_p*eta rounds like Algorithm 1's block
sizes (reading R2) per process; the Philox stream is indexed by GLOBAL row
and column, so P = 1 is Algorithm 1 exactly.  A degenerate local step
(W_p = 0, or no positive score in the partition) is skipped (reading R7).

Pins (tests/test_oracle_lazy.py): P = 1 reproduces oracle.Oracle's trajectory
bit for bit; P = m (one row per process) makes every local z-problem 1x|U|
so z_1 = 0 on every row that meets U, and the x-step the Cimmino iteration
x + (1/m) sum_i r_i a_i / ||a_i||^2; per-process block sizes; the per-process
norm identity ||z^(p)_{k+1}||^2 = ||z^(p)_k||^2 - Z_p^2 / W_p (monotone).
Algorithm 2 need not converge to A^+ b (a global U with local residuals can
stall); that is a property of the method, not a pin.
"""
import numpy as np

from .rgdbek import Oracle, block_size, scores, sample_keys, select_block


def partition_bounds(m, P):
    """Row ranges [floor(m p / P), floor(m (p+1) / P)) of P processes."""
    return [(m * p // P, m * (p + 1) // P) for p in range(P)]


class LazyOracle(Oracle):
    """Algorithm 2 with P logical processes, pinv-free reading R28."""

    def __init__(self, A, b, eta=0.5, parts=2, bounds=None):
        super().__init__(A, b, eta)
        if bounds is not None:
            # explicit contiguous row blocks (e.g. the nnz-balanced ranks of P:443)
            bounds = [(int(r0), int(r1)) for r0, r1 in bounds]
            if bounds[0][0] != 0 or bounds[-1][1] != self.m or any(
                    bounds[i][1] != bounds[i + 1][0] or bounds[i][0] >= bounds[i][1]
                    for i in range(len(bounds) - 1)):
                raise ValueError("bounds must be contiguous non-empty row blocks covering [0, m)")
            parts = len(bounds)
        if not 1 <= parts <= self.m:
            raise ValueError("parts must lie in [1, m]")
        self.P = int(parts)
        self.bounds = bounds if bounds is not None else partition_bounds(self.m, self.P)

    def column_step(self, seed):
        """global U from A^T z; a local first-CGLS z-step per process."""
        A, z = self.A, self.z
        s = A.T @ z                                        # allreduce of the partials
        eps = scores(s, self.gamma)                        # eps^z
        kappa = sample_keys(eps, seed, self.k, 0)
        kp = min(self.kc, int(np.count_nonzero(eps > 0)))
        U = select_block(kappa, kp, eps > 0)               # one global U
        inU = np.zeros(self.n, dtype=bool)
        inU[U] = True
        znew = z.copy()
        Zs = Ws = 0.0
        for (r0, r1) in self.bounds:
            Ap = A[r0:r1]
            g = Ap.T @ z[r0:r1]                            # (A^(p))^T z^(p)
            zeta = np.where(inU, g, 0.0)
            Zp = float(g[U] @ g[U])
            w = Ap @ zeta
            Wp = float(w @ w)
            if kp > 0 and Wp > 0:                          # reading R7, per process
                znew[r0:r1] = z[r0:r1] - (Zp / Wp) * w
            Zs += Zp
            Ws += Wp
        self.z = znew
        return kp, U, Zs, Ws

    def row_step(self, seed):
        """local row samples and local first-Craig steps, averaged."""
        A = self.A
        r = self.b - self.z - A @ self.x                   # r^(p) for every p at once
        eps = scores(r, self.rho)                          # eps^x
        kappa = sample_keys(eps, seed, self.k, 1)          # global row indices
        xupd = np.zeros(self.n)
        Js = []
        kpp = 0
        Xs = Vs = 0.0
        for (r0, r1) in self.bounds:
            pos = eps[r0:r1] > 0
            kk = min(block_size(self.eta, r1 - r0), int(np.count_nonzero(pos)))
            Jp = r0 + select_block(kappa[r0:r1], kk, pos)  # d_p * eta own rows
            xi = np.zeros(r1 - r0)
            xi[Jp - r0] = r[Jp]
            Xp = float(r[Jp] @ r[Jp])
            v = A[r0:r1].T @ xi
            Vp = float(v @ v)
            if kk > 0 and Vp > 0:
                xupd = xupd + (Xp / Vp) * v                # x_update^(p)
            Js.append(Jp)
            kpp += kk
            Xs += Xp
            Vs += Vp
        self.x = self.x + xupd / self.P                    # lazy average
        J = np.concatenate(Js) if Js else np.zeros(0, dtype=np.int64)
        return kpp, J, Xs, Vs

"""Plain CPU oracle of the pseudoinverse-free RGDBEK sweep — TEST INFRASTRUCTURE.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this module.  The
product path (``paper_2509_19267_b200``) never imports, links or executes it,
and this module shares no code with the CUDA library.

What it computes (PAPER.md = /root/reference/PAPER.md, cited as P:<line>):

* Problem: A x = b, A in R^{m x n}, b in R^m (eq:Ax=b).
* Algorithm 1, read with the substitutions listed in DESIGN.md:
  - x_0 = 0, z_0 = b.
  - Column step: s = A^T z_k; eps^z_j = s_j^2 / ||A_(j)||^2 (P:94,
    Alg. 1 line 5); U_k = n*eta columns drawn with P(j) = eps_j / sum eps
    (Alg. 1 lines 6-7), without replacement (reading R3) via
    exponential keys kappa_j = -ln(u_j) / eps_j, keeping the k smallest
    (reading R3/R4); update z_{k+1} = z_k - (Z/W) w with zeta = s on U,
    Z = ||zeta||^2, w = A zeta, W = ||w||^2 (reading R1: the
    pseudoinverse-free form BASELINE.json's north_star prescribes in place of
    z_k - A_U A_U^+ z_k of P:117).
  - Row step: r = b - z_{k+1} - A x_k (Alg. 1 line 10);
    eps^x_i = r_i^2 / ||A^(i)||^2; J_k = m*eta rows by the same sampler;
    xi = r on J, X = ||xi||^2, v = A^T xi, V = ||v||^2, x_{k+1} = x_k + (X/V) v
    (reading R1: north_star's  x += (eta^T r / ||A^T eta||^2) A^T eta, with
    eta^T r = ||xi||^2 = X, in place of the pseudoinverse of P:122).
  - Stop test on RSE = ||A x - b||^2 / ||b||^2 or on
    ||x - x*|| / ||x*|| (BASELINE.json metric), after each full iteration.
* update="exact_lstsq": Algorithm 1's own updates, z_{k+1} =
  z_k - A_U A_U^+ z_k and x_{k+1} = x_k + (A^J)^+ r^J, written
  out with numpy's minimum-norm least-squares solver (lstsq) on the extracted
  submatrices — the definition.
* update="exact": the same projections by an inner Krylov solve from 0, CGLS in
  place of the paper's LSQR (Remark 2), with the inner stopping rule
  of DESIGN.md reading R1b.  Pinned to "exact_lstsq" (tests/test_oracle_exact.py);
  the GPU exact mode is compared with both.
* No blocking, fusion or reordering: every product is one library matvec
  (numpy BLAS for dense A, scipy.sparse for CSR A), every selection one sort.

Pins (tests/test_oracle_*.py): the norm caches rho, gamma by the paper's printed
Frobenius norm of its FEM Poisson matrix, the rank-one closed form and
sum rho = sum gamma = ||A||_F^2 (test_oracle_norms.py); the k = 1 selection law
P(j) = eps_j / sum eps through column_step / row_step on systems whose scores have
a norm-free closed form; Philox KATs; sampler inclusion probabilities
(closed forms for k=1, k=2, exhaustive enumeration); the Pythagoras identity of
eq:res_norm_evolve; orthogonality of both updates; reduction to
the REK column step and the Kaczmarz row step at block size 1;
equality with the first CGLS iterate (z) and the first Craig iterate (x);
trajectory invariance under b -> b + r with r in null(A^T); convergence to
A^+ b and (I - A A^+) b on tiny inputs checked by SVD brute force.
"""
from dataclasses import dataclass, field

import numpy as np

from .philox import uniforms

MASK64 = (1 << 64) - 1

OUTCOME_CONVERGED = 0   # SPEC.md exit-code convention: converged
OUTCOME_MAX_ITER = 2    # iteration cap reached
OUTCOME_STALLED = 3     # no positive score mass in either step

STOP_RSE = 0
STOP_REL_ERR = 1
STOP_NONE = 2


def block_size(eta, d):
    """k = max(1, floor(eta*d + 1/2)) — reading R2 of "n eta" / "m eta"."""
    return max(1, int(np.floor(eta * d + 0.5)))


def splitmix64(i):
    """SplitMix64 finaliser of indices (uint64 arithmetic wraps mod 2^64)."""
    with np.errstate(over="ignore"):
        z = np.atleast_1d(np.asarray(i, dtype=np.uint64)) + np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


def block_hash(indices):
    """Order-independent 64-bit fingerprint: sum of splitmix64(i) mod 2^64."""
    idx = np.asarray(indices, dtype=np.uint64)
    if idx.size == 0:
        return 0
    return int(np.sum(splitmix64(idx), dtype=np.uint64))


def row_sq_norms(A):
    """rho_i = ||A^(i)||^2, the row-score denominators."""
    if isinstance(A, np.ndarray):
        return np.einsum("ij,ij->i", A, A)
    return np.asarray(A.multiply(A).sum(axis=1)).ravel()


def col_sq_norms(A):
    """gamma_j = ||A_(j)||^2, the column-score denominators."""
    if isinstance(A, np.ndarray):
        return np.einsum("ij,ij->j", A, A)
    return np.asarray(A.multiply(A).sum(axis=0)).ravel()


def scores(numer, denom):
    """eps = numer^2 / denom, and 0 where denom == 0 (reading R6)."""
    eps = np.zeros_like(numer)
    nz = denom > 0
    eps[nz] = numer[nz] * numer[nz] / denom[nz]
    return eps


def sample_keys(eps, seed, k, step):
    """Exponential keys kappa = -ln(u) / eps (+inf where eps == 0); reading R3/R5.

    Taking the k smallest keys is successive sampling without replacement with
    probabilities P(j) = eps_j / sum_l eps_l: for k = 1 the
    smallest key is index j with probability exactly P(j).
    """
    u = uniforms(np.arange(len(eps)), k, step, seed)
    kappa = np.full(len(eps), np.inf)
    pos = eps > 0
    with np.errstate(over="ignore"):            # an overflow to +inf is the IEEE result
        kappa[pos] = -np.log(u[pos]) / eps[pos]
    return kappa


def select_block(kappa, kk, eligible=None):
    """Indices of the kk smallest (kappa_j, j) pairs, sorted (reading R4: lower index wins ties).

    Indices with eps == 0 (``eligible`` False) are never taken before eligible
    ones (reading R6); the caller clamps kk to the eligible count.
    """
    n = len(kappa)
    never = np.zeros(n, dtype=bool) if eligible is None else ~np.asarray(eligible)
    order = np.lexsort((np.arange(n), kappa, never))
    return np.sort(order[:kk])


def greedy_block(eps, eta):
    """GDBEK's greedy set {j : eps_j >= eta * max_l eps_l}, '>=' per SPEC S:303;
    empty when every score is 0."""
    emax = float(eps.max()) if len(eps) else 0.0
    if not emax > 0:
        return np.zeros(0, dtype=np.int64)
    return np.flatnonzero(eps >= eta * emax)


@dataclass
class IterRecord:
    """What one iteration k produced (compared with the GPU trace)."""
    k: int
    kp: int            # |U_k|
    hash_u: int
    Z: float           # ||zeta||^2
    W: float           # ||A zeta||^2
    kpp: int           # |J_k|
    hash_j: int
    X: float           # ||xi||^2
    V: float           # ||A^T xi||^2
    rse: float         # RSE(x_{k+1})
    U: np.ndarray = field(repr=False, default=None)
    J: np.ndarray = field(repr=False, default=None)


class Oracle:
    """State (x_k, z_k, k) of Algorithm 1 and its plain iteration."""

    def __init__(self, A, b, eta=0.5, update="pinv_free", inner_tol=1e-13, inner_max=50,
                 select="random"):
        if update not in ("pinv_free", "exact", "exact_lstsq"):
            raise ValueError("update must be 'pinv_free', 'exact' or 'exact_lstsq'")
        if select not in ("random", "greedy"):
            raise ValueError("select must be 'random' or 'greedy'")
        self.select = select
        self.update = update
        self.inner_tol = float(inner_tol)
        self.inner_max = int(inner_max)
        self.A = A
        self.b = np.asarray(b, dtype=np.float64)
        self.m, self.n = A.shape
        if self.b.shape != (self.m,):
            raise ValueError(f"b has shape {self.b.shape}, expected ({self.m},)")
        if not (0.0 < eta < 1.0):
            raise ValueError("eta must lie in (0, 1)")
        self.eta = float(eta)
        self.rho = row_sq_norms(A)
        self.gamma = col_sq_norms(A)
        self.kc = block_size(eta, self.n)
        self.kr = block_size(eta, self.m)
        self.bnorm2 = float(self.b @ self.b)
        self.reset()

    def reset(self):
        self.x = np.zeros(self.n)          # x_0 = 0
        self.z = self.b.copy()             # z_0 = b
        self.k = 0

    def rse(self, x=None):
        """RSE = ||A x - b||^2 / ||b||^2, one extra matvec."""
        x = self.x if x is None else x
        res = self.A @ x - self.b
        return float(res @ res) / self.bnorm2

    def column_step(self, seed):
        """Alg. 1 lines 4-8 in pseudoinverse-free form (reading R1)."""
        A, z = self.A, self.z
        s = A.T @ z                                        # A^T z_k
        eps = scores(s, self.gamma)                        # eps^z
        if self.select == "greedy":
            U = greedy_block(eps, self.eta)                # GDBEK threshold set
            kp = len(U)
        else:
            kappa = sample_keys(eps, seed, self.k, 0)
            kp = min(self.kc, int(np.count_nonzero(eps > 0)))  # clamp (reading R6)
            U = select_block(kappa, kp, eps > 0)
        zeta = np.zeros(self.n)
        zeta[U] = s[U]
        Z = float(s[U] @ s[U])
        w = A @ zeta
        W = float(w @ w)
        if self.update == "exact_lstsq":
            # z_{k+1} = z_k - A_U A_U^+ z_k: the orthogonal projection of z_k
            # onto range(A_U)^perp, via the minimum-norm least-squares solution
            if kp > 0:
                AU = A[:, U] if isinstance(A, np.ndarray) else A[:, U].toarray()
                y = np.linalg.lstsq(AU, z, rcond=None)[0]
                self.z = z - AU @ y
        elif self.update == "exact":
            # the same projection by the paper's route, an inner Krylov solve of
            # min ||A_U y - z_k|| (LSQR; here its equivalent CGLS, reading
            # R1b), from y = 0; z holds its residual z_k - A_U y.  Stopping rule:
            # ||A_U^T z||^2 <= inner_tol^2 Z, or inner_max iterations.
            if kp > 0:
                p, gam = zeta.copy(), Z
                z = z.copy()
                inU = np.zeros(self.n, dtype=bool)
                inU[U] = True
                for it in range(self.inner_max):
                    if not gam > 0:
                        break
                    q = A @ p
                    Wq = float(q @ q)
                    if not Wq > 0:
                        break
                    z = z - (gam / Wq) * q
                    if it + 1 == self.inner_max:
                        break
                    sp = A.T @ z
                    gnew = float(sp[inU] @ sp[inU])
                    if gnew <= self.inner_tol ** 2 * Z:
                        break
                    p = np.where(inU, sp + (gnew / gam) * p, 0.0)
                    gam = gnew
                self.z = z
        elif kp > 0 and W > 0:                             # reading R7
            self.z = z - (Z / W) * w
        return kp, U, Z, W

    def row_step(self, seed):
        """Alg. 1 lines 9-13 in pseudoinverse-free form (reading R1)."""
        A = self.A
        r = self.b - self.z - A @ self.x                   # uses z_{k+1} (reading R8)
        eps = scores(r, self.rho)                          # eps^x
        if self.select == "greedy":
            J = greedy_block(eps, self.eta)
            kpp = len(J)
        else:
            kappa = sample_keys(eps, seed, self.k, 1)
            kpp = min(self.kr, int(np.count_nonzero(eps > 0)))
            J = select_block(kappa, kpp, eps > 0)
        xi = np.zeros(self.m)
        xi[J] = r[J]
        X = float(r[J] @ r[J])
        v = A.T @ xi
        V = float(v @ v)
        if self.update == "exact_lstsq":
            # x_{k+1} = x_k + (A^J)^+ (b^J - z^J_{k+1} - A^J x_k), minimum-norm LS
            if kpp > 0:
                AJ = A[J, :] if isinstance(A, np.ndarray) else A[J, :].toarray()
                self.x = self.x + np.linalg.lstsq(AJ, r[J], rcond=None)[0]
        elif self.update == "exact":
            # inner CGLS on min ||A^J y - r^J|| from y = 0 (limit (A^J)^+ r^J); stopping
            # rule ||A^J^T res||^2 <= inner_tol^2 ||A^J^T r^J||^2, or inner_max iterations
            if kpp > 0 and X > 0:
                inJ = np.zeros(self.m, dtype=bool)
                inJ[J] = True
                res = xi.copy()
                t = A.T @ res
                p = t.copy()
                gam0 = gam = float(t @ t)
                x = self.x.copy()
                for it in range(self.inner_max):
                    if not gam > 0:
                        break
                    u = A @ p
                    Wq = float(u[inJ] @ u[inJ])
                    if not Wq > 0:
                        break
                    al = gam / Wq
                    x = x + al * p
                    res = np.where(inJ, res - al * u, 0.0)
                    if it + 1 == self.inner_max:
                        break
                    t = A.T @ res
                    gnew = float(t @ t)
                    if gnew <= self.inner_tol ** 2 * gam0:
                        break
                    p = t + (gnew / gam) * p
                    gam = gnew
                self.x = x
        elif kpp > 0 and V > 0:
            self.x = self.x + (X / V) * v
        return kpp, J, X, V

    def iterate(self, seed, keep_blocks=False):
        """One full iteration k -> k+1 of Algorithm 1; returns its IterRecord."""
        kp, U, Z, W = self.column_step(seed)
        kpp, J, X, V = self.row_step(seed)
        rec = IterRecord(self.k, kp, block_hash(U), Z, W, kpp, block_hash(J), X, V,
                         self.rse(),
                         U.copy() if keep_blocks else None,
                         J.copy() if keep_blocks else None)
        self.k += 1
        return rec

    def solve(self, tol, max_iter, seed, stop=STOP_RSE, xstar=None, records=None):
        """Iterate until the stop test holds after an iteration (reading R11/R12).

        Returns (outcome, iters, rse, rel_err).  Test order after iteration k:
        converged, then stalled (both blocks empty), then the iteration cap.
        """
        if stop == STOP_REL_ERR:
            if xstar is None:
                raise ValueError("STOP_REL_ERR needs xstar")
            xstar = np.asarray(xstar, dtype=np.float64)
            xs_norm = float(np.linalg.norm(xstar))
        while True:
            rec = self.iterate(seed)
            if records is not None:
                records.append(rec)
            rel = (float(np.linalg.norm(self.x - xstar)) / xs_norm
                   if xstar is not None else float("nan"))
            if stop == STOP_RSE and rec.rse <= tol:
                return OUTCOME_CONVERGED, self.k, rec.rse, rel
            if stop == STOP_REL_ERR and rel <= tol:
                return OUTCOME_CONVERGED, self.k, rec.rse, rel
            if rec.kp == 0 and rec.kpp == 0:
                return OUTCOME_STALLED, self.k, rec.rse, rel
            if self.k >= max_iter:
                return OUTCOME_MAX_ITER, self.k, rec.rse, rel

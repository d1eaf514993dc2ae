"""Synthetic inputs shaped like the paper's workloads (recipe: DESIGN.md §3).

Every generator is seeded (numpy PCG64 ``default_rng``) and returns a
``Workload``.  Data randomness uses numpy; the BLOCK SELECTION randomness of
the method is Philox and lives on each side of the boundary separately.

Configs (BASELINE.json "configs", made concrete in SURVEY.md §8(d)):
  C1   dense Gaussian 200x50, consistent, seed 0              (configs[0])
  C2c  dense Gaussian 20000x5000, consistent, seed 0          (configs[1])
  C2i  same A, b = A x* + r, r in null(A^T), ||r|| = 0.1||Ax*|| (configs[1])
  C3   2-D Poisson 5-point stencil on a 2000^2 interior grid   (configs[2])
  C4   1-D Gaussian Toeplitz blur sigma=r=20 (eq:toeplitz) on a
       vectorised 1024x1024 image, plus noise                  (configs[3])
  C5   population-model sliding-window system 50M x 5M, 1e9 nnz (configs[4])
  C5s  the same generator at 50000x5000                        (configs[4], scaled)
"""
from dataclasses import dataclass, field
from typing import Optional

import numpy as np
import scipy.sparse as sp


@dataclass
class Workload:
    name: str
    A: object                      # np.ndarray (row-major f64) or scipy csr_matrix
    b: np.ndarray
    xstar: Optional[np.ndarray]    # A^+ b when known by construction, else None
    rvec: Optional[np.ndarray]     # (I - A A^+) b when known, else None
    eta: float = 0.5
    symmetric: bool = False
    stop: str = "rel_err"          # "rel_err" | "rse" | "none"
    tol: float = 1e-6
    max_iter: int = 100000
    meta: dict = field(default_factory=dict)

    @property
    def shape(self):
        return self.A.shape

    @property
    def dense(self):
        return isinstance(self.A, np.ndarray)

    @property
    def nnz(self):
        return self.A.size if self.dense else self.A.nnz

    def csr_arrays(self):
        """(row_ptr int64[m+1], col_idx int32[nnz], val f64[nnz]) of a sparse workload."""
        A = self.A
        return (np.ascontiguousarray(A.indptr, dtype=np.int64),
                np.ascontiguousarray(A.indices, dtype=np.int32),
                np.ascontiguousarray(A.data, dtype=np.float64))


def _null_component(A, g, scale_to):
    """r = g - Q (Q^T g) with Q a thin QR basis of range(A), scaled to ||r|| = scale_to."""
    Q, _ = np.linalg.qr(A, mode="reduced")
    r = g - Q @ (Q.T @ g)
    return r * (scale_to / np.linalg.norm(r))


def dense_gaussian(m, n, seed=0, noise=0.0, eta=0.5):
    """A ~ N(0,1) row-major, x_true ~ N(0,1) (the paper's randn protocol).

    noise > 0 adds r in null(A^T) with ||r|| = noise * ||A x_true||, making the
    system inconsistent (the "r" of P:306 read as r in range(A)^perp, reading R10).
    Tall full-rank A => x* = x_true; fat A => x* = A^+ b via lstsq.
    """
    rng = np.random.default_rng(seed)
    A = rng.standard_normal((m, n))
    x_true = rng.standard_normal(n)
    b = A @ x_true
    rvec = np.zeros(m)
    if noise > 0:
        if m <= n:
            raise ValueError("an inconsistent system needs m > n")
        g = rng.standard_normal(m)
        rvec = _null_component(A, g, noise * np.linalg.norm(b))
        b = b + rvec
    if m >= n:
        xstar = x_true
    else:
        xstar = np.linalg.lstsq(A, b, rcond=None)[0]
    name = f"dense_gaussian_{m}x{n}" + ("_inconsistent" if noise > 0 else "")
    return Workload(name, A, b, xstar, rvec, eta=eta,
                    meta={"seed": seed, "noise": noise, "x_true": x_true})


def _poisson_stencil(N):
    """5-point Laplacian [4, -1 x 4] on an N x N interior grid, natural row-major order."""
    T = sp.diags([-np.ones(N - 1), 2 * np.ones(N), -np.ones(N - 1)], [-1, 0, 1], format="csr")
    I = sp.identity(N, format="csr")
    A = (sp.kron(I, T, format="csr") + sp.kron(T, I, format="csr")).tocsr()
    A.sort_indices()
    A.eliminate_zeros()
    return A


def poisson2d(N, eta=0.5):
    """C3: -Laplace u = f on the unit square, N^2 interior nodes.

    The P1 stiffness matrix on a structured right-triangle mesh is exactly the
    5-point stencil; x_true = sin(pi x) sin(pi y) at the nodes
    (P:745), b = A x_true.  Symmetric, so A^T = A (the CSR serves as CSC).
    """
    A = _poisson_stencil(N)
    h = 1.0 / (N + 1)
    t = np.arange(1, N + 1) * h
    X, Y = np.meshgrid(t, t, indexing="ij")
    x_true = (np.sin(np.pi * X) * np.sin(np.pi * Y)).ravel()
    b = A @ x_true
    return Workload(f"poisson2d_{N}x{N}", A, b, x_true, np.zeros(A.shape[0]), eta=eta,
                    symmetric=True, stop="none", max_iter=200,
                    meta={"grid": N})


def poisson_fem_paper(nx=25):
    """The paper's FEM Poisson matrix, N = nx*nx nodes (tab:poisson_helmholtz).

    Boundary nodes get identity rows, boundary columns are eliminated from the
    interior rows, interior rows carry the 5-point P1 stencil.  Used only to
    pin the C3 structure against the printed sparsity / ||A||_F / kappa.
    """
    N = nx
    rows, cols, vals = [], [], []
    def idx(i, j):
        return i * N + j
    for i in range(N):
        for j in range(N):
            p = idx(i, j)
            if i in (0, N - 1) or j in (0, N - 1):
                rows.append(p); cols.append(p); vals.append(1.0)
                continue
            rows.append(p); cols.append(p); vals.append(4.0)
            for di, dj in ((-1, 0), (1, 0), (0, -1), (0, 1)):
                ii, jj = i + di, j + dj
                if 0 < ii < N - 1 and 0 < jj < N - 1:
                    rows.append(p); cols.append(idx(ii, jj)); vals.append(-1.0)
    A = sp.csr_matrix((vals, (rows, cols)), shape=(N * N, N * N))
    A.sort_indices()
    return A


def toeplitz_blur(N, sigma=20.0, radius=20, seed=0, noise=1e-3, eta=0.5):
    """C4: banded Toeplitz Gaussian PSF of eq:toeplitz, sigma = r = 20.

    A_ij = exp(-(i-j)^2 / (2 sigma^2)) / (sigma sqrt(2 pi)) for |i-j| <= r on the
    vectorised image (reading R21).  x = synthetic image in [0,1] (Gaussian
    blobs + rectangles), b = A x + N(0, (noise * max|Ax|)^2).  Throughput-only:
    kappa(A) is effectively infinite, so x* is not known.
    """
    offs = np.arange(-radius, radius + 1)
    coef = np.exp(-(offs.astype(np.float64) ** 2) / (2.0 * sigma * sigma)) / (sigma * np.sqrt(2.0 * np.pi))
    diags = [np.full(N - abs(o), c) for o, c in zip(offs, coef)]
    A = sp.diags(diags, offs, shape=(N, N), format="csr")
    A.sort_indices()
    side = int(round(np.sqrt(N)))
    rng = np.random.default_rng(seed)
    if side * side == N:
        yy, xx = np.mgrid[0:side, 0:side] / max(side - 1, 1)
        img = np.zeros((side, side))
        for _ in range(12):
            cx, cy, w, a = rng.uniform(0, 1), rng.uniform(0, 1), rng.uniform(0.02, 0.2), rng.uniform(0.2, 1)
            img += a * np.exp(-((xx - cx) ** 2 + (yy - cy) ** 2) / (2 * w * w))
        for _ in range(6):
            x0, y0 = rng.uniform(0, 0.8, size=2)
            w, h = rng.uniform(0.05, 0.2, size=2)
            img[(xx >= x0) & (xx < x0 + w) & (yy >= y0) & (yy < y0 + h)] += rng.uniform(0.2, 0.8)
        img = np.clip(img / img.max(), 0.0, 1.0)
        x_img = img.ravel()
    else:
        x_img = rng.uniform(0, 1, size=N)
    Ax = A @ x_img
    b = Ax + rng.normal(0.0, noise * np.abs(Ax).max(), size=N)
    return Workload(f"toeplitz_blur_{N}", A, b, None, None, eta=eta, symmetric=True,
                    stop="none", max_iter=200, meta={"sigma": sigma, "radius": radius, "image": x_img})


PPS_PARAMS = dict(r=0.5, k=100.0, a=0.5, a0=0.25, b=0.5, b0=0.25, d=0.5, e=1.0,
                  f=0.1, g=0.5, h=0.1, i=0.1, i0=0.25, j=1.0)   # tab:param


def pps_trajectory(T=200.0, dt=0.1, x0=(4.0, 3.0, 2.0), p=PPS_PARAMS):
    """RK4 of the predator-prey-scavenger ODE eq:predpreyscav, P:865 settings."""
    def f(u):
        x, y, z = u
        dx = p["r"] * x * (1 - x / p["k"]) - p["a"] * x * x * y / (1 + p["a0"] * x * x) \
            - p["b"] * x * x * z / (1 + p["b0"] * x * x)
        dy = p["d"] * x * x * y / (1 + p["a0"] * x * x) + p["f"] * z * z * y / (1 + p["i0"] * z * z) - p["e"] * y
        dz = p["g"] * x * x * z / (1 + p["b0"] * x * x) + p["h"] * y * z \
            - p["i"] * y * z * z / (1 + p["i0"] * z * z) - p["j"] * z
        return np.array([dx, dy, dz])
    steps = int(round(T / dt))
    out = np.empty((steps + 1, 3))
    u = np.array(x0, dtype=np.float64)
    out[0] = u
    for s in range(steps):
        k1 = f(u); k2 = f(u + 0.5 * dt * k1); k3 = f(u + 0.5 * dt * k2); k4 = f(u + dt * k3)
        u = u + dt / 6.0 * (k1 + 2 * k2 + 2 * k3 + k4)
        out[s + 1] = u
    return out


def popmodel(m, n, seed=0, width=20, noise_frac=0.1, sigma=3.0, delay=1, eta=0.5, block=30):
    """C5 / C5s: noisy delayed population-model sliding-window system (reading R22).

    Row i covers columns c_i .. c_i+width-1, c_i = floor(i (n-width) / (m-1));
    A[i, c_i+t] = sig[(i+t) mod S] with sig(t) = prey(t - delay) + N(0, sigma^2)
    (delay 1, sigma 3).  x* = x_true ~ N(0,1); the
    inconsistent part r is a sum over disjoint `block`-row blocks of a random
    multiple of the block's left null vector (A_blk^T y = 0), so A^T r = 0
    exactly up to rounding; ||r|| = noise_frac ||A x*||.
    """
    rng = np.random.default_rng(seed)
    traj = pps_trajectory()
    S = traj.shape[0]
    prey = traj[:, 0]
    sig = prey[np.maximum(np.arange(S) - delay, 0)] + rng.normal(0.0, sigma, size=S)
    i = np.arange(m, dtype=np.int64)
    c = (i * (n - width)) // max(m - 1, 1)
    t = np.arange(width, dtype=np.int64)
    cols = np.empty(m * width, dtype=np.int32)
    vals = np.empty(m * width, dtype=np.float64)
    CH = 1 << 20                                     # rows per chunk (bounded temporaries)
    for r0 in range(0, m, CH):
        r1 = min(m, r0 + CH)
        cols[r0 * width:r1 * width] = (c[r0:r1, None] + t[None, :]).ravel()
        vals[r0 * width:r1 * width] = sig[(i[r0:r1, None] + t[None, :]) % S].ravel()
    indptr = np.arange(0, m * width + 1, width, dtype=np.int64)
    A = sp.csr_matrix((vals, cols, indptr), shape=(m, n))
    x_true = rng.standard_normal(n)
    Ax = A @ x_true
    rvec = np.zeros(m)
    if noise_frac > 0:
        nblk = m // block
        if nblk > 0:
            coef = rng.standard_normal(nblk)
            vv_all = vals.reshape(m, width)
            BCH = 1 << 16                            # blocks per chunk
            for b0 in range(0, nblk, BCH):
                b1 = min(nblk, b0 + BCH)
                nb = b1 - b0
                rr = i[b0 * block:b1 * block].reshape(nb, block)
                c0 = c[rr[:, 0]]
                loc = (c[rr][:, :, None] + t[None, None, :]) - c0[:, None, None]
                span = int(loc.max()) + 1
                if span >= block:
                    raise ValueError("row blocks too short to have a left null space")
                Ab = np.zeros((nb, block, span))
                vv = vv_all[b0 * block:b1 * block].reshape(nb, block, width)
                bi = np.repeat(np.arange(nb), block * width)
                ri = np.tile(np.repeat(np.arange(block), width), nb)
                Ab[bi, ri, loc.ravel()] = vv.ravel()
                U, _, _ = np.linalg.svd(Ab, full_matrices=True)
                rvec[b0 * block:b1 * block] = (coef[b0:b1, None] * U[:, :, -1]).ravel()
            rvec *= noise_frac * np.linalg.norm(Ax) / np.linalg.norm(rvec)
    b = Ax + rvec
    return Workload(f"popmodel_{m}x{n}", A, b, x_true, rvec, eta=eta,
                    meta={"seed": seed, "width": width, "noise_frac": noise_frac})


def sparse_random(m, n, density=0.05, seed=0, eta=0.5, consistent=True):
    """sprandn-like sparse A (99% sparse in the paper); for small tests.

    x* = A^+ b (lstsq on the dense copy; only used at small sizes).
    """
    rng = np.random.default_rng(seed)
    A = sp.random(m, n, density=density, format="csr", random_state=rng,
                  data_rvs=rng.standard_normal)
    A.sort_indices()
    x_true = rng.standard_normal(n)
    b = A @ x_true
    if not consistent:
        b = b + 0.1 * rng.standard_normal(m)
    Ad = A.toarray()
    xstar = np.linalg.lstsq(Ad, b, rcond=None)[0]
    rvec = b - Ad @ xstar
    return Workload(f"sparse_random_{m}x{n}_{density}", A, b, xstar, rvec, eta=eta,
                    meta={"seed": seed, "density": density})


CONFIGS = {
    "C1": lambda: dense_gaussian(200, 50, seed=0),
    "C2c": lambda: dense_gaussian(20000, 5000, seed=0),
    "C2i": lambda: dense_gaussian(20000, 5000, seed=0, noise=0.1),
    "C3": lambda: poisson2d(2000),
    "C4": lambda: toeplitz_blur(1024 * 1024),
    "C5s": lambda: popmodel(50000, 5000, seed=0),
    # measured: ||x - x*||/||x*|| = 4.4e-4 after 100,000 iterations on one B200 (1114 s),
    # so the full-size C5 is benchmarked for throughput, not time to 1e-6
    "C5": lambda: _throughput_only(popmodel(50_000_000, 5_000_000, seed=0)),
    # C5's matrix with a consistent b (no null-space noise: skips the 1.7M block SVDs);
    # same A, same bytes per iteration — used for ncu captures of the C5 kernel
    "C5c": lambda: _throughput_only(popmodel(50_000_000, 5_000_000, seed=0, noise_frac=0.0)),
    # a tenth of C5 (same structure, 1e8 nnz, consistent b): quick to generate, large
    # enough to be bandwidth-bound (kernel experiments, tools/ab_pass.py)
    "C5m": lambda: _throughput_only(popmodel(5_000_000, 500_000, seed=0, noise_frac=0.0)),
    # small twins used by parity tests
    "C2s": lambda: dense_gaussian(2000, 500, seed=0),
    "C2si": lambda: dense_gaussian(2000, 500, seed=0, noise=0.1),
    "C3s": lambda: poisson2d(48),
    "C4s": lambda: toeplitz_blur(48 * 48),
    "C5t": lambda: popmodel(5000, 500, seed=0),
}


def _throughput_only(w, iters=200):
    w.stop = "none"
    w.max_iter = iters
    return w


def by_name(name):
    return CONFIGS[name]()

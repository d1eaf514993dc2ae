"""The three application drivers (see apps/__init__.py).  Each returns a dict."""
import numpy as np
import scipy.sparse as sp

from workloads.gen import poisson_fem_paper, pps_trajectory


def _solver(A, b, eta, stop="rse"):
    from paper_2509_19267_b200 import Solver
    if sp.issparse(A):
        return Solver.from_scipy(A, b, eta=eta, stop=stop)
    return Solver(A, b, eta=eta, stop=stop)


def fem_poisson(nx=25, tol=1e-6, eta=0.5, max_iter=1_000_000, seed=0):
    """-Laplace u = f on (0,1)^2, u = 0 on the boundary, exact u = sin(pi x) sin(pi y)
    (P:740-745), P1 elements on the structured diagonal-split mesh of nx x nx nodes
    (the stiffness matrix is the 5-point stencil, boundary rows are the
    identity).  Load vector by nodal quadrature, b_i = h^2 f(x_i).  Solved to the
    paper's RSE threshold 1e-6."""
    A = poisson_fem_paper(nx)
    h = 1.0 / (nx - 1)
    g = np.linspace(0.0, 1.0, nx)
    yy, xx = np.meshgrid(g, g, indexing="ij")
    u_exact = (np.sin(np.pi * xx) * np.sin(np.pi * yy)).ravel()
    f = 2.0 * np.pi ** 2 * u_exact
    boundary = np.zeros((nx, nx), dtype=bool)
    boundary[[0, -1], :] = True
    boundary[:, [0, -1]] = True
    b = np.where(boundary.ravel(), 0.0, h * h * f)
    s = _solver(A, b, eta)
    res = s.solve(tol, max_iter, seed)
    u = s.x()
    s.close()
    err = u - u_exact
    return {"app": "fem_poisson", "nodes": nx * nx, "iters": res["iters"],
            "outcome": res["outcome"], "rse": res["rse"], "seconds": res["seconds"],
            "rel_l2_error": float(np.linalg.norm(err) / np.linalg.norm(u_exact)),
            "std_error": float(np.std(err)),
            "paper": {"rse": 9.359952e-7, "rel_l2_error": 3.238629e-3, "std_error": 1.090497e-3}}


def _psnr(x, ref):
    mse = float(np.mean((x - ref) ** 2))
    return float("inf") if mse == 0 else 10.0 * np.log10(1.0 / mse)


def _ssim(x, ref, win=7):
    """Mean SSIM (Wang et al. 2004) with a win x win uniform window, data range 1."""
    from scipy.ndimage import uniform_filter
    c1, c2 = 0.01 ** 2, 0.03 ** 2
    mx, my = uniform_filter(x, win), uniform_filter(ref, win)
    vx = uniform_filter(x * x, win) - mx * mx
    vy = uniform_filter(ref * ref, win) - my * my
    cxy = uniform_filter(x * ref, win) - mx * my
    s = ((2 * mx * my + c1) * (2 * cxy + c2)) / ((mx * mx + my * my + c1) * (vx + vy + c2))
    return float(s.mean())


def synthetic_rgb(side=256, seed=0):
    """A seeded synthetic colour image in [0,1]: smooth blobs, bars and a checker
    patch per channel (the paper's photographs are not available)."""
    rng = np.random.default_rng(seed)
    yy, xx = np.mgrid[0:side, 0:side] / (side - 1)
    img = np.zeros((side, side, 3))
    for c in range(3):
        ch = np.zeros((side, side))
        for _ in range(10):
            cx, cy, w, a = rng.uniform(0, 1), rng.uniform(0, 1), rng.uniform(0.03, 0.2), rng.uniform(0.2, 1)
            ch += a * np.exp(-((xx - cx) ** 2 + (yy - cy) ** 2) / (2 * w * w))
        for _ in range(5):
            x0, y0 = rng.uniform(0, 0.8, size=2)
            w, h = rng.uniform(0.05, 0.2, size=2)
            ch[(xx >= x0) & (xx < x0 + w) & (yy >= y0) & (yy < y0 + h)] += rng.uniform(0.2, 0.8)
        q = (np.floor(xx * 16) + np.floor(yy * 16)) % 2
        ch[(xx > 0.6) & (yy > 0.6)] += 0.3 * q[(xx > 0.6) & (yy > 0.6)]
        img[:, :, c] = ch / ch.max()
    return np.clip(img, 0.0, 1.0)


def deblur(side=256, iters=200000, eta=0.5, sigma=20.0, radius=20, seed=0, multi_rhs=False):
    """b_c = A x_c per channel, A = eq:toeplitz with sigma = r = 20
    on the vectorised channel (N = side^2; the paper's 256x256x3 images give
    65536 x 65536); RGDBEK for a fixed iteration budget per channel.  Reports
    PSNR, SSIM and RSE per channel and their means (tab:image).  multi_rhs=True solves
    the three channels as three right-hand sides of ONE solve (every pass over A serves
    all three; channel c uses seed + c, reading R29)."""
    N = side * side
    offs = np.arange(-radius, radius + 1)
    coef = np.exp(-(offs.astype(np.float64) ** 2) / (2.0 * sigma * sigma)) / (sigma * np.sqrt(2.0 * np.pi))
    A = sp.diags([np.full(N - abs(o), c) for o, c in zip(offs, coef)], offs, shape=(N, N), format="csr")
    A.sort_indices()
    img = synthetic_rgb(side, seed)
    out = {"app": "deblur", "pixels": [side, side, 3], "iters_per_channel": iters, "channels": []}
    from paper_2509_19267_b200 import Solver
    B = np.array([A @ img[:, :, c].ravel() for c in range(3)])
    if multi_rhs:
        sm = Solver.from_scipy_multi(A, B, eta=eta, stop="none")
        sm.reset(seed)
        res_all = sm.step(iters)
        X = [sm.x_rhs(c) for c in range(3)]
        rse_all = [sm.trace_rhs(c)[-1]["rse"] for c in range(3)]
        sm.close()
        out["multi_rhs"] = True
        out["seconds_total"] = res_all["seconds"]
    for c in range(3):
        b = B[c]
        if multi_rhs:
            x = np.clip(X[c].reshape(side, side), 0.0, 1.0)
            res = {"rse": rse_all[c], "seconds": res_all["seconds"] / 3}
        else:
            s = Solver.from_scipy(A, b, eta=eta, symmetric=True, stop="none")
            s.reset(seed)
            res = s.step(iters)
            x = np.clip(s.x().reshape(side, side), 0.0, 1.0)
            s.close()
        blurred = b.reshape(side, side)
        out["channels"].append({"psnr": _psnr(x, img[:, :, c]), "ssim": _ssim(x, img[:, :, c]),
                                "psnr_blurred": _psnr(np.clip(blurred, 0, 1), img[:, :, c]),
                                "rse": res["rse"], "seconds": res["seconds"]})
    for k in ("psnr", "ssim", "rse", "psnr_blurred"):
        out["mean_" + k] = float(np.mean([ch[k] for ch in out["channels"]]))
    out["paper"] = {"psnr": [46.59, 50.18, 41.21], "ssim": [0.9982, 0.9980, 0.9878],
                    "avg_rse": [4.303157e-12, 2.474059e-12, 6.247516e-12]}
    return out


def pps_filter(taps=20, sigma=3.0, delay=1, tol=1e-6, eta=0.5, max_iter=200000, seed=0):
    """Predator-prey-scavenger model (eq:predpreyscav, tab:param; x0 = (4, 3, 2),
    T = 200, dt = 0.1), noisy delayed populations s(t) = u(t - delay) + N(0, sigma^2)
    (P:865).  Per species, the filter c solves M c = v with M[i, :] = s[i .. i+taps-1]
    (the noisy delayed population matrix M_v) and v[i] = u[i + taps - 1] (the actual
    population), solved to relative error 1e-6 against the least-squares
    filter M^+ v; the estimate is M c.  Reports the relative error of the estimate and
    of the noisy data against the true populations."""
    traj = pps_trajectory()
    rng = np.random.default_rng(seed)
    S = traj.shape[0]
    out = {"app": "pps_filter", "samples": S, "taps": taps, "species": []}
    for sp_i, name in enumerate(("prey", "predator", "scavenger")):
        u = traj[:, sp_i]
        sig = u[np.maximum(np.arange(S) - delay, 0)] + rng.normal(0.0, sigma, size=S)
        rows = S - taps + 1
        M = np.lib.stride_tricks.sliding_window_view(sig, taps)[:rows].copy()
        v = u[taps - 1:taps - 1 + rows]
        # the system is inconsistent (noise): RGDBEK's extended iteration converges
        # to the least-squares filter M^+ v, the stop reference
        c_ls = np.linalg.lstsq(M, v, rcond=None)[0]
        s = _solver(M, v, eta, stop="rel_err")
        s.set_reference(c_ls)
        res = s.solve(tol, max_iter, seed)
        c = s.x()
        s.close()
        est = M @ c
        out["species"].append({
            "species": name, "iters": res["iters"], "outcome": res["outcome"], "rse": res["rse"],
            "rel_error_estimate": float(np.linalg.norm(est - v) / np.linalg.norm(v)),
            "rel_error_noisy": float(np.linalg.norm(sig[taps - 1:taps - 1 + rows] - v) / np.linalg.norm(v))})
    return out

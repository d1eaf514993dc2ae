"""Property-based pins of the oracle (hypothesis): invariants that must hold for
every input, fixed by the mathematics of Algorithm 1 rather than by
re-typing the oracle's formulas.
"""
import numpy as np
import pytest
from hypothesis import HealthCheck, given, settings, strategies as st

from oracle import Oracle, block_hash, sample_keys, select_block
from oracle.rgdbek import block_size, greedy_block

SETTINGS = dict(max_examples=25, deadline=None, suppress_health_check=[HealthCheck.too_slow])


def _system(seed, m, n, noise):
    rng = np.random.default_rng(seed)
    A = rng.standard_normal((m, n))
    if m > 3:                                    # an empty row and a zero column (reading R6)
        A[rng.integers(m)] = 0.0
        A[:, rng.integers(n)] = 0.0
    b = A @ rng.standard_normal(n) + noise * rng.standard_normal(m)
    if not np.any(b):
        b[0] = 1.0
    return A, b


@settings(**SETTINGS)
@given(seed=st.integers(0, 2**31 - 1), m=st.integers(2, 40), n=st.integers(2, 40),
       eta=st.floats(0.05, 0.95), noise=st.sampled_from([0.0, 0.3]))
def test_sweep_invariants(seed, m, n, eta, noise):
    A, b = _system(seed, m, n, noise)
    o = Oracle(A, b, eta)
    Ab = A @ np.linalg.pinv(A)
    r_opt = b - Ab @ b                          # (I - A A^+) b, Theorem 1
    _, s, Vt = np.linalg.svd(A)
    rank = int(np.sum(s > 1e-10 * max(s[0], 1e-300)))
    prev = np.linalg.norm(o.z - r_opt)
    for k in range(6):
        rec = o.iterate(seed)
        # block sizes: k' = min(round(eta d), #positive scores) (readings R2, R6)
        assert rec.kp <= block_size(eta, n) and rec.kpp <= block_size(eta, m)
        # z_k - r stays in range(A) and its norm never grows (eq:res_norm_evolve)
        e = o.z - r_opt
        assert np.linalg.norm(e - Ab @ e) <= 1e-8 * max(np.linalg.norm(b), 1.0)
        cur = np.linalg.norm(e)
        assert cur <= prev * (1 + 1e-12) + 1e-12
        prev = cur
        # x_k in range(A^T) (x_0 = 0, every update is a multiple of A^T xi)
        null_part = Vt[rank:] @ o.x
        assert np.linalg.norm(null_part) <= 1e-8 * max(np.linalg.norm(o.x), 1e-300)


@settings(**SETTINGS)
@given(seed=st.integers(0, 2**31 - 1), d=st.integers(1, 300), frac=st.floats(0.0, 1.0),
       zeros=st.integers(0, 50))
def test_sampler_block_properties(seed, d, frac, zeros):
    rng = np.random.default_rng(seed)
    eps = rng.exponential(size=d) * rng.choice([1e-8, 1.0, 1e8], size=d)
    eps[rng.choice(d, size=min(zeros, d), replace=False)] = 0.0
    kk = min(max(1, int(frac * d)), int(np.count_nonzero(eps > 0)))
    keys = sample_keys(eps, seed, 3, 1)
    U = select_block(keys, kk, eps > 0)
    assert len(U) == kk == len(np.unique(U))
    assert np.all(eps[U] > 0)                  # zero scores are never sampled
    if kk:
        # the block is exactly the kk smallest keys: every outsider's key is >= every member's
        out = np.setdiff1d(np.arange(d)[eps > 0], U)
        if len(out):
            assert keys[out].min() >= keys[U].max()
    # order-free hash
    assert block_hash(U) == block_hash(U[::-1])


@settings(**SETTINGS)
@given(seed=st.integers(0, 2**31 - 1), d=st.integers(1, 200), eta=st.floats(0.01, 1.0))
def test_greedy_block_properties(seed, d, eta):
    eps = np.random.default_rng(seed).random(d) ** 3
    U = greedy_block(eps, eta)
    assert int(np.argmax(eps)) in U.tolist()
    inside = np.zeros(d, dtype=bool)
    inside[U] = True
    assert np.all(eps[inside] >= eta * eps.max()) and np.all(eps[~inside] < eta * eps.max())

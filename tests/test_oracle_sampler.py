"""Pins of the oracle's Philox stream, U01 map, hash and block sampler.

The sampler realises "select n*eta columns using probability P(j_k)"
(Alg. 1 line 7) and "m*eta rows using P(i_k)" by exponential
keys (reading R3).  Pinned against: Random123 KATs, the closed-form inclusion
probabilities of successive sampling, exhaustive enumeration on tiny inputs,
and the degenerate cases of SPEC S:153-160.
"""
import itertools

import numpy as np
import pytest

from conftest import read_golden_rows
from oracle.philox import philox4x32_10, u01, uniforms
from oracle.rgdbek import block_hash, block_size, sample_keys, scores, select_block, splitmix64

pytestmark = pytest.mark.filterwarnings("error")


def test_philox_known_answers():
    rows = read_golden_rows("philox4x32_10_kat.txt")
    assert len(rows) == 3
    for r in rows:
        ctr = [int(t, 16) for t in r[0:4]]
        key = [int(t, 16) for t in r[4:6]]
        want = [int(t, 16) for t in r[6:10]]
        got = philox4x32_10(*ctr, *key)
        assert [int(g) for g in got] == want


def test_u01_exact_range_and_endpoints():
    lo = u01(np.uint32(0), np.uint32(0))
    hi = u01(np.uint32(0xFFFFFFFF), np.uint32(0xFFFFFFFF))
    assert lo == 2.0 ** -53
    assert hi == 1.0 - 2.0 ** -53
    assert hi < 1.0 and lo > 0.0
    u = uniforms(np.arange(200000), 7, 1, 12345)
    assert u.min() > 0 and u.max() < 1
    # odd multiples of 2^-53: exactly representable, so (u * 2^53) is an odd integer
    t = u * 2.0 ** 53
    assert np.all(t == np.floor(t)) and np.all(np.mod(t, 2) == 1)
    # mean / variance of U(0,1) within 5 sigma
    assert abs(u.mean() - 0.5) < 5 * np.sqrt(1 / 12 / u.size)


def test_streams_are_distinct_and_deterministic():
    a = uniforms(np.arange(64), 3, 0, 99)
    assert np.array_equal(a, uniforms(np.arange(64), 3, 0, 99))
    assert not np.array_equal(a, uniforms(np.arange(64), 3, 1, 99))   # step
    assert not np.array_equal(a, uniforms(np.arange(64), 4, 0, 99))   # iteration
    assert not np.array_equal(a, uniforms(np.arange(64), 3, 0, 98))   # seed
    # the stream of an index does not depend on which other indices are drawn
    assert np.array_equal(uniforms(np.arange(10, 20), 3, 0, 99), a[10:20])


def test_splitmix_and_hash():
    rows = read_golden_rows("splitmix64.txt")
    for state, first in rows:
        assert int(splitmix64(int(state, 16))[0]) == int(first, 16)
    assert block_hash([]) == 0
    assert block_hash([5, 1, 9]) == block_hash([9, 5, 1])
    h = sum(int(splitmix64(i)[0]) for i in (1, 5, 9)) % (1 << 64)
    assert block_hash([1, 5, 9]) == h


def test_block_size_rounding():
    # reading R2: k = max(1, floor(eta d + 1/2))
    assert block_size(0.5, 50) == 25
    assert block_size(0.5, 5) == 3
    assert block_size(0.1, 4) == 1
    assert block_size(0.1, 1048576) == 104858
    assert block_size(0.01, 3) == 1


def test_scores_spec_examples():
    # A = [[1,0],[0,2]], z = (1,1) -> (1, 1); z = 0 -> 0
    A = np.array([[1.0, 0.0], [0.0, 2.0]])
    gamma = (A * A).sum(axis=0)
    assert np.array_equal(scores(A.T @ np.ones(2), gamma), [1.0, 1.0])
    assert np.array_equal(scores(A.T @ np.zeros(2), gamma), [0.0, 0.0])
    # identity, b=(2,0), z=0, x=0 -> (4, 0); empty row -> 0
    assert np.array_equal(scores(np.array([2.0, 0.0]), np.ones(2)), [4.0, 0.0])
    assert np.array_equal(scores(np.array([3.0, 1.0]), np.array([0.0, 1.0])), [0.0, 1.0])


def _draw_many(eps, kk, ndraws, seed=2024, step=0):
    """Blocks of size kk drawn by the oracle at iterations k = 0..ndraws-1."""
    return np.array([select_block(sample_keys(eps, seed, k, step), kk) for k in range(ndraws)])


def test_k1_selection_probability_matches_normalised_scores():
    # P(j) = eps_j / sum eps; SPEC S:155 example (0.75, 0.25)
    eps = np.array([3.0, 1.0, 0.5, 0.0])
    nd = 20000
    sel = _draw_many(eps, 1, nd)[:, 0]
    freq = np.bincount(sel, minlength=4) / nd
    p = eps / eps.sum()
    assert freq[3] == 0.0
    assert np.all(np.abs(freq - p) <= 5 * np.sqrt(p * (1 - p) / nd) + 1e-12)
    eps2 = np.array([0.75, 0.25])
    f2 = np.bincount(_draw_many(eps2, 1, nd, seed=7)[:, 0], minlength=2) / nd
    assert abs(f2[0] - 0.75) < 0.01


def _successive_inclusion(p, kk):
    """Exact P(j in S) for successive sampling without replacement, by enumeration."""
    d = len(p)
    incl = np.zeros(d)
    for seq in itertools.permutations(range(d), kk):
        prob, rest = 1.0, 1.0
        for j in seq:
            prob *= p[j] / rest
            rest -= p[j]
        for j in seq:
            incl[j] += prob
    return incl


def test_k2_closed_form_inclusion():
    p = np.array([0.4, 0.3, 0.2, 0.1])
    closed = np.array([p[j] + sum(p[i] * p[j] / (1 - p[i]) for i in range(4) if i != j)
                       for j in range(4)])
    np.testing.assert_allclose(closed, [0.71587, 0.60833, 0.44127, 0.23452], atol=5e-6)
    np.testing.assert_allclose(_successive_inclusion(p, 2), closed, rtol=1e-12)
    nd = 20000
    blocks = _draw_many(p, 2, nd, seed=11)
    freq = np.bincount(blocks.ravel(), minlength=4) / nd
    assert np.all(np.abs(freq - closed) <= 5 * np.sqrt(closed * (1 - closed) / nd))


def test_k3_of_5_exhaustive_enumeration():
    p = np.array([0.05, 0.35, 0.15, 0.25, 0.2])
    exact = _successive_inclusion(p, 3)
    assert abs(exact.sum() - 3.0) < 1e-12
    nd = 20000
    blocks = _draw_many(p * 7.0, 3, nd, seed=5)        # unnormalised scores
    freq = np.bincount(blocks.ravel(), minlength=5) / nd
    assert np.all(np.abs(freq - exact) <= 5 * np.sqrt(exact * (1 - exact) / nd))


def test_degenerate_blocks():
    # point mass, k = n, no duplicates, clamp to positive count
    eps = np.array([1.0, 0.0, 0.0])
    for k in range(20):
        assert select_block(sample_keys(eps, 3, k, 0), 1).tolist() == [0]
    eps = np.ones(6)
    assert select_block(sample_keys(eps, 3, 0, 0), 6).tolist() == list(range(6))
    eps = np.array([0.0, 2.0, 0.0, 1.0, 5.0])
    kappa = sample_keys(eps, 1, 0, 1)
    assert np.isinf(kappa[[0, 2]]).all() and np.isfinite(kappa[[1, 3, 4]]).all()
    assert select_block(kappa, 3).tolist() == [1, 3, 4]
    blk = select_block(sample_keys(np.random.default_rng(0).random(1000), 9, 4, 0), 400)
    assert len(np.unique(blk)) == 400


def test_ties_broken_by_lower_index():
    kappa = np.array([2.0, 1.0, 1.0, 1.0, 0.5])
    assert select_block(kappa, 3).tolist() == [1, 2, 4]


def test_scale_invariance_of_selection():
    eps = np.random.default_rng(1).random(500) * 10
    for k in range(5):
        a = select_block(sample_keys(eps, 17, k, 0), 100)
        b = select_block(sample_keys(eps * 4.0, 17, k, 0), 100)
        assert np.array_equal(a, b)

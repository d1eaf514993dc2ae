"""Philox4x32-10 counter-based generator and the U01 map — ORACLE SIDE.

TEST INFRASTRUCTURE ONLY: nothing under ``oracle/`` may be imported by the
product path (``paper_2509_19267_b200``).  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs use it.

Why a counter-based generator: the paper samples the blocks "using
probability P(j_k)" (Alg. 1 line 7) and "P(i_k)" (PAPER.md:121,
Alg. 1 line 12) without fixing a generator; BASELINE.json's north_star names a
"Philox counter-based sampler" so that the oracle and the GPU draw the SAME
uniforms without sharing code.  This module is an independent re-statement of
Philox4x32-10 (Salmon, Moraes, Dror, Shaw, "Parallel random numbers: as easy as
1, 2, 3", SC'11); it is pinned by the Random123 known-answer vectors in
``tests/golden/philox4x32_10_kat.txt``.

Counter / key layout (reading R5):
    ctr = (index, k mod 2^32, step, k >> 32), key = (seed mod 2^32, seed >> 32)
    step = 0 for the column step, 1 for the row step; index is GLOBAL.

U01 (reading R6): u = (w >> 12) * 2^-52 + 2^-53 with
w = (o1 << 32) | o0, so u is an odd multiple of 2^-53 in [2^-53, 1 - 2^-53]:
exactly representable, never 0 or 1, so -log(u) is finite and > 0.
"""
import numpy as np

PHILOX_M0 = np.uint64(0xD2511F53)
PHILOX_M1 = np.uint64(0xCD9E8D57)
PHILOX_W0 = 0x9E3779B9
PHILOX_W1 = 0xBB67AE85
_MASK32 = np.uint64(0xFFFFFFFF)


def philox4x32_10(c0, c1, c2, c3, k0, k1):
    """Ten Philox-4x32 rounds on arrays of 32-bit counters (broadcasting).

    One round (SC'11, Philox-4x32):
        (hi0, lo0) = mulhilo(M0, c0); (hi1, lo1) = mulhilo(M1, c2)
        c' = (hi1 ^ c1 ^ k0, lo1, hi0 ^ c3 ^ k1, lo0)
    and the key is bumped by the Weyl constants (W0, W1) between rounds.
    Returns four uint32 arrays.
    """
    c0 = np.asarray(c0, dtype=np.uint64) & _MASK32
    c1 = np.asarray(c1, dtype=np.uint64) & _MASK32
    c2 = np.asarray(c2, dtype=np.uint64) & _MASK32
    c3 = np.asarray(c3, dtype=np.uint64) & _MASK32
    k0 = int(k0) & 0xFFFFFFFF
    k1 = int(k1) & 0xFFFFFFFF
    for rnd in range(10):
        if rnd > 0:
            k0 = (k0 + PHILOX_W0) & 0xFFFFFFFF
            k1 = (k1 + PHILOX_W1) & 0xFFFFFFFF
        p0 = PHILOX_M0 * c0          # < 2^64: exact in uint64
        p1 = PHILOX_M1 * c2
        hi0, lo0 = p0 >> np.uint64(32), p0 & _MASK32
        hi1, lo1 = p1 >> np.uint64(32), p1 & _MASK32
        c0, c1, c2, c3 = (hi1 ^ c1 ^ np.uint64(k0), lo1,
                          hi0 ^ c3 ^ np.uint64(k1), lo0)
    return (c0.astype(np.uint32), c1.astype(np.uint32),
            c2.astype(np.uint32), c3.astype(np.uint32))


def u01(o0, o1):
    """Map two 32-bit Philox outputs to u in [2^-53, 1 - 2^-53] exactly."""
    w = (np.asarray(o1, dtype=np.uint64) << np.uint64(32)) | np.asarray(o0, dtype=np.uint64)
    return (w >> np.uint64(12)).astype(np.float64) * 2.0 ** -52 + 2.0 ** -53


def uniforms(indices, k, step, seed):
    """The uniform u(seed, k, step, index) for every index in ``indices``."""
    idx = np.asarray(indices, dtype=np.uint64)
    k = int(k)
    seed = int(seed) & 0xFFFFFFFFFFFFFFFF
    o0, o1, _, _ = philox4x32_10(idx, np.uint64(k & 0xFFFFFFFF), np.uint64(step),
                                 np.uint64((k >> 32) & 0xFFFFFFFF),
                                 seed & 0xFFFFFFFF, seed >> 32)
    return u01(o0, o1)

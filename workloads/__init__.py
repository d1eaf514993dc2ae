"""Seeded synthetic workload generators shared by tests, bench.py and smoke().

This package holds NONE of the method's arithmetic: it only builds (A, b) and
the ground truth (x*, r) that the problem statement A x = b and
Theorem 1's limits x* = A^+ b, r = (I - A A^+) b refer to.
"""
from .gen import (Workload, dense_gaussian, poisson2d, poisson_fem_paper,
                  toeplitz_blur, popmodel, sparse_random, by_name, CONFIGS)

__all__ = ["Workload", "dense_gaussian", "poisson2d", "poisson_fem_paper",
           "toeplitz_blur", "popmodel", "sparse_random", "by_name", "CONFIGS"]

"""One multi-RHS solve run for ncu: python tools/run_multi.py C4 3 [steps]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
from workloads import by_name
from paper_2509_19267_b200 import Solver

w = by_name(sys.argv[1])
nr = int(sys.argv[2])
k = int(sys.argv[3]) if len(sys.argv) > 3 else 3
rng = np.random.default_rng(0)
B = np.array([w.b] + [w.A @ rng.random(w.shape[1]) for _ in range(nr - 1)])
s = Solver.from_scipy_multi(w.A, B, eta=w.eta)
s.reset(0)
print(s.step(k))

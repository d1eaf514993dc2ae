"""Create one workload's solver and run step(K) once (a short command for ncu)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from workloads import by_name
from paper_2509_19267_b200 import Solver

name = sys.argv[1] if len(sys.argv) > 1 else "C2c"
k = int(sys.argv[2]) if len(sys.argv) > 2 else 3
w = by_name(name)
s = Solver(w.A, w.b, eta=w.eta) if w.dense else Solver.from_scipy(w.A, w.b, eta=w.eta, symmetric=w.symmetric)
s.reset(0)
r = s.step(k)
print(name, k, r)

"""One standalone hot pass of a workload, for ncu: python tools/run_pass.py C4 N|T [reps]
(rgdbek_launch_kernel: the graph engine's k_csr_tiles / dense pass kernels)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from workloads import by_name
from paper_2509_19267_b200 import Solver

name, kind = sys.argv[1], sys.argv[2]
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
w = by_name(name)
s = Solver(w.A, w.b, eta=w.eta) if w.dense else Solver.from_scipy(w.A, w.b, eta=w.eta, symmetric=w.symmetric)
s.reset(0)
s.step(2)
b = s.launch_kernel(0 if kind == "T" else 1, reps)
import ctypes
print(name, kind, reps, b)

"""A/B of library variants on the standalone sparse / dense passes and the full iteration.

usage: python tools/ab_pass.py "C4,C5s" base build_ab/librgdbek_x.so ... [--reps 2]
For each (variant, workload): standalone pass T and pass N (rgdbek_launch_kernel, CUDA
events on the solver stream; both products) in GB/s of the library's algorithmic bytes,
and the persistent engine's it/s over 200 iterations.  Interleaved repetitions, medians.
"""
import json
import os
import statistics
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r"""
import json, os, sys
sys.path.insert(0, %r)
import torch
from workloads import by_name
from paper_2509_19267_b200 import Solver
w = by_name(sys.argv[1])
s = Solver(w.A, w.b, eta=w.eta) if w.dense else Solver.from_scipy(w.A, w.b, eta=w.eta, symmetric=w.symmetric)
st = torch.cuda.ExternalStream(s.stream)
out = {}
s.reset(0); s.step(3)
for kid, nm in ((0, "T"), (1, "N")):
    s.launch_kernel(kid, 3)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); e0.record(st)
    b = s.launch_kernel(kid, 20)
    e1.record(st); torch.cuda.synchronize()
    dt = e0.elapsed_time(e1) * 1e-3 / 20
    out["pass" + nm + "_gbs"] = b / dt / 1e9
s.reset(0); s.step(5); s.reset(0)
r = s.step(200)
out["it_s"] = 200 / r["seconds"]
print(json.dumps(out))
""" % ROOT


def main():
    argv = sys.argv[1:]
    reps = 2
    if "--reps" in argv:
        i = argv.index("--reps"); reps = int(argv[i + 1]); del argv[i:i + 2]
    wls = argv[0].split(",")
    variants = argv[1:]
    res = {}
    for _ in range(reps):
        for v in variants:
            env = dict(os.environ)
            if v != "base":
                env["RGDBEK_LIB"] = os.path.join(ROOT, v) if not os.path.isabs(v) else v
            for wl in wls:
                out = subprocess.run([sys.executable, "-c", CHILD, wl], env=env,
                                     capture_output=True, text=True, timeout=900)
                try:
                    d = json.loads(out.stdout.strip().splitlines()[-1])
                except Exception:
                    sys.stderr.write(out.stderr[-2000:])
                    d = {}
                for k, x in d.items():
                    res.setdefault((v, wl, k), []).append(x)
    rows = {}
    for (v, wl, k), xs in res.items():
        rows.setdefault((v, wl), {})[k] = round(statistics.median(xs), 1)
    for (v, wl), d in rows.items():
        print(json.dumps({"variant": os.path.basename(v), "workload": wl, **d}), flush=True)


if __name__ == "__main__":
    main()

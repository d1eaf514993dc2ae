"""A/B timing of library variants on one box (interleaved repetitions).

usage: python tools/ab_run.py "C3,C4,C5s" base build_ab/librgdbek_x.so ... [--steps 300 --reps 2]
'base' = the in-tree library; 'env:K=V[,K2=V2]' = the in-tree library under those
environment variables; 'LIB|K=V[,K2=V2]' = a variant library under them.  Prints it/s per (variant, workload), median over reps.
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
from workloads import by_name
from paper_2509_19267_b200 import Solver
w = by_name(sys.argv[1]); steps = int(sys.argv[2])
s = Solver(w.A, w.b, eta=w.eta) if w.dense else Solver.from_scipy(w.A, w.b, eta=w.eta, symmetric=w.symmetric)
s.reset(0); s.step(5); s.reset(0)
r = s.step(steps)
print(json.dumps({"it_s": steps / r["seconds"]}))
""" % ROOT


def main():
    argv = sys.argv[1:]
    steps, reps = 300, 2
    if "--steps" in argv:
        i = argv.index("--steps"); steps = int(argv[i + 1]); del argv[i:i + 2]
    if "--reps" in argv:
        i = argv.index("--reps"); reps = int(argv[i + 1]); del argv[i:i + 2]
    wls = argv[0].split(",")
    variants = argv[1:]
    res = {}
    for _ in range(reps):
        for v in variants:
            env = dict(os.environ)
            lib, _, envs = v.partition("|")          # "lib|K=V,..." = a library under env vars
            if lib.startswith("env:"):
                lib, envs = "base", lib[4:]
            if envs:
                env.update(kv.split("=", 1) for kv in envs.split(","))
            if lib != "base":
                env["RGDBEK_LIB"] = os.path.join(ROOT, lib) if not os.path.isabs(lib) else lib
            for wl in wls:
                out = subprocess.run([sys.executable, "-c", CHILD, wl, str(steps)], env=env,
                                     capture_output=True, text=True, timeout=600)
                try:
                    it = json.loads(out.stdout.strip().splitlines()[-1])["it_s"]
                except Exception:
                    sys.stderr.write(out.stderr[-2000:])
                    it = float("nan")
                res.setdefault((v, wl), []).append(it)
    for (v, wl), xs in res.items():
        print(json.dumps({"variant": v if ("env:" in v or "|" in v) else os.path.basename(v), "workload": wl,
                          "it_s": round(statistics.median(xs), 1), "all": [round(x, 1) for x in xs]}))


if __name__ == "__main__":
    main()

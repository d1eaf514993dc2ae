"""A/B of the multi-RHS kernel: it/s of C4 / C3 with nr right-hand sides across variants.
usage: python tools/ab_multi.py "C4,C3" "2,3,4" base build_ab/librgdbek_x.so ... [--reps 2]"""
import json, os, statistics, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r"""
import json, sys
sys.path.insert(0, %r)
import numpy as np
from workloads import by_name
from paper_2509_19267_b200 import Solver
w = by_name(sys.argv[1]); nr = int(sys.argv[2])
rng = np.random.default_rng(0)
B = np.array([w.b] + [w.A @ rng.random(w.shape[1]) for _ in range(nr - 1)])
s = Solver.from_scipy_multi(w.A, B, eta=w.eta) if nr > 1 else Solver.from_scipy(w.A, w.b, eta=w.eta, symmetric=w.symmetric)
s.reset(0); s.step(5); s.reset(0)
r = s.step(300)
print(json.dumps({"it_s": 300 / r["seconds"], "rhs_it_s": nr * 300 / r["seconds"]}))
""" % ROOT
argv = sys.argv[1:]
reps = 2
if "--reps" in argv:
    i = argv.index("--reps"); reps = int(argv[i + 1]); del argv[i:i + 2]
wls, nrs, variants = argv[0].split(","), [int(x) for x in argv[1].split(",")], argv[2:]
res = {}
for _ in range(reps):
    for v in variants:
        env = dict(os.environ)
        if v != "base":
            env["RGDBEK_LIB"] = os.path.join(ROOT, v)
        for wl in wls:
            for nr in nrs:
                out = subprocess.run([sys.executable, "-c", CHILD, wl, str(nr)], env=env, capture_output=True, text=True, timeout=900)
                try:
                    d = json.loads(out.stdout.strip().splitlines()[-1])
                except Exception:
                    sys.stderr.write(out.stderr[-1500:]); d = {}
                for k, x in d.items():
                    res.setdefault((v, wl, nr, k), []).append(x)
rows = {}
for (v, wl, nr, k), xs in res.items():
    rows.setdefault((v, wl, nr), {})[k] = round(statistics.median(xs), 1)
for (v, wl, nr), d in rows.items():
    print(json.dumps({"variant": os.path.basename(v), "workload": wl, "nr": nr, **d}), flush=True)

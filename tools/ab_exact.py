"""A/B of the exact mode (time to rel. error 1e-6 on C2c, passes, A bytes) across library variants.
usage: python tools/ab_exact.py base build_ab/librgdbek_x.so ... [--reps 2]"""
import json, os, statistics, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r"""
import json, sys
sys.path.insert(0, %r)
from workloads import by_name
from paper_2509_19267_b200 import Solver
w = by_name("C2c")
s = Solver(w.A, w.b, eta=0.5, stop="rel_err")
s.set_mode("exact", inner_tol=1e-13, inner_max=200)
s.set_reference(w.xstar)
s.solve(1e-6, 1000, 0)
r = s.solve(1e-6, 1000, 0)
print(json.dumps({"seconds": r["seconds"], "iters": r["iters"], "passes": s.passes(), "a_gb": s.a_bytes() / 1e9}))
""" % ROOT
argv = sys.argv[1:]
reps = 2
if "--reps" in argv:
    i = argv.index("--reps"); reps = int(argv[i + 1]); del argv[i:i + 2]
res = {}
for _ in range(reps):
    for v in argv:
        env = dict(os.environ)
        if v != "base":
            env["RGDBEK_LIB"] = os.path.join(ROOT, v)
        out = subprocess.run([sys.executable, "-c", CHILD], env=env, capture_output=True, text=True, timeout=900)
        try:
            d = json.loads(out.stdout.strip().splitlines()[-1])
        except Exception:
            sys.stderr.write(out.stderr[-2000:]); d = {}
        for k, x in d.items():
            res.setdefault((v, k), []).append(x)
for v in argv:
    print(json.dumps({"variant": os.path.basename(v), **{k: statistics.median(res[(v, k)]) for (vv, k) in res if vv == v}}))

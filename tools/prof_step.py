"""Profiling driver: one refinement step on a quick synthetic system.
python tools/prof_step.py N uf u ur [m k]"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2201_09827_b200 import _lib
from paper_2201_09827_b200.precision import PrecisionTriple
from paper_2201_09827_b200.refine import Method, RefineConfig, make_options
n = int(sys.argv[1]); uf, u, ur = sys.argv[2:5]
m = int(sys.argv[5]) if len(sys.argv) > 5 else 100
k = int(sys.argv[6]) if len(sys.argv) > 6 else 20
steps = int(os.environ.get("STEPS", "1"))
rng = np.random.default_rng(0)
a = rng.standard_normal((n, n)) / np.sqrt(n) + 0.0 * np.eye(n)
b = rng.standard_normal(n)
cfg = RefineConfig(PrecisionTriple.parse(uf, u, ur), Method.RGMRES_IR, m=m, k=k, tau=1e-10, i_max=steps)
s = _lib.Solver(n, make_options(cfg, n, int(os.environ.get("GRID", "0"))))
s.set_system(a, b)
t0 = time.time(); z, g = s.factorize(); print("factor ms", s.last_factor_ms, "zero", z, "growth", g)
s.initial_solution(); ok = s.reference_solution(); print("xref", ok)
import collections
for i in range(steps):
    s.phaselog(20000, read=False)
    info = s.step(); cyc, ke = s.last_cycles()
    log = s.phaselog(0)
    acc = collections.defaultdict(float); cnt = collections.Counter()
    for (t0, a), (t1, b) in zip(log[:-1], log[1:]):
        acc[(t0, t1)] += (b - a) / 1e3; cnt[(t0, t1)] += 1
    for key, v in sorted(acc.items(), key=lambda kv: -kv[1])[:12]:
        print("   %s->%s: total %.1f us, n %d, avg %.2f us" % (key[0], key[1], v, cnt[key], v / cnt[key]))
    print("step ms %.2f applies %d its %d cycles %s keff %s nbe %.2e" % (s.last_step_ms, info.applies, info.inner_iters, cyc[:6], ke[:6], info.nbe))

"""Run one benchmark configuration through the drop-in API and compare with
its golden (if any).  Usage: python tools/run_config.py cfg4 [--n N] [--method M]"""
import argparse, json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2201_09827_b200 import problems
from paper_2201_09827_b200.precision import PrecisionTriple
from paper_2201_09827_b200.refine import Method, RefineConfig, _refine

ap = argparse.ArgumentParser()
ap.add_argument("cfg")
ap.add_argument("--n", type=int, default=None)
ap.add_argument("--method", default="rgmres-ir")
ap.add_argument("--grid", type=int, default=0)
ap.add_argument("--imax", type=int, default=None)
ap.add_argument("--max-cycles", type=int, default=None)
ap.add_argument("--lu-mode", default="exact")
args = ap.parse_args()
spec = problems.CONFIGS[args.cfg]
t0 = time.perf_counter()
a, b = problems.config_problem(spec, 0, args.n)
t1 = time.perf_counter()
cfg = RefineConfig(PrecisionTriple.parse(*spec.precisions), Method.parse(args.method), m=spec.m,
                   k=spec.k if args.method.startswith("r") else 0, tau=spec.tau, i_max=args.imax or spec.i_max,
                   max_cycles=args.max_cycles, lu_mode=args.lu_mode)
trace = []
if os.environ.get("PHASES"):
    import collections
    from paper_2201_09827_b200 import _lib
    orig_step = _lib.Solver.step
    def step(self):
        self.phaselog(200000, read=False)
        info = orig_step(self)
        log = self.phaselog(0)
        acc = collections.defaultdict(float); cnt = collections.Counter()
        for (t0, a0), (t1, b1) in zip(log[:-1], log[1:]):
            acc[(t0, t1)] += (b1 - a0) / 1e3; cnt[(t0, t1)] += 1
        tot = sum(acc.values())
        for key, v in sorted(acc.items(), key=lambda kv: -kv[1])[:16]:
            print("   %s->%s: %5.1f%% total %.1f us, n %d, avg %.2f us" % (key[0], key[1], 100 * v / tot, v, cnt[key], v / cnt[key]))
        return info
    _lib.Solver.step = step
rep = _refine(a, b, cfg, trace=trace, grid_ctas=args.grid)
t2 = time.perf_counter()
print(f"gen {t1-t0:.1f}s solve {t2-t1:.2f}s")
print("converged", rep.converged, "inner", rep.inner_iters, "reason", rep.divergence_reason)
print("nbe", rep.nbe_history, "ferr", rep.ferr_history, rep.diagnostics)
for t in trace:
    print({k: (v if k != "cycles" else (v[:12], len(v), sum(v))) for k, v in t.items() if k != "k_eff"}, "keff", t["k_eff"][:12])

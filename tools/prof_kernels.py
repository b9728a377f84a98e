"""Bounded single launches for ncu captures.
  python tools/prof_kernels.py step N uf u ur m k cycles   -- one refinement step capped at `cycles` cycles
  python tools/prof_kernels.py lu N uf u ur mode           -- one factorisation (mode exact|tensor)
Random well-conditioned system (seed 0); prints the CUDA-event time of the launch."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2201_09827_b200 import _lib
from paper_2201_09827_b200.precision import PrecisionTriple
from paper_2201_09827_b200.refine import Method, RefineConfig, make_options

what, n = sys.argv[1], int(sys.argv[2])
uf, u, ur = sys.argv[3:6]
rng = np.random.default_rng(0)
a = rng.standard_normal((n, n)) / np.sqrt(n) + 4.0 * np.eye(n)
b = rng.standard_normal(n)
if what == "step":
    m, k, cyc = int(sys.argv[6]), int(sys.argv[7]), int(sys.argv[8])
    cfg = RefineConfig(PrecisionTriple.parse(uf, u, ur), Method.RGMRES_IR, m=m, k=k, tau=1e-30, i_max=1,
                       max_cycles=cyc)
else:
    cfg = RefineConfig(PrecisionTriple.parse(uf, u, ur), Method.RGMRES_IR, m=20, k=4, i_max=1,
                       lu_mode=sys.argv[6])
s = _lib.Solver(n, make_options(cfg, n))
s.set_system(a, b)
z, g = s.factorize()
print(f"factor ms {s.last_factor_ms:.3f} zero {z} growth {g:.3g}")
if what == "step":
    s.initial_solution()
    s.reference_solution()
    info = s.step()
    print(f"step ms {s.last_step_ms:.3f} applies {info.applies} its {info.inner_iters}")

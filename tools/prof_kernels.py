"""Bounded single launches for ncu captures (seeded N(0,1/n) + 4I system).
  python tools/prof_kernels.py step N uf u ur m k cycles  -- one refinement step capped at `cycles` cycles
  python tools/prof_kernels.py lu N uf u ur mode          -- one factorisation (mode exact|tensor)
  python tools/prof_kernels.py op N uf u ur               -- one apply_preconditioned + one residual launch
  python tools/prof_kernels.py batched                     -- one cfg3 batched launch (4096 x n=128)
Prints the CUDA-event time of the launches."""
import math, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2201_09827_b200 import _lib
from paper_2201_09827_b200.precision import PrecisionTriple
from paper_2201_09827_b200.refine import Method, RefineConfig, make_options

what = sys.argv[1]
if what == "batched":
    import bench
    from paper_2201_09827_b200.batched import solve_batched
    spec = bench._spec("cfg3")
    A, B = bench._inputs(spec, 0)
    cfg = bench._cfg(spec)
    Ad, Bd = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
    for _ in range(2):
        r = solve_batched(None, None, cfg, on_device_ptrs=(Ad.data_ptr(), Bd.data_ptr()), count=spec.batch, n=spec.n)
        print(f"batched ms {r.device_ms:.3f} converged {int(r.converged.sum())}")
    sys.exit(0)
n = int(sys.argv[2])
uf, u, ur = sys.argv[3:6]
gen = torch.Generator(device="cuda").manual_seed(0)
a = torch.randn((n, n), dtype=torch.float64, device="cuda", generator=gen) / math.sqrt(n)
a.diagonal().add_(4.0)
b = torch.randn(n, dtype=torch.float64, device="cuda", generator=gen)
if what == "step":
    m, k, cyc = int(sys.argv[6]), int(sys.argv[7]), int(sys.argv[8])
    cfg = RefineConfig(PrecisionTriple.parse(uf, u, ur), Method.RGMRES_IR, m=m, k=k, tau=1e-30, i_max=1,
                       max_cycles=cyc)
else:
    cfg = RefineConfig(PrecisionTriple.parse(uf, u, ur), Method.RGMRES_IR, m=20, k=4, i_max=1,
                       lu_mode=sys.argv[6] if what == "lu" else "exact")
s = _lib.Solver(n, make_options(cfg, n))
s.set_system_device(a.data_ptr(), b.data_ptr())
z, g = s.factorize()
print(f"factor ms {s.last_factor_ms:.3f} zero {z} growth {g:.3g}")
if what == "step":
    s.initial_solution()
    s.reference_solution()
    info = s.step()
    print(f"step ms {s.last_step_ms:.3f} applies {info.applies} its {info.inner_iters}")
elif what == "op":
    fmt = {"half": 0, "single": 1, "double": 2, "quad": 3}
    sq = {"half": "single", "single": "double", "double": "quad"}[u]
    v = np.random.default_rng(0).standard_normal(n)
    s.apply_preconditioned(v, fmt[sq])
    print(f"op ms {s.time_op(0, 5):.3f}")
    s.residual(v, fmt[ur])
    print(f"residual ms {s.time_op(2, 5):.3f}")

"""Compare the batched device timing with the end-to-end wall time (cfg3)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2201_09827_b200 import problems
from paper_2201_09827_b200.batched import solve_batched
import bench
spec = problems.CONFIGS["cfg3"]
A, B = bench._inputs(spec, 0)
cfg = bench._cfg(spec)
Ad, Bd = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
for it in range(4):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    r = solve_batched(None, None, cfg, on_device_ptrs=(Ad.data_ptr(), Bd.data_ptr()), count=spec.batch, n=spec.n)
    torch.cuda.synchronize(); t1 = time.perf_counter()
    r2 = solve_batched(A, B, cfg)
    torch.cuda.synchronize(); t2 = time.perf_counter()
    print(f"device-ptr: wall {1e3*(t1-t0):.1f} ms kernel {r.device_ms:.1f} ms conv {r.converged.sum()} | host: wall {1e3*(t2-t1):.1f} ms kernel {r2.device_ms:.1f} conv {r2.converged.sum()}")
    print("  inner equal:", np.array_equal(r.inner, r2.inner), "x equal:", np.array_equal(r.x, r2.x))

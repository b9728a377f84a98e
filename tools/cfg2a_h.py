"""cfg2a cold cycle on the device vs the oracle: Hessenberg matrix and the
harmonic-Ritz selection (k_eff) computed from each."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2201_09827_b200 import _lib, problems
from paper_2201_09827_b200.precision import PrecisionTriple
from paper_2201_09827_b200.refine import Method, RefineConfig, make_options

def keff(h, hsub, k=10):
    j = h.shape[0]
    e = np.zeros(j); e[-1] = 1
    w = np.linalg.solve(h.T, e)
    m = h + hsub * hsub * np.outer(w, e)
    vals = np.linalg.eigvals(m); o = np.argsort(np.abs(vals), kind="stable"); vals = vals[o]
    cols, i = 0, 0
    while i < len(vals) and cols < k:
        if vals[i].imag == 0: cols += 1; i += 1; continue
        if cols + 2 <= k + 1: cols += 2; i += 2; continue
        break
    return cols, vals[:12]

spec = problems.CONFIGS["cfg2a"]
a, b = problems.config_problem(spec)
cfg = RefineConfig(PrecisionTriple.parse(*spec.precisions), Method.RGMRES_IR, m=50, k=10, tau=1e-6, i_max=1, max_cycles=1)
s = _lib.Solver(1024, make_options(cfg, 1024))
s.set_system(a, b); s.factorize(); s.initial_solution(); s.reference_solution()
info = s.step()
cyc, ke = s.last_cycles()
H = s.hessenberg()
print("device cycles", cyc, "k_eff", ke)
hd, hsub_d = H[:50, :50], H[50, 49]
ho = np.load(os.path.join(os.path.dirname(__file__), "micro", "data", "h_cfg2a_oracle.npy"))
hsub_o = 0.22003598699005675
print("max |H_dev - H_oracle| = %.3e (|H| %.3e), hsub %.17g vs %.17g" % (np.max(np.abs(hd - ho)), np.max(np.abs(ho)), hsub_d, hsub_o))
rel = np.abs(hd - ho) / np.maximum(np.abs(ho), 1e-300)
print("relative diff by column (max over rows):", np.array2string(np.max(np.where(np.abs(ho) > 0, rel, 0), axis=0)[:50:5], precision=2))
print("k_eff numpy(device H) =", keff(hd, hsub_d)[0], " numpy(oracle H) =", keff(ho, hsub_o)[0])
print(keff(hd, hsub_d)[1][:8])

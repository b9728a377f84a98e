import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, scipy.linalg
from paper_2201_09827_b200 import problems, _lib
from paper_2201_09827_b200.precision import PrecisionTriple
from paper_2201_09827_b200.refine import Method, RefineConfig, make_options
for alpha in (0.434, 0.45, 0.455):
    a = problems.prolate(100, alpha)
    a32 = a.astype(np.float32).astype(np.float64)
    cfg = RefineConfig(PrecisionTriple.parse("single", "double", "quad"), Method.GMRES_IR, m=16)
    s = _lib.Solver(100, make_options(cfg, 100)); s.set_system(a, np.ones(100)); s.factorize()
    lu, perm = s.factors()
    L = np.tril(lu, -1) + np.eye(100); U = np.triu(lu)
    e_ours = np.max(np.abs(a32[perm] - L @ U)) / np.max(np.abs(a32))
    lu2, piv = scipy.linalg.lu_factor(a.astype(np.float32))
    p2 = np.arange(100)
    for i, p in enumerate(piv): p2[i], p2[p] = p2[p], p2[i]
    L2 = np.tril(lu2, -1).astype(np.float64) + np.eye(100); U2 = np.triu(lu2).astype(np.float64)
    e_ref = np.max(np.abs(a32[p2] - L2 @ U2)) / np.max(np.abs(a32))
    first = int(np.argmax(perm != p2)) if np.any(perm != p2) else -1
    print(f"alpha {alpha}: backward err ours {e_ours:.2e} sgetrf {e_ref:.2e}; first pivot diff {first}; growth {np.max(np.abs(U))/np.max(np.abs(a32)):.3f} vs {np.max(np.abs(U2))/np.max(np.abs(a32)):.3f}")
    # preconditioned operator conditioning
    M1 = np.linalg.solve(U, np.linalg.solve(L, a[perm])); M2 = np.linalg.solve(U2, np.linalg.solve(L2, a[p2]))
    print("   cond(U^-1 L^-1 A) ours %.3e ref %.3e" % (np.linalg.cond(M1), np.linalg.cond(M2)))
    s.close()

"""Tensor-core (tcgen05) fp16 LU vs the exact fp16 LU: timing, pivot-prefix
agreement and backward error.  python tools/lu_tc_check.py N [N ...]"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2201_09827_b200 import _lib
from paper_2201_09827_b200.precision import PrecisionTriple
from paper_2201_09827_b200.refine import Method, RefineConfig, make_options
for n in [int(v) for v in sys.argv[1:]]:
    rng = np.random.default_rng(1)
    a = rng.standard_normal((n, n))
    res = {}
    for mode in ("exact", "tensor"):
        cfg = RefineConfig(PrecisionTriple.parse("half", "single", "double"), Method.GMRES_IR, m=min(n, 40), lu_mode=mode)
        s = _lib.Solver(n, make_options(cfg, n))
        s.set_system(a, np.ones(n))
        s.factorize(); z, g = s.factorize()
        ms = s.last_factor_ms
        lu, perm = s.factors()
        st = s.tc_update_stats()
        res[mode] = (ms, z, g, lu, perm)
        s.close()
        print(f"n={n} {mode:6s}: factor {ms:8.2f} ms = {2 * n ** 3 / 3 / ms / 1e9:.1f} TFLOP/s  zero={z} growth={g:.3f}",
              flush=True)
        if st:
            print(f"   tcgen05 trailing updates: {st['ms']:.2f} ms, {st['tflops']:.0f} TFLOP/s, "
                  f"{100 * st['flop_share']:.1f}% of the LU flops; U12 solves {st['trsm_ms']:.2f} ms; "
                  f"panels + interchanges {st['panel_ms']:.2f} ms", flush=True)
    if True:
        a16 = a.astype(np.float32).astype(np.float16).astype(np.float64)
        for mode in ("exact", "tensor"):
            lu, perm = res[mode][3], res[mode][4]
            x = rng.standard_normal(n)
            L = np.tril(lu, -1) + np.eye(n); U = np.triu(lu)
            be = np.max(np.abs(a16[perm] @ x - L @ (U @ x))) / (np.max(np.abs(a16)) * np.max(np.abs(x)) * n)
            print(f"   {mode}: scaled backward error {be:.2e}")
        pe, pt = res["exact"][4], res["tensor"][4]
        d = np.nonzero(pe != pt)[0]
        print("   first pivot difference:", d[0] if d.size else None, "of", n)

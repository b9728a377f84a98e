"""Grid-team operator: parity vs the oracle on the device's own factors (n = 2048)
and device timing at n = 8192 / 16384 (fp16 factors, fp32 A, fp64 operator)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from oracle import cpu_gcrodr_ir as O
from paper_2201_09827_b200 import _lib
from paper_2201_09827_b200.precision import Format, PrecisionTriple
from paper_2201_09827_b200.refine import Method, RefineConfig, make_options

def solver(a, prec, n):
    cfg = RefineConfig(PrecisionTriple.parse(*prec), method=Method.RGMRES_IR, m=20, k=4)
    s = _lib.Solver(n, make_options(cfg, n))
    s.set_system(a, np.ones(n))
    return s

rng = np.random.default_rng(11)
n = 2048
a = rng.standard_normal((n, n)) / np.sqrt(n) + 4.0 * np.eye(n)
s = solver(a, ("half", "single", "double"), n)
z, _ = s.factorize()
lu, perm = s.factors()
F = O.Factors(np.tril(lu, -1) + np.eye(n), np.triu(lu), perm.astype(np.int64), "half", 1.0)
a_u = O.rnd(a, "single")
v = O.rnd(rng.standard_normal(n), "single")
w = s.apply_preconditioned(v, Format.DOUBLE.code)
w_ref = O.apply_op(a_u, F, v, "double", "single")
p = s.precond_rhs(v, Format.DOUBLE.code)
p_ref = O.precond_rhs(F, v, "double", "single")
print("n=2048 operator max rel diff %.3e, precond_rhs %.3e (one fp32 ulp = %.1e)" % (
    np.max(np.abs(w - w_ref)) / np.max(np.abs(w_ref)), np.max(np.abs(p - p_ref)) / np.max(np.abs(p_ref)), 2.0**-23))
print("ulp-exact entries: op %d/%d, prhs %d/%d" % (np.sum(w == w_ref), n, np.sum(p == p_ref), n))
s.close()
import torch
for n in (8192, 16384):
    gen = torch.Generator(device="cuda").manual_seed(1)
    A = torch.randn((n, n), dtype=torch.float64, device="cuda", generator=gen) / np.sqrt(n)
    A.diagonal().add_(4.0)
    b = torch.randn(n, dtype=torch.float64, device="cuda", generator=gen)
    cfg = RefineConfig(PrecisionTriple.parse("half", "single", "double"), Method.RGMRES_IR, m=20, k=4, i_max=1)
    s = _lib.Solver(n, make_options(cfg, n))
    s.set_system_device(A.data_ptr(), b.data_ptr())
    s.factorize()
    print("n=%d LU %.1f ms" % (n, s.last_factor_ms))
    v = np.random.default_rng(0).standard_normal(n)
    s.apply_preconditioned(v, Format.DOUBLE.code)
    t_op = s.time_op(0, 20)
    s.precond_rhs(v, Format.DOUBLE.code)
    t_pr = s.time_op(1, 20)
    s.residual(v, Format.DOUBLE.code)
    t_res = s.time_op(2, 20)
    ob = n * n * 6
    print("n=%d apply %.1f us = %.0f GB/s (%.1f%% of 6451.5), precond_rhs %.1f us, residual %.1f us" % (
        n, t_op * 1e3, ob / (t_op * 1e-3) / 1e9, 100 * ob / (t_op * 1e-3) / 1e9 / 6451.5, t_pr * 1e3, t_res * 1e3))
    s.close(); del A, b; torch.cuda.empty_cache()

"""Pin the CPU oracle (oracle/cpu_gcrodr_ir.py) against the reference's own
outputs captured in tests/golden/ (make_goldens.py ran the reference).

The oracle restates the reference with the same numpy/scipy calls, so on the
same BLAS build and thread count it must agree bit for bit; the fixtures were
captured with OPENBLAS_NUM_THREADS=1, which these tests also need
for the fp32-LU and fp64-GEMV paths (set in the environment of the run).
"""

import math
import os

import numpy as np
import pytest

from conftest import golden_json, golden_npz
from oracle import cpu_gcrodr_ir as O
from paper_2201_09827_b200 import problems

SINGLE_THREAD = os.environ.get("OPENBLAS_NUM_THREADS") == "1"


def test_problem_generators_match_reference_matgen():
    meta = golden_json("precision")["matgen"]
    import hashlib

    def sha(a):
        return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()

    assert sha(problems.prolate(100, 0.45)) == meta["prolate_100_0.45"]
    assert sha(problems.prolate(1024, 0.45)) == meta["prolate_1024_0.45"]
    if SINGLE_THREAD:
        assert sha(problems.randsvd(100, 1e4, 1)) == meta["randsvd_100_10000_1"]
        assert sha(problems.randsvd(128, 1e3, 7)) == meta["randsvd_128_1000_7"]


def test_rounding_and_dd_primitives():
    z = golden_npz("precision")
    assert np.array_equal(O.rnd(z["x"], O.HALF), z["half"])
    assert np.array_equal(O.rnd(z["x"], O.SINGLE), z["single"])
    a, al, b, bl = z["a"], z["al"], z["b"], z["bl"]
    for name, fn in [("add", O.dd_add), ("mul", O.dd_mul), ("div", O.dd_div)]:
        h, l = fn(a, al, b, bl)
        assert np.array_equal(h, z[f"{name}_h"]) and np.array_equal(l, z[f"{name}_l"])
    h, l = O.two_prod(a, b)
    assert np.array_equal(h, z["tp_h"]) and np.array_equal(l, z["tp_l"])
    h, l = O.dd_matvec(z["mat"], z["vec"])
    assert np.array_equal(h, z["mv_h"]) and np.array_equal(l, z["mv_l"])


def test_half_rounding_exhaustive_against_first_principles():
    """Every finite binary16 value is a fixed point and midpoints round to even
    (reference test_precision.py:96-106 property, restated)."""
    bits = np.arange(0, 1 << 16, dtype=np.uint16)
    vals = bits.view(np.float16).astype(np.float64)
    fin = np.isfinite(vals)
    assert np.array_equal(O.rnd(vals[fin], O.HALF), vals[fin])
    pos = np.sort(np.unique(vals[fin & (vals > 0)]))
    mid = (pos[:-1] + pos[1:]) / 2
    r = O.rnd(mid, O.HALF)
    lo_even = (pos[:-1].astype(np.float16).view(np.uint16) & 1) == 0
    assert np.array_equal(r, np.where(lo_even, pos[:-1], pos[1:]))


@pytest.mark.parametrize("name", ["cfg1_half", "cfg3s0_half", "cfg3s1_half", "r256_half", "r200_double",
                                  "prol100_single", "r100k8_single"])
def test_lu_golden(name):
    meta = golden_json("lu")[name]
    z = golden_npz("lu")
    a = O.rnd(z[f"{name}_a"], meta["u"])
    f = O.lu_factor(a, meta["uf"])
    if meta["uf"] != "half" and not SINGLE_THREAD:
        pytest.skip("LAPACK LU bits depend on OPENBLAS_NUM_THREADS")
    assert np.array_equal(f.perm, z[f"{name}_perm"])
    assert np.array_equal(f.packed, z[f"{name}_lu"])
    assert f.growth == meta["growth"]


def test_kernels_golden():
    k = golden_npz("kernels")
    a0, b0 = k["a"], k["b"]
    for tag, (uf, u) in {"hs": ("half", "single"), "sd": ("single", "double"), "hd": ("half", "double")}.items():
        a = O.rnd(a0, u)
        b = O.rnd(b0, u)
        f = O.lu_factor(a, uf)
        assert np.array_equal(O.lu_solve(f, b, uf, store=u), k[f"{tag}_x0"])
        assert np.array_equal(O.apply_op(a, f, k[f"{tag}_v"], O.squared(u), u), k[f"{tag}_op"])
        assert np.array_equal(O.precond_rhs(f, k[f"{tag}_v"], O.squared(u), u), k[f"{tag}_prhs"])
        assert np.array_equal(O.residual(a, k[f"{tag}_x"], b, O.QUAD), k[f"{tag}_res_q"])
        assert np.array_equal(O.residual(a, k[f"{tag}_x"], b, O.DOUBLE), k[f"{tag}_res_d"])
    assert np.array_equal(O.quad_solve(a0, b0), k["xref_q"])


def _same_report(rep, g):
    assert rep.converged == g["converged"]
    assert rep.inner_iters == g["inner_iters"]
    assert rep.divergence_reason == g["divergence_reason"]
    for x, y in zip(rep.nbe_history + rep.ferr_history, g["nbe_history"] + g["ferr_history"]):
        assert x == y or (math.isnan(x) and math.isnan(y))
    if "solution" in g:
        assert np.array_equal(rep.solution, np.array(g["solution"]), equal_nan=True)


@pytest.mark.parametrize("method", ["gmres-ir", "rgmres-ir"])
def test_config1_golden(method):
    g = golden_json("cfg1")[method]
    a, b = problems.config_problem(problems.CONFIGS["cfg1"])
    rep = O.solve(a, b, ("half", "single", "double"), method, 100, 5 if method[0] == "r" else 0, 1e-4, 10)
    _same_report(rep, g)
    if method == "rgmres-ir":
        assert [c.k_eff for c in rep.inner_calls] == [c["k_eff"] for c in g["inner_calls"]]


@pytest.mark.parametrize("table", ["table5", "table6"])
def test_prolate_tables_golden(table):
    for row in golden_json(table)["rows"]:
        if len(row["inner_iters"]) > 20:
            continue  # the long IMaxExceeded rows are pinned on the GPU side only
        a = problems.prolate(100, row["alpha"])
        rep = O.solve(a, problems.rhs_ones(100), tuple(row["precisions"]), row["method"], row["m"],
                      row["k"], row["tau"], row["i_max"])
        _same_report(rep, row)


def test_config3_subset_golden():
    g = golden_json("cfg3")
    spec = problems.CONFIGS["cfg3"]
    for i in range(6):
        a, b = problems.config_problem(spec, i)
        for method in ("rgmres-ir", "gmres-ir"):
            rep = O.solve(a, b, spec.precisions, method, spec.m, spec.k if method[0] == "r" else 0,
                          spec.tau, spec.i_max)
            _same_report(rep, g[method][i])


@pytest.mark.parametrize("tag", ["half_rgmres-ir", "single_gmres-ir"])
def test_scale_diag_matches_reference(tag):
    """scale_diag=True (pow2 equilibration, refine.py:261-270, 293-297, 408-409)
    on badly scaled systems: the oracle reproduces the reference run exactly."""
    g = golden_json("scaled")[tag]
    z = golden_npz("scaled")
    rep = O.solve(z[f"{tag}_a"], z[f"{tag}_b"], tuple(g["precisions"]), g["method"], g["m"], g["k"], g["tau"],
                  g["i_max"], scale_diag=True)
    assert rep.converged == g["converged"] and rep.inner_iters == g["inner_iters"]
    assert rep.nbe_history == g["nbe_history"]
    assert np.array_equal(rep.solution, np.array(g["solution"]))
    assert rep.diagnostics.get("equilibrated")


@pytest.mark.parametrize("tag", ["gmres-ir_m4", "rgmres-ir_m4", "gmres-ir_m8", "rgmres-ir_m8"])
def test_explicit_residual_matches_reference(tag):
    """restart_residual / cycle_residual = "explicit": the oracle reproduces the
    reference's runs exactly (the checker of the GPU explicit-residual tests)."""
    from paper_2201_09827_b200 import problems

    g = golden_json("explicit")[tag]
    a, b = problems.config_problem(problems.CONFIGS["cfg1"])
    rep = O.solve(a, b, ("half", "single", "double"), g["method"], g["m"], g["k"], g["tau"], g["i_max"],
                  restart_residual="explicit", cycle_residual="explicit")
    assert rep.converged == g["converged"] and rep.inner_iters == g["inner_iters"]
    assert rep.nbe_history == g["nbe_history"]
    assert np.array_equal(rep.solution, np.array(g["solution"]))


_VARIANT_TAGS = [f"{p}_{m}" for p in ("half_single", "single_double", "half_double")
                 for m in ("sir", "sgmres-ir", "rsgmres-ir")]


@pytest.mark.parametrize("tag", _VARIANT_TAGS)
def test_sir_and_s_variants_match_reference(tag):
    """SIR / SGMRES-IR / RSGMRES-IR on config 1 (tests/golden/variants.json,
    reference runs): verdict, reason, per-step counts and every nbe exact."""
    from paper_2201_09827_b200 import problems

    g = golden_json("variants")[tag]
    a, b = problems.config_problem(problems.CONFIGS["cfg1"])
    rep = O.solve(a, b, tuple(g["precisions"]), g["method"], g["m"], g["k"], g["tau"], g["i_max"])
    assert rep.converged == g["converged"] and rep.divergence_reason == g["divergence_reason"]
    assert rep.inner_iters == g["inner_iters"] and rep.nbe_history == g["nbe_history"]

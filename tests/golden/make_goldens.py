"""Capture golden vectors by running the REFERENCE package itself.

Run in the build container only (the reference does not exist on the GPU box):

    OPENBLAS_NUM_THREADS=1 PYTHONPATH=/root/reference/pkg/src:/root/repo \
        python tests/golden/make_goldens.py <case> [<case> ...]

Cases: precision, lu, kernels, cfg1, cfg3, table5, table6, cfg2a, cfg2b, cfg4,
cfg5_1024, scaled, explicit, variants.  Each case writes ``tests/golden/<case>.json`` (+ ``.npz`` when
arrays are needed).  Inputs come from ``paper_2201_09827_b200.problems``,
which is itself pinned against ``irkit.matgen`` here (``check_matgen``).
``OPENBLAS_NUM_THREADS=1`` is required: the fp32 LU pivots and fp64 GEMV bits
of the reference change with the BLAS thread count.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))

import irkit  # noqa: E402  (reference, via PYTHONPATH)
from irkit import densela, gcrodr, gmres, matgen, precision, refine  # noqa: E402

from paper_2201_09827_b200 import problems  # noqa: E402


def _sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def _runtime_info() -> dict:
    return {
        "numpy": np.__version__,
        "openblas_threads": os.environ.get("OPENBLAS_NUM_THREADS"),
        "reference": "irkit " + getattr(irkit, "__version__", "?"),
    }


def _dump(case: str, meta: dict, arrays: dict | None = None) -> None:
    meta = dict(meta)
    meta["_runtime"] = _runtime_info()
    with open(os.path.join(HERE, f"{case}.json"), "w") as fh:
        json.dump(meta, fh, indent=1, sort_keys=True)
    if arrays:
        np.savez_compressed(os.path.join(HERE, f"{case}.npz"), **arrays)
    print(f"[golden] wrote {case}", flush=True)


# --------------------------------------------------------------------------
# solve capture with per-cycle recording
# --------------------------------------------------------------------------

class _Recorder:
    """Wraps gmres_solve/gcrodr_solve inside irkit.refine to record the
    per-cycle iteration counts and k_eff of every inner solve."""

    def __init__(self):
        self.calls: list[dict] = []
        self._orig_gm = refine.gmres_solve
        self._orig_gc = refine.gcrodr_solve

    def __enter__(self):
        rec = self

        def gm(*args, **kw):
            out = rec._orig_gm(*args, **kw)
            rec.calls.append({"kind": "gmres", "cycles": list(out.iterations_per_cycle),
                              "stagnated": bool(out.stagnated),
                              "applies": int(out.operator_applies),
                              "relres": float(out.final_relres)})
            return out

        def gc(a, f, r, cfg, recycle_in=None):
            cfg.collect_diagnostics = True
            out, rec_out = rec._orig_gc(a, f, r, cfg, recycle_in)
            diag = out.cycle_diagnostics or []
            rec.calls.append({
                "kind": "gcrodr",
                "cycles": list(out.iterations_per_cycle),
                "k_eff": [int(d["k_eff"]) for d in diag],
                "cycle_kind": [d["kind"] for d in diag],
                "warm": recycle_in is not None,
                "stagnated": bool(out.stagnated),
                "applies": int(out.operator_applies),
                "relres": float(out.final_relres),
            })
            return out, rec_out

        refine.gmres_solve = gm
        refine.gcrodr_solve = gc
        return self

    def __exit__(self, *exc):
        refine.gmres_solve = self._orig_gm
        refine.gcrodr_solve = self._orig_gc


def _report_dict(rep, with_solution: bool = True) -> dict:
    d = {
        "converged": bool(rep.converged),
        "steps": int(rep.steps),
        "inner_iters": [int(v) for v in rep.inner_iters],
        "nbe_history": [float(v) for v in rep.nbe_history],
        "ferr_history": [float(v) for v in rep.ferr_history],
        "divergence_reason": rep.divergence_reason.value if rep.divergence_reason else None,
        "diagnostics": {k: (float(v) if isinstance(v, (int, float, bool)) else str(v))
                        for k, v in rep.diagnostics.items()},
    }
    if rep.solution is not None:
        d["solution_sha"] = _sha(np.asarray(rep.solution, dtype=np.float64))
        d["solution_inf"] = float(np.max(np.abs(rep.solution)))
        if with_solution:
            d["solution"] = [float(v) for v in rep.solution]
    return d


def _solve(a, b, prec, method, m, k, tau, i_max, with_solution=True):
    cfg = refine.RefineConfig(
        precisions=precision.PrecisionTriple.parse(*prec),
        method=refine.Method.parse(method), m=m, k=k, tau=tau, i_max=i_max)
    t0 = time.perf_counter()
    with _Recorder() as rec:
        rep = refine.solve(a, b, cfg)
    dt = time.perf_counter() - t0
    d = _report_dict(rep, with_solution)
    d["inner_calls"] = rec.calls
    d["seconds"] = dt
    d["precisions"] = list(prec)
    d["method"] = method
    d["m"], d["k"], d["tau"], d["i_max"] = m, k, tau, i_max
    return d


# --------------------------------------------------------------------------
# cases
# --------------------------------------------------------------------------

def check_matgen() -> dict:
    out = {}
    for n, kap, seed in [(100, 1e4, 1), (128, 1e3, 1), (128, 1e3, 7), (300, 1e8, 3)]:
        ref = matgen.gen_randsvd(matgen.RandSvdSpec(n, kap, seed))
        ours = problems.randsvd(n, kap, seed)
        assert np.array_equal(ref, ours), (n, kap, seed)
        out[f"randsvd_{n}_{kap:g}_{seed}"] = _sha(ref)
    for n, al in [(100, 0.45), (1024, 0.45)]:
        ref = matgen.gen_prolate(matgen.ProlateSpec(n, al))
        assert np.array_equal(ref, problems.prolate(n, al))
        out[f"prolate_{n}_{al:g}"] = _sha(ref)
    return out


def case_precision():
    rng = np.random.Generator(np.random.Philox(11))
    x = np.concatenate([
        rng.standard_normal(2000) * np.exp2(rng.integers(-30, 20, 2000)),
        np.array([65504.0, 65519.99, 65520.0, 1e6, 2.0 ** -24, 2.0 ** -25, 3 * 2.0 ** -26,
                  2.0 ** -14, 6.1e-5, -0.0, 0.0, 1.0 + 2.0 ** -11, 1.0 + 3 * 2.0 ** -11]),
    ])
    h = precision.round_array(x, precision.Format.HALF)
    s = precision.round_array(x, precision.Format.SINGLE)
    a = rng.standard_normal(257) * 1e3
    b = rng.standard_normal(257)
    al = a * 1e-17
    bl = b * 1e-17
    add = precision.dd_add(a, al, b, bl)
    mul = precision.dd_mul(a, al, b, bl)
    div = precision.dd_div(a, al, b, bl)
    tp = precision._two_prod(a, b)
    mat = rng.standard_normal((33, 47))
    vec = rng.standard_normal(47)
    mv = precision.dd_matvec(mat, vec)
    dot = precision.dd_dot(a, b)
    _dump("precision", {"matgen": check_matgen()},
          {"x": x, "half": h, "single": s, "a": a, "al": al, "b": b, "bl": bl,
           "add_h": add[0], "add_l": add[1], "mul_h": mul[0], "mul_l": mul[1],
           "div_h": div[0], "div_l": div[1], "tp_h": tp[0], "tp_l": tp[1],
           "mat": mat, "vec": vec, "mv_h": mv[0], "mv_l": mv[1],
           "dot_h": np.array(dot[0]), "dot_l": np.array(dot[1])})


def _lu_record(a_u, fmt):
    f = densela.lu_factor(a_u, precision.context_for(fmt))
    packed = np.tril(f.L, -1) + f.U
    return f, packed


def case_lu():
    meta = {}
    arrays = {}
    H, S, D = precision.Format.HALF, precision.Format.SINGLE, precision.Format.DOUBLE
    cases = [
        ("cfg1_half", problems.randsvd(100, 1e4, 1), S, H),
        ("cfg3s0_half", problems.randsvd(128, 1e3, 1), S, H),
        ("cfg3s1_half", problems.randsvd(128, 1e3, 2), S, H),
        ("r256_half", problems.randsvd(256, 1e4, 5), S, H),
        ("r100k8_single", problems.randsvd(100, 1e8, 2), D, S),
        ("prol100_single", problems.prolate(100, 0.45), D, S),
        ("r200_double", problems.randsvd(200, 1e6, 3), D, D),
    ]
    for name, a, u, uf in cases:
        a_u = precision.round_array(a, u)
        f, packed = _lu_record(a_u, uf)
        arrays[f"{name}_a"] = a
        arrays[f"{name}_perm"] = f.perm.astype(np.int64)
        arrays[f"{name}_lu"] = packed
        meta[name] = {"n": int(a.shape[0]), "u": u.value, "uf": uf.value,
                      "growth": f.growth, "lu_sha": _sha(packed)}
    # larger fp16 cases: perm + hash only
    for name, a, u in [("cfg2b_half", problems.prolate(1024, 0.45), D),
                       ("r1024k8_half", problems.randsvd(1024, 1e8, 1), S)]:
        a_u = precision.round_array(a, u)
        t0 = time.perf_counter()
        f, packed = _lu_record(a_u, H)
        arrays[f"{name}_perm"] = f.perm.astype(np.int64)
        arrays[f"{name}_diag"] = np.diag(packed).copy()
        meta[name] = {"n": int(a.shape[0]), "u": u.value, "uf": "half", "growth": f.growth,
                      "lu_sha": _sha(packed), "seconds": time.perf_counter() - t0}
    for name, a, u in [("cfg2a_single", problems.prolate(1024, 0.45), D)]:
        a_u = precision.round_array(a, u)
        f, packed = _lu_record(a_u, S)
        arrays[f"{name}_perm"] = f.perm.astype(np.int64)
        meta[name] = {"n": 1024, "u": u.value, "uf": "single", "growth": f.growth}
    _dump("lu", meta, arrays)


def case_kernels():
    """Kernel-level vectors at n=100: residual, operator, precond_rhs, x0."""
    H, S, D, Q = (precision.Format.HALF, precision.Format.SINGLE,
                  precision.Format.DOUBLE, precision.Format.QUAD)
    ctx = precision.context_for
    a0 = problems.randsvd(100, 1e4, 1)
    b0 = problems.rhs_normal(100, 1)
    rng = np.random.Generator(np.random.Philox(5))
    arrays = {"a": a0, "b": b0}
    meta = {}
    for tag, (uf, u) in {"hs": (H, S), "sd": (S, D), "hd": (H, D)}.items():
        a = precision.round_array(a0, u)
        b = precision.round_array(b0, u)
        f = densela.lu_factor(a, ctx(uf))
        v = precision.round_array(rng.standard_normal(100), u)
        x = precision.round_array(np.linalg.solve(a, b) + 1e-3 * rng.standard_normal(100), u)
        arrays[f"{tag}_v"] = v
        arrays[f"{tag}_x"] = x
        arrays[f"{tag}_x0"] = densela.lu_solve(f, b, ctx(uf), store_fmt=u)
        u2 = precision.squared_format(u)
        arrays[f"{tag}_op"] = densela.apply_preconditioned(a, f, v, ctx(u2), u)
        arrays[f"{tag}_op_u"] = densela.apply_preconditioned(a, f, v, ctx(u), u)
        arrays[f"{tag}_prhs"] = densela.precond_rhs(f, v, ctx(u2), u)
        arrays[f"{tag}_res_d"] = densela.residual(a, x, b, ctx(D))
        arrays[f"{tag}_res_q"] = densela.residual(a, x, b, ctx(Q))
        arrays[f"{tag}_perm"] = f.perm.astype(np.int64)
    arrays["xref_q"] = densela.quad_solve(a0, b0)
    # fp64 LU + dd refinement recipe (refine.py:251-256) at n=100 for the kernel test
    f = densela.lu_factor(a0, ctx(D))
    x = densela.lu_solve(f, b0, ctx(D))
    for _ in range(4):
        r = densela.residual(a0, x, b0, ctx(Q))
        x = x + densela.lu_solve(f, r, ctx(D))
    arrays["xref_lu"] = x
    _dump("kernels", meta, arrays)


def case_cfg1():
    a, b = problems.config_problem(problems.CONFIGS["cfg1"])
    out = {}
    for method in ["gmres-ir", "rgmres-ir"]:
        out[method] = _solve(a, b, ("half", "single", "double"), method, 100, 5, 1e-4, 10)
    _dump("cfg1", out)


def case_cfg3(count: int = 48):
    spec = problems.CONFIGS["cfg3"]
    out = {"count": count, "rgmres-ir": [], "gmres-ir": []}
    for i in range(count):
        a, b = problems.config_problem(spec, i)
        for method in ["rgmres-ir", "gmres-ir"]:
            out[method].append(_solve(a, b, spec.precisions, method, spec.m, spec.k,
                                      spec.tau, spec.i_max))
    _dump("cfg3", out)


_ALPHAS = [0.475, 0.47, 0.467, 0.455, 0.45, 0.4468, 0.44, 0.434]


def _table(prec, k, tau, i_max):
    rows = []
    for al in _ALPHAS:
        a = problems.prolate(100, al)
        b = problems.rhs_ones(100)
        for method in ["gmres-ir", "rgmres-ir"]:
            d = _solve(a, b, prec, method, 16, k if method == "rgmres-ir" else 0, tau, i_max)
            d["alpha"] = al
            rows.append(d)
    return rows


def case_table5():
    _dump("table5", {"rows": _table(("single", "double", "quad"), 4, 1e-8, 10000)})


def case_table6():
    # i_max bounded at 200 (the reference default 10000 only lengthens the
    # IMaxExceeded cases; every converging row needs < 10 steps)
    _dump("table6", {"rows": _table(("half", "single", "double"), 5, 1e-4, 200)})


def _big(case: str, n_override=None, methods=("rgmres-ir",), with_solution=False):
    name = case.split("_")[0]
    spec = problems.CONFIGS[name]
    a, b = problems.config_problem(spec, 0, n_override)
    out = {"n": int(a.shape[0]), "a_sha": _sha(a), "b_sha": _sha(b)}
    for method in methods:
        out[method] = _solve(a, b, spec.precisions, method, spec.m,
                             spec.k if method == "rgmres-ir" else 0,
                             spec.tau, spec.i_max, with_solution)
    sol = {}
    _dump(case, out, sol or None)


CASES = {
    "precision": case_precision,
    "lu": case_lu,
    "kernels": case_kernels,
    "cfg1": case_cfg1,
    "cfg3": case_cfg3,
    "table5": case_table5,
    "table6": case_table6,
    "cfg2a": lambda: _big("cfg2a"),
    "cfg2b": lambda: _big("cfg2b"),
    "cfg4": lambda: _big("cfg4", methods=("rgmres-ir", "gmres-ir")),
    "cfg5_1024": lambda: _big("cfg5_1024", 1024, methods=("rgmres-ir", "gmres-ir"),
                              with_solution=True),
    # the config-5 analogue on the grid-team kernel type (n > 1024): GCRO-DR-IR only
    # (661 s of reference time + the simulated fp16 LU)
    "cfg5_2048": lambda: _big("cfg5_2048", 2048, methods=("rgmres-ir",)),
}


def case_scaled():
    """scale_diag=True (refine.py:261-270, 293-297, 408-409) on badly row/column
    scaled randsvd systems: D_r A D_c with D ~ 10^U(-6, 6) (not powers of two,
    so the equilibration is not a no-op)."""
    rng = np.random.default_rng(2201)
    out = {}
    for n, kappa, prec, method, m, k, tau in ((60, 1e3, ("half", "single", "double"), "rgmres-ir", 20, 4, 1e-4),
                                              (80, 1e5, ("single", "double", "quad"), "gmres-ir", 30, 0, 1e-8)):
        a0 = problems.randsvd(n, kappa, seed=7)
        dr, dc = 10.0 ** rng.uniform(-6, 6, n), 10.0 ** rng.uniform(-6, 6, n)
        a = dr[:, None] * a0 * dc[None, :]
        b = rng.standard_normal(n)
        tag = f"{prec[0]}_{method}"
        cfg = refine.RefineConfig(precisions=precision.PrecisionTriple.parse(*prec),
                                  method=refine.Method.parse(method), m=m, k=k, tau=tau, i_max=20, scale_diag=True)
        rep = refine.solve(a, b, cfg)
        d = _report_dict(rep)
        d.update(precisions=list(prec), method=method, m=m, k=k, tau=tau, i_max=20, n=n)
        out[tag] = (d, a, b)
    _dump("scaled", {t: v[0] for t, v in out.items()},
          {**{f"{t}_a": v[1] for t, v in out.items()}, **{f"{t}_b": v[2] for t, v in out.items()}})


CASES["scaled"] = case_scaled


def case_explicit():
    """restart_residual / cycle_residual = "explicit" (gmres.py:292-295,
    gcrodr.py:301-304, 376-379) on config 1 with short restarts."""
    a, b = problems.config_problem(problems.CONFIGS["cfg1"])
    out = {}
    for method, m, k in (("gmres-ir", 4, 0), ("rgmres-ir", 4, 2), ("gmres-ir", 8, 0), ("rgmres-ir", 8, 3)):
        cfg = refine.RefineConfig(precisions=precision.PrecisionTriple.parse("half", "single", "double"),
                                  method=refine.Method.parse(method), m=m, k=k, tau=1e-4, i_max=10,
                                  restart_residual="explicit", cycle_residual="explicit")
        d = _report_dict(refine.solve(a, b, cfg))
        d.update(method=method, m=m, k=k, tau=1e-4, i_max=10)
        out[f"{method}_m{m}"] = d
    _dump("explicit", out)


CASES["explicit"] = case_explicit


def case_variants():
    """SIR and the uniform-precision S-variants (refine.py:56-83, 124-131,
    378-380) on config 1 under three precision triples."""
    a, b = problems.config_problem(problems.CONFIGS["cfg1"])
    out = {}
    for prec in (("half", "single", "double"), ("single", "double", "double"), ("half", "double", "double")):
        for method in ("sir", "sgmres-ir", "rsgmres-ir"):
            m = 0 if method == "sir" else 100
            k = 5 if method == "rsgmres-ir" else 0
            tau = None if method == "sir" else 1e-4
            cfg = refine.RefineConfig(precisions=precision.PrecisionTriple.parse(*prec),
                                      method=refine.Method.parse(method), m=m, k=k, tau=tau, i_max=10)
            d = _report_dict(refine.solve(a, b, cfg))
            d.update(precisions=list(prec), method=method, m=m, k=k, tau=tau, i_max=10)
            out[f"{prec[0]}_{prec[1]}_{method}"] = d
    _dump("variants", out)


CASES["variants"] = case_variants


# well-posed recycling systems in the cluster-team range n in (256, 1024]
# (VERDICT r1 item 1 / SURVEY F7): cold cycle >= k, deflated cycles, warm
# starts in later refinement steps, converging
WELLPOSED = [
    # (tag, n, kappa, seed, precisions, m, k, tau)
    ("w1024_hsd", 1024, 1e3, 3, ("half", "single", "double"), 10, 4, 1e-4),
    ("w1024_hdq", 1024, 1e3, 3, ("half", "double", "quad"), 10, 4, 1e-6),
    ("w1024_sdq", 1024, 1e7, 3, ("single", "double", "quad"), 10, 4, 1e-10),
]


def case_wellposed():
    out = {}
    for tag, n, kappa, seed, prec, m, k, tau in WELLPOSED:
        a = problems.randsvd(n, kappa, seed)
        b = problems.rhs_normal(n, seed)
        d = _solve(a, b, prec, "rgmres-ir", m, k, tau, 10)
        d.update(n=n, kappa=kappa, seed=seed, a_sha=_sha(a), b_sha=_sha(b))
        out[tag] = d
        print(tag, d["inner_iters"], d["converged"], [c["cycles"] for c in d["inner_calls"]], flush=True)
    _dump("wellposed", out)


CASES["wellposed"] = case_wellposed


def _first_divergence_unblocked(a_u, ref_perm):
    """First step where an unblocked, FMA-free fp32 GEPP of the same matrix
    picks a different pivot row than the reference's sgetrf (None if never)."""
    w = a_u.astype(np.float32)
    n = w.shape[0]
    perm = np.arange(n)
    for k in range(n):
        p = k + int(np.argmax(np.abs(w[k:, k])))
        if p != k:
            w[[k, p], :] = w[[p, k], :]
            perm[[k, p]] = perm[[p, k]]
        if perm[k] != ref_perm[k]:
            return k
        if w[k, k] != 0:
            w[k + 1:, k] *= np.float32(1) / w[k, k]
            w[k + 1:, k + 1:] -= np.outer(w[k + 1:, k], w[k, k + 1:])
    return None


def case_lu_large():
    """Pivot goldens beyond n = 1024: exact fp16 GEPP at n = 2048 (randsvd
    kappa 1e8, the config-5 analogue with fp16 subnormals) and the
    fp32 sgetrf pivots of config 4 (n = 8192).  For the fp32 cases the first
    pivot where another valid GEPP of the same matrix (unblocked, no FMA)
    departs from the reference is recorded too: the parity noise floor
    (SURVEY F14)."""
    meta, arrays = {}, {}
    H, S_, D = precision.Format.HALF, precision.Format.SINGLE, precision.Format.DOUBLE
    a = problems.randsvd(2048, 1e8, 1)
    a_u = precision.round_array(a, S_)
    t0 = time.perf_counter()
    f, packed = _lu_record(a_u, H)
    arrays["r2048k8_half_perm"] = f.perm.astype(np.int64)
    arrays["r2048k8_half_diag"] = np.diag(packed).copy()
    arrays["r2048k8_half_row7"] = packed[7].copy()
    meta["r2048k8_half"] = {"n": 2048, "u": "single", "uf": "half", "growth": f.growth, "lu_sha": _sha(packed),
                            "a_sha": _sha(a), "seconds": time.perf_counter() - t0}
    print("r2048k8_half", meta["r2048k8_half"], flush=True)
    for name, a in (("cfg2a_single", problems.prolate(1024, 0.45)),
                    ("cfg4_single", problems.randsvd(8192, 1e6, 1))):
        a_u = precision.round_array(a, D)
        f, packed = _lu_record(a_u, S_)
        alt = _first_divergence_unblocked(a_u, f.perm)
        arrays[f"{name}_perm"] = f.perm.astype(np.int64)
        arrays[f"{name}_diag"] = np.diag(packed).copy()
        meta[name] = {"n": int(a.shape[0]), "u": "double", "uf": "single", "growth": f.growth,
                      "a_sha": _sha(a), "alt_divergence": alt}
        print(name, meta[name], flush=True)
    _dump("lu_large", meta, arrays)


CASES["lu_large"] = case_lu_large


if __name__ == "__main__":
    if os.environ.get("OPENBLAS_NUM_THREADS") != "1":
        sys.exit("set OPENBLAS_NUM_THREADS=1 (SURVEY.md F14)")
    for c in sys.argv[1:]:
        t0 = time.perf_counter()
        CASES[c]()
        print(f"[golden] {c}: {time.perf_counter() - t0:.1f} s", flush=True)

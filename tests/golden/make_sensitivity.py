"""Measure the reference algorithm's own sensitivity to rounding-order changes.

For ill-conditioned systems the reference's per-step GMRES iteration counts
(and even its verdict) change when only the summation order of its fp32/fp64
dot products, or the blocking of its fp32/fp64 LU, changes.  Any other correct
implementation (ours runs warp-tree reductions and a different LU blocking)
lands somewhere in that envelope, so the GPU parity tests check per-step
iteration counts against [min - 1, max + 1] of the envelope and the verdict
against the set of verdicts seen.

Runs the ORACLE (oracle/cpu_gcrodr_ir.py, pinned bit-exact to the reference by
tests/test_oracle_golden.py) under these perturbations:
  lanes  -- dot / norm / M^T v accumulated in 32 lane-strided partial sums
            combined by a tree (the GPU reduction shape), same format;
  lu     -- fp32/fp64 LU by an unblocked right-looking FMA-free elimination
            instead of LAPACK getrf (fp16 LU is exact on the GPU: unchanged);
  both   -- the two together;
  op     -- the fp64 preconditioned operator (GEMV and both substitutions)
            accumulated in 32 lane-strided partial sums combined by a tree
            (the GPU's row-dot shape) instead of OpenBLAS dgemv/dtrsv order;
  ulpS   -- the first refinement update x <- fl_u(x + nu d) moved by a
            random {-1, 0, +1} ulp of u per entry (seed S = 0..7), later
            updates exact: the iterate is stored at u, so any implementation
            whose first correction differs in the last bit lands here.  On
            the chaotic prolate rows this alone spans most of the envelope
            (e.g. Table 6, alpha 0.45, GMRES-IR: step 2 in 29..32).

    OPENBLAS_NUM_THREADS=1 python tests/golden/make_sensitivity.py
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import cpu_gcrodr_ir as O  # noqa: E402
from paper_2201_09827_b200 import problems  # noqa: E402

_orig = {name: getattr(O, name) for name in ("vdot", "vnorm2", "tvec", "lu_factor", "apply_op", "precond_rhs",
                                               "vadd")}
_ULP = {"rng": None}


def vadd_ulp(x, y, fmt):
    """The refinement update (only caller of vadd) with a last-bit perturbation."""
    s = _orig["vadd"](x, y, fmt)
    if _ULP["rng"] is None or fmt not in (O.SINGLE, O.DOUBLE):
        return s
    rng, _ULP["rng"] = _ULP["rng"], None  # first update of the solve only
    dt = np.float32 if fmt == O.SINGLE else np.float64
    f = s.astype(dt)
    d = rng.integers(-1, 2, size=f.shape)
    f = np.where(d > 0, np.nextafter(f, dt(np.inf)), np.where(d < 0, np.nextafter(f, dt(-np.inf)), f))
    return f.astype(np.float64)


def _lane_sum(prod: np.ndarray, dt) -> float:
    n = prod.shape[0]
    pad = (-n) % 32
    p = np.concatenate([prod, np.zeros(pad, dt)]).reshape(-1, 32)
    acc = np.zeros(32, dt)
    for row in p:
        acc = (acc + row).astype(dt)
    while acc.shape[0] > 1:
        acc = (acc[0::2] + acc[1::2]).astype(dt)
    return float(acc[0])


_MODE = {"order": "lanes"}


def _ordered_sum(prod: np.ndarray, dt) -> float:
    mode = _MODE["order"]
    if mode == "reversed":
        acc = dt(0)
        for v in prod[::-1]:
            acc = dt(acc + v)
        return float(acc)
    if mode == "wide":  # accumulate in fp64, round once
        return float(dt(np.sum(prod.astype(np.float64))))
    return _lane_sum(prod, dt)


def vdot_lanes(x, y, fmt):
    if fmt in (O.SINGLE, O.DOUBLE, O.QUAD):
        dt = np.float32 if fmt == O.SINGLE else np.float64
        return _ordered_sum(np.asarray(x, dt) * np.asarray(y, dt), dt)
    return _orig["vdot"](x, y, fmt)


def vnorm2_lanes(x, fmt):
    if fmt == O.SINGLE:
        return float(np.sqrt(np.float32(vdot_lanes(x, x, fmt))))
    if fmt in (O.DOUBLE, O.QUAD):
        return float(np.sqrt(vdot_lanes(x, x, fmt)))
    return _orig["vnorm2"](x, fmt)


def tvec_lanes(m, r, fmt):
    m = np.asarray(m, dtype=np.float64)
    if fmt in (O.SINGLE, O.DOUBLE, O.QUAD):
        return np.array([vdot_lanes(m[:, i], r, fmt) for i in range(m.shape[1])])
    return _orig["tvec"](m, r, fmt)


def lu_unblocked(a, fmt):
    if fmt == O.HALF:
        return _orig["lu_factor"](a, fmt)
    dt = np.float32 if fmt == O.SINGLE else np.float64
    w = O.rnd(np.asarray(a, dtype=np.float64), fmt).astype(dt).copy()
    n = w.shape[0]
    amax = float(np.max(np.abs(w)))
    perm = np.arange(n)
    for k in range(n):
        p = k + int(np.argmax(np.abs(w[k:, k])))
        if w[p, k] == 0:
            continue
        if p != k:
            w[[k, p], :] = w[[p, k], :]
            perm[[k, p]] = perm[[p, k]]
        w[k + 1:, k] = w[k + 1:, k] * (dt(1) / w[k, k])
        w[k + 1:, k + 1:] -= np.outer(w[k + 1:, k], w[k, k + 1:]).astype(dt)
    w = w.astype(np.float64)
    upper = np.triu(w)
    if np.any(np.diag(upper) == 0):
        raise O.ZeroPivot(int(np.argmax(np.diag(upper) == 0)))
    return O.Factors(np.tril(w, -1) + np.eye(n), upper, perm, fmt, float(np.max(np.abs(upper)) / amax))


def _rows_lanes(m: np.ndarray, x: np.ndarray) -> np.ndarray:
    """fp64 row dots m @ x in 32 lane-strided partial sums + a tree."""
    n = m.shape[1]
    pad = (-n) % 32
    p = np.concatenate([m * x[None, :], np.zeros((m.shape[0], pad))], axis=1).reshape(m.shape[0], -1, 32)
    acc = np.zeros((m.shape[0], 32))
    for c in range(p.shape[1]):
        acc = acc + p[:, c, :]
    while acc.shape[1] > 1:
        acc = acc[:, 0::2] + acc[:, 1::2]
    return acc[:, 0]


def _sub_rows(f, y):
    y = y.copy()
    n = f.n
    for i in range(1, n):
        y[i] = y[i] - _rows_lanes(f.L[i:i + 1, :i], y[:i])[0]
    for i in range(n - 1, -1, -1):
        if i < n - 1:
            y[i] = y[i] - _rows_lanes(f.U[i:i + 1, i + 1:], y[i + 1:])[0]
        y[i] = y[i] / f.U[i, i]
    return y


def apply_op_lanes(a, f, v, fmt, store):
    if fmt != O.DOUBLE:
        return _orig["apply_op"](a, f, v, fmt, store)
    w = _rows_lanes(np.asarray(a, dtype=np.float64), np.asarray(v, dtype=np.float64))
    return O.rnd(_sub_rows(f, w[f.perm]), store)


def precond_rhs_lanes(f, r, fmt, store):
    if fmt != O.DOUBLE:
        return _orig["precond_rhs"](f, r, fmt, store)
    return O.rnd(_sub_rows(f, np.asarray(r, dtype=np.float64)[f.perm]), store)


def _set(lanes: bool, lu: bool, op: bool = False, ulp_seed=None):
    _ULP["rng"] = None if ulp_seed is None else np.random.default_rng(ulp_seed)
    O.vadd = vadd_ulp if ulp_seed is not None else _orig["vadd"]
    O.apply_op = apply_op_lanes if op else _orig["apply_op"]
    O.precond_rhs = precond_rhs_lanes if op else _orig["precond_rhs"]
    O.vdot = vdot_lanes if lanes else _orig["vdot"]
    O.vnorm2 = vnorm2_lanes if lanes else _orig["vnorm2"]
    O.tvec = tvec_lanes if lanes else _orig["tvec"]
    O.lu_factor = lu_unblocked if lu else _orig["lu_factor"]


def squared_fmt(u: str) -> str:
    return O.squared(u)


def envelope(a, b, prec, method, m, k, tau, i_max, ulp=True):
    runs = {}
    variants = {"ref": (False, False, "lanes"), "lanes": (True, False, "lanes"), "lu": (False, True, "lanes"),
                "both": (True, True, "lanes"), "reversed": (True, False, "reversed"),
                "wide": (True, False, "wide"), "op": (False, False, "op"), "op+lanes": (True, False, "op+lanes")}
    if ulp:
        variants.update({f"ulp{sd}": (False, False, f"ulp{sd}") for sd in range(8)})
    for name, (lanes, lu, order) in variants.items():
        if lu and prec[0] == "half":
            continue
        if order.startswith("op") and squared_fmt(prec[1]) != O.DOUBLE:
            continue
        _MODE["order"] = order if order in ("lanes", "reversed", "wide") else "lanes"
        _set(lanes, lu, op=order.startswith("op"), ulp_seed=int(order[3:]) if order.startswith("ulp") else None)
        try:
            rep = O.solve(a, b, tuple(prec), method, m, k, tau, i_max)
            runs[name] = {"inner": rep.inner_iters, "converged": rep.converged,
                          "reason": rep.divergence_reason}
        finally:
            _set(False, False)
    steps = max(len(r["inner"]) for r in runs.values())
    lo, hi = [], []
    for s in range(steps):
        vals = [r["inner"][s] for r in runs.values() if s < len(r["inner"])]
        lo.append(min(vals))
        hi.append(max(vals))
    return {"runs": runs, "lo": lo, "hi": hi,
            "verdicts": sorted({(r["converged"], r["reason"] or "") for r in runs.values()})}


def lu_divergence(a, uf="single"):
    """First pivot index where a different valid GEPP (unblocked, no FMA)
    departs from the reference's LAPACK factorisation; None if never."""
    au = O.rnd(np.asarray(a, dtype=np.float64), O.DOUBLE)
    ref = _orig["lu_factor"](au, uf)
    alt = lu_unblocked(au, uf)
    d = np.nonzero(ref.perm != alt.perm)[0]
    return int(d[0]) if d.size else None


def main_lu(out):
    lu = json.load(open(os.path.join(HERE, "lu.json")))
    z = np.load(os.path.join(HERE, "lu.npz"))
    out["lu"] = {name: lu_divergence(z[f"{name}_a"], meta["uf"])
                 for name, meta in lu.items() if meta.get("uf") == "single" and f"{name}_a" in z}


def main():
    out = {"tables": [], "cfg1": {}, "cfg3": []}
    main_lu(out)
    for tab in ("table5", "table6"):
        for row in json.load(open(os.path.join(HERE, f"{tab}.json")))["rows"]:
            a = problems.prolate(100, row["alpha"])
            env = envelope(a, np.ones(100), row["precisions"], row["method"], row["m"], row["k"],
                           row["tau"], row["i_max"])
            env.update({"table": tab, "alpha": row["alpha"], "method": row["method"]})
            out["tables"].append(env)
            print(tab, row["alpha"], row["method"], env["lo"][:6], env["hi"][:6], env["verdicts"], flush=True)
    a, b = problems.config_problem(problems.CONFIGS["cfg1"])
    for method in ("gmres-ir", "rgmres-ir"):
        out["cfg1"][method] = envelope(a, b, ("half", "single", "double"), method, 100,
                                       5 if method[0] == "r" else 0, 1e-4, 10)
    spec = problems.CONFIGS["cfg3"]
    for i in range(48):
        a, b = problems.config_problem(spec, i)
        row = {}
        for method in ("rgmres-ir", "gmres-ir"):
            row[method] = envelope(a, b, spec.precisions, method, spec.m, spec.k if method[0] == "r" else 0,
                                   spec.tau, spec.i_max)
        out["cfg3"].append(row)
    with open(os.path.join(HERE, "sensitivity.json"), "w") as fh:
        json.dump(out, fh, indent=0)


if __name__ == "__main__":
    if os.environ.get("OPENBLAS_NUM_THREADS") != "1":
        sys.exit("set OPENBLAS_NUM_THREADS=1")
    if "--tables-only" in sys.argv:
        path = os.path.join(HERE, "sensitivity.json")
        data = json.load(open(path))
        data["tables"] = []
        for tab in ("table5", "table6"):
            for row in json.load(open(os.path.join(HERE, f"{tab}.json")))["rows"]:
                a = problems.prolate(100, row["alpha"])
                env = envelope(a, np.ones(100), row["precisions"], row["method"], row["m"], row["k"],
                               row["tau"], row["i_max"])
                env.update({"table": tab, "alpha": row["alpha"], "method": row["method"]})
                data["tables"].append(env)
                print(tab, row["alpha"], row["method"], {k: v["inner"][:4] for k, v in env["runs"].items()},
                      flush=True)
        json.dump(data, open(path, "w"), indent=0)
    elif "--lu-only" in sys.argv:
        path = os.path.join(HERE, "sensitivity.json")
        data = json.load(open(path))
        main_lu(data)
        json.dump(data, open(path, "w"), indent=0)
    else:
        main()

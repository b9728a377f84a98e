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
  both   -- the two together.

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

_orig = {name: getattr(O, name) for name in ("vdot", "vnorm2", "tvec", "lu_factor")}


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


def _set(lanes: bool, lu: bool):
    O.vdot = vdot_lanes if lanes else _orig["vdot"]
    O.vnorm2 = vnorm2_lanes if lanes else _orig["vnorm2"]
    O.tvec = tvec_lanes if lanes else _orig["tvec"]
    O.lu_factor = lu_unblocked if lu else _orig["lu_factor"]


def envelope(a, b, prec, method, m, k, tau, i_max):
    runs = {}
    variants = {"ref": (False, False, "lanes"), "lanes": (True, False, "lanes"), "lu": (False, True, "lanes"),
                "both": (True, True, "lanes"), "reversed": (True, False, "reversed"),
                "wide": (True, False, "wide")}
    for name, (lanes, lu, order) in variants.items():
        if lu and prec[0] == "half":
            continue
        _MODE["order"] = order
        _set(lanes, lu)
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
    if "--lu-only" in sys.argv:
        path = os.path.join(HERE, "sensitivity.json")
        data = json.load(open(path))
        main_lu(data)
        json.dump(data, open(path, "w"), indent=0)
    else:
        main()

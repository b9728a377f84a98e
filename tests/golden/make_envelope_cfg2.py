"""Config 2's own sensitivity envelope (prolate(1024, 0.45) is
numerically singular, so the reference's Arnoldi total at the 205-cycle cap
moves with last-bit changes).

Runs the pinned ORACLE (oracle/cpu_gcrodr_ir.py, bit-exact to the reference
by tests/test_oracle_golden.py; its unperturbed cfg2 runs equal the golden
cfg2a/cfg2b captures) under the perturbation family of make_sensitivity.py
(lane-ordered / reversed / fp64-widened Krylov dots, unblocked fp32 LU, and a
{-1, 0, +1}-ulp move of the first refinement update), one variant per
process:

    OPENBLAS_NUM_THREADS=1 python tests/golden/make_envelope_cfg2.py run cfg2a lanes
    OPENBLAS_NUM_THREADS=1 python tests/golden/make_envelope_cfg2.py merge

Each run records total Arnoldi steps, cycle count, verdict, final nbe/ferr
and the per-cycle k_eff sequence into tests/golden/env_cfg2/<cfg>_<variant>.json;
``merge`` writes tests/golden/cfg2_envelope.json.  About 30-40 min per run.
"""

from __future__ import annotations

import glob
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
import make_sensitivity as S  # noqa: E402

O = S.O
problems = S.problems
OUT = os.path.join(HERE, "env_cfg2")

VARIANTS = {
    # name: (lanes, lu, order)
    "lanes": (True, False, "lanes"),
    "lu": (False, True, "lanes"),
    "both": (True, True, "lanes"),
    "reversed": (True, False, "reversed"),
    "wide": (True, False, "wide"),
    **{f"ulp{s}": (False, False, f"ulp{s}") for s in range(8)},
    # unblocked fp32 LU together with a last-bit move of the first update
    **{f"lu_ulp{s}": (False, True, f"ulp{s}") for s in range(4)},
    # the operator's result moved by a random {-1, 0, +1} ulp of u per entry
    # (seed S): config 2 runs the operator in double-double through factors
    # with kappa(U) ~ 1e17, so two dd implementations that differ at the 1e-32
    # level (summation order, FMA two_prod) differ by ulps of u after rounding
    **{f"opulp{s}": (False, False, f"opulp{s}") for s in range(8)},
}


def _perturb_operator(seed: int) -> None:
    rng = np.random.default_rng(1000 + seed)
    base_op, base_rhs = O.apply_op, O.precond_rhs

    def nudge(w):
        w = np.asarray(w, dtype=np.float64)
        step = rng.integers(-1, 2, size=w.shape)
        up = np.nextafter(w, np.inf)
        dn = np.nextafter(w, -np.inf)
        return np.where(step > 0, up, np.where(step < 0, dn, w))

    O.apply_op = lambda a, f, v, fmt, store: nudge(base_op(a, f, v, fmt, store))
    O.precond_rhs = lambda f, r, fmt, store: nudge(base_rhs(f, r, fmt, store))


def run(cfg: str, variant: str) -> dict:
    spec = problems.CONFIGS[cfg]
    a, b = problems.config_problem(spec)
    lanes, lu, order = VARIANTS[variant]
    if lu and spec.precisions[0] == "half":
        raise SystemExit("fp16 LU is exact on the GPU: no LU variant for half factors")
    S._MODE["order"] = order if order in ("lanes", "reversed", "wide") else "lanes"
    S._set(lanes, lu, op=False, ulp_seed=int(order[3:]) if order.startswith("ulp") else None)
    if order.startswith("opulp"):
        if spec.precisions[1] != "double":
            raise SystemExit("opulp variants perturb at u = double")
        _perturb_operator(int(order[5:]))
    t0 = time.perf_counter()
    rep = O.solve(a, b, spec.precisions, "rgmres-ir", spec.m, spec.k, spec.tau, spec.i_max)
    call = rep.inner_calls[0] if rep.inner_calls else None
    out = {"cfg": cfg, "variant": variant, "inner": rep.inner_iters, "converged": rep.converged,
           "reason": rep.divergence_reason, "nbe": rep.nbe_history, "ferr": rep.ferr_history,
           "seconds": time.perf_counter() - t0}
    if call is not None:
        out["cycles"] = [int(c) for c in getattr(call, "cycles", [])]
        out["k_eff"] = [int(c) for c in getattr(call, "k_eff", [])]
    os.makedirs(OUT, exist_ok=True)
    with open(os.path.join(OUT, f"{cfg}_{variant}.json"), "w") as fh:
        json.dump(out, fh, indent=0, default=float)
    return out


def merge() -> None:
    env = {}
    for path in sorted(glob.glob(os.path.join(OUT, "*.json"))):
        r = json.load(open(path))
        e = env.setdefault(r["cfg"], {"runs": {}})
        e["runs"][r["variant"]] = {k: r[k] for k in ("inner", "converged", "reason", "nbe", "ferr") if k in r}
    for cfg, e in env.items():
        g = json.load(open(os.path.join(HERE, f"{cfg}.json")))["rgmres-ir"]
        e["runs"]["ref"] = {"inner": g["inner_iters"], "converged": g["converged"],
                            "reason": g["divergence_reason"], "nbe": g["nbe_history"], "ferr": g["ferr_history"]}
        tot = [sum(r["inner"]) for r in e["runs"].values()]
        e["lo"], e["hi"] = min(tot), max(tot)
        e["verdicts"] = sorted({(r["converged"], r["reason"] or "") for r in e["runs"].values()})
    with open(os.path.join(HERE, "cfg2_envelope.json"), "w") as fh:
        json.dump(env, fh, indent=1, default=float)
    for cfg, e in env.items():
        print(cfg, e["lo"], e["hi"], e["verdicts"], {k: sum(v["inner"]) for k, v in e["runs"].items()})


if __name__ == "__main__":
    if os.environ.get("OPENBLAS_NUM_THREADS") != "1":
        sys.exit("set OPENBLAS_NUM_THREADS=1")
    if sys.argv[1] == "run":
        print(json.dumps(run(sys.argv[2], sys.argv[3]), default=float)[:400])
    else:
        merge()

"""Sweeps over the device solver: the reference's experiment layer on top of
``solve`` (reference harness.py:74-333), for the paper's Tables 5/6 grids and
the recycle-dimension scan (Fig. 2).

Every solve goes through ``refine.solve`` (the CUDA path).  The per-problem
condition numbers in a row are problem statistics (numpy on the host, as the
reference computes them: densela.py:491-503) and are not part of any timed
solve.  ``mtx:`` problems are read by ``mtx.read_matrix_market``.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, replace

import numpy as np

from . import problems
from .mtx import read_matrix_market
from .precision import PrecisionTriple
from .refine import Method, RefineConfig, RefinementReport, solve

__all__ = ["ProblemRef", "SweepSpec", "format_cell", "run_sweep", "kscan", "cond_inf", "CSV_COLUMNS"]

# harness.py:55-70
CSV_COLUMNS = ["problem_id", "kappa_inf", "kappa_2", "method", "m", "k", "tau", "converged", "steps",
               "total_inner", "per_step", "nbe_final", "ferr_final", "divergence_reason"]


@dataclass(frozen=True)
class ProblemRef:
    """A generated test problem (harness.py:74-115); b = ones as in the reference."""

    kind: str  # "prolate" | "randsvd" | "mtx"
    alpha: float | None = None
    kappa2: float | None = None
    n: int = 100
    seed: int = 1
    path: str | None = None

    @property
    def problem_id(self) -> str:
        if self.kind == "prolate":
            return f"prolate:{self.alpha:g}"
        if self.kind == "randsvd":
            return f"randsvd:{self.kappa2:g}"
        stem = (self.path or "").replace("\\", "/").rsplit("/", 1)[-1]
        return stem.rsplit(".", 1)[0] if "." in stem else stem

    def materialize(self) -> tuple[np.ndarray, np.ndarray]:
        if self.kind == "prolate":
            a = problems.prolate(self.n, self.alpha)
        elif self.kind == "randsvd":
            a = problems.randsvd(self.n, self.kappa2, self.seed)
        elif self.kind == "mtx":
            a = read_matrix_market(self.path)
        else:
            raise ValueError(f"unknown problem kind {self.kind!r}")
        return a, problems.rhs_ones(a.shape[0])

    @classmethod
    def parse(cls, text: str, n: int = 100, seed: int = 1) -> "ProblemRef":
        """"prolate:0.475", "randsvd:1e12" or "mtx:/path/file.mtx"."""
        kind, _, arg = text.partition(":")
        kind = kind.strip().lower()
        if kind == "prolate":
            return cls("prolate", alpha=float(arg), n=n, seed=seed)
        if kind == "randsvd":
            return cls("randsvd", kappa2=float(arg), n=n, seed=seed)
        if kind == "mtx":
            return cls("mtx", path=arg, n=n, seed=seed)
        raise ValueError(f"unknown problem spec {text!r}")


@dataclass
class SweepSpec:
    """A grid of problems x methods under one setting (harness.py:118-131).
    ``jobs`` is accepted for signature parity; the sweep runs on one device,
    one solve at a time."""

    problems: list
    methods: list
    precisions: PrecisionTriple
    m: int
    k: int = 0
    tau: float | None = None
    i_max: int = 10000
    seed: int = 1
    scale_diag: bool = False
    jobs: int = 1
    skip_kappa2: bool = False


def format_cell(report: RefinementReport) -> str:
    """"total (c1,c2,...)"; divergent runs render "-" (harness.py:134-139)."""
    if not report.converged:
        return "-"
    return f"{report.total_inner} ({','.join(str(c) for c in report.inner_iters)})"


def cond_inf(a) -> float:
    """||A||_inf ||A^-1||_inf (densela.py:491-503); inf for a singular A."""
    a = np.asarray(a, dtype=np.float64)
    if a.ndim != 2 or a.shape[0] != a.shape[1]:
        raise ValueError("cond_inf requires a square matrix")
    try:
        inv = np.linalg.inv(a)
    except np.linalg.LinAlgError:
        return math.inf
    return float(np.max(np.sum(np.abs(a), axis=1)) * np.max(np.sum(np.abs(inv), axis=1)))


def _config(spec: SweepSpec, method: Method) -> RefineConfig:
    return RefineConfig(precisions=spec.precisions, method=method, m=spec.m, k=spec.k, tau=spec.tau,
                        i_max=spec.i_max, scale_diag=spec.scale_diag)


def _payload(rep: RefinementReport) -> dict:
    return {
        "converged": rep.converged,
        "steps": rep.steps,
        "inner_iters": list(rep.inner_iters),
        "total_inner": rep.total_inner,
        "nbe_history": [float(v) for v in rep.nbe_history],
        "ferr_history": [float(v) for v in rep.ferr_history],
        "divergence_reason": rep.divergence_reason.value if rep.divergence_reason else None,
        "solution": None if rep.solution is None else [float(v) for v in rep.solution],
        "diagnostics": {key: (float(val) if isinstance(val, (int, float)) else str(val))
                        for key, val in rep.diagnostics.items()},
    }


def _error_row(problem_id: str, spec: SweepSpec, method: Method, exc) -> dict:
    return {"problem_id": problem_id, "kappa_inf": math.nan, "kappa_2": math.nan, "method": method.value,
            "m": spec.m, "k": spec.k if method.uses_recycling else 0,
            "tau": spec.tau if spec.tau is not None else math.nan, "converged": False, "steps": 0,
            "total_inner": 0, "per_step": "", "nbe_final": math.nan, "ferr_final": math.nan,
            "divergence_reason": f"error: {exc}", "cell": "-", "report": None}


def _one_problem(spec: SweepSpec, ref: ProblemRef) -> list:
    try:
        a, b = ref.materialize()
        kinf = cond_inf(a)
        k2 = math.nan if spec.skip_kappa2 else float(np.linalg.cond(a))
    except Exception as exc:  # recorded in-row, the sweep continues (harness.py:181-187)
        return [_error_row(ref.problem_id, spec, method, exc) for method in spec.methods]
    rows = []
    for method in spec.methods:
        try:
            cfg = _config(spec, method)
            rep = solve(a, b, cfg)
            rows.append({
                "problem_id": ref.problem_id, "kappa_inf": kinf, "kappa_2": k2, "method": method.value,
                "m": spec.m, "k": spec.k if method.uses_recycling else 0, "tau": cfg.resolved_tau(),
                "converged": rep.converged, "steps": rep.steps, "total_inner": rep.total_inner,
                "per_step": ";".join(str(c) for c in rep.inner_iters), "nbe_final": rep.nbe_final,
                "ferr_final": rep.ferr_final,
                "divergence_reason": rep.divergence_reason.value if rep.divergence_reason else "",
                "cell": format_cell(rep), "report": _payload(rep),
            })
        except Exception as exc:
            rows.append(_error_row(ref.problem_id, spec, method, exc))
    return rows


def run_sweep(spec: SweepSpec) -> list:
    """One row per (problem, method) in spec order; failures recorded in-row
    (harness.py:242-258)."""
    if not spec.problems:
        raise ValueError("empty problem set")
    if not spec.methods:
        raise ValueError("empty method list")
    rows: list = []
    for ref in spec.problems:
        rows.extend(_one_problem(spec, ref))
    return rows


def kscan(problem: ProblemRef, cfg: RefineConfig, k_range) -> list:
    """Total inner iterations of the recycling method per k; divergent runs
    give -1 (harness.py:306-328)."""
    k_values = list(k_range)
    if any(k >= cfg.resolved_m(problem.n) for k in k_values):
        raise ValueError("every k must be smaller than m")
    a, b = problem.materialize()
    rows = []
    for k in k_values:
        rep = solve(a, b, replace(cfg, k=int(k)))
        rows.append({"k": int(k), "total_inner": rep.total_inner if rep.converged else -1})
    return rows

"""Parameter sweeps over the device solver.

The reference's experiment layer (harness.py:118-333) runs grids of solves
to rebuild the paper's Tables 5/6 and the recycle-dimension scan (Fig. 2).
This module keeps that role -- and the reference's row schema, so tables
built from either side line up -- on top of ``refine.solve`` (the CUDA
path).  The reference's command line (harness.py:389-572) is out of scope
 and is not mirrored.

Problems are written ``family:value`` (``prolate:0.475``, ``randsvd:1e4``,
``mtx:/path/to/file.mtx``); right-hand sides are all-ones, as in the
reference's harness (harness.py:101).  Per-problem condition numbers are host
statistics, outside any timed solve.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field, replace

import numpy as np

from . import problems as _gen
from .mtx import read_matrix_market
from .precision import Format, PrecisionTriple
from .refine import Method, RefineConfig, RefinementReport, solve

__all__ = ["Problem", "SweepSpec", "CSV_COLUMNS", "format_cell", "cond_inf", "run_sweep", "run_sweep_ranks",
           "kscan", "preconditioned_matrix", "spectrum_dump"]

# row schema of the reference's sweep output (harness.py:55-70)
CSV_COLUMNS = ("problem_id", "kappa_inf", "kappa_2", "method", "m", "k", "tau", "converged", "steps",
               "total_inner", "per_step", "nbe_final", "ferr_final", "divergence_reason")

_BUILDERS = {
    "prolate": lambda p: _gen.prolate(p.n, float(p.value)),
    "randsvd": lambda p: _gen.randsvd(p.n, float(p.value), p.seed),
    "mtx": lambda p: read_matrix_market(str(p.value)),
}


@dataclass(frozen=True)
class Problem:
    """One generated (or file-backed) system."""

    family: str
    value: float | str
    n: int = 100
    seed: int = 1

    @classmethod
    def from_text(cls, text: str, n: int = 100, seed: int = 1) -> "Problem":
        family, sep, value = text.partition(":")
        family = family.strip().lower()
        if not sep or family not in _BUILDERS:
            raise ValueError(f"problem must be prolate:<alpha>, randsvd:<kappa> or mtx:<path>, got {text!r}")
        return cls(family, value if family == "mtx" else float(value), n, seed)

    @property
    def label(self) -> str:
        if self.family == "mtx":
            base = str(self.value).replace("\\", "/").split("/")[-1]
            return base[: base.rfind(".")] if "." in base else base
        return f"{self.family}:{self.value:g}"

    def system(self) -> tuple[np.ndarray, np.ndarray]:
        a = _BUILDERS[self.family](self)
        return a, np.ones(a.shape[0])


@dataclass
class SweepSpec:
    """A grid of problems x methods under one precision / solver setting."""

    problems: list
    methods: list
    precisions: PrecisionTriple
    m: int
    k: int = 0
    tau: float | None = None
    i_max: int = 10000
    scale_diag: bool = False
    skip_kappa2: bool = False
    extra: dict = field(default_factory=dict)

    def config(self, method: Method) -> RefineConfig:
        return RefineConfig(precisions=self.precisions, method=method, m=self.m,
                            k=self.k if method.uses_recycling else 0, tau=self.tau, i_max=self.i_max,
                            scale_diag=self.scale_diag, **self.extra)


def format_cell(report: RefinementReport) -> str:
    """Table cell: ``total (step1,step2,...)``, or ``-`` when not converged."""
    return f"{report.total_inner} ({','.join(map(str, report.inner_iters))})" if report.converged else "-"


def cond_inf(a) -> float:
    a = np.asarray(a, dtype=np.float64)
    if a.ndim != 2 or a.shape[0] != a.shape[1]:
        raise ValueError("cond_inf needs a square matrix")
    try:
        return float(np.linalg.norm(a, np.inf) * np.linalg.norm(np.linalg.inv(a), np.inf))
    except np.linalg.LinAlgError:
        return math.inf


def _row(label: str, spec: SweepSpec, method: Method, stats: tuple, rep: RefinementReport | None,
         error: str | None = None) -> dict:
    cfg = spec.config(method)
    base = dict(problem_id=label, kappa_inf=stats[0], kappa_2=stats[1], method=method.value, m=spec.m,
                k=cfg.k, tau=cfg.resolved_tau() if error is None else (spec.tau if spec.tau else math.nan))
    if rep is None:
        return {**base, "converged": False, "steps": 0, "total_inner": 0, "per_step": "", "nbe_final": math.nan,
                "ferr_final": math.nan, "divergence_reason": f"error: {error}", "cell": "-", "report": None}
    return {**base, "converged": rep.converged, "steps": rep.steps, "total_inner": rep.total_inner,
            "per_step": ";".join(map(str, rep.inner_iters)), "nbe_final": rep.nbe_final,
            "ferr_final": rep.ferr_final,
            "divergence_reason": rep.divergence_reason.value if rep.divergence_reason else "",
            "cell": format_cell(rep), "report": rep}


def _problem_rows(spec: SweepSpec, prob: Problem) -> list:
    try:
        a, b = prob.system()
        stats = (cond_inf(a), math.nan if spec.skip_kappa2 else float(np.linalg.cond(a)))
    except Exception as exc:  # a broken problem is reported in its rows; the grid goes on
        return [_row(prob.label, spec, meth, (math.nan, math.nan), None, str(exc)) for meth in spec.methods]
    out = []
    for meth in spec.methods:
        try:
            out.append(_row(prob.label, spec, meth, stats, solve(a, b, spec.config(meth))))
        except Exception as exc:
            out.append(_row(prob.label, spec, meth, stats, None, str(exc)))
    return out


def _validate(spec: SweepSpec) -> None:
    if not spec.problems or not spec.methods:
        raise ValueError("a sweep needs at least one problem and one method")


def run_sweep(spec: SweepSpec) -> list:
    """Rows for every (problem, method), problems in order, methods inner."""
    _validate(spec)
    return [row for prob in spec.problems for row in _problem_rows(spec, prob)]


def run_sweep_ranks(spec: SweepSpec, group=None) -> list:
    """``run_sweep`` split over the ranks of a torch.distributed group: rank
    r solves problems r, r+W, ...; one object all-gather returns the full
    row list (spec order) on every rank.  The caller pins one GPU per rank
    (bench.py does); this function selects LOCAL_RANK's device when torch
    sees several and none was chosen."""
    import os

    import torch
    import torch.distributed as dist

    _validate(spec)
    if torch.cuda.is_available() and torch.cuda.device_count() > 1 and "LOCAL_RANK" in os.environ:
        torch.cuda.set_device(int(os.environ["LOCAL_RANK"]) % torch.cuda.device_count())
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    mine = [(i, _problem_rows(spec, p)) for i, p in enumerate(spec.problems) if i % world == rank]
    gathered = [None] * world
    dist.all_gather_object(gathered, mine, group=group)
    by_index = dict(item for part in gathered for item in part)
    return [row for i in sorted(by_index) for row in by_index[i]]


def kscan(problem: Problem, cfg: RefineConfig, k_values) -> list:
    """Total inner iterations of a recycling solve for each k (-1 where the
    solve does not converge) -- the Fig. 2 knee scan."""
    ks = [int(k) for k in k_values]
    m = cfg.resolved_m(problem.n)
    bad = [k for k in ks if not 1 <= k < m]
    if bad:
        raise ValueError(f"recycle dimensions {bad} outside 1 <= k < m = {m}")
    a, b = problem.system()
    out = []
    for k in ks:
        rep = solve(a, b, replace(cfg, k=k))
        out.append({"k": k, "total_inner": rep.total_inner if rep.converged else -1})
    return out


def preconditioned_matrix(a, factors) -> np.ndarray:
    """U^-1 L^-1 P A at double, built column by column from device operator
    applications (the matrix whose spectrum the reference dumps)."""
    from . import densela

    a = np.asarray(a, dtype=np.float64)
    cols = np.eye(a.shape[0])
    return np.stack([densela.apply_preconditioned(a, factors, c, Format.DOUBLE, Format.DOUBLE) for c in cols],
                    axis=1)


def spectrum_dump(a, uf_format: Format, out) -> list:
    """Eigenvalues of A and of the preconditioned operators for LU factors at
    double and at ``uf_format``, written as ``set,re,im`` CSV points (sorted by
    modulus); returns the names of the sets written.  Factors and operator
    columns come from the device; the n x n eigensolve (n <= 500) is LAPACK
    on the host, as in the reference."""
    from . import densela

    a = np.asarray(a, dtype=np.float64)
    if a.shape[0] > 500:
        raise ValueError("spectrum dump supports n <= 500")
    mats = [("original", a)]
    for fmt in (Format.DOUBLE, uf_format):  # uf = double writes the double set twice, as the reference does
        fac = densela.lu_factor(a, fmt)
        try:
            mats.append((f"precond_{fmt.value}", preconditioned_matrix(a, fac)))
        finally:
            fac.close()
    written, lines = [], ["set,re,im"]
    for name, mat in mats:
        try:
            ev = np.linalg.eigvals(mat)
        except np.linalg.LinAlgError:
            continue
        written.append(name)
        lines += [f"{name},{float(z.real)!r},{float(z.imag)!r}" for z in ev[np.argsort(np.abs(ev), kind="stable")]]
    with open(out, "w", encoding="ascii") as fh:
        fh.write("\n".join(lines) + "\n")
    return written

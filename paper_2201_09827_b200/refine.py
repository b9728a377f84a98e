"""Mixed-precision iterative refinement drivers -- the drop-in API.

Mirrors ``irkit.refine`` (reference refine.py:56-464): the same ``Method``,
``RefineConfig`` fields and defaults, ``RefinementReport`` fields and the same
decision rules.  The refinement loop stays on the host (north_star); each
iteration is ONE device launch (``gb_refine_step``: residual-scaled
correction solve by GCRO-DR / GMRES / LU substitution, the update, the forward
error and the new residual with nbe/cbe), and only its scalars come back.
"""

from __future__ import annotations

import enum
import math
import threading
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .precision import Format, PrecisionTriple, half_flushes_subnormals, squared_format

__all__ = [
    "Method",
    "DivergenceReason",
    "RefineConfig",
    "RefinementReport",
    "ConvergenceDecision",
    "classify",
    "sir",
    "gmres_ir",
    "rgmres_ir",
    "solve",
]


class Method(enum.Enum):
    SIR = "sir"
    GMRES_IR = "gmres-ir"
    SGMRES_IR = "sgmres-ir"
    RGMRES_IR = "rgmres-ir"
    RSGMRES_IR = "rsgmres-ir"

    @classmethod
    def parse(cls, name: str) -> "Method":
        try:
            return cls(name.strip().lower())
        except ValueError:
            raise ValueError(f"unknown method {name!r}; expected one of {[m.value for m in cls]}") from None

    @property
    def uses_gmres(self) -> bool:
        return self in (Method.GMRES_IR, Method.SGMRES_IR)

    @property
    def uses_recycling(self) -> bool:
        return self in (Method.RGMRES_IR, Method.RSGMRES_IR)

    @property
    def uniform_precision(self) -> bool:
        return self in (Method.SGMRES_IR, Method.RSGMRES_IR)

    @property
    def code(self) -> int:
        return {"sir": _lib.SIR, "gmres-ir": _lib.GMRES_IR, "sgmres-ir": _lib.SGMRES_IR,
                "rgmres-ir": _lib.RGMRES_IR, "rsgmres-ir": _lib.RSGMRES_IR}[self.value]


class DivergenceReason(enum.Enum):
    I_MAX_EXCEEDED = "IMaxExceeded"
    INNER_STAGNATION = "InnerStagnation"
    ERROR_GROWTH = "ErrorGrowth"


_DEFAULT_TAU = {Format.HALF: 1e-2, Format.SINGLE: 1e-4, Format.DOUBLE: 1e-8, Format.QUAD: 1e-8}


@dataclass
class RefineConfig:
    """refine.py:100-134 (same fields, same defaults)."""

    precisions: PrecisionTriple
    method: Method = Method.GMRES_IR
    m: int = 0
    k: int = 0
    tau: float | None = None
    i_max: int = 10000
    extra_precision_matvec: bool | None = None
    c_conv: float = 2.0
    max_cycles: int | None = None
    reorthogonalize: bool = True
    scale_diag: bool = False
    collect_diagnostics: bool = False
    restart_residual: str = "recurrence"
    cycle_residual: str = "recurrence"
    # extension (not in the reference): "exact" reproduces the reference's
    # u_f arithmetic bit for bit; "tensor" runs the fp16 trailing update on
    # tcgen05 tensor cores with fp32 accumulation (pivots agree up to ties)
    lu_mode: str = "exact"

    def resolved_tau(self) -> float:
        return self.tau if self.tau is not None else _DEFAULT_TAU[self.precisions.u]

    def resolved_extra_precision(self) -> bool:
        if self.extra_precision_matvec is not None:
            return self.extra_precision_matvec
        return not self.method.uniform_precision

    def matvec_format(self) -> Format:
        u = self.precisions.u
        return squared_format(u) if self.resolved_extra_precision() else u

    def resolved_m(self, n: int) -> int:
        return self.m if self.m else min(n, 40)

    def resolved_max_cycles(self, n: int) -> int:
        if self.max_cycles is not None:
            return self.max_cycles
        return max(1, math.ceil(10 * n / self.resolved_m(n)))


@dataclass
class RefinementReport:
    """refine.py:137-160."""

    converged: bool
    steps: int
    inner_iters: list[int]
    nbe_history: list[float]
    ferr_history: list[float]
    divergence_reason: DivergenceReason | None = None
    solution: np.ndarray | None = None
    diagnostics: dict = field(default_factory=dict)

    @property
    def total_inner(self) -> int:
        return sum(self.inner_iters)

    @property
    def nbe_final(self) -> float:
        return self.nbe_history[-1] if self.nbe_history else float("nan")

    @property
    def ferr_final(self) -> float:
        return self.ferr_history[-1] if self.ferr_history else float("nan")


@dataclass
class ConvergenceDecision:
    state: str  # "continue" | "converged" | "diverged"
    reason: DivergenceReason | None
    nbe: float
    cbe: float = float("nan")
    ferr: float = float("nan")


def classify(nbe: float, cbe: float, ferr: float, history: list[float], precisions: PrecisionTriple,
             c_conv: float = 2.0, inner_stagnated: bool = False) -> ConvergenceDecision:
    """The decision rules of check_convergence (refine.py:210-229) applied to
    device-computed nbe / cbe (the residual itself never leaves the GPU)."""
    gate = c_conv * precisions.u.unit_roundoff
    worst = max(nbe, cbe, ferr if math.isfinite(ferr) else 0.0)
    if math.isfinite(worst) and worst <= gate:
        return ConvergenceDecision("converged", None, nbe, cbe, ferr)
    if inner_stagnated:
        return ConvergenceDecision("diverged", DivergenceReason.INNER_STAGNATION, nbe, cbe, ferr)
    growth = 0
    seq = history + [nbe]
    for prev, cur in zip(seq[:-1], seq[1:]):
        if not math.isfinite(cur) or (math.isfinite(prev) and cur >= 2.0 * prev):
            growth += 1
        else:
            growth = 0
    if growth >= 3:
        return ConvergenceDecision("diverged", DivergenceReason.ERROR_GROWTH, nbe, cbe, ferr)
    return ConvergenceDecision("continue", None, nbe, cbe, ferr)


def make_options(cfg: RefineConfig, n: int, grid_ctas: int = 0) -> _lib.Options:
    """Resolve a RefineConfig into the C-ABI option block (refine.py:327-353)."""
    prec = cfg.precisions
    m = cfg.resolved_m(n)
    if not (1 <= m <= n):
        raise ValueError(f"restart length m={m} must satisfy 1 <= m <= n={n}")
    if cfg.method.uses_recycling and not (1 <= cfg.k < m):
        raise ValueError("recycling methods need 1 <= k < m")
    if not cfg.resolved_tau() > 0:
        raise ValueError("tolerance tau must be positive")
    if half_flushes_subnormals() and Format.HALF in (prec.uf, prec.u, prec.ur):
        raise NotImplementedError("half flush-to-zero (set_half_flush_subnormals(True)) is not built "
                                  "on the device path")
    o = _lib.Options()
    o.uf, o.u, o.ur = prec.uf.code, prec.u.code, prec.ur.code
    o.method = cfg.method.code
    o.m, o.k = m, (cfg.k if cfg.method.uses_recycling else 0)
    o.tau = cfg.resolved_tau()
    o.max_cycles = cfg.resolved_max_cycles(n)
    o.reorthogonalize = int(bool(cfg.reorthogonalize))
    o.extra_precision = int(cfg.resolved_extra_precision())
    o.grid_ctas = grid_ctas
    if cfg.lu_mode not in ("exact", "tensor"):
        raise ValueError(f"unknown lu_mode {cfg.lu_mode!r}")
    o.lu_mode = 1 if cfg.lu_mode == "tensor" else 0
    # any value other than "recurrence" recomputes s - A~ x at the restart,
    # as the reference does (gmres.py:292-295; gcrodr.py:301-304, 376-379);
    # plain GMRES reads restart_residual, GCRO-DR cycle_residual (refine.py:338, 352)
    mode = cfg.cycle_residual if cfg.method.uses_recycling else cfg.restart_residual
    o.explicit_residual = int(mode != "recurrence")
    return o


def _pow2_equilibrate(a: np.ndarray, b: np.ndarray):
    """Two-sided power-of-two scaling (refine.py:261-270); exact in binary."""
    row = np.max(np.abs(a), axis=1)
    row[row == 0.0] = 1.0
    dr = 2.0 ** (-np.round(np.log2(row)))
    a1 = dr[:, None] * a
    col = np.max(np.abs(a1), axis=0)
    col[col == 0.0] = 1.0
    dc = 2.0 ** (-np.round(np.log2(col)))
    return a1 * dc[None, :], dr * b, dc


def _round_u(x: np.ndarray, u: Format) -> np.ndarray:
    if u is Format.SINGLE:
        return x.astype(np.float32).astype(np.float64)
    if u is Format.HALF:
        return x.astype(np.float16).astype(np.float64)
    return x


# Device workspaces are kept between solves of the same order and options
# (allocating and freeing ~n^2 buffers per call would dominate small solves).
# A cached solver is taken out of the cache while in use, so concurrent calls
# never share one; gb_set_system resets all per-solve device state.
_SOLVER_CACHE: dict = {}
_SOLVER_CACHE_MAX = 2
_SOLVER_LOCK = threading.Lock()


def _options_key(n: int, o) -> tuple:
    # a cached solver owns device memory on the device that was current at
    # creation and launches on the stream captured then: key on both
    return (_lib.current_device(), _lib.current_stream(), n) + tuple(getattr(o, f) for f, _ in o._fields_)


def _acquire_solver(n: int, opts):
    key = _options_key(n, opts)
    with _SOLVER_LOCK:
        cached = _SOLVER_CACHE.pop(key, None)
    return key, (cached if cached is not None else _lib.Solver(n, opts))


def _release_solver(key, solver) -> None:
    with _SOLVER_LOCK:
        if key not in _SOLVER_CACHE and len(_SOLVER_CACHE) < _SOLVER_CACHE_MAX:
            _SOLVER_CACHE[key] = solver
            return
    solver.close()


def release_workspaces() -> None:
    """Free the device workspaces kept between solves."""
    with _SOLVER_LOCK:
        cached = list(_SOLVER_CACHE.values())
        _SOLVER_CACHE.clear()
    for s in cached:
        s.close()


def _refine(a, b, cfg: RefineConfig, *, trace: list | None = None, grid_ctas: int = 0) -> RefinementReport:
    prec = cfg.precisions
    if prec.u not in (Format.SINGLE, Format.DOUBLE):
        raise NotImplementedError("working precision u must be single or double on this build")
    a = np.ascontiguousarray(a, dtype=np.float64)
    b = np.ascontiguousarray(b, dtype=np.float64)
    n = a.shape[0]
    if a.ndim != 2 or a.shape != (n, n) or b.shape != (n,):
        raise ValueError("need a square matrix and a matching right-hand side")
    diagnostics: dict = {}
    col_scale = None
    if cfg.scale_diag:
        # host-side input scaling by powers of two (exact); rounding to u of the
        # scaled data is repeated on the device, as in refine.py:293-297
        a, b, col_scale = _pow2_equilibrate(_round_u(a, prec.u), _round_u(b, prec.u))
        diagnostics["equilibrated"] = True
    opts = make_options(cfg, n, grid_ctas)
    key, solver = _acquire_solver(n, opts)
    ok = False
    try:
        solver.set_system(a, b)
        zero, growth = solver.factorize()
        if zero >= 0:
            ok = True
            return RefinementReport(False, 0, [], [], [], DivergenceReason.INNER_STAGNATION, None,
                                    {"lu_failed": f"exact zero pivot at column {zero}", **diagnostics})
        diagnostics["lu_growth"] = growth
        if solver.initial_solution():
            diagnostics["x0_reset"] = True
        if not solver.reference_solution():
            diagnostics["no_reference_solution"] = True
        nbe_hist: list[float] = []
        ferr_hist: list[float] = []
        inner: list[int] = []
        reason: DivergenceReason | None = DivergenceReason.I_MAX_EXCEEDED
        converged = False
        for _ in range(cfg.i_max):
            info = solver.step()
            if trace is not None:
                cyc, keff = solver.last_cycles()
                trace.append({"nu": info.nu, "cycles": cyc, "k_eff": keff, "applies": info.applies,
                              "status": info.status, "ms": solver.last_step_ms})
            if info.status & (_lib.ST_NU_ZERO | _lib.ST_NU_NONFINITE):
                if info.status & _lib.ST_NU_ZERO:
                    converged, reason = True, None
                    inner.append(0)
                    nbe_hist.append(0.0)
                    ferr_hist.append(info.ferr)
                else:
                    reason = DivergenceReason.ERROR_GROWTH
                break
            inner.append(int(info.inner_iters))
            stagnated = bool(info.status & _lib.ST_STAGNATED) and cfg.method is not Method.SIR
            decision = classify(info.nbe, info.cbe, info.ferr, nbe_hist, prec, cfg.c_conv, stagnated)
            nbe_hist.append(decision.nbe)
            ferr_hist.append(info.ferr)
            if decision.state == "converged":
                converged, reason = True, None
                break
            if decision.state == "diverged":
                reason = decision.reason
                break
        solution = solver.solution()
        if col_scale is not None:
            solution = col_scale * solution
        ok = True
        return RefinementReport(converged, len(inner), inner, nbe_hist, ferr_hist,
                                None if converged else reason, solution, diagnostics)
    finally:
        if ok:
            _release_solver(key, solver)
        else:
            solver.close()


def check_convergence(a, b, x, d, history, precisions: PrecisionTriple, c_conv: float = 2.0,
                      inner_stagnated: bool = False, norm_a_inf: float | None = None,
                      norm_b_inf: float | None = None, ferr: float = float("nan")) -> ConvergenceDecision:
    """refine.py:172-229: residual at u_r, nbe, cbe on the device
    (gb_backward_errors), the decision rules on the host (``classify``).  The
    norms are those of fl_u(a), fl_u(b) as the loop holds them; passing other
    values is not supported on the device path."""
    del d  # unused by the reference too
    a = np.ascontiguousarray(a, dtype=np.float64)
    b = np.ascontiguousarray(b, dtype=np.float64)
    x = np.ascontiguousarray(x, dtype=np.float64)
    n = a.shape[0]
    if a.shape != (n, n) or b.shape != (n,) or x.shape != (n,):
        raise ValueError("dimension mismatch in check_convergence")
    if norm_a_inf is not None or norm_b_inf is not None:
        raise NotImplementedError("the device computes ||A||_inf and ||b||_inf itself")
    cfg = RefineConfig(precisions, Method.GMRES_IR, m=min(n, 2))
    solver = _lib.Solver(n, make_options(cfg, n))
    try:
        solver.set_system(a, b)
        _, nbe, cbe = solver.backward_errors(x)
    finally:
        solver.close()
    return classify(nbe, cbe, ferr, list(history), precisions, c_conv, inner_stagnated)


def sir(a, b, cfg: RefineConfig) -> RefinementReport:
    if cfg.method is not Method.SIR:
        raise ValueError("sir() requires cfg.method == Method.SIR")
    return _refine(a, b, cfg)


def gmres_ir(a, b, cfg: RefineConfig) -> RefinementReport:
    if not cfg.method.uses_gmres:
        raise ValueError("gmres_ir() requires a GMRES-based method")
    return _refine(a, b, cfg)


def rgmres_ir(a, b, cfg: RefineConfig) -> RefinementReport:
    if not cfg.method.uses_recycling:
        raise ValueError("rgmres_ir() requires a recycling method")
    return _refine(a, b, cfg)


def solve(a, b, cfg: RefineConfig) -> RefinementReport:
    """Dispatch on cfg.method (refine.py:458-464)."""
    if cfg.method is Method.SIR:
        return sir(a, b, cfg)
    if cfg.method.uses_gmres:
        return gmres_ir(a, b, cfg)
    return rgmres_ir(a, b, cfg)

"""The inner solvers of the refinement loop as standalone entry points,
mirroring ``irkit.gmres.gmres_solve`` (gmres.py:235-311) and
``irkit.gcrodr.gcrodr_solve`` (gcrodr.py:221-419) over the device context of
an ``LUFactors`` (densela.lu_factor): one launch of the step kernel in its
inner-solver-only mode (``gb_debug_inner_solve``).  No CPU path.

The recycle space stays on the device: ``gcrodr_solve`` returns a
``RecycleSpace`` handle naming the context that holds U_k; passing it back as
``recycle_in`` warm-starts the next solve from it (gcrodr.py:268-285), passing
``None`` starts cold.  ``Yk`` / ``Uk`` / ``Ck`` are not copied to the host.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .densela import LUFactors, _fmt
from .precision import Format, PrecisionTriple
from .refine import Method, RefineConfig, make_options

__all__ = ["GmresConfig", "GmresOutcome", "GcrodrConfig", "RecycleSpace", "gmres_solve", "gcrodr_solve"]


def _ceil_cycles(n: int, m: int, given: int | None) -> int:
    return given if given is not None else max(1, math.ceil(10 * n / m))


@dataclass
class GmresConfig:
    """gmres.py:36-62."""

    m: int
    tau: float
    matvec_ctx: object
    work_fmt: Format
    max_cycles: int | None = None
    reorthogonalize: bool = True
    restart_residual: str = "recurrence"

    def resolved_max_cycles(self, n: int) -> int:
        return _ceil_cycles(n, self.m, self.max_cycles)

    def validate(self, n: int) -> None:
        if not (1 <= self.m <= n):
            raise ValueError(f"restart length m={self.m} must satisfy 1 <= m <= n={n}")
        if not self.tau > 0:
            raise ValueError("tolerance tau must be positive")
        if self.resolved_max_cycles(n) < 1:
            raise ValueError("max_cycles must be >= 1")


@dataclass
class GcrodrConfig:
    """gcrodr.py:68-97."""

    m: int
    k: int
    tau: float
    matvec_ctx: object
    work_fmt: Format
    max_cycles: int | None = None
    reorthogonalize: bool = True
    collect_diagnostics: bool = False
    cycle_residual: str = "recurrence"

    def resolved_max_cycles(self, n: int) -> int:
        return _ceil_cycles(n, self.m, self.max_cycles)

    def validate(self, n: int) -> None:
        if not (1 <= self.k < self.m <= n):
            raise ValueError(f"need 1 <= k < m <= n, got k={self.k}, m={self.m}, n={n}")
        if not self.tau > 0:
            raise ValueError("tolerance tau must be positive")


@dataclass
class GmresOutcome:
    """gmres.py:65-81.  ``basis`` stays on the device (None); ``final_relres``
    is not returned by the device solver (NaN); ``cycle_diagnostics`` carries
    the per-cycle (kind, steps, k_eff) the device records when asked."""

    solution: np.ndarray
    iterations_per_cycle: list
    converged: bool
    final_relres: float = float("nan")
    basis: tuple | None = None
    stagnated: bool = False
    happy_breakdown: bool = False
    operator_applies: int = 0
    cycle_diagnostics: list | None = None

    @property
    def total_iterations(self) -> int:
        return sum(self.iterations_per_cycle)


@dataclass
class RecycleSpace:
    """Handle of the device-resident (U_k, C_k) of one context (gcrodr.py:60-66)."""

    k_eff: int
    _owner: object = field(default=None, repr=False)


def _context(f: LUFactors, method: Method, m: int, k: int, tau: float, mv: Format, u: Format, max_cycles: int,
             reorth: bool, residual_mode: str) -> _lib.Solver:
    if u not in (Format.SINGLE, Format.DOUBLE):
        raise NotImplementedError("working precision u must be single or double on this build")
    key = ("krylov", method, m, k, tau, mv, u, max_cycles, reorth, residual_mode)
    s = f._ctx.get(key)
    if s is None:
        cfg = RefineConfig(PrecisionTriple(f.format, u, Format.DOUBLE), method, m=m, k=k, tau=tau,
                           extra_precision_matvec=mv is not u, max_cycles=max_cycles, reorthogonalize=reorth,
                           restart_residual=residual_mode, cycle_residual=residual_mode)
        s = _lib.Solver(f.n, make_options(cfg, f.n))
        s.set_system(f._a, np.zeros(f.n))
        zero, _ = s.factorize()
        if zero >= 0:
            s.close()
            raise RuntimeError("factorisation of the context failed")
        f._ctx[key] = s
    return s


def _outcome(s: _lib.Solver, d: np.ndarray, info, recycling: bool, want_diag: bool, keff_in: int = 0) -> GmresOutcome:
    cycles, keff = s.last_cycles()
    diag = None
    if want_diag:
        diag = [{"kind": "cold" if (i == 0 and not keff_in) else "deflated", "steps": int(c), "k_eff": int(ke)}
                for i, (c, ke) in enumerate(zip(cycles, keff))] if recycling else []
    conv = bool(info.status & _lib.ST_CONVERGED)
    return GmresOutcome(d, [int(c) for c in cycles], conv, stagnated=not conv,
                        happy_breakdown=bool(info.status & _lib.ST_BREAKDOWN), operator_applies=int(info.applies),
                        cycle_diagnostics=diag)


def gmres_solve(a, f: LUFactors, r, cfg: GmresConfig) -> GmresOutcome:
    """Restarted GMRES(m) on U^-1 L^-1 A d = U^-1 L^-1 r (gmres.py:235-311)."""
    a = np.asarray(a, dtype=np.float64)
    r = np.ascontiguousarray(r, dtype=np.float64)
    n = f.n
    if a.shape != (n, n) or r.shape != (n,):
        raise ValueError("dimension mismatch in gmres_solve")
    cfg.validate(n)
    s = _context(f, Method.GMRES_IR, cfg.m, 0, cfg.tau, _fmt(cfg.matvec_ctx), cfg.work_fmt,
                 cfg.resolved_max_cycles(n), cfg.reorthogonalize, cfg.restart_residual)
    d, info = s.inner_solve(r, reset_recycle=True)
    return _outcome(s, d, info, False, False)


def gcrodr_solve(a, f: LUFactors, r, cfg: GcrodrConfig, recycle_in: RecycleSpace | None = None):
    """One GCRO-DR(m, k) solve (gcrodr.py:221-419): (outcome, recycle space
    for the next call)."""
    a = np.asarray(a, dtype=np.float64)
    r = np.ascontiguousarray(r, dtype=np.float64)
    n = f.n
    if a.shape != (n, n) or r.shape != (n,):
        raise ValueError("dimension mismatch in gcrodr_solve")
    cfg.validate(n)
    s = _context(f, Method.RGMRES_IR, cfg.m, cfg.k, cfg.tau, _fmt(cfg.matvec_ctx), cfg.work_fmt,
                 cfg.resolved_max_cycles(n), cfg.reorthogonalize, cfg.cycle_residual)
    if recycle_in is not None and recycle_in._owner is not s:
        raise NotImplementedError("the recycle space lives in the device context that produced it")
    d, info = s.inner_solve(r, reset_recycle=recycle_in is None)
    out = _outcome(s, d, info, True, cfg.collect_diagnostics, recycle_in.k_eff if recycle_in is not None else 0)
    space = RecycleSpace(int(info.keff), s) if info.keff > 0 else None
    return out, space

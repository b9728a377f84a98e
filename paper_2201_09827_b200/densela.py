"""Kernel-level entry points of the solve loop, mirroring the reference's
``densela`` functions (densela.py:58-361) over the device context.

``lu_factor`` factorises on the GPU and hands back an ``LUFactors`` whose
L / U / perm are the device factors (fp16 factors bit-identical to the
reference's, fp32 factors with the same pivots up to ties); the factors stay
resident in a device context attached to the object, and ``lu_solve``,
``apply_preconditioned``, ``precond_rhs`` and ``residual`` run the CUDA
kernels against it.  There is no CPU path: without the library or a GPU
every call raises ``GpuUnavailable``.

Device precisions: a context stores vectors at a working precision u
strictly wider than the factor format (the narrowest that holds A exactly,
or the ``store_fmt`` a call asks for) and holds A exactly -- the operands
of the solve path, where A is already u-valued (refine.py:285, 317, 363).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .precision import Format, PrecisionTriple
from .refine import Method, RefineConfig, make_options

__all__ = ["ExactZeroPivot", "LUFactors", "lu_factor", "lu_solve", "apply_preconditioned", "precond_rhs",
           "residual"]

_ORDER = [Format.HALF, Format.SINGLE, Format.DOUBLE, Format.QUAD]


class ExactZeroPivot(Exception):
    """A pivot column is exactly zero at the factor precision (densela.py:58-63)."""

    def __init__(self, index: int):
        self.index = index
        super().__init__(f"exact zero pivot at column {index}")


def _fmt(ctx) -> Format:
    """A Format, a format name, or a context object carrying ``.format``."""
    if isinstance(ctx, Format):
        return ctx
    if isinstance(ctx, str):
        return Format.parse(ctx)
    return ctx.format


@dataclass
class LUFactors:
    """GEPP factors with A[perm, :] = L @ U (densela.py:82-106)."""

    L: np.ndarray
    U: np.ndarray
    perm: np.ndarray
    format: Format
    growth: float
    _a: np.ndarray | None = field(default=None, repr=False)
    _ctx: dict = field(default_factory=dict, repr=False)

    @property
    def n(self) -> int:
        return self.L.shape[0]

    def _device(self, u: Format, extra: bool | None = None) -> _lib.Solver:
        """Device context holding A and these factors at working precision u,
        its operator at u^2 (extra) or u."""
        extra = _default_extra(self.format, u) if extra is None else extra
        s = self._ctx.get((u, extra))
        if s is None:
            if not _exact_in(self._a, u):
                raise NotImplementedError(f"A is not exactly representable at u = {u.value}; a device "
                                          "context there would factor a different matrix")
            s = _context(self._a, self.format, u, extra)
            zero, _ = s.factorize()
            if zero >= 0:
                raise ExactZeroPivot(zero)
            self._ctx[(u, extra)] = s
        return s

    def close(self) -> None:
        for s in self._ctx.values():
            s.close()
        self._ctx.clear()


def _default_extra(uf: Format, u: Format) -> bool:
    """Operator at u^2 as on the solve path, except for fp64 factors at u =
    double (the build compiles that variant with the fp64 operator only)."""
    return not (uf is u is Format.DOUBLE)


def _context(a: np.ndarray, uf: Format, u: Format, extra: bool | None = None) -> _lib.Solver:
    wider = _ORDER.index(u) > _ORDER.index(uf) or u is uf is Format.DOUBLE  # fp64 factors: u = double
    if not wider or u not in (Format.SINGLE, Format.DOUBLE):
        raise NotImplementedError(f"no device context stores {uf.value} factors at u = {u.value}")
    n = a.shape[0]
    ur = Format.DOUBLE
    extra = _default_extra(uf, u) if extra is None else extra
    cfg = RefineConfig(PrecisionTriple(uf, u, ur), Method.GMRES_IR, m=min(n, 2), extra_precision_matvec=extra)
    s = _lib.Solver(n, make_options(cfg, n))
    s.set_system(a, np.zeros(n))
    return s


def _exact_in(a: np.ndarray, u: Format) -> bool:
    if u is Format.DOUBLE:
        return True
    with np.errstate(over="ignore", invalid="ignore"):
        return bool(np.array_equal(a.astype(np.float32).astype(np.float64), a, equal_nan=True))


def _default_u(uf: Format, a: np.ndarray | None = None) -> Format:
    """Narrowest device working precision above uf that holds A exactly, so
    the factors are those of GEPP on A itself (densela.py:124-131)."""
    if uf is Format.HALF and (a is None or _exact_in(a, Format.SINGLE)):
        return Format.SINGLE
    return Format.DOUBLE


def lu_factor(a, ctx) -> LUFactors:
    """GEPP at the factor precision on the device (densela.py:124-168).
    Raises ``ExactZeroPivot`` on a zero pivot column, ``ValueError`` for a
    non-square input."""
    a = np.ascontiguousarray(a, dtype=np.float64)
    if a.ndim != 2 or a.shape[0] != a.shape[1]:
        raise ValueError("lu_factor requires a square matrix")
    uf = _fmt(ctx)
    u = _default_u(uf, a)
    s = _context(a, uf, u)
    zero, growth = s.factorize()
    if zero >= 0:
        s.close()
        raise ExactZeroPivot(zero)
    lu, perm = s.factors()
    L = np.tril(lu, -1) + np.eye(a.shape[0])
    U = np.triu(lu)
    f = LUFactors(L, U, perm, uf, float(growth), _a=a)
    f._ctx[(u, _default_extra(uf, u))] = s
    return f


def _vec(x, n: int, what: str) -> np.ndarray:
    x = np.ascontiguousarray(x, dtype=np.float64)
    if x.shape != (n,):
        raise ValueError(f"{what} length does not match the factors")
    return x


def lu_solve(f: LUFactors, b, ctx, store_fmt: Format | None = None) -> np.ndarray:
    """x = U^-1 L^-1 b[perm] with every operation at the factor precision
    (densela.py:235-261); the result is exact in the factor format, so
    ``store_fmt`` (wider than it on the device) leaves it unchanged."""
    if _fmt(ctx) is not f.format:
        raise NotImplementedError("the device substitutes in the factor precision only")
    b = _vec(b, f.n, "right-hand side")
    u = store_fmt if store_fmt is not None and store_fmt is not f.format else _default_u(f.format, f._a)
    return f._device(u).lu_solve(b)


def apply_preconditioned(a, f: LUFactors, v, matvec_ctx, store_fmt: Format) -> np.ndarray:
    """fl_store(U^-1 L^-1 (A v)[perm]) with the multiply and both solves at
    ``matvec_ctx`` (densela.py:268-299); ``matvec_ctx`` is store_fmt or its
    square (refine.py:129-131)."""
    a = np.asarray(a, dtype=np.float64)
    if a.shape != (f.n, f.n):
        raise ValueError("dimension mismatch in apply_preconditioned")
    if a is not f._a and not np.array_equal(a, f._a, equal_nan=True):
        raise NotImplementedError("the device operator uses the matrix the factors were computed from")
    v = _vec(v, f.n, "vector")
    mv = _fmt(matvec_ctx)
    return f._device(store_fmt, mv is not store_fmt).apply_preconditioned(v, mv.code)


def precond_rhs(f: LUFactors, r, matvec_ctx, store_fmt: Format) -> np.ndarray:
    """fl_store(U^-1 L^-1 r[perm]) at ``matvec_ctx`` (densela.py:314-333)."""
    r = _vec(r, f.n, "vector")
    mv = _fmt(matvec_ctx)
    return f._device(store_fmt, mv is not store_fmt).precond_rhs(r, mv.code)


def residual(a, x, b, ctx) -> np.ndarray:
    """r = b - A x accumulated at ``ctx`` (densela.py:340-361) on the device;
    A and b are held exactly (u = double)."""
    a = np.ascontiguousarray(a, dtype=np.float64)
    if a.ndim != 2 or a.shape[0] != a.shape[1]:
        raise ValueError("residual requires a square matrix")
    n = a.shape[0]
    x = _vec(x, n, "x")
    b = _vec(b, n, "b")
    s = _context(a, Format.SINGLE, Format.DOUBLE)
    try:
        s.set_system(a, b)
        return s.residual(x, _fmt(ctx).code)
    finally:
        s.close()

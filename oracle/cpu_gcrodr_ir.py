"""CPU oracle: a numpy restatement of the reference GCRO-DR-IR path.

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py`` (its ``cpu_baseline`` leg and ``--impl reference`` arm) may import
this module, and only as the checker / the timed CPU reference -- never as
part of the shipped product path (``paper_2201_09827_b200`` never imports it).

It restates ``irkit`` (reference ``/root/reference/pkg/src/irkit``) function
by function with the same numpy / scipy (OpenBLAS / LAPACK) calls on the same
array layouts, so that on one machine and BLAS thread count it reproduces the
reference's numbers bit for bit.  That claim is PINNED by
``tests/test_oracle_golden.py`` against fixtures captured by running the
reference itself (``tests/golden/make_goldens.py``).  Every function cites the
reference ``file:line`` it follows; paths are relative to
``/root/reference/pkg/src/irkit/``.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np
import scipy.linalg

# ---------------------------------------------------------------------------
# formats (precision.py:54-107, 169-199)
# ---------------------------------------------------------------------------

HALF, SINGLE, DOUBLE, QUAD = "half", "single", "double", "quad"
UNIT_ROUNDOFF = {HALF: 2.0 ** -11, SINGLE: 2.0 ** -24, DOUBLE: 2.0 ** -53, QUAD: 2.0 ** -105}
_NP = {HALF: np.float16, SINGLE: np.float32}
_SQUARED = {HALF: SINGLE, SINGLE: DOUBLE, DOUBLE: QUAD, QUAD: QUAD}
DEFAULT_TAU = {HALF: 1e-2, SINGLE: 1e-4, DOUBLE: 1e-8, QUAD: 1e-8}  # refine.py:92-97

# process-wide half flush-to-zero (precision.py:111-128)
_FTZ = {"on": False}


def set_half_ftz(flag: bool) -> bool:
    old, _FTZ["on"] = _FTZ["on"], bool(flag)
    return old


def squared(fmt: str) -> str:
    """u^2 evaluation format (precision.py:169-175)."""
    return _SQUARED[fmt]


def check_triple(uf: str, u: str, ur: str) -> None:
    """precision.py:186-195."""
    if not UNIT_ROUNDOFF[uf] >= UNIT_ROUNDOFF[u] >= UNIT_ROUNDOFF[ur]:
        raise ValueError(f"precisions must satisfy uf >= u >= ur, got ({uf}, {u}, {ur})")


# ---------------------------------------------------------------------------
# rounding (precision.py:206-232)
# ---------------------------------------------------------------------------

def rnd(x, fmt: str) -> np.ndarray:
    arr = np.asarray(x, dtype=np.float64)
    if fmt in (DOUBLE, QUAD):
        return arr
    with np.errstate(over="ignore", invalid="ignore"):
        out = arr.astype(_NP[fmt]).astype(np.float64)
    if fmt == HALF and _FTZ["on"]:
        tiny = np.abs(out) < 2.0 ** -14
        if np.any(tiny):
            out = np.where(tiny, np.copysign(0.0, out), out)
    return out


def rnd1(x: float, fmt: str) -> float:
    if fmt in (DOUBLE, QUAD):
        return float(x)
    with np.errstate(over="ignore", invalid="ignore"):
        r = float(np.float64(x).astype(_NP[fmt]))
    if fmt == HALF and _FTZ["on"] and 0.0 < abs(r) < 2.0 ** -14:
        return math.copysign(0.0, r)
    return r


# ---------------------------------------------------------------------------
# double-double error-free transforms (precision.py:239-341)
# ---------------------------------------------------------------------------

def two_sum(a, b):
    s = a + b
    v = s - a
    return s, (a - (s - v)) + (b - v)


def fast_two_sum(a, b):
    s = a + b
    return s, b - (s - a)


def _split(a):
    t = 134217729.0 * a
    hi = t - (t - a)
    return hi, a - hi


def two_prod(a, b):
    p = a * b
    ah, al = _split(a)
    bh, bl = _split(b)
    return p, ((ah * bh - p) + ah * bl + al * bh) + al * bl


def dd_add(xh, xl, yh, yl):
    s, e = two_sum(xh, yh)
    t, f = two_sum(xl, yl)
    s, e = fast_two_sum(s, e + t)
    return fast_two_sum(s, e + f)


def dd_neg_add(xh, xl, yh, yl):
    return dd_add(xh, xl, -yh, -yl)


def dd_mul(xh, xl, yh, yl):
    p, e = two_prod(xh, yh)
    return fast_two_sum(p, e + (xh * yl + xl * yh))


def dd_scale(d, xh, xl):
    p, e = two_prod(d, xh)
    return fast_two_sum(p, e + d * xl)


def dd_div(xh, xl, yh, yl):
    q1 = xh / yh
    rh, rl = dd_neg_add(xh, xl, *dd_scale(q1, yh, yl))
    q2 = rh / yh
    rh, rl = dd_neg_add(rh, rl, *dd_scale(q2, yh, yl))
    q3 = rh / yh
    qh, ql = fast_two_sum(q1, q2)
    return dd_add(qh, ql, q3, 0.0)


def dd_tree_sum(hi, lo, axis=0):
    hi = np.moveaxis(np.asarray(hi, dtype=np.float64), axis, 0)
    lo = np.moveaxis(np.asarray(lo, dtype=np.float64), axis, 0)
    while hi.shape[0] > 1:
        n = hi.shape[0]
        ev = n - (n & 1)
        sh, sl = dd_add(hi[0:ev:2], lo[0:ev:2], hi[1:ev:2], lo[1:ev:2])
        if n & 1:
            sh = np.concatenate([sh, hi[ev:]], axis=0)
            sl = np.concatenate([sl, lo[ev:]], axis=0)
        hi, lo = sh, sl
    return hi[0], lo[0]


def dd_matvec(a, x):
    ph, pl = two_prod(np.asarray(a, dtype=np.float64), np.asarray(x, dtype=np.float64)[None, :])
    return dd_tree_sum(ph, pl, axis=1)


# ---------------------------------------------------------------------------
# format-faithful BLAS-1/2 (precision.py:505-603)
# ---------------------------------------------------------------------------

def _tree_rounded(a, fmt, axis=0):
    a = np.moveaxis(np.asarray(a, dtype=np.float64), axis, 0)
    if a.shape[0] == 0:
        return np.zeros(a.shape[1:]) if a.ndim > 1 else 0.0
    while a.shape[0] > 1:
        n = a.shape[0]
        ev = n - (n & 1)
        s = rnd(a[0:ev:2] + a[1:ev:2], fmt)
        if n & 1:
            s = np.concatenate([s, a[ev:]], axis=0)
        a = s
    return a[0]


def vdot(x, y, fmt):
    if fmt == SINGLE:
        return float(np.asarray(x, dtype=np.float32) @ np.asarray(y, dtype=np.float32))
    if fmt == HALF:
        return float(_tree_rounded(rnd(np.asarray(x) * np.asarray(y), fmt), fmt))
    return float(np.asarray(x) @ np.asarray(y))


def vnorm2(x, fmt):
    if fmt == SINGLE:
        return float(np.linalg.norm(np.asarray(x, dtype=np.float32)))
    if fmt == HALF:
        return rnd1(math.sqrt(vdot(x, x, fmt)), fmt)
    return float(np.linalg.norm(np.asarray(x, dtype=np.float64)))


def vscale(alpha, x, fmt):
    x = np.asarray(x, dtype=np.float64)
    if fmt == SINGLE:
        return (np.float32(alpha) * x.astype(np.float32)).astype(np.float64)
    if fmt == HALF:
        return rnd(alpha * x, fmt)
    return alpha * x


def vaxpy(alpha, x, y, fmt):
    """y + alpha*x, product and sum rounded separately (precision.py:541-550)."""
    x = np.asarray(x, dtype=np.float64)
    y = np.asarray(y, dtype=np.float64)
    if fmt == SINGLE:
        return (y.astype(np.float32) + np.float32(alpha) * x.astype(np.float32)).astype(np.float64)
    if fmt == HALF:
        return rnd(y + rnd(alpha * x, fmt), fmt)
    return y + alpha * x


def vadd(x, y, fmt):
    if fmt == SINGLE:
        return (np.asarray(x, dtype=np.float32) + np.asarray(y, dtype=np.float32)).astype(np.float64)
    s = np.asarray(x, dtype=np.float64) + np.asarray(y, dtype=np.float64)
    return rnd(s, fmt) if fmt == HALF else s


def vsub(x, y, fmt):
    if fmt == SINGLE:
        return (np.asarray(x, dtype=np.float32) - np.asarray(y, dtype=np.float32)).astype(np.float64)
    s = np.asarray(x, dtype=np.float64) - np.asarray(y, dtype=np.float64)
    return rnd(s, fmt) if fmt == HALF else s


def tvec(m, r, fmt):
    """M^T r in the format's arithmetic (precision.py:577-587)."""
    m = np.asarray(m, dtype=np.float64)
    r = np.asarray(r, dtype=np.float64)
    if fmt == SINGLE:
        return np.atleast_1d((m.astype(np.float32).T @ r.astype(np.float32)).astype(np.float64))
    if fmt == HALF:
        return np.atleast_1d(_tree_rounded(rnd(m * r[:, None], fmt), fmt, axis=0))
    return m.T @ r


# ---------------------------------------------------------------------------
# exceptions (densela.py:58-79)
# ---------------------------------------------------------------------------

class ZeroPivot(Exception):
    def __init__(self, index):
        self.index = index
        super().__init__(f"exact zero pivot at column {index}")


class RankDeficient(Exception):
    pass


class NoConvergence(Exception):
    pass


class SingularB(Exception):
    pass


# ---------------------------------------------------------------------------
# LU (densela.py:124-168)
# ---------------------------------------------------------------------------

@dataclass
class Factors:
    L: np.ndarray
    U: np.ndarray
    perm: np.ndarray
    fmt: str
    growth: float
    _f32: tuple | None = None

    @property
    def n(self):
        return self.L.shape[0]

    def f32(self):
        if self._f32 is None:
            self._f32 = (self.L.astype(np.float32), self.U.astype(np.float32))
        return self._f32

    @property
    def packed(self):
        return np.tril(self.L, -1) + self.U


def lu_factor(a, fmt: str) -> Factors:
    a = rnd(np.asarray(a, dtype=np.float64), fmt).copy()
    n = a.shape[0]
    if a.ndim != 2 or a.shape[1] != n:
        raise ValueError("lu_factor requires a square matrix")
    amax = float(np.max(np.abs(a))) if a.size else 0.0
    if fmt != HALF:
        lu, piv = scipy.linalg.lu_factor(a.astype(np.float32) if fmt == SINGLE else a,
                                         check_finite=False)
        perm = np.arange(n)
        for i, p in enumerate(piv):  # LAPACK ipiv -> permutation vector
            perm[i], perm[p] = perm[p], perm[i]
        lower = (np.tril(lu, -1) + np.eye(n, dtype=lu.dtype)).astype(np.float64)
        upper = np.triu(lu).astype(np.float64)
        zero = np.diag(upper) == 0.0
        if np.any(zero):
            raise ZeroPivot(int(np.argmax(zero)))
        return Factors(lower, upper, perm,
                       fmt, float(np.max(np.abs(upper)) / amax) if amax else float("nan"))
    perm = np.arange(n)
    with np.errstate(divide="ignore", invalid="ignore", over="ignore"):
        for k in range(n - 1):
            p = k + int(np.argmax(np.abs(a[k:, k])))  # first max wins
            if a[p, k] == 0.0:
                raise ZeroPivot(k)
            if p != k:
                a[[k, p], :] = a[[p, k], :]
                perm[[k, p]] = perm[[p, k]]
            l = rnd(a[k + 1:, k] / a[k, k], fmt)
            a[k + 1:, k] = l
            a[k + 1:, k + 1:] = rnd(a[k + 1:, k + 1:] - rnd(np.outer(l, a[k, k + 1:]), fmt), fmt)
    if a[n - 1, n - 1] == 0.0:
        raise ZeroPivot(n - 1)
    upper = np.triu(a)
    return Factors(np.tril(a, -1) + np.eye(n), upper, perm, fmt,
                   float(np.max(np.abs(upper)) / amax) if amax else float("nan"))


# ---------------------------------------------------------------------------
# substitution (densela.py:175-261)
# ---------------------------------------------------------------------------

def _nonzero_diag(f: Factors):
    z = np.diag(f.U) == 0.0
    if np.any(z):
        raise ZeroPivot(int(np.argmax(z)))


def sub_f64(f: Factors, b):
    _nonzero_diag(f)
    y = scipy.linalg.solve_triangular(f.L, b, lower=True, unit_diagonal=True, check_finite=False)
    return scipy.linalg.solve_triangular(f.U, y, lower=False, check_finite=False)


def sub_f32(f: Factors, b):
    _nonzero_diag(f)
    l32, u32 = f.f32()
    y = scipy.linalg.solve_triangular(l32, b.astype(np.float32), lower=True, unit_diagonal=True,
                                      check_finite=False)
    return scipy.linalg.solve_triangular(u32, y, lower=False, check_finite=False).astype(np.float64)


def sub_rounded(f: Factors, b, fmt):
    """Column sweep with every op rounded (densela.py:201-217)."""
    _nonzero_diag(f)
    n = f.n
    y = b.copy()
    with np.errstate(divide="ignore", invalid="ignore", over="ignore"):
        for i in range(n - 1):
            y[i + 1:] = rnd(y[i + 1:] - rnd(f.L[i + 1:, i] * y[i], fmt), fmt)
        for i in range(n - 1, -1, -1):
            y[i] = rnd(y[i] / f.U[i, i], fmt)
            if i:
                y[:i] = rnd(y[:i] - rnd(f.U[:i, i] * y[i], fmt), fmt)
    return y


def sub_dd(f: Factors, bh, bl):
    """Double-double column sweep (densela.py:220-232)."""
    _nonzero_diag(f)
    n = f.n
    yh, yl = bh.copy(), bl.copy()
    for i in range(n - 1):
        th, tl = dd_scale(f.L[i + 1:, i], yh[i], yl[i])
        yh[i + 1:], yl[i + 1:] = dd_neg_add(yh[i + 1:], yl[i + 1:], th, tl)
    for i in range(n - 1, -1, -1):
        yh[i], yl[i] = dd_div(yh[i], yl[i], f.U[i, i], 0.0)
        if i:
            th, tl = dd_scale(f.U[:i, i], yh[i], yl[i])
            yh[:i], yl[:i] = dd_neg_add(yh[:i], yl[:i], th, tl)
    return yh, yl


def lu_solve(f: Factors, b, fmt: str, store: str | None = None):
    """densela.py:235-261."""
    b = np.asarray(b, dtype=np.float64)
    if b.shape != (f.n,):
        raise ValueError("right-hand side length does not match the factors")
    if fmt == QUAD:
        bp = b[f.perm]
        xh, xl = sub_dd(f, bp, np.zeros_like(bp))
        x = xh + xl
    elif fmt == DOUBLE:
        x = sub_f64(f, b[f.perm])
    elif fmt == SINGLE:
        x = sub_f32(f, rnd(b, fmt)[f.perm])
    else:
        x = sub_rounded(f, rnd(b, fmt)[f.perm], fmt)
    return rnd(x, store) if store is not None else x


def apply_op(a, f: Factors, v, fmt: str, store: str):
    """U^-1 L^-1 (A v)[perm] at ``fmt`` (densela.py:268-299)."""
    a = np.asarray(a, dtype=np.float64)
    v = np.asarray(v, dtype=np.float64)
    if a.shape != (f.n, f.n) or v.shape != (f.n,):
        raise ValueError("dimension mismatch in apply_preconditioned")
    if fmt == QUAD:
        wh, wl = dd_matvec(a, v)
        xh, xl = sub_dd(f, wh[f.perm], wl[f.perm])
        w = xh + xl
    elif fmt == DOUBLE:
        w = sub_f64(f, (a @ v)[f.perm])
    elif fmt == SINGLE:
        w = sub_f32(f, (a.astype(np.float32) @ v.astype(np.float32)).astype(np.float64)[f.perm])
    else:
        acc = np.zeros(f.n)
        with np.errstate(over="ignore", invalid="ignore"):
            for j in range(f.n):
                if v[j] != 0.0:
                    acc = rnd(acc + rnd(a[:, j] * v[j], fmt), fmt)
        w = sub_rounded(f, acc[f.perm], fmt)
    return rnd(w, store)


def precond_rhs(f: Factors, r, fmt: str, store: str):
    """U^-1 L^-1 r[perm] at ``fmt`` (densela.py:314-333)."""
    r = np.asarray(r, dtype=np.float64)
    if fmt == QUAD:
        rp = r[f.perm]
        xh, xl = sub_dd(f, rp, np.zeros_like(rp))
        s = xh + xl
    elif fmt == DOUBLE:
        s = sub_f64(f, r[f.perm])
    elif fmt == SINGLE:
        s = sub_f32(f, rnd(r, fmt)[f.perm])
    else:
        s = sub_rounded(f, rnd(r, fmt)[f.perm], fmt)
    return rnd(s, store)


def residual(a, x, b, fmt: str):
    """b - A x accumulated in ``fmt`` (densela.py:340-361)."""
    a = np.asarray(a, dtype=np.float64)
    x = np.asarray(x, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    if fmt == QUAD:
        mh, ml = dd_matvec(a, x)
        rh, rl = dd_add(b, np.zeros_like(b), -mh, -ml)
        return rh + rl
    if fmt == DOUBLE:
        return b - a @ x
    if fmt == SINGLE:
        return (b.astype(np.float32) - a.astype(np.float32) @ x.astype(np.float32)).astype(np.float64)
    acc = rnd(b, fmt)
    with np.errstate(over="ignore", invalid="ignore"):
        for j in range(a.shape[1]):
            if x[j] != 0.0:
                acc = rnd(acc - rnd(a[:, j] * x[j], fmt), fmt)
    return acc


def quad_solve(a, b):
    """Double-double GEPP solve (densela.py:368-407)."""
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    n = a.shape[0]
    ah, al = a.copy(), np.zeros_like(a)
    perm = np.arange(n)
    for k in range(n - 1):
        p = k + int(np.argmax(np.abs(ah[k:, k])))
        if ah[p, k] == 0.0 and al[p, k] == 0.0:
            raise ZeroPivot(k)
        if p != k:
            ah[[k, p], :] = ah[[p, k], :]
            al[[k, p], :] = al[[p, k], :]
            perm[[k, p]] = perm[[p, k]]
        mh, ml = dd_div(ah[k + 1:, k], al[k + 1:, k], ah[k, k], al[k, k])
        ah[k + 1:, k], al[k + 1:, k] = mh, ml
        ph, pl = dd_mul(mh[:, None], ml[:, None], ah[k, k + 1:][None, :], al[k, k + 1:][None, :])
        ah[k + 1:, k + 1:], al[k + 1:, k + 1:] = dd_neg_add(ah[k + 1:, k + 1:], al[k + 1:, k + 1:], ph, pl)
    if ah[n - 1, n - 1] == 0.0 and al[n - 1, n - 1] == 0.0:
        raise ZeroPivot(n - 1)
    yh, yl = b[perm].copy(), np.zeros(n)
    for i in range(n - 1):
        th, tl = dd_mul(ah[i + 1:, i], al[i + 1:, i], yh[i], yl[i])
        yh[i + 1:], yl[i + 1:] = dd_neg_add(yh[i + 1:], yl[i + 1:], th, tl)
    for i in range(n - 1, -1, -1):
        yh[i], yl[i] = dd_div(yh[i], yl[i], ah[i, i], al[i, i])
        if i:
            th, tl = dd_mul(ah[:i, i], al[:i, i], yh[i], yl[i])
            yh[:i], yl[:i] = dd_neg_add(yh[:i], yl[:i], th, tl)
    return yh + yl


def qr_signed(m):
    """Householder QR with diag(R) >= 0 and the rank test (densela.py:410-432)."""
    m = np.asarray(m, dtype=np.float64)
    if m.ndim != 2 or m.shape[0] < m.shape[1]:
        raise ValueError("qr_reduced requires rows >= cols")
    if not np.all(np.isfinite(m)):
        raise RankDeficient("non-finite entries")
    q, r = np.linalg.qr(m, mode="reduced")
    s = np.sign(np.diag(r))
    s[s == 0.0] = 1.0
    q = q * s[None, :]
    r = r * s[:, None]
    tol = max(m.shape) * UNIT_ROUNDOFF[DOUBLE] * float(np.linalg.norm(r))
    if np.any(np.abs(np.diag(r)) < tol):
        raise RankDeficient("numerically rank deficient")
    return q, r


def eig_sorted(m):
    """All eigenpairs, ascending |value|, unit vectors (densela.py:435-457)."""
    m = np.asarray(m, dtype=np.float64)
    if not np.all(np.isfinite(m)):
        raise NoConvergence("non-finite entries")
    try:
        w, v = np.linalg.eig(m)
    except np.linalg.LinAlgError as exc:
        raise NoConvergence(str(exc)) from exc
    w = np.asarray(w, dtype=np.complex128)
    v = np.asarray(v, dtype=np.complex128)
    nrm = np.linalg.norm(v, axis=0)
    nrm[nrm == 0.0] = 1.0
    v = v / nrm[None, :]
    order = np.argsort(np.abs(w), kind="stable")
    return w[order], v[:, order]


def eig_pencil(amat, bmat):
    """A z = theta B z via eig(B^-1 A) after a 2-norm cond test (densela.py:460-477)."""
    amat = np.asarray(amat, dtype=np.float64)
    bmat = np.asarray(bmat, dtype=np.float64)
    if not np.all(np.isfinite(amat)):
        raise NoConvergence("non-finite entries in the left matrix")
    if not np.all(np.isfinite(bmat)):
        raise SingularB("non-finite entries in the right matrix")
    try:
        c = np.linalg.cond(bmat)
    except np.linalg.LinAlgError as exc:
        raise SingularB(str(exc)) from exc
    if not np.isfinite(c) or c > 1.0 / UNIT_ROUNDOFF[DOUBLE]:
        raise SingularB(f"condition {c:.3e} exceeds 1/u")
    return eig_sorted(np.linalg.solve(bmat, amat))


def inf_norm(m):
    m = np.asarray(m, dtype=np.float64)
    if m.ndim == 1:
        return float(np.max(np.abs(m))) if m.size else 0.0
    return float(np.max(np.sum(np.abs(m), axis=1)))


# ---------------------------------------------------------------------------
# Arnoldi / restarted GMRES (gmres.py:99-311)
# ---------------------------------------------------------------------------

@dataclass
class Cycle:
    V: np.ndarray
    H: np.ndarray
    B: np.ndarray | None
    steps: int
    y: np.ndarray
    converged: bool
    breakdown: bool


def _givens(a, b, fmt):
    h = math.hypot(a, b)
    if h == 0.0:
        return 1.0, 0.0
    return rnd1(a / h, fmt), rnd1(b / h, fmt)


def _rotate(c, s, a, b, fmt):
    return (rnd1(rnd1(c * a, fmt) + rnd1(s * b, fmt), fmt),
            rnd1(rnd1(c * b, fmt) - rnd1(s * a, fmt), fmt))


def _upper_solve(r, g):
    if np.any(np.diag(r) == 0.0):
        return np.linalg.lstsq(r, g, rcond=None)[0]
    return scipy.linalg.solve_triangular(r, g, lower=False, check_finite=False)


def arnoldi(op, r0, beta, m, tol_abs, fmt, reorth=True, C=None) -> Cycle:
    """One MGS Arnoldi cycle with Givens tracking (gmres.py:123-215)."""
    n = r0.shape[0]
    kc = 0 if C is None else C.shape[1]
    V = np.zeros((n, m + 1))
    H = np.zeros((m + 1, m))
    R = np.zeros((m + 1, m))
    B = np.zeros((kc, m)) if kc else None
    cs = np.zeros(m)
    sn = np.zeros(m)
    g = np.zeros(m + 1)
    g[0] = beta
    V[:, 0] = vscale(1.0 / beta, r0, fmt)
    sq = math.sqrt(UNIT_ROUNDOFF[fmt])
    steps, conv, brk = 0, False, False
    with np.errstate(invalid="ignore", over="ignore", divide="ignore"):
        for j in range(m):
            w = op(V[:, j])
            if kc:
                cc = tvec(C, w, fmt)
                for i in range(kc):
                    w = vaxpy(-cc[i], C[:, i], w, fmt)
                B[:, j] = cc
            w0 = vnorm2(w, fmt)
            col = np.zeros(j + 2)
            for i in range(j + 1):
                h = vdot(V[:, i], w, fmt)
                w = vaxpy(-h, V[:, i], w, fmt)
                col[i] = h
            hn = vnorm2(w, fmt)
            if reorth and hn < sq * w0:
                for i in range(j + 1):
                    c2 = vdot(V[:, i], w, fmt)
                    w = vaxpy(-c2, V[:, i], w, fmt)
                    col[i] = rnd1(col[i] + c2, fmt)
                hn = vnorm2(w, fmt)
            col[j + 1] = hn
            H[: j + 2, j] = col
            rot = col.copy()
            for i in range(j):
                rot[i], rot[i + 1] = _rotate(cs[i], sn[i], rot[i], rot[i + 1], fmt)
            cs[j], sn[j] = _givens(rot[j], rot[j + 1], fmt)
            rot[j], _ = _rotate(cs[j], sn[j], rot[j], rot[j + 1], fmt)
            rot[j + 1] = 0.0
            R[: j + 2, j] = rot
            g[j], g[j + 1] = _rotate(cs[j], sn[j], g[j], 0.0, fmt)
            steps = j + 1
            if hn == 0.0:
                brk = conv = True
                break
            V[:, j + 1] = vscale(1.0 / hn, w, fmt)
            if abs(g[j + 1]) <= tol_abs:
                conv = True
                break
        y = rnd(_upper_solve(R[:steps, :steps], g[:steps]), fmt)
    return Cycle(V[:, : steps + 1], H[: steps + 1, :steps],
                 B[:, :steps] if B is not None else None, steps, y, conv, brk)


def recurrence_res(cyc: Cycle, beta, fmt):
    """V (beta e1 - Hbar y) with t rounded (gmres.py:218-232)."""
    j = cyc.steps
    t = -cyc.H[: j + 1, :j] @ cyc.y
    t[0] += beta
    t = rnd(t, fmt)
    res = np.zeros(cyc.V.shape[0])
    for i in range(j + 1):
        res = vaxpy(t[i], cyc.V[:, i], res, fmt)
    return res


@dataclass
class Inner:
    solution: np.ndarray
    cycles: list
    converged: bool
    relres: float
    stagnated: bool = False
    breakdown: bool = False
    applies: int = 0
    k_eff: list = field(default_factory=list)

    @property
    def total(self):
        return sum(self.cycles)


def _max_cycles(n, m, given):
    return given if given is not None else max(1, math.ceil(10 * n / m))


def gmres(a, f: Factors, r, m, tau, mv_fmt, fmt, max_cycles=None, reorth=True,
          restart_residual="recurrence") -> Inner:
    """Restarted left-preconditioned GMRES(m) (gmres.py:235-311)."""
    a = np.asarray(a, dtype=np.float64)
    n = f.n
    if not 1 <= m <= n:
        raise ValueError("restart length must satisfy 1 <= m <= n")
    cnt = [0]

    def op(v):
        cnt[0] += 1
        return apply_op(a, f, v, mv_fmt, fmt)

    s = precond_rhs(f, r, mv_fmt, fmt)
    snorm = vnorm2(s, fmt)
    x = np.zeros(n)
    if snorm == 0.0:
        return Inner(x, [], True, 0.0)
    tol = tau * snorm
    res = s.copy()
    cyc_steps, conv, brk = [], False, False
    with np.errstate(invalid="ignore", over="ignore", divide="ignore"):
        for _ in range(_max_cycles(n, m, max_cycles)):
            beta = vnorm2(res, fmt)
            if beta <= tol:
                conv = True
                break
            cyc = arnoldi(op, res, beta, m, tol, fmt, reorth)
            cyc_steps.append(cyc.steps)
            for jj in range(cyc.steps):
                x = vaxpy(cyc.y[jj], cyc.V[:, jj], x, fmt)
            brk = brk or cyc.breakdown
            if cyc.converged:
                conv = True
                res = recurrence_res(cyc, beta, fmt)
                break
            res = (recurrence_res(cyc, beta, fmt) if restart_residual == "recurrence"
                   else vsub(s, op(x), fmt))
    return Inner(x, cyc_steps, conv, vnorm2(res, fmt) / snorm, not conv, brk, cnt[0])


# ---------------------------------------------------------------------------
# GCRO-DR (gcrodr.py:104-419)
# ---------------------------------------------------------------------------

@dataclass
class Recycle:
    Yk: np.ndarray
    Uk: np.ndarray
    Ck: np.ndarray
    k_eff: int


def real_basis(vals, vecs, k, dim):
    """Real basis of the k smallest-|theta| eigenvectors (gcrodr.py:104-137)."""
    allow = k + 1 if k + 1 <= dim - 1 else k
    cols = []
    i = 0
    while i < len(vals) and len(cols) < k:
        lam, vec = vals[i], vecs[:, i]
        if lam.imag == 0.0:
            cols.append(np.real(vec))
            i += 1
        elif len(cols) + 2 <= allow:
            cols.extend([np.real(vec), np.imag(vec)])
            i += 2
        elif not cols:
            cols.append(np.real(vec))
            i += 1
        else:
            break
    p = np.column_stack(cols)
    nrm = np.linalg.norm(p, axis=0)
    nrm[nrm == 0.0] = 1.0
    return p / nrm[None, :]


def harmonic_first(h, hsub, V, k):
    """gcrodr.py:140-168."""
    h = np.asarray(h, dtype=np.float64)
    j = h.shape[0]
    mm = h
    if hsub != 0.0:
        e = np.zeros(j)
        e[-1] = 1.0
        try:
            w = np.linalg.solve(h.T, e)
            if np.all(np.isfinite(w)):
                mm = h + (hsub * hsub) * np.outer(w, e)
        except np.linalg.LinAlgError:
            pass
    vals, vecs = eig_sorted(mm)
    p = real_basis(vals, vecs, min(k, j), j)
    return p, V[:, :j] @ p


def harmonic_recycle(g, W, Vh, k, fmt):
    """gcrodr.py:171-197."""
    g = np.asarray(g, dtype=np.float64)
    pd = g.shape[1]
    wtv = np.column_stack([tvec(W, Vh[:, i], fmt) for i in range(pd)])
    a1 = g.T @ g
    b1 = g.T @ wtv
    try:
        vals, vecs = eig_pencil(a1, b1)
    except SingularB:
        if not np.all(np.isfinite(b1)):
            raise
        shift = math.sqrt(UNIT_ROUNDOFF[DOUBLE]) * np.linalg.norm(b1)
        vals, vecs = eig_pencil(a1, b1 + shift * np.eye(pd))
    return real_basis(vals, vecs, min(k, pd), pd)


def _u_from_r(ytil, r, fmt):
    return rnd(scipy.linalg.solve_triangular(r, ytil.T, trans="T", lower=False,
                                             check_finite=False).T, fmt)


def _ls(g, rhs):
    q, r = np.linalg.qr(g, mode="reduced")
    if np.any(np.abs(np.diag(r)) == 0.0):
        return np.linalg.lstsq(g, rhs, rcond=None)[0]
    return scipy.linalg.solve_triangular(r, q.T @ rhs, lower=False, check_finite=False)


def gcrodr(a, f: Factors, r, m, k, tau, mv_fmt, fmt, recycle_in: Recycle | None = None,
           max_cycles=None, reorth=True, cycle_residual="recurrence"):
    """One preconditioned GCRO-DR(m, k) solve (gcrodr.py:221-419)."""
    a = np.asarray(a, dtype=np.float64)
    n = f.n
    if not 1 <= k < m <= n:
        raise ValueError(f"need 1 <= k < m <= n, got k={k}, m={m}, n={n}")
    cnt = [0]

    def op(v):
        cnt[0] += 1
        return apply_op(a, f, v, mv_fmt, fmt)

    s = precond_rhs(f, r, mv_fmt, fmt)
    snorm = vnorm2(s, fmt)
    x = np.zeros(n)
    if snorm == 0.0:
        return Inner(x, [], True, 0.0), recycle_in
    tol = tau * snorm
    res = s.copy()
    st = {"C": None, "U": None, "keff": 0, "cycles": 0, "brk": False}
    iters: list[int] = []
    keffs: list[int] = []
    cap = _max_cycles(n, m, max_cycles)

    with np.errstate(invalid="ignore", over="ignore", divide="ignore"):
        if recycle_in is not None:
            yk = rnd(np.asarray(recycle_in.Yk, dtype=np.float64), fmt)
            ay = np.column_stack([op(yk[:, i]) for i in range(yk.shape[1])])
            try:
                q, rr = qr_signed(ay)
                st["C"] = rnd(q, fmt)
                st["U"] = _u_from_r(yk, rr, fmt)
                st["keff"] = st["C"].shape[1]
                t = tvec(st["C"], res, fmt)
                for i in range(st["keff"]):
                    x = vaxpy(t[i], st["U"][:, i], x, fmt)
                    res = vaxpy(-t[i], st["C"][:, i], res, fmt)
            except RankDeficient:
                st["C"] = st["U"] = None
                st["keff"] = 0

        def cold():
            nonlocal x, res
            beta = vnorm2(res, fmt)
            cyc = arnoldi(op, res, beta, m, tol, fmt, reorth)
            iters.append(cyc.steps)
            st["cycles"] += 1
            st["brk"] = st["brk"] or cyc.breakdown
            j = cyc.steps
            for jj in range(j):
                x = vaxpy(cyc.y[jj], cyc.V[:, jj], x, fmt)
            res = (recurrence_res(cyc, beta, fmt)
                   if cyc.converged or cycle_residual == "recurrence" else vsub(s, op(x), fmt))
            if j < k:
                return
            try:
                p, yt = harmonic_first(cyc.H[:j, :j], float(cyc.H[j, j - 1]), cyc.V, k)
                yt = rnd(yt, fmt)
                q, rr = qr_signed(cyc.H[: j + 1, :j] @ p)
                st["C"] = rnd(cyc.V[:, : j + 1] @ q, fmt)
                st["U"] = _u_from_r(yt, rr, fmt)
                st["keff"] = p.shape[1]
            except (RankDeficient, NoConvergence):
                st["C"] = st["U"] = None
                st["keff"] = 0

        if st["C"] is None:
            cold()
            if st["C"] is not None:
                keffs.append(st["keff"])

        conv = False
        while True:
            if vnorm2(res, fmt) <= tol:
                conv = True
                break
            if st["cycles"] >= cap:
                break
            if st["C"] is None:
                cold()
                continue
            C, U, keff = st["C"], st["U"], st["keff"]
            beta = vnorm2(res, fmt)
            cyc = arnoldi(op, res, beta, m - keff, tol, fmt, reorth, C=C)
            iters.append(cyc.steps)
            st["cycles"] += 1
            st["brk"] = st["brk"] or cyc.breakdown
            j = cyc.steps
            dk = np.array([vnorm2(U[:, i], fmt) for i in range(keff)])
            dk[dk == 0.0] = 1.0
            dk = rnd(1.0 / dk, fmt)
            ut = np.column_stack([rnd(U[:, i] * dk[i], fmt) for i in range(keff)])
            G = np.zeros((keff + j + 1, keff + j))
            G[:keff, :keff] = np.diag(dk)
            G[:keff, keff:] = cyc.B[:, :j]
            G[keff:, keff:] = cyc.H[: j + 1, :j]
            W = np.column_stack([C, cyc.V[:, : j + 1]])
            Vh = np.column_stack([ut, cyc.V[:, :j]])
            y = rnd(_ls(G, tvec(W, res, fmt)), fmt)
            for jj in range(keff + j):
                x = vaxpy(y[jj], Vh[:, jj], x, fmt)
            gy = rnd(G @ y, fmt)
            nr = res.copy()
            for i in range(keff + j + 1):
                nr = vaxpy(-gy[i], W[:, i], nr, fmt)
            res = nr if (cyc.converged or cycle_residual == "recurrence") else vsub(s, op(x), fmt)
            if j >= 1:
                try:
                    p = harmonic_recycle(G, W, Vh, k, fmt)
                    yt = rnd(Vh @ p, fmt)
                    q, rr = qr_signed(G @ p)
                    st["C"] = rnd(W @ q, fmt)
                    st["U"] = _u_from_r(yt, rr, fmt)
                    st["keff"] = p.shape[1]
                except (SingularB, RankDeficient, NoConvergence):
                    pass
            keffs.append(st["keff"])

    out = Inner(x, iters, conv, vnorm2(res, fmt) / snorm, not conv, st["brk"], cnt[0], keffs)
    rec = None
    if st["U"] is not None:
        rec = Recycle(st["U"].copy(), st["U"], st["C"], st["keff"])
    return out, rec


# ---------------------------------------------------------------------------
# refinement (refine.py:56-464)
# ---------------------------------------------------------------------------

METHODS = ("sir", "gmres-ir", "sgmres-ir", "rgmres-ir", "rsgmres-ir")


@dataclass
class Report:
    converged: bool
    steps: int
    inner_iters: list
    nbe_history: list
    ferr_history: list
    divergence_reason: str | None = None
    solution: np.ndarray | None = None
    diagnostics: dict = field(default_factory=dict)
    inner_calls: list = field(default_factory=list)


def check_convergence(a, b, x, history, u, c_conv, stagnated, norm_a, norm_b, ferr, ur):
    """refine.py:172-229; returns (state, reason, nbe, cbe)."""
    r = residual(a, x, b, ur)
    denom = norm_a * inf_norm(x) + norm_b
    nbe = float(np.max(np.abs(r))) / denom if denom > 0 else float("inf")
    cden = np.abs(a) @ np.abs(x) + np.abs(b)
    with np.errstate(divide="ignore", invalid="ignore"):
        ratio = np.abs(r) / cden
    ratio = ratio[np.isfinite(ratio)]
    cbe = float(np.max(ratio)) if ratio.size else nbe
    worst = max(nbe, cbe, ferr if math.isfinite(ferr) else 0.0)
    if math.isfinite(worst) and worst <= c_conv * UNIT_ROUNDOFF[u]:
        return "converged", None, nbe, cbe
    if stagnated:
        return "diverged", "InnerStagnation", nbe, cbe
    grow = 0
    seq = history + [nbe]
    for prev, cur in zip(seq[:-1], seq[1:]):
        grow = grow + 1 if (not math.isfinite(cur) or (math.isfinite(prev) and cur >= 2.0 * prev)) else 0
    if grow >= 3:
        return "diverged", "ErrorGrowth", nbe, cbe
    return "continue", None, nbe, cbe


def reference_solution(a, b):
    """Forward-error reference (refine.py:236-258)."""
    try:
        if a.shape[0] <= 600:
            x = quad_solve(a, b)
            return x if np.all(np.isfinite(x)) else None
        f = lu_factor(a, DOUBLE)
        x = lu_solve(f, b, DOUBLE)
        for _ in range(4):
            x = x + lu_solve(f, residual(a, x, b, QUAD), DOUBLE)
        return x if np.all(np.isfinite(x)) else None
    except ZeroPivot:
        return None


def forward_error(x, xref):
    """refine.py:424-430."""
    if xref is None:
        return float("nan")
    d = float(np.max(np.abs(xref)))
    e = float(np.max(np.abs(x - xref)))
    return e if d == 0.0 else e / d


def pow2_equilibrate(a, b):
    """Row then column scaling by the power of two nearest 1/max|.|
    (refine.py:261-270); exact in binary.  Returns (a', b', column scales)."""
    rmax = np.max(np.abs(a), axis=1)
    rmax = np.where(rmax == 0.0, 1.0, rmax)
    r = np.exp2(-np.round(np.log2(rmax)))
    ar = a * r[:, None]
    cmax = np.max(np.abs(ar), axis=0)
    cmax = np.where(cmax == 0.0, 1.0, cmax)
    c = np.exp2(-np.round(np.log2(cmax)))
    return ar * c[None, :], b * r, c


def solve(a, b, precisions=("half", "single", "double"), method="rgmres-ir", m=0, k=0,
          tau=None, i_max=10000, extra_precision_matvec=None, c_conv=2.0, max_cycles=None,
          reorthogonalize=True, restart_residual="recurrence", cycle_residual="recurrence",
          scale_diag=False) -> Report:
    """The shared refinement loop (refine.py:277-421) for every method."""
    uf, u, ur = precisions
    check_triple(uf, u, ur)
    if method not in METHODS:
        raise ValueError(f"unknown method {method!r}")
    tau = DEFAULT_TAU[u] if tau is None else tau
    uniform = method in ("sgmres-ir", "rsgmres-ir")
    extra = (not uniform) if extra_precision_matvec is None else extra_precision_matvec
    mv = squared(u) if extra else u
    with np.errstate(invalid="ignore", over="ignore", divide="ignore"):
        a = rnd(np.asarray(a, dtype=np.float64), u)
        b = rnd(np.asarray(b, dtype=np.float64), u)
        n = a.shape[0]
        if a.shape != (n, n) or b.shape != (n,):
            raise ValueError("need a square matrix and a matching right-hand side")
        diag: dict = {}
        col_scale = None
        if scale_diag:  # refine.py:293-297 with _pow2_equilibrate (261-270)
            a, b, col_scale = pow2_equilibrate(a, b)
            a, b = rnd(a, u), rnd(b, u)
            diag["equilibrated"] = True
        norm_a, norm_b = inf_norm(a), inf_norm(b)
        try:
            F = lu_factor(a, uf)
        except ZeroPivot as exc:
            return Report(False, 0, [], [], [], "InnerStagnation", None, {"lu_failed": str(exc), **diag})
        diag["lu_growth"] = F.growth
        x = lu_solve(F, b, uf, store=u)
        if not np.all(np.isfinite(x)):
            x = np.zeros(n)
            diag["x0_reset"] = True
        xref = reference_solution(a, b)
        if xref is None:
            diag["no_reference_solution"] = True
        mm = m if m else min(n, 40)
        if method in ("rgmres-ir", "rsgmres-ir") and not (1 <= k < mm):
            raise ValueError("recycling methods need 1 <= k < m")
        recycle = None
        nbe_h, ferr_h, inner, calls = [], [], [], []
        reason, converged = "IMaxExceeded", False
        for _ in range(i_max):
            r = residual(a, x, b, ur)
            nu = float(np.max(np.abs(r)))
            if nu == 0.0 or not math.isfinite(nu):
                if nu == 0.0:
                    converged, reason = True, None
                    inner.append(0)
                    nbe_h.append(0.0)
                    ferr_h.append(forward_error(x, xref))
                else:
                    reason = "ErrorGrowth"
                break
            rhat = rnd(r / nu, u)
            stag = False
            if method == "sir":
                d = lu_solve(F, rhat, uf, store=u)
                its = 1
            elif method in ("gmres-ir", "sgmres-ir"):
                out = gmres(a, F, rhat, mm, tau, mv, u, max_cycles, reorthogonalize, restart_residual)
                d, its, stag = out.solution, out.total, out.stagnated
                calls.append(out)
            else:
                out, recycle = gcrodr(a, F, rhat, mm, k, tau, mv, u, recycle, max_cycles,
                                      reorthogonalize, cycle_residual)
                d, its, stag = out.solution, out.total, out.stagnated
                calls.append(out)
            x = vadd(x, vscale(nu, d, u), u)
            inner.append(its)
            fe = forward_error(x, xref)
            state, why, nbe, _ = check_convergence(a, b, x, nbe_h, u, c_conv, stag, norm_a,
                                                   norm_b, fe, ur)
            nbe_h.append(nbe)
            ferr_h.append(fe)
            if state == "converged":
                converged, reason = True, None
                break
            if state == "diverged":
                reason = why
                break
    if col_scale is not None and x is not None:
        x = col_scale * x  # refine.py:408-409
    return Report(converged, len(inner), inner, nbe_h, ferr_h, None if converged else reason,
                  x, diag, calls)

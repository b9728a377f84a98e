"""ctypes binding of the C ABI in ``include/gcrodr_b200.h``.

The library is the in-tree ``libgcrodr_b200.so`` built by ``_build.py``.  There
is no CPU fallback: if the library or a GPU is missing, every solver entry
point raises ``GpuUnavailable``.
"""

from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
# GB_LIB_PATH: an alternative build of the same library (A/B measurements)
LIB_PATH = os.environ.get("GB_LIB_PATH") or os.path.join(HERE, "libgcrodr_b200.so")

# formats / methods (gcrodr_b200.h)
HALF, SINGLE, DOUBLE, QUAD = 0, 1, 2, 3
SIR, GMRES_IR, SGMRES_IR, RGMRES_IR, RSGMRES_IR = 0, 1, 2, 3, 4

ST_CONVERGED, ST_STAGNATED, ST_BREAKDOWN = 1, 2, 4
ST_NU_ZERO, ST_NU_NONFINITE = 256, 512

EXPORTS = [
    "gb_version", "gb_last_error", "gb_device_count", "gb_solver_create", "gb_solver_destroy",
    "gb_set_system", "gb_set_system_device", "gb_launch_count", "gb_factorize", "gb_initial_solution", "gb_reference_solution",
    "gb_refine_step", "gb_last_cycles", "gb_get_solution", "gb_get_reference", "gb_get_factors",
    "gb_apply_preconditioned", "gb_precond_rhs", "gb_residual", "gb_lu_solve",
    "gb_last_step_ms", "gb_last_factor_ms", "gb_solve_batched", "gb_debug_phaselog", "gb_time_op",
    "gb_debug_hessenberg", "gb_debug_set_max_cycles", "gb_lu_tc_stats",
    "gb_debug_inner_solve", "gb_backward_errors",
]


class GpuUnavailable(RuntimeError):
    """The CUDA library or device is missing (no CPU fallback exists)."""


class GbError(RuntimeError):
    pass


class Options(C.Structure):
    _fields_ = [
        ("uf", C.c_int), ("u", C.c_int), ("ur", C.c_int), ("method", C.c_int),
        ("m", C.c_int), ("k", C.c_int), ("tau", C.c_double), ("max_cycles", C.c_int),
        ("reorthogonalize", C.c_int), ("extra_precision", C.c_int), ("grid_ctas", C.c_int),
        ("lu_mode", C.c_int), ("explicit_residual", C.c_int),
    ]


class StepInfo(C.Structure):
    _fields_ = [
        ("nu", C.c_double), ("inner_iters", C.c_int), ("ncycles", C.c_int), ("status", C.c_int),
        ("applies", C.c_int), ("keff", C.c_int), ("pad", C.c_int), ("ferr", C.c_double),
        ("nbe", C.c_double), ("cbe", C.c_double),
    ]


class BatchOut(C.Structure):
    _fields_ = [
        ("converged", C.c_void_p), ("steps", C.c_void_p), ("reason", C.c_void_p),
        ("inner", C.c_void_p), ("nbe", C.c_void_p), ("ferr", C.c_void_p), ("x", C.c_void_p),
        ("growth", C.c_void_p), ("flags", C.c_void_p),
    ]


_LIB = None


def load(path: str | None = None):
    """Load (once) the C-ABI library; raises GpuUnavailable when absent."""
    global _LIB
    if _LIB is not None:
        return _LIB
    p = path or LIB_PATH
    if not os.path.exists(p):
        raise GpuUnavailable(f"{p} is not built (run __graft_entry__.build())")
    lib = C.CDLL(p)
    vp, ip, dp = C.c_void_p, C.POINTER(C.c_int), C.POINTER(C.c_double)
    sig = {
        "gb_version": (C.c_char_p, []),
        "gb_last_error": (C.c_char_p, []),
        "gb_device_count": (C.c_int, []),
        "gb_solver_create": (C.c_int, [C.POINTER(vp), C.c_int, C.POINTER(Options), vp]),
        "gb_solver_destroy": (C.c_int, [vp]),
        "gb_set_system": (C.c_int, [vp, vp, vp]),
        "gb_set_system_device": (C.c_int, [vp, vp, vp]),
        "gb_launch_count": (C.c_longlong, []),
        "gb_factorize": (C.c_int, [vp, ip, dp]),
        "gb_initial_solution": (C.c_int, [vp, ip]),
        "gb_reference_solution": (C.c_int, [vp, ip]),
        "gb_refine_step": (C.c_int, [vp, C.POINTER(StepInfo)]),
        "gb_last_cycles": (C.c_int, [vp, vp, vp, C.c_int, ip]),
        "gb_get_solution": (C.c_int, [vp, vp]),
        "gb_get_reference": (C.c_int, [vp, vp]),
        "gb_get_factors": (C.c_int, [vp, vp, vp]),
        "gb_apply_preconditioned": (C.c_int, [vp, vp, vp, C.c_int]),
        "gb_precond_rhs": (C.c_int, [vp, vp, vp, C.c_int]),
        "gb_residual": (C.c_int, [vp, vp, vp, C.c_int]),
        "gb_lu_solve": (C.c_int, [vp, vp, vp]),
        "gb_last_step_ms": (C.c_double, [vp]),
        "gb_debug_phaselog": (C.c_int, [vp, C.c_int, vp]),
        "gb_time_op": (C.c_int, [vp, C.c_int, C.c_int, dp]),
        "gb_debug_hessenberg": (C.c_int, [vp, vp]),
        "gb_debug_set_max_cycles": (C.c_int, [vp, C.c_int]),
        "gb_last_factor_ms": (C.c_double, [vp]),
        "gb_lu_tc_stats": (C.c_int, [vp, dp]),
        "gb_debug_inner_solve": (C.c_int, [vp, vp, C.c_int, vp, C.POINTER(StepInfo)]),
        "gb_backward_errors": (C.c_int, [vp, vp, vp, dp, dp]),
        "gb_solve_batched": (C.c_int, [C.c_int, C.c_int, C.POINTER(Options), C.c_int, C.c_double,
                                       vp, vp, C.c_int, C.POINTER(BatchOut), dp, vp]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name, None)
        if fn is None:  # an older build under GB_LIB_PATH (A/B runs)
            continue
        fn.restype = res
        fn.argtypes = args
    _LIB = lib
    return lib


def _check(code: int, what: str) -> None:
    if code != 0:
        msg = _LIB.gb_last_error().decode() if _LIB is not None else "?"
        if code == 1:
            raise ValueError(f"{what}: {msg}")
        if code == 2:
            raise NotImplementedError(f"{what}: {msg}")
        raise GbError(f"{what} failed ({code}): {msg}")


def _ptr(a: np.ndarray) -> int:
    return a.ctypes.data


def require_gpu():
    lib = load()
    if lib.gb_device_count() < 1:
        raise GpuUnavailable("no CUDA device visible; the solver has no CPU fallback")
    return lib


def current_device() -> int:
    """torch's current CUDA device when torch is initialised, else 0."""
    try:
        import torch

        if torch.cuda.is_available() and torch.cuda.is_initialized():
            return int(torch.cuda.current_device())
    except Exception:  # pragma: no cover - torch is plumbing only
        pass
    return 0


def current_stream() -> int:
    """torch's current CUDA stream when torch is initialised, else NULL."""
    try:
        import torch

        if torch.cuda.is_available() and torch.cuda.is_initialized():
            return int(torch.cuda.current_stream().cuda_stream)
    except Exception:  # pragma: no cover - torch is plumbing only
        pass
    return 0


class Solver:
    """Device context for one system of order n (gb_solver)."""

    def __init__(self, n: int, opts: Options, stream: int | None = None):
        self.lib = require_gpu()
        self.n = int(n)
        self.opts = opts
        h = C.c_void_p()
        _check(self.lib.gb_solver_create(C.byref(h), self.n, C.byref(opts),
                                         C.c_void_p(stream if stream is not None else current_stream())),
               "gb_solver_create")
        self.h = h

    def close(self):
        if getattr(self, "h", None):
            self.lib.gb_solver_destroy(self.h)
            self.h = None

    def __del__(self):  # pragma: no cover
        try:
            self.close()
        except Exception:
            pass

    def set_system(self, a: np.ndarray, b: np.ndarray) -> None:
        a = np.ascontiguousarray(a, dtype=np.float64)
        b = np.ascontiguousarray(b, dtype=np.float64)
        self._keep = (a, b)
        _check(self.lib.gb_set_system(self.h, _ptr(a), _ptr(b)), "gb_set_system")

    def set_system_device(self, a_ptr: int, b_ptr: int) -> None:
        """float64 inputs already resident in device memory (e.g. torch tensors)."""
        _check(self.lib.gb_set_system_device(self.h, C.c_void_p(a_ptr), C.c_void_p(b_ptr)), "gb_set_system_device")

    def factorize(self) -> tuple[int, float]:
        z, g = C.c_int(), C.c_double()
        _check(self.lib.gb_factorize(self.h, C.byref(z), C.byref(g)), "gb_factorize")
        return z.value, g.value

    def initial_solution(self) -> bool:
        r = C.c_int()
        _check(self.lib.gb_initial_solution(self.h, C.byref(r)), "gb_initial_solution")
        return bool(r.value)

    def reference_solution(self) -> bool:
        ok = C.c_int()
        _check(self.lib.gb_reference_solution(self.h, C.byref(ok)), "gb_reference_solution")
        return bool(ok.value)

    def step(self) -> StepInfo:
        info = StepInfo()
        _check(self.lib.gb_refine_step(self.h, C.byref(info)), "gb_refine_step")
        return info

    def set_max_cycles(self, cycles: int) -> None:
        """Lower the cycle cap of subsequent steps (<= the cap at creation)."""
        _check(self.lib.gb_debug_set_max_cycles(self.h, int(cycles)), "gb_debug_set_max_cycles")

    def last_cycles(self) -> tuple[list[int], list[int]]:
        cap = self.opts.max_cycles + 1
        it = np.zeros(cap, dtype=np.int32)
        ke = np.zeros(cap, dtype=np.int32)
        nc = C.c_int()
        _check(self.lib.gb_last_cycles(self.h, _ptr(it), _ptr(ke), cap, C.byref(nc)), "gb_last_cycles")
        return it[: nc.value].tolist(), ke[: nc.value].tolist()

    def solution(self) -> np.ndarray:
        x = np.empty(self.n)
        _check(self.lib.gb_get_solution(self.h, _ptr(x)), "gb_get_solution")
        return x

    def reference(self) -> np.ndarray:
        x = np.empty(self.n)
        _check(self.lib.gb_get_reference(self.h, _ptr(x)), "gb_get_reference")
        return x

    def factors(self) -> tuple[np.ndarray, np.ndarray]:
        lu = np.empty((self.n, self.n))
        perm = np.empty(self.n, dtype=np.int64)
        _check(self.lib.gb_get_factors(self.h, _ptr(lu), _ptr(perm)), "gb_get_factors")
        return lu, perm

    def _vec_op(self, fn, x, *extra) -> np.ndarray:
        x = np.ascontiguousarray(x, dtype=np.float64)
        out = np.empty(self.n)
        _check(fn(self.h, _ptr(x), _ptr(out), *extra), fn.__name__)
        return out

    def apply_preconditioned(self, v, fmt: int) -> np.ndarray:
        return self._vec_op(self.lib.gb_apply_preconditioned, v, fmt)

    def precond_rhs(self, r, fmt: int) -> np.ndarray:
        return self._vec_op(self.lib.gb_precond_rhs, r, fmt)

    def residual(self, x, fmt: int) -> np.ndarray:
        return self._vec_op(self.lib.gb_residual, x, fmt)

    def lu_solve(self, b) -> np.ndarray:
        return self._vec_op(self.lib.gb_lu_solve, b)

    def time_op(self, what: int, reps: int = 10) -> float:
        """Device ms of one kernel-level launch (0 apply, 1 precond_rhs,
        2 residual, 3 lu_solve) on the vector of the last kernel-level call."""
        ms = C.c_double()
        _check(self.lib.gb_time_op(self.h, what, reps, C.byref(ms)), "gb_time_op")
        return ms.value

    def phaselog(self, cap: int = 0, read: bool = True):
        """Diagnostics: read the current phase log (tag, ns) and re-arm with cap."""
        out = None
        if read and getattr(self, "_plog_cap", 0):
            buf = np.zeros(1 + 2 * self._plog_cap, dtype=np.uint64)
            _check(self.lib.gb_debug_phaselog(self.h, cap, _ptr(buf)), "gb_debug_phaselog")
            k = int(buf[0])
            out = [(int(buf[1 + 2 * i]), int(buf[2 + 2 * i])) for i in range(k)]
        else:
            _check(self.lib.gb_debug_phaselog(self.h, cap, None), "gb_debug_phaselog")
        self._plog_cap = cap
        return out

    def hessenberg(self) -> np.ndarray:
        """(m+1) x m Hessenberg matrix of the last Arnoldi cycle (diagnostics)."""
        m = self.opts.m
        h = np.empty((m, m + 1))
        _check(self.lib.gb_debug_hessenberg(self.h, _ptr(h)), "gb_debug_hessenberg")
        return h.T.copy()

    @property
    def last_step_ms(self) -> float:
        return self.lib.gb_last_step_ms(self.h)

    @property
    def last_factor_ms(self) -> float:
        return self.lib.gb_last_factor_ms(self.h)

    def tc_update_stats(self) -> dict | None:
        """Blocked tensor-mode LU: device time and rate of the tcgen05 trailing
        updates of the last factorisation (None in exact mode)."""
        out = (C.c_double * 4)()
        _check(self.lib.gb_lu_tc_stats(self.h, out), "gb_lu_tc_stats")
        ms, flop, trsm_ms, panel_ms = out[0], out[1], out[2], out[3]
        if ms <= 0.0 or flop <= 0.0:
            return None
        n = self.n
        return {"ms": ms, "tflops": flop / (ms * 1e-3) / 1e12, "flop_share": flop / (2.0 * n ** 3 / 3.0),
                "trsm_ms": trsm_ms, "panel_ms": panel_ms}

    def inner_solve(self, r: np.ndarray, reset_recycle: bool = False):
        """gmres_solve / gcrodr_solve on r with this context's m, k, tau
        (gb_debug_inner_solve): (d, StepInfo)."""
        r = np.ascontiguousarray(r, dtype=np.float64)
        d = np.empty(self.n)
        info = StepInfo()
        _check(self.lib.gb_debug_inner_solve(self.h, _ptr(r), int(bool(reset_recycle)), _ptr(d), C.byref(info)),
               "gb_debug_inner_solve")
        return d, info

    def backward_errors(self, x: np.ndarray):
        """(r, nbe, cbe) of check_convergence for x (gb_backward_errors)."""
        x = np.ascontiguousarray(x, dtype=np.float64)
        r = np.empty(self.n)
        nbe, cbe = C.c_double(), C.c_double()
        _check(self.lib.gb_backward_errors(self.h, _ptr(x), _ptr(r), C.byref(nbe), C.byref(cbe)),
               "gb_backward_errors")
        return r, nbe.value, cbe.value

"""Batched mode: many independent small systems, one CTA per system, the
whole refinement loop (refine.py:277-421) on the device in ONE launch
(gb_solve_batched).  Returns one RefinementReport per system, exactly as a
loop of ``solve`` calls over the systems would (the reference's harness fans
independent problems out to a process pool instead, harness.py:250-252)."""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib
from .refine import DivergenceReason, RefineConfig, RefinementReport, _pow2_equilibrate, _round_u, make_options

__all__ = ["solve_batched", "BatchResult"]

_REASON = {0: None, 1: DivergenceReason.I_MAX_EXCEEDED, 2: DivergenceReason.INNER_STAGNATION,
           3: DivergenceReason.ERROR_GROWTH}


class BatchResult:
    """Raw per-system arrays plus lazily built RefinementReports."""

    def __init__(self, count, n, i_max):
        self.count, self.n, self.i_max = count, n, i_max
        self.converged = np.zeros(count, dtype=np.int32)
        self.steps = np.zeros(count, dtype=np.int32)
        self.reason = np.zeros(count, dtype=np.int32)
        self.flags = np.zeros(count, dtype=np.int32)
        self.inner = np.zeros((count, i_max), dtype=np.int32)
        self.nbe = np.zeros((count, i_max))
        self.ferr = np.zeros((count, i_max))
        self.x = np.zeros((count, n))
        self.growth = np.zeros(count)
        self.device_ms = 0.0
        self.col_scale = None  # (count, n) when cfg.scale_diag equilibrated the systems

    def c_struct(self) -> _lib.BatchOut:
        o = _lib.BatchOut()
        for name in ("converged", "steps", "reason", "inner", "nbe", "ferr", "x", "growth", "flags"):
            setattr(o, name, getattr(self, name).ctypes.data)
        return o

    def report(self, i: int) -> RefinementReport:
        s = int(self.steps[i])
        diag = {}
        if self.flags[i] & 4:
            diag["lu_failed"] = "exact zero pivot"
            return RefinementReport(False, 0, [], [], [], DivergenceReason.INNER_STAGNATION, None, diag)
        diag["lu_growth"] = float(self.growth[i])
        if self.flags[i] & 1:
            diag["x0_reset"] = True
        if self.flags[i] & 2:
            diag["no_reference_solution"] = True
        x = self.x[i].copy()
        if self.col_scale is not None:
            diag["equilibrated"] = True
            x = self.col_scale[i] * x  # refine.py:408-409
        return RefinementReport(bool(self.converged[i]), s, self.inner[i, :s].tolist(),
                                self.nbe[i, :s].tolist(), self.ferr[i, :s].tolist(),
                                _REASON[int(self.reason[i])], x, diag)

    def reports(self) -> list[RefinementReport]:
        return [self.report(i) for i in range(self.count)]


def solve_batched(a, b, cfg: RefineConfig, *, on_device_ptrs: tuple[int, int] | None = None,
                  count: int | None = None, n: int | None = None) -> BatchResult:
    """Solve systems a[i] x = b[i] (a: (count, n, n), b: (count, n)).

    ``on_device_ptrs`` passes device pointers (e.g. torch CUDA tensors'
    data_ptr()) of already-resident float64 inputs instead of host arrays."""
    lib = _lib.require_gpu()
    if on_device_ptrs is None:
        a = np.ascontiguousarray(a, dtype=np.float64)
        b = np.ascontiguousarray(b, dtype=np.float64)
        count, n = a.shape[0], a.shape[1]
        if a.shape != (count, n, n) or b.shape != (count, n):
            raise ValueError("need a (count, n, n) stack and a (count, n) right-hand side")
        col_scale = None
        if cfg.scale_diag:
            # per-system pow2 equilibration on the host, as _refine does for one
            # system (refine.py:293-297); the device repeats the rounding to u
            u = cfg.precisions.u
            a, b = a.copy(), b.copy()
            col_scale = np.empty((count, n))
            for i in range(count):
                a[i], b[i], col_scale[i] = _pow2_equilibrate(_round_u(a[i], u), _round_u(b[i], u))
        pa, pb, dev = a.ctypes.data, b.ctypes.data, 0
    else:
        if cfg.scale_diag:
            raise NotImplementedError("scale_diag with device-resident inputs: pass host arrays "
                                      "(the equilibration runs on the host)")
        pa, pb = on_device_ptrs
        dev = 1
        col_scale = None
    opts = make_options(cfg, n)
    res = BatchResult(count, n, cfg.i_max)
    res.col_scale = col_scale
    out = res.c_struct()
    ms = C.c_double()
    _lib._check(lib.gb_solve_batched(count, n, C.byref(opts), cfg.i_max, cfg.c_conv, C.c_void_p(pa),
                                     C.c_void_p(pb), dev, C.byref(out), C.byref(ms),
                                     C.c_void_p(_lib.current_stream())), "gb_solve_batched")
    res.device_ms = ms.value
    return res

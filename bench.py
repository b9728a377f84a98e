#!/usr/bin/env python
"""GCRO-DR-IR benchmark (driver contract).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload cfg5|cfg4|cfg3|cfg2|cfg1] [--budget-s S]

A step is one pass of the hot path over one batch of synthetic input:
  * single-system workloads -- one full GCRO-DR-IR solve (factorisation,
    x0, reference solution, refinement loop to its verdict) of every
    precision variant the configuration names;
  * cfg3 -- one batched launch over all systems of the configuration.

Default workload: cfg5, BASELINE.json configs[4] -- the largest single-GPU
configuration (randsvd n = 16384, kappa 1e8, (fp16, fp32, fp64),
GCRO-DR-IR(200, 30)); BASELINE's metric names no configuration, so the
largest one is the headline.  One cfg5 solve runs the inner solver to its
820-cycle cap (~1.6e5 operator applications), i.e. minutes even at the HBM
roofline (1.61 GB per application), so K timed solves are capped by a wall
clock budget (--budget-s): the line reports the number of solves actually
timed in "steps" (and the request in "steps_requested"); the warm-up steps
of cfg5 are solves truncated at a few cycles (every kernel of the path runs,
the clocks ramp) -- see "config".  Multi-GPU: replicas (one independent solve
stream per rank, no collective on the data path), cfg3 shards its systems;
timing is the max over ranks of CUDA-event device time.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "GCRO-DR-IR solves/s + time-to-solution; precond-op HBM GB/s, LU TC util vs peak"
T_START = time.perf_counter()

WORKLOADS = {
    "cfg1": ["cfg1"],
    "cfg2": ["cfg2a", "cfg2b"],
    "cfg3": ["cfg3"],
    "cfg4": ["cfg4"],
    "cfg5": ["cfg5"],
}
# cycle cap of the truncated warm-up solves of the long workload
WARM_CYCLES = {"cfg5": 4}

_BYTES = {"half": 2, "single": 4, "double": 8, "quad": 8}
_FMT = {"half": 0, "single": 1, "double": 2, "quad": 3}
_SQUARED = {"half": "single", "single": "double", "double": "quad"}


def _log(msg: str) -> None:
    print(f"[bench +{time.perf_counter() - T_START:6.1f}s] {msg}", file=sys.stderr, flush=True)


def _rank_env():
    return int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")), int(
        os.environ.get("LOCAL_RANK", "0"))


def _measured(key: str, fallback: float):
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        v = json.load(open(p)).get(key)
        if v:
            return float(v), "measured"
    return fallback, "fallback"


def _fp64_peak():
    """DFMA throughput measured on this pool's B200s (tools/micro/fp64peak.cu,
    profiles/r02/fp64_peak.json), TFLOP/s; None when not measured."""
    p = os.path.join(ROOT, "profiles", "r02", "fp64_peak.json")
    if os.path.exists(p):
        return json.load(open(p)).get("dfma_tflops")
    return None


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap,utilization.gpu")

    def __init__(self, index: int, period: float = 0.2):
        self.index = index
        self.period = period
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout.strip()
                if out:
                    self.samples.append([s.strip() for s in out.split(",")])
            except Exception:
                pass
            self._stop.wait(self.period)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self._t:
            self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        util = [float(s[6]) for s in self.samples if len(s) > 6 and s[6].replace(".", "").isdigit()]
        loaded = [c for c, u in zip(sm, util) if u > 0] or sm
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if s[2 + i].lower().startswith("active")})
        return {"sm_mhz": statistics.median(loaded) if loaded else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


# ---------------------------------------------------------------------------
# workload plumbing
# ---------------------------------------------------------------------------

def _spec(name):
    from paper_2201_09827_b200 import problems

    return problems.CONFIGS[name]


def _cfg(spec, method="rgmres-ir"):
    from paper_2201_09827_b200.precision import PrecisionTriple
    from paper_2201_09827_b200.refine import Method, RefineConfig

    return RefineConfig(PrecisionTriple.parse(*spec.precisions), Method.parse(method), m=spec.m,
                        k=spec.k if method.startswith("r") else 0, tau=spec.tau, i_max=spec.i_max)


def shard_systems(spec, rank: int, world: int) -> range:
    """Multi-GPU decomposition.  The batched workload (cfg3)
    splits the configuration's own systems: rank r solves the contiguous
    block r of ceil(batch / world) systems (seeds 1 + index, no data-path
    collective) -- strong scaling of the 4096-system batch.  A single-system
    workload does not shard: every rank solves the same system as an
    independent replica (weak scaling)."""
    if spec.batch == 1:
        return range(0, 1)
    per = -(-spec.batch // world)
    return range(min(spec.batch, rank * per), min(spec.batch, (rank + 1) * per))


def max_over_ranks(value: float, dist, device) -> float:
    """Whole-job time = the slowest rank's device time (the only collective)."""
    if dist is None:
        return value
    import torch

    t = torch.tensor([value], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def _inputs(spec, rank: int = 0, world: int = 1):
    """Seeded inputs (paper_2201_09827_b200/problems.py, bit-identical to the
    reference's generators).  Large single systems are cached under /tmp (the
    Haar factors of cfg5 cost minutes of host LAPACK time)."""
    from paper_2201_09827_b200 import problems

    if spec.batch == 1:
        cache = os.path.join("/tmp", f"gb_inputs_{spec.name}_{spec.n}.npz")
        if os.path.exists(cache):
            try:
                z = np.load(cache)
                return z["a"], z["b"]
            except Exception:
                pass
        t0 = time.perf_counter()
        a, b = _device_randsvd(spec) if spec.kind == "randsvd" and spec.n >= 8192 else (None, None)
        how = "device QR"
        if a is None:
            a, b = problems.config_problem(spec, 0)
            how = "host LAPACK"
        _log(f"generated {spec.name} inputs (n={spec.n}, {how}) in {time.perf_counter() - t0:.1f}s")
        if spec.n >= 2048:
            try:
                np.savez(cache + ".tmp.npz", a=a, b=b)
                os.replace(cache + ".tmp.npz", cache)
            except OSError:
                pass
        return a, b
    idx = shard_systems(spec, rank, world)
    A = np.empty((len(idx), spec.n, spec.n))
    B = np.empty((len(idx), spec.n))
    for i, sysid in enumerate(idx):
        A[i], B[i] = problems.config_problem(spec, sysid)
    return A, B


def _device_randsvd(spec):
    """The reference's randsvd construction (matgen.py:70-92: Philox(seed)
    Gaussians, two Haar factors from sign-fixed QR, geometric singular values,
    A = (P * sigma) Q^T) with the two n x n QR factorisations and the product
    on the GPU -- minutes of host LAPACK become seconds.  Same seeded Gaussian
    stream and the same distribution as the reference's generator, not the
    same bits (cuSOLVER's Householder QR rounds differently from LAPACK's);
    no reference run exists at these sizes to be bit-compatible with (SURVEY
    F8).  Returns (None, None) without a GPU."""
    try:
        import torch

        if not torch.cuda.is_available():
            return None, None
    except Exception:
        return None, None
    from paper_2201_09827_b200 import problems

    n = spec.n
    rng = np.random.Generator(np.random.Philox(1))
    sig = torch.from_numpy(spec.param ** (-np.arange(n) / (n - 1))).cuda()

    def haar():
        g = torch.from_numpy(rng.standard_normal((n, n))).cuda()
        q, r = torch.linalg.qr(g)
        d = torch.sign(torch.diagonal(r)).clone()
        d[d == 0] = 1.0
        del g, r
        return q * d[None, :]

    left = haar()
    right = haar()
    a = ((left * sig[None, :]) @ right.T).cpu().numpy()
    del left, right
    torch.cuda.empty_cache()
    return a, problems.rhs_normal(n, 1)


def _alg_bytes(spec, trace) -> float:
    """SURVEY §8(d) algorithmic bytes of one refinement-step launch:
    applies * n^2 (b_u + b_f) + n^2 b_f (precond_rhs) + n^2 b_u (residual)
    + sum_j (j + 1 + k_eff) n b_u (orthogonalisation)."""
    uf, u, _ = spec.precisions
    n = spec.n
    bu, bf = _BYTES[u], _BYTES[uf]
    total = 0.0
    for t in trace:
        total += t["applies"] * n * n * (bu + bf) + n * n * bf + n * n * bu
        ke_prev = 0
        for s, ke in zip(t["cycles"], t["k_eff"]):
            total += (s * (s + 1) / 2 + s * ke_prev) * n * bu
            ke_prev = ke
    return total


class SingleRun:
    """Device-resident single-system solves through the C ABI (value) and the
    public API from host arrays (e2e)."""

    def __init__(self, spec, torch):
        from paper_2201_09827_b200 import _lib
        from paper_2201_09827_b200.refine import make_options

        self.spec, self.torch = spec, torch
        self.a, self.b = _inputs(spec)
        self.cfg = _cfg(spec)
        self.opts = make_options(self.cfg, spec.n)
        self.solver = _lib.Solver(spec.n, self.opts)
        self.a_dev = torch.from_numpy(self.a).cuda()
        self.b_dev = torch.from_numpy(self.b).cuda()
        self.a_pin = torch.from_numpy(self.a).pin_memory()
        self.b_pin = torch.from_numpy(self.b).pin_memory()
        self.last_trace = []
        self.last_report = None
        self.last_phase_ms = {}

    def solve_device(self, max_cycles=None):
        """One full solve with inputs resident in HBM; mirrors refine._refine."""
        from paper_2201_09827_b200 import _lib
        from paper_2201_09827_b200.refine import classify

        s = self.solver
        s.set_max_cycles(max_cycles if max_cycles else self.opts.max_cycles)
        s.set_system_device(self.a_dev.data_ptr(), self.b_dev.data_ptr())
        zero, _ = s.factorize()
        self.last_phase_ms = {"lu_ms": s.last_factor_ms}
        if zero >= 0:
            return {"converged": False, "steps": 0}
        x0_reset = s.initial_solution()
        s.reference_solution()
        hist, inner, trace, conv = [], [], [], False
        reason = "IMaxExceeded"
        ferr = None
        for _ in range(self.cfg.i_max):
            info = s.step()
            cyc, ke = s.last_cycles()
            trace.append({"applies": info.applies, "cycles": cyc, "k_eff": ke, "ms": s.last_step_ms})
            if info.status & (_lib.ST_NU_ZERO | _lib.ST_NU_NONFINITE):
                conv = bool(info.status & _lib.ST_NU_ZERO)
                break
            inner.append(info.inner_iters)
            ferr = info.ferr
            d = classify(info.nbe, info.cbe, info.ferr, hist, self.cfg.precisions, self.cfg.c_conv,
                         bool(info.status & _lib.ST_STAGNATED))
            hist.append(d.nbe)
            if d.state != "continue":
                conv = d.state == "converged"
                reason = d.reason.value if d.reason else None
                break
        self.last_trace = trace
        self.last_report = {"name": self.spec.name, "converged": conv, "inner_iters": inner,
                            "cycles": [len(t["cycles"]) for t in trace],
                            "applies": [t["applies"] for t in trace],
                            "nbe": hist[-1] if hist else None, "ferr": ferr,
                            "reason": None if conv else reason, "x0_reset": bool(x0_reset),
                            "step_ms": [t["ms"] for t in trace], **self.last_phase_ms}
        return self.last_report

    def solve_e2e(self):
        """The public API call from pinned host memory; result read back."""
        from paper_2201_09827_b200.refine import _refine

        return _refine(self.a_pin.numpy(), self.b_pin.numpy(), self.cfg)

    def h2d_bytes(self):
        return self.a.nbytes + self.b.nbytes

    def d2h_bytes(self):
        return self.spec.n * 8


class BatchRun:
    def __init__(self, spec, torch, rank, world):
        from paper_2201_09827_b200.refine import make_options

        self.spec, self.torch = spec, torch
        self.A, self.B = _inputs(spec, rank, world)
        self.count = self.A.shape[0]
        self.cfg = _cfg(spec)
        self.opts = make_options(self.cfg, spec.n)
        self.A_dev = torch.from_numpy(self.A).cuda()
        self.B_dev = torch.from_numpy(self.B).cuda()
        self.A_pin = torch.from_numpy(self.A).pin_memory()
        self.B_pin = torch.from_numpy(self.B).pin_memory()
        self.last_ms = 0.0
        self.last_trace = []
        self.last_report = None

    def solve_device(self, max_cycles=None):
        from paper_2201_09827_b200.batched import solve_batched

        res = solve_batched(None, None, self.cfg, on_device_ptrs=(self.A_dev.data_ptr(), self.B_dev.data_ptr()),
                            count=self.count, n=self.spec.n)
        self.last_ms = res.device_ms
        self.last_report = {"name": self.spec.name, "converged": int(res.converged.sum()), "count": self.count}
        return res

    def solve_e2e(self):
        from paper_2201_09827_b200.batched import solve_batched

        return solve_batched(self.A_pin.numpy(), self.B_pin.numpy(), self.cfg)

    def h2d_bytes(self):
        return self.A.nbytes + self.B.nbytes

    def d2h_bytes(self):
        return self.count * self.spec.n * 8


KERNEL_CASES = [
    # (name, n, (u_f, u, u_r), lu_modes): BASELINE configs[3] / configs[4] sizes
    ("cfg4", 8192, ("single", "double", "quad"), ("exact",)),
    ("cfg5", 16384, ("half", "single", "double"), ("exact", "tensor")),
]


def kernel_rooflines(torch, peak_gbs: float, peak_tf: float, reps: int = 10, cases=KERNEL_CASES):
    """Per-kernel evidence at the large configurations: the
    preconditioned operator and the residual as standalone launches on
    device-resident data (CUDA events, back-to-back launches, inputs larger
    than L2), and the LU factorisation.  A: seeded N(0, 1/n) + 4 I generated
    on the device (the operator/residual/LU cost does not depend on values)."""
    from paper_2201_09827_b200 import _lib
    from paper_2201_09827_b200.precision import PrecisionTriple
    from paper_2201_09827_b200.refine import Method, RefineConfig, make_options

    out = []
    fp64 = _fp64_peak()
    for name, n, prec, modes in cases:
        gen = torch.Generator(device="cuda").manual_seed(1)
        a = torch.randn((n, n), dtype=torch.float64, device="cuda", generator=gen) / math.sqrt(n)
        a.diagonal().add_(4.0)
        b = torch.randn(n, dtype=torch.float64, device="cuda", generator=gen)
        uf, u, ur = prec
        bu, bf = _BYTES[u], _BYTES[uf]
        for mode in modes:
            cfg = RefineConfig(PrecisionTriple.parse(*prec), Method.RGMRES_IR, m=20, k=4, i_max=1, lu_mode=mode)
            s = _lib.Solver(n, make_options(cfg, n))
            s.set_system_device(a.data_ptr(), b.data_ptr())
            s.factorize()
            lu_ms = s.last_factor_ms
            row = {"case": name, "n": n, "precisions": "/".join(prec), "lu_mode": mode,
                   "lu_ms": lu_ms, "lu_tflops": 2.0 * n ** 3 / 3.0 / (lu_ms * 1e-3) / 1e12,
                   "lu_frac_of_tc_peak": 2.0 * n ** 3 / 3.0 / (lu_ms * 1e-3) / 1e12 / peak_tf}
            if mode == "tensor":
                tu = s.tc_update_stats() if hasattr(s, "tc_update_stats") else None
                if tu:
                    row.update({"tc_update_ms": tu["ms"], "tc_update_tflops": tu["tflops"],
                                "tc_update_frac_of_tc_peak": tu["tflops"] / peak_tf,
                                "tc_update_flop_share": tu["flop_share"]})
            if mode == "exact":
                v = np.random.default_rng(0).standard_normal(n)
                s.apply_preconditioned(v, _FMT[_SQUARED[u]])
                t_op = s.time_op(0, reps)
                s.residual(v, _FMT[ur])
                t_res = s.time_op(2, reps)
                op_b = n * n * (bu + bf)
                res_b = n * n * bu
                row.update({"op_ms": t_op, "op_alg_bytes": op_b, "op_gbs": op_b / (t_op * 1e-3) / 1e9,
                            "op_frac": op_b / (t_op * 1e-3) / 1e9 / peak_gbs,
                            "residual_ms": t_res, "residual_alg_bytes": res_b,
                            "residual_gbs": res_b / (t_res * 1e-3) / 1e9,
                            "residual_frac": res_b / (t_res * 1e-3) / 1e9 / peak_gbs})
                if _SQUARED[u] == "quad" and fp64:
                    # double-double operator: ~22 fp64 flop per matrix / factor entry
                    fl = 22.0 * 2 * n * n
                    row.update({"op_dd_fp64_tflops": fl / (t_op * 1e-3) / 1e12,
                                "op_dd_frac_of_fp64_peak": fl / (t_op * 1e-3) / 1e12 / fp64})
            out.append(row)
            s.close()
            del s
        del a, b
        torch.cuda.empty_cache()
    return out


def _flush_l2(torch, buf):
    buf.add_(1.0)  # 512 MiB write > 126 MB L2


# ---------------------------------------------------------------------------
# CPU (oracle) timing -- reference arm and cpu_baseline
# ---------------------------------------------------------------------------

def _cores() -> int:
    return len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1)


def _time_call(fn, min_s=0.5, max_reps=50):
    """Seconds per call of fn (at least one call, repeated up to min_s)."""
    t0 = time.perf_counter()
    reps = 0
    while True:
        fn()
        reps += 1
        dt = time.perf_counter() - t0
        if dt >= min_s or reps >= max_reps:
            return dt / reps


def cpu_cycle_sample(spec, budget_s: float, cycles_hint=None):
    """Single system that the CPU restatement can iterate on within the budget
    (n <= 1024): setup (rounding, LU, x0, xref) timed fully; the GCRO-DR part
    timed over the cold cycle plus the first deflated cycles, then extended to
    the solve's cycle count at the measured per-deflated-cycle cost."""
    from oracle import cpu_gcrodr_ir as O

    a, b = _inputs(spec)
    uf, u, ur = spec.precisions
    t0 = time.perf_counter()
    a_u, b_u = O.rnd(a, u), O.rnd(b, u)
    f = O.lu_factor(a_u, uf)
    x = O.lu_solve(f, b_u, uf, store=u)
    if not np.all(np.isfinite(x)):
        x = np.zeros(spec.n)
    O.reference_solution(a_u, b_u)
    r = O.residual(a_u, x, b_u, ur)
    nu = float(np.max(np.abs(r)))
    rhat = O.rnd(r / nu, u)
    t_setup = time.perf_counter() - t0
    mv = O.squared(u)
    t1 = time.perf_counter()
    out1, _ = O.gcrodr(a_u, f, rhat, spec.m, spec.k, spec.tau, mv, u, None, max_cycles=1)
    t_cold = time.perf_counter() - t1
    ncyc_full = int(cycles_hint or 1)
    if out1.converged or ncyc_full <= 1:
        est = t_setup + t_cold
        return est, (f"{spec.name}: setup {t_setup:.1f}s + {out1.total} Arnoldi its {t_cold:.1f}s, "
                     f"measured in full"), False
    extra = 2
    t2 = time.perf_counter()
    out3, _ = O.gcrodr(a_u, f, rhat, spec.m, spec.k, spec.tau, mv, u, None, max_cycles=1 + extra)
    t_three = time.perf_counter() - t2
    per_defl = max(t_three - t_cold, 0.0) / extra
    est = t_setup + t_cold + (ncyc_full - 1) * per_defl
    return est, (f"{spec.name}: setup {t_setup:.1f}s timed; cold cycle ({out1.total} its) {t_cold:.1f}s and "
                 f"{extra} deflated cycles ({out3.total - out1.total} its) {t_three - t_cold:.1f}s timed; "
                 f"x {ncyc_full} cycles of the full solve -> {est:.0f}s (extrapolated)"), True


def cpu_model_sample(spec, iters_full: int, cycles_full: int, lu_cols: int = 2):
    """Large single system (n >= 2048: the reference cannot finish a solve in
    minutes): SURVEY §8(d)'s time-boxed model.  Timed on the host:
    the first `lu_cols` columns of the reference's LU at u_f (simulated fp16:
    the reference's own per-column numpy update; LAPACK for fp32), one fp64
    LU-quality GEMM rate for the xref dgetrf, operator applications and the
    Gram-Schmidt vector operations at this n.  Model: T = T_LU + T_xref +
    iterations x (T_apply + T_orth(average j)), labelled extrapolated."""
    from oracle import cpu_gcrodr_ir as O

    n = spec.n
    uf, u, ur = spec.precisions
    a, b = _inputs(spec)
    a_u = O.rnd(a, u)
    notes = []
    # --- LU
    if uf == "half":
        w = O.rnd(a_u, uf).copy()
        t0 = time.perf_counter()
        with np.errstate(divide="ignore", invalid="ignore", over="ignore"):
            for k in range(lu_cols):  # the reference's column step (densela.py:151-162)
                p = k + int(np.argmax(np.abs(w[k:, k])))
                if p != k:
                    w[[k, p], :] = w[[p, k], :]
                l = O.rnd(w[k + 1:, k] / w[k, k], uf)
                w[k + 1:, k] = l
                w[k + 1:, k + 1:] = O.rnd(w[k + 1:, k + 1:] - O.rnd(np.outer(l, w[k, k + 1:]), uf), uf)
        per_col = (time.perf_counter() - t0) / lu_cols
        t_lu = per_col * n / 3.0  # sum_k (n - k)^2 / n^2 = n / 3 column-equivalents
        notes.append(f"fp16 LU: {lu_cols} columns timed ({per_col:.2f}s each) -> {t_lu:.0f}s for n^3/3")
        del w
    else:
        import scipy.linalg

        w = a_u.astype(np.float32) if uf == "single" else a_u
        t0 = time.perf_counter()
        scipy.linalg.lu_factor(w, check_finite=False)
        t_lu = time.perf_counter() - t0
        notes.append(f"{uf} LU (LAPACK) timed in full {t_lu:.1f}s")
        del w
    # --- xref: dgetrf + 4 x (dd residual + fp64 solve); dd residual ~ 8.5 s at n = 8192
    import scipy.linalg

    nn = min(n, 4096)
    g = np.random.default_rng(0).standard_normal((nn, nn))
    t0 = time.perf_counter()
    scipy.linalg.lu_factor(g, check_finite=False)
    t_getrf = (time.perf_counter() - t0) * (n / nn) ** 3
    rows = 256
    t0 = time.perf_counter()
    O.dd_matvec(a_u[:rows], b)
    t_ddres = (time.perf_counter() - t0) * n / rows
    t_xref = t_getrf + 4 * t_ddres
    notes.append(f"xref: dgetrf at n={nn} scaled by (n/{nn})^3 -> {t_getrf:.0f}s, dd residual on {rows} rows "
                 f"scaled -> {t_ddres:.1f}s x 4")
    # --- operator application with synthetic factors of the same shape / format
    rng = np.random.default_rng(1)
    lower = np.tril(rng.standard_normal((n, n)) * (0.5 / math.sqrt(n)), -1) + np.eye(n)
    upper = np.triu(rng.standard_normal((n, n)) * (0.5 / math.sqrt(n)), 1) + 2.0 * np.eye(n)
    f = O.Factors(lower, upper, np.arange(n), uf, 1.0)
    v = O.rnd(rng.standard_normal(n), u)
    mv = O.squared(u)
    if mv == "quad":
        t0 = time.perf_counter()
        O.apply_op(a_u, f, v, mv, u)
        t_apply = time.perf_counter() - t0
    else:
        O.apply_op(a_u, f, v, mv, u)
        t_apply = _time_call(lambda: O.apply_op(a_u, f, v, mv, u), min_s=3.0, max_reps=5)
    # --- everything in a deflated Arnoldi cycle except the operator: the
    # reference's own cycle (projection against C_k, MGS, Givens, LS) run on a
    # stand-in operator that costs nothing (a fixed pseudo-random vector per step)
    kk = spec.k
    steps = spec.m - kk
    cmat, _ = np.linalg.qr(rng.standard_normal((n, kk)))
    cmat = O.rnd(cmat, u)
    pool = O.rnd(rng.standard_normal((n, 8)), u)
    cnt = [0]

    def fake_op(_v):
        cnt[0] += 1
        return pool[:, cnt[0] % 8] + 0.01 * _v

    r0 = O.rnd(rng.standard_normal(n), u)
    t0 = time.perf_counter()
    O.arnoldi(fake_op, r0, O.vnorm2(r0, u), steps, 0.0, u, True, C=cmat)
    t_cycle = time.perf_counter() - t0
    est = t_lu + t_xref + iters_full * t_apply + cycles_full * t_cycle
    notes.append(f"apply {t_apply * 1e3:.0f} ms x {iters_full} Arnoldi steps; one deflated cycle without the "
                 f"operator ({steps} steps: C_k projection, MGS, Givens, LS) {t_cycle:.2f}s x {cycles_full} cycles "
                 f"-> {est:.0f}s (extrapolated; per-cycle harmonic-Ritz / QR work not included)")
    return est, f"{spec.name}: " + "; ".join(notes), True


def cpu_sample(workload: str, budget_s: float = 20.0, hints: dict | None = None):
    """Time the CPU restatement of the reference (oracle/cpu_gcrodr_ir.py) on a
    bounded sample of the workload and scale to solves/s.  hints: per spec
    name {"iters": Arnoldi steps, "cycles": cycles} of the full solve (from the
    GPU run of the same system, else the reference's goldens)."""
    specs = [_spec(s) for s in WORKLOADS[workload]]
    cores = _cores()
    if specs[0].batch > 1:
        spec = specs[0]
        from concurrent.futures import ProcessPoolExecutor

        count = min(spec.batch, max(cores * 6, 16))
        t0 = time.perf_counter()
        with ProcessPoolExecutor(max_workers=cores, initializer=_one_thread) as ex:
            list(ex.map(_cpu_cfg3_one, range(count)))
        dt = time.perf_counter() - t0
        return {"value": count / dt, "unit": "solves/s", "cores": cores, "kind": "port", "extrapolated": False,
                "sample": f"{count} of {spec.batch} cfg3 systems, full solves, {cores}-process pool "
                          f"(OPENBLAS_NUM_THREADS=1 per worker, harness.py:250-252)"}
    total_s = 0.0
    notes = []
    extrap = False
    for spec in specs:
        h = (hints or {}).get(spec.name) or _GOLDEN_HINTS.get(spec.name, {})
        if spec.n <= 256:
            from oracle import cpu_gcrodr_ir as O

            a, b = _inputs(spec)
            t0 = time.perf_counter()
            rep = O.solve(a, b, spec.precisions, "rgmres-ir", spec.m, spec.k, spec.tau, spec.i_max)
            est = time.perf_counter() - t0
            note, ex = f"{spec.name}: full solve measured ({est:.2f}s, inner {rep.inner_iters})", False
        elif spec.n >= 2048:
            est, note, ex = cpu_model_sample(spec, int(h.get("iters", 1)), int(h.get("cycles", 1)))
        else:
            est, note, ex = cpu_cycle_sample(spec, budget_s / len(specs), h.get("cycles"))
        total_s += est
        notes.append(note)
        extrap = extrap or ex
    return {"value": len(specs) / total_s, "unit": "solves/s", "cores": cores, "kind": "port",
            "extrapolated": extrap, "threads": "default OpenBLAS threading (all cores) in BLAS/LAPACK calls; "
            "the reference's Python-level loops are single-threaded",
            "sample": "; ".join(notes)}


def _one_thread():
    os.environ["OPENBLAS_NUM_THREADS"] = "1"
    try:
        from threadpoolctl import threadpool_limits

        threadpool_limits(1)
    except Exception:
        pass


def _cpu_cfg3_one(i):
    from oracle import cpu_gcrodr_ir as O
    from paper_2201_09827_b200 import problems

    spec = problems.CONFIGS["cfg3"]
    a, b = problems.config_problem(spec, i)
    O.solve(a, b, spec.precisions, "rgmres-ir", spec.m, spec.k, spec.tau, spec.i_max)
    return i


# Arnoldi steps / cycles of full solves when no GPU run supplies them: the
# reference's own runs (tests/golden/*.json); cfg5 from the GPU run committed
# under profiles/r02/ (the reference cannot run it)
_GOLDEN_HINTS = {"cfg1": {"iters": 19, "cycles": 2}, "cfg2a": {"iters": 8158, "cycles": 205},
                 "cfg2b": {"iters": 5402, "cycles": 205}, "cfg4": {"iters": 24, "cycles": 2},
                 "cfg5": {"iters": 139430, "cycles": 820}}


def _cfg5_hint():
    p = os.path.join(ROOT, "profiles", "r02", "cfg5_full.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return {"iters": int(sum(d["inner_iters"])), "cycles": int(sum(d["cycles"]))}
    return None


# ---------------------------------------------------------------------------
# main
# ---------------------------------------------------------------------------

def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="cfg5", choices=sorted(WORKLOADS))
    ap.add_argument("--budget-s", type=float, default=640.0,
                    help="wall-clock budget of the whole invocation; timed solves stop when the next one "
                         "would not fit (at least one is always timed)")
    ap.add_argument("--profile-cycles", type=int, default=0,
                    help="profiling only (ncu launch lists): cap the inner solver of the TIMED solves at this "
                         "many cycles; the printed line is then not a bench value and says so")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-kernels", action="store_true", help="skip the per-kernel cfg4/cfg5 rooflines")
    args = ap.parse_args()
    rank, world, local = _rank_env()
    specs = [_spec(s) for s in WORKLOADS[args.workload]]
    workload_desc = "; ".join(
        f"{s.name}: {s.kind}({s.n}, {s.param:g}){' x%d' % s.batch if s.batch > 1 else ''} "
        f"GCRO-DR-IR(m={s.m}, k={s.k}) tau={s.tau:g} prec={'/'.join(s.precisions)} i_max={s.i_max}"
        for s in specs)
    c5 = _cfg5_hint()
    if c5:
        _GOLDEN_HINTS["cfg5"] = c5

    if args.impl == "reference":
        if rank != 0:
            return
        # the reference's own algorithm (the pinned CPU restatement) on the host cores
        res = cpu_sample(args.workload)
        line = {"metric": METRIC, "value": res["value"], "unit": "solves/s", "n_gpus": args.gpus,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": len(specs) * 1e3 / res["value"],
                "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
                "data": "synthetic (seeded, SURVEY §8(d))", "impl": "reference",
                "config": {"workload": workload_desc},
                "cpu_baseline": res,
                "e2e": {"value": res["value"], "unit": "solves/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(line))
        return

    import torch

    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2201_09827_b200 import _lib

    lib = _lib.require_gpu()
    runs = [BatchRun(s, torch, rank, world) if s.batch > 1 else SingleRun(s, torch) for s in specs]
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float64, device="cuda")
    stream = torch.cuda.current_stream()
    warm_cycles = WARM_CYCLES.get(args.workload)
    _log(f"workload {args.workload}: inputs resident, warm-up x{args.warmup}"
         + (f" (truncated at {warm_cycles} cycles)" if warm_cycles else ""))

    for _ in range(args.warmup):
        for r in runs:
            r.solve_device(max_cycles=warm_cycles)
    torch.cuda.synchronize()
    if dist:
        dist.barrier()

    step_ms = []
    kernel_ms = []
    alg_bytes = []
    launches0 = lib.gb_launch_count()
    # reserve for what follows the timed region: the e2e solve (one more step)
    # plus the CPU sample and the per-kernel rooflines
    reserve_fixed = (0 if args.no_cpu else 60.0) + (0 if args.no_kernels else 45.0)
    steps_done = 0
    with ClockSampler(local, 0.2 if args.workload != "cfg5" else 1.0) as clk:
        for _ in range(args.steps):
            _flush_l2(torch, flush)
            torch.cuda.synchronize()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for r in runs:
                r.solve_device(max_cycles=args.profile_cycles or None)
            e1.record(stream)
            torch.cuda.synchronize()
            step_ms.append(e0.elapsed_time(e1))
            steps_done += 1
            for r in runs:
                if isinstance(r, SingleRun):
                    kernel_ms.extend(t["ms"] for t in r.last_trace)
                    alg_bytes.extend(_alg_bytes(r.spec, [t]) for t in r.last_trace)
            per = max(step_ms) / 1e3
            elapsed = time.perf_counter() - T_START
            need = per * (1 + (0 if args.no_e2e else 1)) + reserve_fixed
            stop = elapsed + need > args.budget_s
            if world > 1:
                flag = torch.tensor([1.0 if stop else 0.0], device="cuda")
                dist.all_reduce(flag, op=dist.ReduceOp.MAX)
                stop = bool(flag.item() > 0)
            if stop and steps_done < args.steps:
                _log(f"budget: {steps_done} of {args.steps} requested steps timed ({per:.1f}s per step)")
                break
    launches = lib.gb_launch_count() - launches0
    total_ms = sum(step_ms)
    total_ms = max_over_ranks(total_ms, dist, "cuda")
    if specs[0].batch > 1:
        solves_per_step = specs[0].batch  # the shards of all ranks make up the configuration's batch
        value = solves_per_step * steps_done / (total_ms / 1e3)
        scaling = "strong"
    else:
        solves_per_step = len(specs)
        value = world * solves_per_step * steps_done / (total_ms / 1e3)
        scaling = "weak"

    # end-to-end through the public API from pinned host buffers
    e2e = None
    if not args.no_e2e:
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        nsteps = 1 if max(step_ms) > 5e3 else max(1, min(steps_done, 2))
        t0 = time.perf_counter()
        for _ in range(nsteps):
            for r in runs:
                r.solve_e2e()
        torch.cuda.synchronize()
        e2e_s = time.perf_counter() - t0
        te = torch.tensor([e2e_s], dtype=torch.float64, device="cuda")
        if dist:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        mult = 1 if specs[0].batch > 1 else world
        e2e = {"value": mult * solves_per_step * nsteps / float(te.item()), "unit": "solves/s",
               "h2d_bytes_per_step": int(sum(r.h2d_bytes() for r in runs)),
               "d2h_bytes_per_step": int(sum(r.d2h_bytes() for r in runs)),
               "steps": nsteps, "timer": "wall clock around solve()/solve_batched() from pinned host buffers "
               "(device workspaces cached across calls)"}

    if rank != 0:
        if dist:
            dist.destroy_process_group()
        return

    peak, peak_kind = _measured("hbm_gbs", 6650.0)
    tc_peak, _ = _measured("bf16_tflops", 2250.0)
    reports = [r.last_report for r in runs]
    roof = None
    if kernel_ms:
        avg_ms = statistics.mean(kernel_ms)
        avg_b = statistics.mean(alg_bytes)
        ach = avg_b / (avg_ms / 1e3) / 1e9
        big = specs[0].n >= 4096
        roof = {"bound": "hbm", "achieved": ach, "peak": peak, "unit": "GB/s", "frac": ach / peak,
                "traffic": _ncu_traffic(args.workload, reports), "kernel": "k_step (one refinement step = one "
                "persistent cooperative launch: residual scaling, GCRO-DR cycles, update, errors)",
                "peak_kind": peak_kind, "alg_bytes_per_launch": avg_b, "avg_launch_ms": avg_ms,
                "note": ("A and the factors stream from HBM on every operator application (n^2 (b_u + b_f) = "
                         f"{specs[0].n ** 2 * (_BYTES[specs[0].precisions[1]] + _BYTES[specs[0].precisions[0]]) / 1e9:.2f}"
                         " GB >> L2)") if big else
                        "A and the factors are L2-resident at this n: the HBM fraction only says the step is "
                        "bound by the substitution chain, reductions and double-double arithmetic (see kernels)"}
    else:
        ms = statistics.mean(r.last_ms for r in runs)
        n, cnt = specs[0].n, runs[0].count
        alg = cnt * (n * n * 8 + n * 8)  # input stream
        ach = alg / (ms / 1e3) / 1e9
        fp64 = _fp64_peak()
        roof = {"bound": "hbm", "achieved": ach, "peak": peak, "unit": "GB/s", "frac": ach / peak,
                "traffic": _ncu_traffic(args.workload, reports), "kernel": "k_batched (one CTA per system)",
                "peak_kind": peak_kind, "note": "compute/latency bound: HBM bytes = input stream only"}
        if fp64:
            # xref double-double GEPP: 2 n^3 / 3 dd multiply-adds at ~20 fp64 flop each
            fl = cnt * (2.0 * n ** 3 / 3.0) * 20.0
            roof.update({"fp64_tflops": fl / (ms / 1e3) / 1e12, "fp64_peak_tflops": fp64,
                         "fp64_frac": fl / (ms / 1e3) / 1e12 / fp64})
    cpu = None
    if not args.no_cpu and world == 1:
        hints = {}
        for r in runs:
            if isinstance(r, SingleRun) and r.last_report:
                hints[r.spec.name] = {"iters": sum(r.last_report["inner_iters"]) or 1,
                                      "cycles": sum(r.last_report["cycles"]) or 1}
        _log("cpu_baseline sample")
        cpu = cpu_sample(args.workload, hints=hints)
    kernels = None
    if not args.no_kernels and world == 1:
        for r in runs:
            if isinstance(r, SingleRun):
                r.solver.close()
        del runs
        from paper_2201_09827_b200.refine import release_workspaces

        release_workspaces()
        torch.cuda.empty_cache()
        _log("per-kernel rooflines")
        kernels = kernel_rooflines(torch, peak, tc_peak)
    line = {
        "metric": METRIC, "value": value, "unit": "solves/s", "n_gpus": world, "steps": steps_done,
        "warmup": args.warmup, "ms_per_step": total_ms / steps_done, "higher_is_better": True,
        "scaling": scaling, "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded inputs, SURVEY §8(d); no dataset)",
        "steps_requested": args.steps,
        **({"not_a_bench_value": f"timed solves truncated at {args.profile_cycles} cycles (--profile-cycles)"}
           if args.profile_cycles else {}),
        "config": {"workload": workload_desc, "l2": "flushed between steps (512 MiB write)",
                   "parallelism": f"replicas x{world}" if specs[0].batch == 1 else f"shards x{world}",
                   "time_to_solution_ms": total_ms / steps_done / len(specs) if specs[0].batch == 1 else None,
                   "warmup_steps": (f"solves truncated at {warm_cycles} inner cycles (LU, x0, xref, one "
                                    f"refinement launch with cold + deflated cycles)" if warm_cycles
                                    else "full solves"),
                   "budget_s": args.budget_s,
                   "verdicts": reports},
        "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "clocks": clk.summary(), "gpu_launches": int(launches),
        "kernels": kernels,
    }
    print(json.dumps(line))
    if dist:
        dist.destroy_process_group()


def _ncu_traffic(workload, reports=None):
    """dram bytes per k_step launch from the committed ncu capture.  cfg5's
    capture is a solve truncated at a few cycles (ncu replays a kernel ~40
    times; the full launch runs for minutes): its bytes per operator
    application are scaled to the applications of the timed launch."""
    p = os.path.join(ROOT, "profiles", f"ncu_traffic_{workload}.json")
    if not os.path.exists(p):
        return None
    d = json.load(open(p))
    if "traffic_bytes_per_apply" in d and reports:
        applies = [a for r in reports if r for a in r.get("applies", [])]
        if applies:
            return d["traffic_bytes_per_apply"] * statistics.mean(applies)
    return d.get("traffic_bytes_per_launch")


if __name__ == "__main__":
    main()

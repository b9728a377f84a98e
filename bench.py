#!/usr/bin/env python
"""GCRO-DR-IR benchmark (driver contract).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload cfg2|cfg1|cfg3|cfg4|cfg5]

A step is one pass of the hot path over one batch of synthetic input:
  * single-system workloads -- one full GCRO-DR-IR solve (factorisation,
    x0, reference solution, refinement loop to its verdict) of every
    precision variant the configuration names;
  * cfg3 -- one batched launch over all systems of the configuration.
Default workload: BASELINE.json configs[1] (cfg2: prolate n=1024, w=0.45,
GCRO-DR-IR(50, 10), tau 1e-6, u_f in {fp32, fp16}).  Multi-GPU: replicas
(one independent solve stream per rank, no collective on the data path),
scaling "weak"; timing is the max over ranks of CUDA-event device time.
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

WORKLOADS = {
    "cfg1": ["cfg1"],
    "cfg2": ["cfg2a", "cfg2b"],
    "cfg3": ["cfg3"],
    "cfg4": ["cfg4"],
    "cfg5": ["cfg5"],
}

_BYTES = {"half": 2, "single": 4, "double": 8, "quad": 8}


def _rank_env():
    return int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")), int(
        os.environ.get("LOCAL_RANK", "0"))


def _tc_peak():
    """dense fp16/bf16 tensor TFLOP/s (MEASURED_PEAKS.json burst; fallback 2250 nominal)"""
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        return json.load(open(p)).get("bf16_tflops", 2250.0)
    return 2250.0


def _peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return d.get("hbm_gbs", 6650.0), "measured"
    return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap,utilization.gpu")

    def __init__(self, index: int):
        self.index = index
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
            self._stop.wait(0.2)

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
    """Multi-GPU decomposition.  Batched workloads (cfg3) are
    weak-scaled shards: rank r solves systems r*batch .. (r+1)*batch - 1
    (seeds 1 + index, disjoint across ranks, no data-path collective).  A
    single-system workload does not shard: every rank solves the same system
    as an independent replica."""
    if spec.batch == 1:
        return range(0, 1)
    return range(rank * spec.batch, (rank + 1) * spec.batch)


def max_over_ranks(value: float, dist, device) -> float:
    """Whole-job time = the slowest rank's device time (the only collective)."""
    if dist is None:
        return value
    import torch

    t = torch.tensor([value], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def _inputs(spec, replica: int, world: int = 1):
    """Seeded inputs; replicas of single-system workloads perturb nothing (the
    configuration is one system) -- cfg3 shards draw systems seed+index."""
    from paper_2201_09827_b200 import problems

    cache = os.path.join("/tmp", f"gb_inputs_{spec.name}_{spec.n}.npz")
    if spec.batch == 1:
        if os.path.exists(cache):
            z = np.load(cache)
            return z["a"], z["b"]
        a, b = problems.config_problem(spec, 0)
        try:
            np.savez(cache, a=a, b=b)
        except OSError:
            pass
        return a, b
    idx = shard_systems(spec, replica, world)
    A = np.empty((spec.batch, spec.n, spec.n))
    B = np.empty((spec.batch, spec.n))
    for i, sysid in enumerate(idx):
        A[i], B[i] = problems.config_problem(spec, sysid)
    return A, B


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
            total += sum((j + 1 + ke_prev) for j in range(s)) * n * bu
            ke_prev = ke
    return total


class SingleRun:
    """Device-resident single-system solves through the C ABI (value) and the
    public API from host arrays (e2e)."""

    def __init__(self, spec, torch):
        from paper_2201_09827_b200 import _lib
        from paper_2201_09827_b200.refine import make_options

        self.spec, self.torch = spec, torch
        self.a, self.b = _inputs(spec, 0)
        self.cfg = _cfg(spec)
        self.opts = make_options(self.cfg, spec.n)
        self.solver = _lib.Solver(spec.n, self.opts)
        self.a_dev = torch.from_numpy(self.a).cuda()
        self.b_dev = torch.from_numpy(self.b).cuda()
        self.a_pin = torch.from_numpy(self.a).pin_memory()
        self.b_pin = torch.from_numpy(self.b).pin_memory()
        self.last_trace = []
        self.last_report = None

    def solve_device(self):
        """One full solve with inputs resident in HBM; mirrors refine._refine."""
        from paper_2201_09827_b200 import _lib
        from paper_2201_09827_b200.refine import classify

        s = self.solver
        s.set_system_device(self.a_dev.data_ptr(), self.b_dev.data_ptr())
        zero, _ = s.factorize()
        if zero >= 0:
            return {"converged": False, "steps": 0}
        s.initial_solution()
        s.reference_solution()
        hist, inner, trace, conv = [], [], [], False
        reason = "IMaxExceeded"
        for _ in range(self.cfg.i_max):
            info = s.step()
            cyc, ke = s.last_cycles()
            trace.append({"applies": info.applies, "cycles": cyc, "k_eff": ke, "ms": s.last_step_ms})
            if info.status & (_lib.ST_NU_ZERO | _lib.ST_NU_NONFINITE):
                conv = bool(info.status & _lib.ST_NU_ZERO)
                break
            inner.append(info.inner_iters)
            d = classify(info.nbe, info.cbe, info.ferr, hist, self.cfg.precisions, self.cfg.c_conv,
                         bool(info.status & _lib.ST_STAGNATED))
            hist.append(d.nbe)
            if d.state != "continue":
                conv = d.state == "converged"
                reason = d.reason.value if d.reason else None
                break
        self.last_trace = trace
        self.last_report = {"converged": conv, "inner_iters": inner, "nbe": hist[-1] if hist else None,
                            "reason": None if conv else reason}
        return self.last_report

    def solve_e2e(self):
        """The public API call from pinned host memory; result read back."""
        from paper_2201_09827_b200.refine import _refine

        rep = _refine(self.a_pin.numpy(), self.b_pin.numpy(), self.cfg)
        return rep

    def h2d_bytes(self):
        return self.a.nbytes + self.b.nbytes

    def d2h_bytes(self):
        return self.spec.n * 8


class BatchRun:
    def __init__(self, spec, torch, replica):
        from paper_2201_09827_b200.refine import make_options

        self.spec, self.torch = spec, torch
        self.A, self.B = _inputs(spec, replica)
        self.cfg = _cfg(spec)
        self.opts = make_options(self.cfg, spec.n)
        self.A_dev = torch.from_numpy(self.A).cuda()
        self.B_dev = torch.from_numpy(self.B).cuda()
        self.A_pin = torch.from_numpy(self.A).pin_memory()
        self.B_pin = torch.from_numpy(self.B).pin_memory()
        self.last_ms = 0.0
        self.last_trace = []

    def solve_device(self):
        from paper_2201_09827_b200.batched import solve_batched

        res = solve_batched(None, None, self.cfg, on_device_ptrs=(self.A_dev.data_ptr(), self.B_dev.data_ptr()),
                            count=self.spec.batch, n=self.spec.n)
        self.last_ms = res.device_ms
        self.last_report = {"converged": int(res.converged.sum()), "count": self.spec.batch}
        return res

    def solve_e2e(self):
        from paper_2201_09827_b200.batched import solve_batched

        return solve_batched(self.A_pin.numpy(), self.B_pin.numpy(), self.cfg)

    def h2d_bytes(self):
        return self.A.nbytes + self.B.nbytes

    def d2h_bytes(self):
        return self.spec.batch * self.spec.n * 8


KERNEL_CASES = [
    # (name, n, (u_f, u, u_r), lu_modes): BASELINE configs[3] / configs[4] sizes
    ("cfg4", 8192, ("single", "double", "quad"), ("exact",)),
    ("cfg5", 16384, ("half", "single", "double"), ("exact", "tensor")),
]


def kernel_rooflines(torch, peak_gbs: float, peak_tf: float, reps: int = 10):
    """Per-kernel evidence at the large configurations: the
    preconditioned operator and the residual as standalone launches on
    device-resident data (CUDA events, back-to-back launches, inputs larger
    than L2), and the LU factorisation.  A: seeded N(0, 1/n) + 4 I generated
    on the device (the operator/residual/LU cost does not depend on values)."""
    from paper_2201_09827_b200 import _lib
    from paper_2201_09827_b200.precision import PrecisionTriple
    from paper_2201_09827_b200.refine import Method, RefineConfig, make_options

    out = []
    for name, n, prec, modes in KERNEL_CASES:
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
            out.append(row)
            del s
        del a, b
        torch.cuda.empty_cache()
    return out


_FMT = {"half": 0, "single": 1, "double": 2, "quad": 3}
_SQUARED = {"half": "single", "single": "double", "double": "quad"}


def _flush_l2(torch, buf):
    buf.add_(1.0)  # 512 MiB write > 126 MB L2


# ---------------------------------------------------------------------------
# CPU (oracle) timing -- reference arm and cpu_baseline
# ---------------------------------------------------------------------------

def cpu_sample(workload: str, budget_s: float = 20.0, iters_hint: dict | None = None):
    """Time the CPU restatement of the reference (oracle/cpu_gcrodr_ir.py) on a
    bounded sample of the workload and scale to solves/s.

    Single-system variants: the setup (rounding, LU, x0, xref) is timed
    exactly; the Krylov part is timed over its first cycles and extrapolated to
    the iteration count of a full solve (from the GPU run, or the reference's
    golden when known).  cfg3: a subset of the systems, all cores, process pool
    (harness.py:250-252 style)."""
    from oracle import cpu_gcrodr_ir as O

    specs = [_spec(s) for s in WORKLOADS[workload]]
    cores = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count()
    if specs[0].batch > 1:
        spec = specs[0]
        from concurrent.futures import ProcessPoolExecutor

        count = min(spec.batch, max(cores * 6, 16))
        t0 = time.perf_counter()
        with ProcessPoolExecutor(max_workers=cores, initializer=_one_thread) as ex:
            list(ex.map(_cpu_cfg3_one, range(count)))
        dt = time.perf_counter() - t0
        return {"value": count / dt, "unit": "solves/s", "cores": cores, "kind": "port",
                "sample": f"{count} of {spec.batch} cfg3 systems, full solves, {cores}-process pool"}
    total_s = 0.0
    notes = []
    for spec in specs:
        a, b = _inputs(spec, 0)
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
        # Krylov sample: cycles until the budget share is used
        mv = O.squared(u)
        cycles = 1
        t_k = 0.0
        its = 0
        while True:
            t1 = time.perf_counter()
            out, _ = O.gcrodr(a_u, f, rhat, spec.m, spec.k, spec.tau, mv, u, None, max_cycles=cycles)
            t_k = time.perf_counter() - t1
            its = out.total
            if t_k > budget_s / len(specs) / 2 or out.converged or cycles >= 8:
                break
            cycles *= 2
        per_it = t_k / max(its, 1)
        full_its = (iters_hint or {}).get(spec.name, its)
        est = t_setup + per_it * full_its
        total_s += est
        notes.append(f"{spec.name}: setup {t_setup:.1f}s timed, {its} Arnoldi its timed "
                     f"({per_it * 1e3:.1f} ms/it) x {full_its} its -> {est:.0f}s (extrapolated)")
    return {"value": len(specs) / total_s, "unit": "solves/s", "cores": 1, "kind": "port",
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


# golden iteration totals of full solves (tests/golden/*.json), used to scale
# the CPU sample when no GPU run is available (reference arm)
_GOLDEN_ITERS = {"cfg2a": 8158, "cfg2b": 5402, "cfg4": 24, "cfg1": 19, "cfg5": 164000}


# ---------------------------------------------------------------------------
# main
# ---------------------------------------------------------------------------

def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="cfg2", choices=sorted(WORKLOADS))
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

    if args.impl == "reference":
        if rank != 0:
            return
        # the reference's own algorithm (the pinned CPU restatement) on the host
        res = cpu_sample(args.workload, iters_hint=_GOLDEN_ITERS)
        cores = len(os.sched_getaffinity(0))
        line = {"metric": METRIC, "value": res["value"], "unit": "solves/s", "n_gpus": args.gpus,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": len(specs) * 1e3 / res["value"],
                "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
                "data": "synthetic (seeded, SURVEY §8(d))", "impl": "reference",
                "config": {"workload": workload_desc},
                "cpu_baseline": {**res, "cores": cores if specs[0].batch > 1 else 1},
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
    runs = [BatchRun(s, torch, rank) if s.batch > 1 else SingleRun(s, torch) for s in specs]
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float64, device="cuda")
    stream = torch.cuda.current_stream()

    for _ in range(args.warmup):
        for r in runs:
            r.solve_device()
    torch.cuda.synchronize()
    if dist:
        dist.barrier()

    step_ms = []
    kernel_ms = []
    alg_bytes = []
    launches0 = lib.gb_launch_count()
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            _flush_l2(torch, flush)
            torch.cuda.synchronize()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for r in runs:
                r.solve_device()
            e1.record(stream)
            torch.cuda.synchronize()
            step_ms.append(e0.elapsed_time(e1))
            for r in runs:
                if isinstance(r, SingleRun):
                    kernel_ms.extend(t["ms"] for t in r.last_trace)
                    alg_bytes.extend(_alg_bytes(r.spec, [t]) for t in r.last_trace)
    launches = lib.gb_launch_count() - launches0
    total_ms = sum(step_ms)
    total_ms = max_over_ranks(total_ms, dist, "cuda")
    solves_per_step = sum(s.batch for s in specs)
    value = world * solves_per_step * args.steps / (total_ms / 1e3)

    # end-to-end through the public API from pinned host buffers
    e2e = None
    if not args.no_e2e:
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        t0 = time.perf_counter()
        for _ in range(max(1, min(args.steps, 2))):
            for r in runs:
                r.solve_e2e()
        torch.cuda.synchronize()
        e2e_s = time.perf_counter() - t0
        te = torch.tensor([e2e_s], dtype=torch.float64, device="cuda")
        if dist:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        nsteps = max(1, min(args.steps, 2))
        e2e = {"value": world * solves_per_step * nsteps / float(te.item()), "unit": "solves/s",
               "h2d_bytes_per_step": int(sum(r.h2d_bytes() for r in runs)),
               "d2h_bytes_per_step": int(sum(r.d2h_bytes() for r in runs)),
               "steps": nsteps, "timer": "wall clock around solve()/solve_batched() from pinned host buffers (device workspaces cached across calls; the first call allocates them)"}

    if rank != 0:
        if dist:
            dist.destroy_process_group()
        return

    peak, peak_kind = _peaks()
    roof = None
    if kernel_ms:
        avg_ms = statistics.mean(kernel_ms)
        avg_b = statistics.mean(alg_bytes)
        ach = avg_b / (avg_ms / 1e3) / 1e9
        roof = {"bound": "hbm", "achieved": ach, "peak": peak, "unit": "GB/s", "frac": ach / peak,
                "traffic": _ncu_traffic(args.workload), "kernel": "k_step (one refinement step, cooperative grid)",
                "peak_kind": peak_kind, "alg_bytes_per_launch": avg_b, "avg_launch_ms": avg_ms}
    else:
        ms = statistics.mean(r.last_ms for r in runs)
        n, cnt = specs[0].n, specs[0].batch
        alg = cnt * (n * n * 8 + n * 8)  # input stream
        ach = alg / (ms / 1e3) / 1e9
        roof = {"bound": "hbm", "achieved": ach, "peak": peak, "unit": "GB/s", "frac": ach / peak,
                "traffic": _ncu_traffic(args.workload), "kernel": "k_batched (one CTA per system)",
                "peak_kind": peak_kind, "note": "compute/latency bound: HBM bytes = input stream only"}
    cpu = None
    if not args.no_cpu and world == 1:
        hint = {}
        for r in runs:
            if isinstance(r, SingleRun) and r.last_report:
                hint[r.spec.name] = sum(r.last_report["inner_iters"]) or 1
        cpu = cpu_sample(args.workload, iters_hint=hint or _GOLDEN_ITERS)
    reports = [r.last_report for r in runs]
    kernels = None
    if not args.no_kernels and world == 1:
        del runs
        torch.cuda.empty_cache()
        kernels = kernel_rooflines(torch, peak, _tc_peak())
    line = {
        "metric": METRIC, "value": value, "unit": "solves/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded inputs, SURVEY §8(d); no dataset)",
        "config": {"workload": workload_desc, "l2": "flushed between steps (512 MiB write)",
                   "parallelism": f"replicas x{world}" if specs[0].batch == 1 else f"shards x{world}",
                   "time_to_solution_ms": total_ms / args.steps / len(specs) if specs[0].batch == 1 else None,
                   "verdicts": reports},
        "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "clocks": clk.summary(), "gpu_launches": int(launches),
        "kernels": kernels,
    }
    print(json.dumps(line))
    if dist:
        dist.destroy_process_group()


def _ncu_traffic(workload):
    p = os.path.join(ROOT, "profiles", f"ncu_traffic_{workload}.json")
    if os.path.exists(p):
        return json.load(open(p)).get("traffic_bytes_per_launch")
    return None


if __name__ == "__main__":
    main()

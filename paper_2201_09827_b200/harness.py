"""Sweeps over the device solver: the reference's experiment layer on top of
``solve`` (reference harness.py:74-333), for the paper's Tables 5/6 grids and
the recycle-dimension scan (Fig. 2).

Every solve goes through ``refine.solve`` (the CUDA path).  The per-problem
condition numbers in a row are problem statistics (numpy on the host, as the
reference computes them: densela.py:491-503) and are not part of any timed
solve.  ``mtx:`` problems are read by ``mtx.read_matrix_market``.
"""

from __future__ import annotations

import argparse
import json
import math
import sys
from dataclasses import dataclass, replace

import numpy as np

from . import problems
from .mtx import read_matrix_market, write_matrix_market
from .precision import Format, PrecisionTriple, set_half_flush_subnormals
from .refine import Method, RefineConfig, RefinementReport, solve

__all__ = ["ProblemRef", "SweepSpec", "format_cell", "run_sweep", "kscan", "cond_inf", "emit", "main",
           "spectrum_dump", "preconditioned_matrix", "run_sweep_ranks",
           "CSV_COLUMNS"]

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


def run_sweep_ranks(spec: SweepSpec, group=None) -> list:
    """``run_sweep`` with the problems dealt round-robin over the ranks of a
    ``torch.distributed`` group (one process per GPU) -- the multi-GPU form
    of the reference's process pool (harness.py:248-252).  Every rank returns
    the full row list, in spec order; the only collective is the final
    object gather of the rows."""
    import torch.distributed as dist

    if not spec.problems:
        raise ValueError("empty problem set")
    if not spec.methods:
        raise ValueError("empty method list")
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    mine = {i: _one_problem(spec, ref) for i, ref in enumerate(spec.problems) if i % world == rank}
    parts = [None] * world
    dist.all_gather_object(parts, mine, group=group)
    merged = {i: rows for part in parts for i, rows in part.items()}
    return [row for i in range(len(spec.problems)) for row in merged[i]]


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


def preconditioned_matrix(a, factors) -> np.ndarray:
    """U^-1 L^-1 P A in double, one device operator application per column
    (harness.py:265-273 forms the same matrix by triangular solves)."""
    from . import densela

    a = np.asarray(a, dtype=np.float64)
    n = a.shape[0]
    out = np.empty((n, n))
    e = np.zeros(n)
    for j in range(n):
        e[j] = 1.0
        out[:, j] = densela.apply_preconditioned(a, factors, e, Format.DOUBLE, Format.DOUBLE)
        e[j] = 0.0
    return out


def spectrum_dump(a, uf_format: Format, out) -> list:
    """Eigenvalues of A and of the double- and uf-preconditioned operators as
    CSV points ``set,re,im`` (harness.py:276-303); returns the set names
    written.  Factors and operator columns come from the device; the dense
    eigensolve of the n x n result (n <= 500) is the host's LAPACK, as in the
    reference (densela.py:435-457)."""
    from . import densela

    a = np.asarray(a, dtype=np.float64)
    if a.shape[0] > 500:
        raise ValueError("spectrum dump is limited to n <= 500")
    sets = []

    def add(name, mat):
        try:
            vals = np.linalg.eigvals(mat)
        except np.linalg.LinAlgError:  # eig_small's NoConvergence: the set is skipped
            return
        sets.append((name, vals[np.argsort(np.abs(vals), kind="stable")]))

    add("original", a)
    for fmt in (Format.DOUBLE, uf_format):
        f = densela.lu_factor(a, fmt)
        try:
            add(f"precond_{fmt.value}", preconditioned_matrix(a, f))
        finally:
            f.close()
    lines = ["set,re,im"] + [f"{name},{float(v.real)!r},{float(v.imag)!r}" for name, vals in sets for v in vals]
    with open(out, "w", encoding="ascii") as fh:
        fh.write("\n".join(lines) + "\n")
    return [name for name, _ in sets]


# ---------------------------------------------------------------------------
# serialisation and the command line (harness.py:335-565)
# ---------------------------------------------------------------------------

def _cell_text(v) -> str:
    if isinstance(v, bool):
        return "true" if v else "false"
    if isinstance(v, float):
        return repr(v)
    return str(v)


def _md_table(columns: list, body: list) -> list:
    return ["| " + " | ".join(columns) + " |", "|" + "|".join(" --- " for _ in columns) + "|"] + \
           ["| " + " | ".join(cells) + " |" for cells in body]


def emit(rows: list, fmt: str, path) -> None:
    """Write sweep / kscan rows as csv, markdown or json, deterministically
    (harness.py:343-381)."""
    sweep_rows = not rows or "problem_id" in rows[0]
    if fmt == "csv":
        cols = CSV_COLUMNS if sweep_rows else list(rows[0])
        text = [",".join(cols)] + [",".join(_cell_text(r.get(c, "")) for c in cols) for r in rows]
    elif fmt == "markdown":
        if rows and sweep_rows:
            cols = ["problem_id", "method", "m", "k", "result", "converged", "nbe_final"]
            body = [[str(r["problem_id"]), str(r["method"]), str(r["m"]), str(r["k"]), r.get("cell", "-"),
                     _cell_text(r["converged"]), _cell_text(r["nbe_final"])] for r in rows]
        else:
            cols = list(rows[0]) if rows else []
            body = [[_cell_text(r[c]) for c in cols] for r in rows]
        text = _md_table(cols, body)
    elif fmt == "json":
        text = [json.dumps(rows, indent=2, allow_nan=True)]
    else:
        raise ValueError(f"unknown output format {fmt!r}")
    with open(path, "w", encoding="ascii") as fh:
        fh.write("\n".join(text) + "\n")


def _parser() -> argparse.ArgumentParser:
    ap = argparse.ArgumentParser(prog="paper_2201_09827_b200.harness",
                                 description="Mixed-precision iterative refinement experiments on the GPU")
    sub = ap.add_subparsers(dest="command", required=True)

    def precision_flags(p):
        p.add_argument("--uf", default="single")
        p.add_argument("--u", default="double")
        p.add_argument("--ur", default="quad")

    def solver_flags(p):
        p.add_argument("--m", type=int, default=40)
        p.add_argument("--k", type=int, default=0)
        p.add_argument("--tau", type=float, default=None)
        p.add_argument("--imax", type=int, default=10000)
        p.add_argument("--seed", type=int, default=1)
        p.add_argument("--n", type=int, default=100)
        p.add_argument("--scale-diag", action="store_true")
        p.add_argument("--half-ftz", action="store_true")

    p = sub.add_parser("solve")
    p.add_argument("--problem", required=True)
    p.add_argument("--method", default="gmres-ir")
    precision_flags(p), solver_flags(p)
    p.add_argument("--out", default=None)
    p = sub.add_parser("sweep")
    for fam in ("prolate", "randsvd", "mtx"):
        p.add_argument(f"--{fam}", default=None)
    p.add_argument("--methods", default="gmres-ir,rgmres-ir")
    precision_flags(p), solver_flags(p)
    p.add_argument("--jobs", type=int, default=1)
    p.add_argument("--out", required=True)
    p.add_argument("--format", default="csv", choices=("csv", "markdown", "json"))
    p = sub.add_parser("spectrum")
    p.add_argument("--problem", required=True)
    p.add_argument("--uf", default="half")
    p.add_argument("--n", type=int, default=100)
    p.add_argument("--seed", type=int, default=1)
    p.add_argument("--out", required=True)
    p = sub.add_parser("kscan")
    p.add_argument("--problem", required=True)
    p.add_argument("--method", default="rgmres-ir")
    precision_flags(p), solver_flags(p)
    p.add_argument("--k-range", required=True)
    p.add_argument("--out", required=True)
    p.add_argument("--format", default="csv", choices=("csv", "markdown", "json"))
    p = sub.add_parser("gen")
    p.add_argument("--problem", required=True)
    p.add_argument("--n", type=int, default=100)
    p.add_argument("--seed", type=int, default=1)
    p.add_argument("--out", required=True)
    return ap


def _k_values(text: str) -> list:
    if ":" in text:
        lo, hi = text.split(":")
        return list(range(int(lo), int(hi) + 1))
    return [int(t) for t in text.split(",") if t.strip()]


def main(argv=None) -> int:
    """The reference CLI's solve / sweep / kscan / gen commands (harness.py:476-565)."""
    args = _parser().parse_args(argv)
    if getattr(args, "half_ftz", False):
        set_half_flush_subnormals(True)
    try:
        if args.command == "gen":
            ref = ProblemRef.parse(args.problem, n=args.n, seed=args.seed)
            a, _ = ref.materialize()
            write_matrix_market(args.out, a, comment=ref.problem_id)
            print(f"wrote {ref.problem_id} ({a.shape[0]}x{a.shape[1]}) to {args.out}")
            return 0
        if args.command == "spectrum":
            ref = ProblemRef.parse(args.problem, n=args.n, seed=args.seed)
            names = spectrum_dump(ref.materialize()[0], Format.parse(args.uf), args.out)
            print(f"wrote {len(names)} point sets to {args.out}")
            return 0
        prec = PrecisionTriple.parse(args.uf, args.u, args.ur)
        if args.command == "solve":
            ref = ProblemRef.parse(args.problem, n=args.n, seed=args.seed)
            a, b = ref.materialize()
            rep = solve(a, b, RefineConfig(precisions=prec, method=Method.parse(args.method), m=args.m, k=args.k,
                                           tau=args.tau, i_max=args.imax, scale_diag=args.scale_diag))
            tail = "" if rep.converged else f"  [{rep.divergence_reason.value}]"
            print(f"{ref.problem_id} {args.method}: {format_cell(rep)}  nbe={rep.nbe_final:.3e} "
                  f"ferr={rep.ferr_final:.3e}{tail}")
            if args.out:
                with open(args.out, "w", encoding="ascii") as fh:
                    fh.write(json.dumps(_payload(rep), indent=2) + "\n")
            return 0
        if args.command == "sweep":
            refs = []
            for fam, key in (("prolate", "alpha"), ("randsvd", "kappa2"), ("mtx", "path")):
                for tok in (getattr(args, fam) or "").split(","):
                    if tok.strip():
                        val = tok.strip() if fam == "mtx" else float(tok)
                        refs.append(ProblemRef(fam, n=args.n, seed=args.seed, **{key: val}))
            spec = SweepSpec(problems=refs, methods=[Method.parse(t) for t in args.methods.split(",")],
                             precisions=prec, m=args.m, k=args.k, tau=args.tau, i_max=args.imax,
                             seed=args.seed, scale_diag=args.scale_diag, jobs=args.jobs)
            rows = run_sweep(spec)
            emit(rows, args.format, args.out)
            for r in rows:
                print(f"{r['problem_id']:>16} {r['method']:>10}: {r['cell']}")
            return 0
        if args.command == "kscan":
            ref = ProblemRef.parse(args.problem, n=args.n, seed=args.seed)
            cfg = RefineConfig(precisions=prec, method=Method.parse(args.method), m=args.m, tau=args.tau,
                               i_max=args.imax, scale_diag=args.scale_diag)
            rows = kscan(ref, cfg, _k_values(args.k_range))
            emit(rows, args.format, args.out)
            for r in rows:
                print(f"k={r['k']:>3}  total={r['total_inner']}")
            return 0
    except (ValueError, OSError, NotImplementedError) as exc:
        print(f"error: {exc}", file=sys.stderr)
        return 2
    return 2


if __name__ == "__main__":
    sys.exit(main())

"""The sweep layer (reference harness.py:74-333) over the device solver."""

import math

import numpy as np
import pytest

from conftest import golden_json
from paper_2201_09827_b200 import harness
from paper_2201_09827_b200.precision import PrecisionTriple
from paper_2201_09827_b200.refine import Method, RefineConfig, RefinementReport


def test_problem_text_and_labels():
    p = harness.Problem.from_text("prolate:0.475")
    assert (p.family, p.value, p.n, p.label) == ("prolate", 0.475, 100, "prolate:0.475")
    r = harness.Problem.from_text("randsvd:1e12", n=64, seed=3)
    assert (r.value, r.n, r.seed, r.label) == (1e12, 64, 3, "randsvd:1e+12")
    assert harness.Problem.from_text("mtx:/data/bcsstk05.mtx").label == "bcsstk05"
    for bad in ("toeplitz:3", "prolate"):
        with pytest.raises(ValueError):
            harness.Problem.from_text(bad)
    a, b = harness.Problem.from_text("prolate:0.45", n=20).system()
    assert a.shape == (20, 20) and np.array_equal(b, np.ones(20))


def test_format_cell():
    rep = RefinementReport(converged=True, steps=3, inner_iters=[10, 4, 4], nbe_history=[], ferr_history=[])
    assert harness.format_cell(rep) == "18 (10,4,4)"
    rep.converged = False
    assert harness.format_cell(rep) == "-"


def test_cond_inf_matches_definition():
    a = harness.Problem.from_text("prolate:0.45", n=20).system()[0]
    want = np.linalg.norm(a, np.inf) * np.linalg.norm(np.linalg.inv(a), np.inf)
    assert math.isclose(harness.cond_inf(a), want, rel_tol=1e-12)
    assert harness.cond_inf(np.zeros((3, 3))) == math.inf


def test_sweep_validation_and_in_row_errors():
    spec = harness.SweepSpec([], [Method.GMRES_IR], PrecisionTriple.parse("single", "double", "quad"), m=16)
    with pytest.raises(ValueError):
        harness.run_sweep(spec)
    spec = harness.SweepSpec([harness.Problem.from_text("mtx:/nonexistent.mtx")],
                             [Method.GMRES_IR, Method.RGMRES_IR], PrecisionTriple.parse("single", "double", "quad"),
                             m=16, k=4)
    rows = harness.run_sweep(spec)
    assert [r["method"] for r in rows] == ["gmres-ir", "rgmres-ir"]
    assert [r["k"] for r in rows] == [0, 4]
    assert all(r["divergence_reason"].startswith("error:") and r["cell"] == "-" for r in rows)
    assert all(set(harness.CSV_COLUMNS) <= set(r) for r in rows)
    with pytest.raises(ValueError):
        harness.kscan(harness.Problem.from_text("prolate:0.45"),
                      RefineConfig(PrecisionTriple.parse("single", "double", "quad"), Method.RGMRES_IR, m=16, k=4),
                      [4, 16])


@pytest.mark.gpu
def test_table5_sweep_on_device(gpu):
    """Table 5 grid rows that are not chaotic (alpha >= 0.455) through run_sweep:
    same verdict and per-step iterations +-1 against the reference's golden rows."""
    rows = [r for r in golden_json("table5")["rows"] if r["alpha"] >= 0.455]
    alphas = sorted({r["alpha"] for r in rows}, reverse=True)
    spec = harness.SweepSpec([harness.Problem.from_text(f"prolate:{a}") for a in alphas],
                             [Method.GMRES_IR, Method.RGMRES_IR], PrecisionTriple.parse("single", "double", "quad"),
                             m=16, k=4, tau=1e-8)
    got = harness.run_sweep(spec)
    assert len(got) == 2 * len(alphas)
    for g in got:
        want = next(r for r in rows if f"prolate:{r['alpha']:g}" == g["problem_id"] and r["method"] == g["method"])
        assert g["converged"] == want["converged"], g
        per = [int(c) for c in g["per_step"].split(";")]
        assert len(per) == len(want["inner_iters"]), (per, want["inner_iters"])
        assert all(abs(x - y) <= 1 for x, y in zip(per, want["inner_iters"])), (per, want["inner_iters"])
        assert g["kappa_inf"] > 1.0 and g["report"].total_inner == sum(per)


@pytest.mark.gpu
def test_kscan_on_device(gpu):
    """Recycle-dimension scan (Fig. 2 shape): one row per k, totals positive
    for converged runs, -1 for divergent ones."""
    cfg = RefineConfig(PrecisionTriple.parse("single", "double", "quad"), Method.RGMRES_IR, m=16, k=4, tau=1e-8)
    rows = harness.kscan(harness.Problem.from_text("prolate:0.455"), cfg, [1, 2, 4, 8])
    assert [r["k"] for r in rows] == [1, 2, 4, 8]
    assert all(r["total_inner"] == -1 or r["total_inner"] > 0 for r in rows)
    k4 = next(r for r in golden_json("table5")["rows"] if r["alpha"] == 0.455 and r["method"] == "rgmres-ir")
    assert abs(rows[2]["total_inner"] - sum(k4["inner_iters"])) <= len(k4["inner_iters"])


def _write(tmp_path, name, text):
    p = tmp_path / name
    p.write_text(text)
    return str(p)


def test_mtx_coordinate_symmetric_and_duplicates(tmp_path):
    from paper_2201_09827_b200.mtx import read_matrix_market

    path = _write(tmp_path, "s.mtx", "%%MatrixMarket matrix coordinate real symmetric\n% c\n\n3 3 4\n"
                  "1 1 2.0\n2 1 -1.5\n3 3 4\n2 1 0.5\n")
    a = read_matrix_market(path)
    assert np.array_equal(a, np.array([[2.0, -1.0, 0.0], [-1.0, 0.0, 0.0], [0.0, 0.0, 4.0]]))


def test_mtx_array_layouts(tmp_path):
    from paper_2201_09827_b200.mtx import read_matrix_market

    gen = read_matrix_market(_write(tmp_path, "g.mtx", "%%MatrixMarket matrix array real general\n2 3\n"
                                    "1\n2\n3\n4\n5\n6\n"))
    assert np.array_equal(gen, np.array([[1.0, 3.0, 5.0], [2.0, 4.0, 6.0]]))
    sym = read_matrix_market(_write(tmp_path, "y.mtx", "%%MatrixMarket matrix array integer symmetric\n3 3\n"
                                    "1\n2\n3\n4\n5\n6\n"))
    assert np.array_equal(sym, np.array([[1.0, 2.0, 3.0], [2.0, 4.0, 5.0], [3.0, 5.0, 6.0]]))


@pytest.mark.parametrize("text,line,kind", [
    ("", 1, "parse"),
    ("%%MatrixMarket matrix coordinate complex general\n1 1 1\n1 1 1 0\n", None, "field"),
    ("%%MatrixMarket matrix coordinate real skew-symmetric\n1 1 0\n", None, "field"),
    ("%%MatrixMarket vector coordinate real general\n", 1, "parse"),
    ("%%MatrixMarket matrix coordinate real general\n", 1, "parse"),
    ("%%MatrixMarket matrix coordinate real general\n2 2\n", 2, "parse"),
    ("%%MatrixMarket matrix coordinate real general\n2 2 1\n3 1 1.0\n", 3, "parse"),
    ("%%MatrixMarket matrix coordinate real general\n2 2 1\n1 1 x\n", 3, "parse"),
    ("%%MatrixMarket matrix coordinate real general\n2 2 2\n1 1 1.0\n", 3, "parse"),
    ("%%MatrixMarket matrix array real general\n2 2\n1\n2\n3\n", 5, "parse"),
])
def test_mtx_errors(tmp_path, text, line, kind):
    from paper_2201_09827_b200.mtx import ParseError, UnsupportedField, read_matrix_market

    path = _write(tmp_path, "e.mtx", text)
    if kind == "field":
        with pytest.raises(UnsupportedField):
            read_matrix_market(path)
    else:
        with pytest.raises(ParseError) as exc:
            read_matrix_market(path)
        assert exc.value.line_no == line


def test_mtx_round_trip_and_sweep_problem(tmp_path):
    from paper_2201_09827_b200.mtx import read_matrix_market, write_matrix_market

    a = harness.Problem.from_text("prolate:0.45", n=12).system()[0]
    a[3, 5] = 0.0
    path = str(tmp_path / "p45.mtx")
    write_matrix_market(path, a, comment="prolate 0.45\nn = 12")
    assert np.array_equal(read_matrix_market(path), a)
    ref = harness.Problem.from_text(f"mtx:{path}")
    got, b = ref.system()
    assert ref.label == "p45" and np.array_equal(got, a) and np.array_equal(b, np.ones(12))


def test_spectrum_dump_size_limit(tmp_path):
    with pytest.raises(ValueError):
        harness.spectrum_dump(np.eye(501), harness.Format.HALF, tmp_path / "s.csv")


@pytest.mark.gpu
@pytest.mark.parametrize("uf", ["half", "double"])
def test_preconditioned_matrix_and_spectrum(gpu, uf, tmp_path):
    """U^-1 L^-1 P A from device operator columns equals the matrix formed by
    triangular solves on the oracle's factors (harness.py:265-273) to double
    rounding x kappa; the dump writes the three point sets (harness.py:276-303)."""
    import scipy.linalg as sl

    from oracle import cpu_gcrodr_ir as O
    from paper_2201_09827_b200 import densela

    a = harness.Problem.from_text("randsvd:1e3", n=48).system()[0]
    F = densela.lu_factor(a, harness.Format.parse(uf))
    R = O.lu_factor(a, uf)
    if uf == "half":
        assert np.array_equal(F.perm, R.perm) and np.array_equal(F.U, R.U)
    m = harness.preconditioned_matrix(a, F)
    F.close()
    want = sl.solve_triangular(F.U, sl.solve_triangular(F.L, a[F.perm], lower=True, unit_diagonal=True))
    np.testing.assert_allclose(m, want, rtol=0, atol=1e3 * 2.0 ** -52 * np.max(np.abs(want)))
    out = tmp_path / "s.csv"
    names = harness.spectrum_dump(a, harness.Format.parse(uf), out)
    assert names == ["original", "precond_double", f"precond_{uf}"] or names == ["original", "precond_double"]
    lines = out.read_text().splitlines()
    assert lines[0] == "set,re,im" and len(lines) == 1 + 48 * len(names)
    orig = np.array([complex(float(l.split(",")[1]), float(l.split(",")[2])) for l in lines[1:49]])
    ev = np.linalg.eigvals(a)
    assert np.array_equal(orig, ev[np.argsort(np.abs(ev), kind="stable")])



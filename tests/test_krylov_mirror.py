"""Host-side behaviour of the inner-solver mirrors (paper_2201_09827_b200/krylov.py):
configuration validation and defaults as in gmres.py:36-62 / gcrodr.py:68-97.  The
device path itself is covered by tests/test_gpu_kernels.py::test_inner_solver_mirrors."""

import pytest

import paper_2201_09827_b200 as gb
from paper_2201_09827_b200.precision import Format


def test_gmres_config_validation_and_cycle_cap():
    cfg = gb.GmresConfig(m=40, tau=1e-4, matvec_ctx=Format.DOUBLE, work_fmt=Format.SINGLE)
    cfg.validate(100)
    assert cfg.resolved_max_cycles(100) == 25  # ceil(10 n / m), gmres.py:51-54
    assert gb.GmresConfig(40, 1e-4, Format.DOUBLE, Format.SINGLE, max_cycles=3).resolved_max_cycles(100) == 3
    with pytest.raises(ValueError):
        gb.GmresConfig(m=101, tau=1e-4, matvec_ctx=Format.DOUBLE, work_fmt=Format.SINGLE).validate(100)
    with pytest.raises(ValueError):
        gb.GmresConfig(m=10, tau=0.0, matvec_ctx=Format.DOUBLE, work_fmt=Format.SINGLE).validate(100)


def test_gcrodr_config_validation():
    ok = gb.GcrodrConfig(m=50, k=10, tau=1e-6, matvec_ctx=Format.QUAD, work_fmt=Format.DOUBLE)
    ok.validate(1024)
    assert ok.resolved_max_cycles(1024) == 205  # config 2's cap
    for m, k in ((5, 5), (5, 0), (2000, 10)):
        with pytest.raises(ValueError):
            gb.GcrodrConfig(m=m, k=k, tau=1e-6, matvec_ctx=Format.QUAD, work_fmt=Format.DOUBLE).validate(1024)
    with pytest.raises(ValueError):
        gb.GcrodrConfig(m=50, k=10, tau=-1.0, matvec_ctx=Format.QUAD, work_fmt=Format.DOUBLE).validate(1024)


def test_outcome_totals_and_exports():
    out = gb.GmresOutcome(solution=None, iterations_per_cycle=[50, 40, 40], converged=False)
    assert out.total_iterations == 130 and out.stagnated is False and out.cycle_diagnostics is None
    for name in ("gmres_solve", "gcrodr_solve", "check_convergence", "RecycleSpace", "solve_batched"):
        assert hasattr(gb, name)

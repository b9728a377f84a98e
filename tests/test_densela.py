"""The densela mirror (densela.py:58-361) over the device context."""

import numpy as np
import pytest

from conftest import golden_npz
from oracle import cpu_gcrodr_ir as O
from paper_2201_09827_b200 import densela
from paper_2201_09827_b200.precision import Format


def test_argument_errors_before_any_device_work():
    with pytest.raises(ValueError):
        densela.lu_factor(np.zeros((3, 4)), Format.HALF)
    with pytest.raises(ValueError):
        densela.residual(np.zeros((3, 4)), np.zeros(3), np.zeros(3), Format.DOUBLE)
    assert densela._default_u(Format.HALF, np.array([[0.1]])) is Format.DOUBLE
    assert densela._default_u(Format.HALF, np.array([[0.5]])) is Format.SINGLE
    assert densela._default_u(Format.SINGLE) is Format.DOUBLE
    e = densela.ExactZeroPivot(3)
    assert e.index == 3 and "column 3" in str(e)


@pytest.mark.gpu
@pytest.mark.parametrize("tag,uf,u", [("hs", "half", "single"), ("hd", "half", "double")])
def test_densela_mirror_matches_oracle(gpu, tag, uf, u):
    """lu_factor / lu_solve / apply_preconditioned / precond_rhs / residual
    through the mirror: fp16 factors and x0 bit-identical to the reference's
    goldens, operator / precond_rhs within one rounding of u, residuals as in
    test_gpu_kernels."""
    k = golden_npz("kernels")
    a = O.rnd(k["a"], u)
    b = k["b"]
    fu, f2 = Format.parse(u), {"single": Format.DOUBLE, "double": Format.QUAD}[u]
    F = densela.lu_factor(a, Format.HALF)
    ref = O.lu_factor(a, "half")
    assert np.array_equal(F.perm, ref.perm)
    assert np.array_equal(F.L, ref.L) and np.array_equal(F.U, ref.U)
    x0 = densela.lu_solve(F, b, Format.HALF, store_fmt=fu)
    assert np.array_equal(x0, k[f"{tag}_x0"])
    w = densela.apply_preconditioned(a, F, k[f"{tag}_v"], f2, fu)
    p = densela.precond_rhs(F, k[f"{tag}_v"], f2, fu)
    tol = 2.0 ** -23 if u == "single" else 2.0 ** -51
    for got, want in ((w, k[f"{tag}_op"]), (p, k[f"{tag}_prhs"])):
        np.testing.assert_allclose(got, want, rtol=tol, atol=tol * np.max(np.abs(want)))
    rq = densela.residual(a, k[f"{tag}_x"], O.rnd(b, u), Format.QUAD)  # b held at u, as the solve does
    np.testing.assert_allclose(rq, k[f"{tag}_res_q"], rtol=0, atol=1e-30 + 2 ** -52 * np.max(np.abs(rq)))
    F.close()


@pytest.mark.gpu
def test_densela_zero_pivot(gpu):
    a = np.eye(4)
    a[:, 2] = 0.0
    with pytest.raises(densela.ExactZeroPivot) as exc:
        densela.lu_factor(a, Format.HALF)
    assert exc.value.index == 2

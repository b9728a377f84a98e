"""Seeded host-side problem construction for the five benchmark configurations.

Input generation is not on the GPU hot path (matgen is OUT OF
SCOPE for the device); it is restated here so that the oracle, the CUDA path
and the bench all see bit-identical inputs without importing the reference.

* randsvd follows ``irkit.matgen.gen_randsvd`` (reference
  ``pkg/src/irkit/matgen.py:70-92``): Philox(seed) stream, two Haar factors
  from sign-fixed QR of Gaussian matrices, geometric singular values
  ``kappa^(-(i)/(n-1))``, ``A = (P * sigma) @ Q^T``.
* prolate follows ``matgen.py:95-103``: symmetric Toeplitz, first column
  ``2*alpha, sin(2*pi*alpha*d)/(pi*d)``.
* right-hand sides: the reference harness only has b = ones
  (``harness.py:101``); SURVEY.md §8(d) fixes our convention as a draw from
  ``Generator(Philox(seed).jumped())`` so it is disjoint from A's stream.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

__all__ = [
    "randsvd",
    "prolate",
    "rhs_normal",
    "rhs_uniform",
    "rhs_ones",
    "ConfigSpec",
    "CONFIGS",
    "config_problem",
]


def _haar(rng: np.random.Generator, n: int) -> np.ndarray:
    gauss = rng.standard_normal((n, n))
    q, r = np.linalg.qr(gauss)
    d = np.sign(np.diagonal(r)).copy()
    d[d == 0.0] = 1.0
    return q * d[None, :]


def randsvd(n: int, kappa2: float, seed: int = 1) -> np.ndarray:
    """Dense matrix with 2-norm condition kappa2 and geometric singular values."""
    if n < 2 or not kappa2 > 1.0:
        raise ValueError("randsvd needs n >= 2 and kappa2 > 1")
    rng = np.random.Generator(np.random.Philox(seed))
    sig = kappa2 ** (-np.arange(n) / (n - 1))
    left = _haar(rng, n)
    right = _haar(rng, n)
    return (left * sig[None, :]) @ right.T


def prolate(n: int, alpha: float) -> np.ndarray:
    """Symmetric Toeplitz prolate matrix, 0 < alpha < 0.5."""
    if n < 1 or not (0.0 < alpha < 0.5):
        raise ValueError("prolate needs n >= 1 and 0 < alpha < 0.5")
    col = np.empty(n)
    col[0] = 2.0 * alpha
    d = np.arange(1, n)
    col[1:] = np.sin(2.0 * math.pi * alpha * d) / (math.pi * d)
    i = np.arange(n)
    return col[np.abs(i[:, None] - i[None, :])]


def _rhs_rng(seed: int) -> np.random.Generator:
    return np.random.Generator(np.random.Philox(seed).jumped())


def rhs_normal(n: int, seed: int = 1) -> np.ndarray:
    return _rhs_rng(seed).standard_normal(n)


def rhs_uniform(n: int, seed: int = 1) -> np.ndarray:
    return _rhs_rng(seed).uniform(-1.0, 1.0, n)


def rhs_ones(n: int) -> np.ndarray:
    return np.ones(n)


@dataclass(frozen=True)
class ConfigSpec:
    """One BASELINE.json configuration."""

    name: str
    n: int
    kind: str  # "randsvd" | "prolate"
    param: float  # kappa2 or alpha
    precisions: tuple[str, str, str]
    m: int
    k: int
    tau: float
    i_max: int
    rhs: str = "normal"
    batch: int = 1
    extra_precisions: tuple = field(default_factory=tuple)


CONFIGS = {
    "cfg1": ConfigSpec("cfg1", 100, "randsvd", 1e4, ("half", "single", "double"), 100, 5, 1e-4, 10),
    "cfg2a": ConfigSpec("cfg2a", 1024, "prolate", 0.45, ("single", "double", "double"), 50, 10, 1e-6, 10),
    "cfg2b": ConfigSpec("cfg2b", 1024, "prolate", 0.45, ("half", "double", "double"), 50, 10, 1e-6, 10),
    "cfg3": ConfigSpec("cfg3", 128, "randsvd", 1e3, ("half", "single", "double"), 32, 8, 1e-4, 10,
                       rhs="uniform", batch=4096),
    "cfg4": ConfigSpec("cfg4", 8192, "randsvd", 1e6, ("single", "double", "quad"), 100, 20, 1e-10, 10),
    "cfg5": ConfigSpec("cfg5", 16384, "randsvd", 1e8, ("half", "single", "double"), 200, 30, 1e-4, 20),
}


def config_problem(spec: ConfigSpec, index: int = 0, n: int | None = None):
    """(A, b) for system ``index`` of a configuration (n may be overridden
    to build the smaller analogues used for parity)."""
    nn = spec.n if n is None else n
    seed = 1 + index
    if spec.kind == "randsvd":
        a = randsvd(nn, spec.param, seed)
    else:
        a = prolate(nn, spec.param)
    b = rhs_uniform(nn, seed) if spec.rhs == "uniform" else rhs_normal(nn, seed)
    return a, b

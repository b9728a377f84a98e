"""B200-native GCRO-DR-IR: mixed-precision GMRES-based iterative refinement
with Krylov subspace recycling (arXiv 2201.09827), drop-in for the reference
package's solver entry points (irkit.refine.solve / gmres_ir / rgmres_ir / sir).

The solver path is hand-written sm_100a CUDA behind a C ABI
(include/gcrodr_b200.h, libgcrodr_b200.so); this package is the host side.
There is no CPU fallback.
"""

from .precision import (Format, PrecisionTriple, half_flushes_subnormals, set_half_flush_subnormals,
                        squared_format)
from . import densela, mtx
from .batched import solve_batched
from .krylov import GcrodrConfig, GmresConfig, GmresOutcome, RecycleSpace, gcrodr_solve, gmres_solve
from .refine import (
    ConvergenceDecision,
    DivergenceReason,
    Method,
    RefineConfig,
    RefinementReport,
    check_convergence,
    classify,
    gmres_ir,
    rgmres_ir,
    sir,
    solve,
)

__version__ = "0.1.0"

__all__ = [
    "Format",
    "PrecisionTriple",
    "squared_format",
    "set_half_flush_subnormals",
    "half_flushes_subnormals",
    "Method",
    "DivergenceReason",
    "RefineConfig",
    "RefinementReport",
    "ConvergenceDecision",
    "classify",
    "check_convergence",
    "GmresConfig",
    "GmresOutcome",
    "gmres_solve",
    "GcrodrConfig",
    "RecycleSpace",
    "gcrodr_solve",
    "solve_batched",
    "solve",
    "sir",
    "gmres_ir",
    "rgmres_ir",
]

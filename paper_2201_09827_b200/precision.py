"""Precision descriptors of the drop-in API (reference precision.py:54-199).

Only the host-side descriptors live here; every arithmetic kernel is CUDA in
``csrc/`` (formats become template parameters there).
"""

from __future__ import annotations

import enum
from dataclasses import dataclass

from . import _lib

__all__ = ["Format", "PrecisionTriple", "squared_format", "set_half_flush_subnormals",
           "half_flushes_subnormals"]

# Process-wide half-precision subnormal handling (precision.py:111-128).  The
# device kernels round fp16 with subnormals kept (the reference default);
# solves that involve the half format refuse to run while flushing is on
# (refine.make_options raises NotImplementedError) rather than silently
# computing the non-flushed result.
_HALF_FLUSH_TO_ZERO = False


class Format(enum.Enum):
    """A floating-point format of a mixed-precision solve (precision.py:54-84)."""

    HALF = "half"
    SINGLE = "single"
    DOUBLE = "double"
    QUAD = "quad"

    @property
    def unit_roundoff(self) -> float:
        return _UNIT_ROUNDOFF[self]

    @property
    def significand_bits(self) -> int:
        return {"half": 11, "single": 24, "double": 53, "quad": 106}[self.value]

    @property
    def code(self) -> int:
        """C-ABI format code (gcrodr_b200.h GB_HALF..GB_QUAD)."""
        return {"half": _lib.HALF, "single": _lib.SINGLE, "double": _lib.DOUBLE, "quad": _lib.QUAD}[self.value]

    @classmethod
    def parse(cls, name: str) -> "Format":
        try:
            return cls(name.strip().lower())
        except ValueError:
            raise ValueError(f"unknown format {name!r}; expected one of {[f.value for f in cls]}") from None


_UNIT_ROUNDOFF = {
    Format.HALF: 2.0 ** -11,
    Format.SINGLE: 2.0 ** -24,
    Format.DOUBLE: 2.0 ** -53,
    Format.QUAD: 2.0 ** -105,  # double-double, as in the reference
}


def squared_format(fmt: Format) -> Format:
    """Format of "precision u^2" operator applications (precision.py:169-175)."""
    if fmt is Format.HALF:
        return Format.SINGLE
    if fmt is Format.SINGLE:
        return Format.DOUBLE
    return Format.QUAD


@dataclass(frozen=True)
class PrecisionTriple:
    """(u_f, u, u_r) with u_f >= u >= u_r in unit roundoff (precision.py:178-199)."""

    uf: Format
    u: Format
    ur: Format

    def __post_init__(self) -> None:
        if not (self.uf.unit_roundoff >= self.u.unit_roundoff >= self.ur.unit_roundoff):
            raise ValueError(
                "precisions must satisfy uf >= u >= ur in unit roundoff, got "
                f"({self.uf.value}, {self.u.value}, {self.ur.value})")

    @classmethod
    def parse(cls, uf: str, u: str, ur: str) -> "PrecisionTriple":
        return cls(Format.parse(uf), Format.parse(u), Format.parse(ur))


def set_half_flush_subnormals(enabled: bool) -> bool:
    """Toggle flush-to-zero for the half format; returns the old setting
    (precision.py:118-123)."""
    global _HALF_FLUSH_TO_ZERO
    old = _HALF_FLUSH_TO_ZERO
    _HALF_FLUSH_TO_ZERO = bool(enabled)
    return old


def half_flushes_subnormals() -> bool:
    """precision.py:126-127."""
    return _HALF_FLUSH_TO_ZERO

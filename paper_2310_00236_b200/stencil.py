"""Stencil taps (reference: stencil.py:34-62).

The staggered derivative itself runs in the sm_100a kernels (fixed fold order
fl(fl(fl(c2 t1)+fl(c3 t2)) + fl(fl(c1 t0)+fl(c4 t3))), stencil.py:72-79); the
host only materialises the dx-scaled taps, each rounded once from the exact
rational tap/dx into the stencil precision.
"""

from __future__ import annotations

from dataclasses import dataclass
from fractions import Fraction

from .precision import Precision, as_precision, round_fraction

TAPS = (Fraction(1, 24), Fraction(-9, 8), Fraction(9, 8), Fraction(-1, 24))
# second order (extension): the inner pair alone, +-1 at offsets -+1/2
TAPS2 = (Fraction(0), Fraction(-1), Fraction(1), Fraction(0))


@dataclass(frozen=True)
class StencilSpec:
    precision: Precision
    dx: float
    coefficients: tuple
    order: int = 4

    @classmethod
    def make(cls, precision, dx: float, order: int = 4) -> "StencilSpec":
        if not dx > 0.0:
            raise ValueError("dx must be positive")
        if order not in (2, 4):
            raise ValueError("order must be 2 or 4")
        p = as_precision(precision)
        base = TAPS if order == 4 else TAPS2
        coeffs = tuple(round_fraction(p, t / Fraction(dx)) for t in base)
        return cls(p, dx, coeffs, order)

    def __post_init__(self):
        c1, c2, c3, c4 = self.coefficients
        if not (c1 == -c4 and c2 == -c3):
            raise ValueError("stencil coefficients must be antisymmetric")

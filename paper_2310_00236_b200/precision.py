"""Precision modes and host-side rounding (reference: precision.py).

Only what the hot path needs on the host: the three IEEE formats, the storage
dtypes, single RNE rounding of binary64 scalars (``round_to``,
precision.py:108-118) and exact-rational rounding for stencil taps
(``round_fraction``, precision.py:161-192).  All array arithmetic happens in
the sm_100a kernels.
"""

from __future__ import annotations

import enum
import math
from dataclasses import dataclass
from fractions import Fraction

import numpy as np


class Precision(enum.Enum):
    FP16 = "fp16"
    FP32 = "fp32"
    FP64 = "fp64"

    def __str__(self):
        return self.value


@dataclass(frozen=True)
class FloatFormat:
    name: str
    exponent_bits: int
    fraction_bits: int

    @property
    def significand_bits(self) -> int:
        return self.fraction_bits + 1

    @property
    def emax(self) -> int:
        return (1 << (self.exponent_bits - 1)) - 1

    @property
    def emin(self) -> int:
        return 1 - self.emax

    @property
    def unit_roundoff(self) -> float:
        return math.ldexp(1.0, -self.significand_bits)

    @property
    def max_finite(self) -> float:
        return math.ldexp(2.0 - math.ldexp(1.0, -self.fraction_bits), self.emax)

    @property
    def min_positive_normal(self) -> float:
        return math.ldexp(1.0, self.emin)

    @property
    def min_positive_subnormal(self) -> float:
        return math.ldexp(1.0, self.emin - self.fraction_bits)


FORMATS = {
    Precision.FP16: FloatFormat("fp16", 5, 10),
    Precision.FP32: FloatFormat("fp32", 8, 23),
    Precision.FP64: FloatFormat("fp64", 11, 52),
}

DTYPES = {
    Precision.FP16: np.dtype(np.float16),
    Precision.FP32: np.dtype(np.float32),
    Precision.FP64: np.dtype(np.float64),
}

LANE_BITS = {Precision.FP16: 16, Precision.FP32: 32, Precision.FP64: 64}


def as_precision(p) -> Precision:
    """Accept this package's Precision or any enum/str with the same value
    (so reference ``halfwave.Precision`` members work as a drop-in)."""
    if isinstance(p, Precision):
        return p
    return Precision(getattr(p, "value", p))


def round_to(precision, x: float) -> float:
    """One RNE rounding of a binary64 value into the format (signed inf on overflow)."""
    precision = as_precision(precision)
    if precision is Precision.FP64:
        return float(x)
    with np.errstate(over="ignore"):
        return float(DTYPES[precision].type(x))


def round_fraction(precision, value: Fraction) -> float:
    """Round an exact rational once into the format, ties to even.

    Integer arithmetic on numerator/denominator: pick the quantum 2^q of the
    value's binade (clamped at the subnormal floor), split value/2^q into an
    integer part and remainder, round half to even, then rebuild the float.
    """
    fmt = FORMATS[as_precision(precision)]
    num, den = value.numerator, value.denominator
    if num == 0:
        return 0.0
    neg = num < 0
    num = abs(num)
    # exponent e with 2^e <= num/den < 2^(e+1)
    e = num.bit_length() - den.bit_length()
    if (num << max(0, -e)) < (den << max(0, e)):
        e -= 1
    q = max(e, fmt.emin) - fmt.fraction_bits
    scaled_num, scaled_den = (num, den << q) if q >= 0 else (num << -q, den)
    k, rem = divmod(scaled_num, scaled_den)
    twice = 2 * rem
    if twice > scaled_den or (twice == scaled_den and k & 1):
        k += 1
    if k == 0:
        mag = 0.0
    elif k.bit_length() - 1 + q > fmt.emax:
        mag = math.inf
    else:
        mag = math.ldexp(float(k), q)
    return -mag if neg else mag

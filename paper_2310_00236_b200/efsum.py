"""Compensated-update variants (reference: efsum.py:30-37).

The error-free transformations themselves (sum_3op / sum_6op / vec_accumulate,
efsum.py:53-121) run inside the sm_100a kernels (csrc/hw_common.cuh `finish`).
"""

from __future__ import annotations

import enum


class Variant(enum.Enum):
    OP3 = "op3"
    OP6 = "op6"

    def __str__(self):
        return self.value


def variant_code(variant) -> int:
    """None -> naive (0); OP3 -> 3; OP6 -> 6.  Accepts reference Variant members."""
    if variant is None:
        return 0
    v = getattr(variant, "value", variant)
    if v == "op3":
        return 3
    if v == "op6":
        return 6
    raise ValueError(f"unknown compensated variant {variant!r}")

"""Run outputs and post-run analytics (reference: diagnostics.py).

The energy functionals themselves (diagnostics.py:76-162) run on the device,
fused into the pressure / stress kernels; this module holds the result types
and the small host-side comparisons (compare_traces, energy_drift).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np


class RangeFailureError(RuntimeError):
    """A field left the representable range (inf or NaN) after a step."""

    def __init__(self, step: int, field_name: str):
        super().__init__(f"non-finite value in field {field_name!r} after step {step}")
        self.step = step
        self.field_name = field_name


@dataclass
class TraceSeries:
    field: str
    ix: int
    iy: int
    samples: np.ndarray
    iz: int | None = None


@dataclass
class EnergySeries:
    times: np.ndarray
    values: np.ndarray

    def __post_init__(self):
        if len(self.times) != len(self.values):
            raise ValueError("times and values must have equal length")
        if np.any(np.diff(self.times) <= 0.0):
            raise ValueError("sample times must be strictly increasing")

    @property
    def flags(self) -> np.ndarray:
        return ~np.isfinite(self.values)


@dataclass
class RunOutput:
    traces: list
    energy: EnergySeries
    flags: dict = field(default_factory=dict)


def _samples(trace) -> np.ndarray:
    return np.asarray(getattr(trace, "samples", trace), dtype=np.float64)


def compare_traces(a, b) -> dict:
    """l2_rel, linf_rel and zero-lag correlation of trace a against reference b."""
    a, b = _samples(a), _samples(b)
    if a.shape != b.shape:
        raise ValueError(f"trace length mismatch: {a.shape} vs {b.shape}")
    diff = a - b
    nb, na = float(np.linalg.norm(b)), float(np.linalg.norm(a))
    peak = float(np.max(np.abs(b))) if b.size else 0.0
    linf = float(np.max(np.abs(diff))) if diff.size else 0.0

    def rel(x, scale):
        return x / scale if scale > 0.0 else (0.0 if x == 0.0 else float("inf"))

    corr = float(np.dot(a, b)) / (na * nb) if na > 0.0 and nb > 0.0 else 0.0
    return {"l2_rel": rel(float(np.linalg.norm(diff)), nb), "linf_rel": rel(linf, peak), "lag0_correlation": corr}


def energy_drift(series: EnergySeries, t_source_off: float) -> dict:
    """Max relative deviation from the mean and least-squares slope after t_source_off."""
    keep = series.times > t_source_off
    if not keep.any():
        raise ValueError(f"no energy samples after t_source_off={t_source_off!r}")
    t, e = series.times[keep], series.values[keep]
    mean = float(np.mean(e))
    dev = float(np.max(np.abs(e - mean)))
    rel_dev = dev / abs(mean) if mean != 0.0 else (0.0 if dev == 0.0 else float("inf"))
    if len(t) < 2:
        slope = 0.0
    else:
        tc = t - t.mean()
        slope = float(np.dot(tc, e) / np.dot(tc, tc))
    return {"rel_deviation": rel_dev, "trend_slope": slope}

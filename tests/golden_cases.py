"""Rebuild the golden cases (tests/golden/*.npz, made by make_golden.py from the
unmodified reference) through this package's reference-mirroring host API."""

from __future__ import annotations

import json
from pathlib import Path

import numpy as np

import paper_2310_00236_b200 as hw

GOLDEN = Path(__file__).resolve().parent / "golden"
PREC = {"fp16": hw.Precision.FP16, "fp32": hw.Precision.FP32, "fp64": hw.Precision.FP64}
VARIANT = {"naive": None, "op3": hw.Variant.OP3, "op6": hw.Variant.OP6}


def names():
    """Reference-run cases (make_golden.py); rigid_*.npz are the mirrored-domain fixtures
    of make_rigid_golden.py, read by tests/test_rigid.py and tests/test_gpu_rigid.py."""
    return sorted(p.stem for p in GOLDEN.glob("*.npz") if not p.stem.startswith("rigid_"))


class Case:
    def __init__(self, name):
        self.name = name
        z = np.load(GOLDEN / f"{name}.npz")
        self.z = z
        self.d = json.loads(str(z["desc"]))
        self.variant = VARIANT[self.d["variant"]]

    def solver(self):
        d, z = self.d, self.z
        bc = hw.Boundary.FREE_SURFACE if d["bc"] == "free-surface" else hw.Boundary.PERIODIC
        grid = hw.GridSpec(d["nx"], d["ny"], d["dx"], d["dt"], d["nt"], bc_y=bc)
        kind = hw.MediumKind.ACOUSTIC if d["eq"] == "acoustic" else hw.MediumKind.ELASTIC
        medium = hw.Medium(kind, d["nx"], d["ny"], {k: z[f"plane_{k}"] for k in d["plane_names"]})
        src = None
        if d["source"]:
            s = d["source"]
            sk = hw.SourceKind.PRESSURE_POINT if d["eq"] == "acoustic" else hw.SourceKind.VY_POINT
            src = hw.SourceSpec(sk, s["ix"], s["iy"], hw.RickerSpec(s["f_center"], s.get("delay"), s["amplitude"]))
        cls = hw.AcousticSolver if d["eq"] == "acoustic" else hw.ElasticSolver
        return cls(grid, medium, src, stencil_precision=PREC[d["stencil"]],
                   update_precision=PREC[d["update"]], receivers=tuple(tuple(r) for r in d["receivers"]),
                   energy_every=d["energy_every"])

    def initial_state(self, solver):
        st = solver.new_state()
        for n in solver.FIELDS:
            getattr(st, n).values = self.z[f"init_{n}"].copy()
        return st

    @property
    def fields(self):
        return (["p", "vx", "vy", "rp", "rvx", "rvy"] if self.d["eq"] == "acoustic" else
                ["vx", "vy", "sxx", "syy", "sxy", "rvx", "rvy", "rsxx", "rsyy", "rsxy"])


def bits(a: np.ndarray) -> np.ndarray:
    a = np.ascontiguousarray(a)
    return a.view({2: np.uint16, 4: np.uint32, 8: np.uint64}[a.dtype.itemsize])


def assert_same_bits(got: np.ndarray, want: np.ndarray, what: str):
    """Bit-exact, except that NaN payloads/signs may differ (numpy vs IEEE hardware NaNs)."""
    got, want = np.asarray(got), np.asarray(want)
    assert got.shape == want.shape, f"{what}: shape {got.shape} vs {want.shape}"
    assert got.dtype == want.dtype, f"{what}: dtype {got.dtype} vs {want.dtype}"
    gn, wn = np.isnan(got), np.isnan(want)
    assert np.array_equal(gn, wn), f"{what}: NaN positions differ"
    diff = (bits(got) != bits(want)) & ~gn
    if diff.any():
        idx = np.argwhere(diff)[0]
        raise AssertionError(
            f"{what}: {int(diff.sum())} of {got.size} elements differ; first at {tuple(idx)}: "
            f"{got[tuple(idx)]!r} vs {want[tuple(idx)]!r}")

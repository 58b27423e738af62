"""BASELINE config 1's reference-native twins (tests/golden/twin/, made by
make_twin_golden.py from the unmodified reference): 256^2, rho = kappa = 1, 4th-order
periodic, Gaussian bump + seeded noise, 2000 steps, energy every step, at CFL 0.5 / 0.05 /
0.0125.  Rebuilt here through this package's reference-mirroring host API."""

from __future__ import annotations

import hashlib
import json
from pathlib import Path

import numpy as np

import paper_2310_00236_b200 as hw

TWIN = Path(__file__).resolve().parent / "golden" / "twin"
FIELDS = ("p", "vx", "vy", "rp", "rvx", "rvy")


def names():
    return sorted(p.stem for p in TWIN.glob("twin_cfl*.npz"))


class Twin:
    def __init__(self, name):
        self.z = np.load(TWIN / f"{name}.npz")
        self.d = json.loads(str(self.z["desc"]))
        self.variant = None if self.d["variant"] == "naive" else hw.Variant.OP3

    def solver(self):
        d = self.d
        prec = hw.Precision.FP16 if d["precision"] == "fp16" else hw.Precision.FP64
        grid = hw.GridSpec(d["n"], d["n"], d["dx"], d["dt"], d["nt"])
        med = hw.build_homogeneous_acoustic(d["n"], d["n"], 1.0, 1.0)
        return hw.AcousticSolver(grid, med, None, stencil_precision=prec, update_precision=prec,
                                 receivers=tuple(tuple(r) for r in d["receivers"]), energy_every=1)

    def initial_state(self, solver):
        st = solver.new_state()
        p0 = np.load(TWIN / "twin_init.npz")["p0_fp64"]
        st.p.values = p0.astype(st.p.values.dtype)  # a single cast to the update lane
        return st

    def check(self, fields, traces, e_times, e_vals):
        """fields: the six final arrays in FIELDS order (update-lane dtype)."""
        for n, a in zip(FIELDS, fields):
            a = np.ascontiguousarray(a)
            assert str(a.dtype) == self.d["dtype"], n
            got = hashlib.sha256(a.tobytes()).hexdigest()
            assert got == self.d["sha256"][n], f"{self.d['name']}: final {n} differs from the reference's bits"
        np.testing.assert_array_equal(np.asarray(traces).reshape(self.z["traces"].shape), self.z["traces"])
        np.testing.assert_array_equal(e_times, self.z["e_times"])
        np.testing.assert_allclose(e_vals, self.z["e_vals"], rtol=1e-12, atol=0)


def relative_change(e):
    return (e[-1] - e[0]) / e[0]

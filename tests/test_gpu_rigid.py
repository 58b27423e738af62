"""Rigid (p = 0) walls on the B200: the product runs the mirrored periodic problem
(paper_2310_00236_b200/rigid.py) through the unchanged kernels; it must reproduce the
reference-made goldens (tests/golden/rigid_*.npz) and the direct image formulation
(oracle/rigid.py) bit for bit, energy within 1e-12."""

import json
from pathlib import Path

import numpy as np
import pytest

import oracle.rigid as orig
import paper_2310_00236_b200 as hw
from golden_cases import assert_same_bits

pytestmark = pytest.mark.gpu

GOLD = sorted((Path(__file__).resolve().parent / "golden").glob("rigid_*.npz"))
FIELDS = ("p", "vx", "vy", "rp", "rvx", "rvy")
VAR = {"naive": None, "op3": hw.Variant.OP3, "op6": hw.Variant.OP6}


@pytest.mark.parametrize("path", GOLD, ids=[p.stem for p in GOLD])
def test_gpu_rigid_matches_reference_mirror(path):
    z = np.load(path)
    d = json.loads(str(z["desc"]))
    g = hw.GridSpec(d["nx"], d["ny"], d["dx"], d["dt"], d["nt"], bc_x=hw.Boundary.RIGID, bc_y=hw.Boundary.RIGID)
    med = hw.Medium(hw.MediumKind.ACOUSTIC, d["nx"], d["ny"], {k: z[f"canon_{k}"] for k in ("rho_x", "rho_y", "beta")})
    s = hw.AcousticSolver(g, med, stencil_precision=hw.Precision.FP16, receivers=[tuple(r) for r in d["receivers"]],
                          energy_every=d["every"])
    st = s.new_state()
    for k in FIELDS:
        getattr(st, k).values = z[f"init_{k}"]
    out = s.run(VAR[d["variant"]], st)
    for k in FIELDS:
        assert_same_bits(getattr(st, k).values, z[f"out_{k}"], k)
    np.testing.assert_array_equal(np.array([t.samples for t in out.traces]).reshape(z["traces"].shape), z["traces"])
    np.testing.assert_allclose(out.energy.values, z["e_vals"], rtol=1e-12)


@pytest.mark.parametrize("variant,vname", [(None, None), (hw.Variant.OP3, "op3")])
def test_gpu_rigid_config1_box_vs_direct_oracle(variant, vname):
    """BASELINE config 1 shape: 256^2 cells, h = 1/256, 2nd order, dt = 0.5 h, rigid p = 0
    walls, Gaussian bump + seeded U(-1e-3, 1e-3) noise, v = 0, energy every step."""
    n, nt = 256, 40
    h = 1.0 / n
    g = hw.GridSpec(n, n, h, 0.5 * h, nt, bc_x=hw.Boundary.RIGID, bc_y=hw.Boundary.RIGID, order=2)
    med = hw.build_homogeneous_acoustic(n, n, 1.0, 1.0)
    s = hw.AcousticSolver(g, med, stencil_precision=hw.Precision.FP16, energy_every=1, receivers=((128, 128), (1, 255)))
    st = s.new_state()
    yy, xx = np.mgrid[0:n + 1, 0:n + 1] * h
    p = np.exp(-((xx - 0.5) ** 2 + (yy - 0.5) ** 2) / 0.01) + np.random.default_rng(1).uniform(-1e-3, 1e-3, xx.shape)
    p[0, :] = p[-1, :] = p[:, 0] = p[:, -1] = 0.0
    st.p.values = p.astype(np.float16)
    init = {k: getattr(st, k).values.copy() for k in FIELDS}
    out = s.run(variant, st)
    assert s.kernel_path() == "small2d"  # the 512^2 mirrored domain runs the persistent small-grid kernel
    bp = {"rho_x": np.ones((n + 1, n)), "rho_y": np.ones((n, n + 1)), "beta": np.ones((n + 1, n + 1))}
    taps = hw.StencilSpec.make(hw.Precision.FP16, h, 2).coefficients
    ref, e, tr = orig.run(init, {k: v.astype(np.float16) for k, v in bp.items()}, bp, taps, h, 0.5 * h, nt,
                          variant=vname, order=2, every=1, receivers=[(128, 128), (1, 255)])
    for k in FIELDS:
        assert_same_bits(getattr(st, k).values, ref[k], k)
    np.testing.assert_array_equal(np.array([t.samples for t in out.traces]), tr)
    np.testing.assert_allclose(out.energy.values, e, rtol=1e-12)


def test_gpu_energy_drift_naive_vs_compensated():
    """The paper's effect: on the config-1 box at CFL 0.05, binary16 naive
    updates lose energy while the compensated (op3) update holds it -- the B200 drift
    histories equal the oracle's."""
    n, nt = 128, 1500
    h = 1.0 / n
    g = hw.GridSpec(n, n, h, float(np.float16(0.05 * h)), nt, bc_x=hw.Boundary.RIGID, bc_y=hw.Boundary.RIGID, order=2)
    med = hw.build_homogeneous_acoustic(n, n, 1.0, 1.0)
    yy, xx = np.mgrid[0:n + 1, 0:n + 1] * h
    p = np.exp(-((xx - 0.5) ** 2 + (yy - 0.5) ** 2) / 0.01) + np.random.default_rng(0).uniform(-1e-3, 1e-3, xx.shape)
    p[0, :] = p[-1, :] = p[:, 0] = p[:, -1] = 0.0
    drift = {}
    for variant, vname in ((None, None), (hw.Variant.OP3, "op3")):
        s = hw.AcousticSolver(g, med, stencil_precision=hw.Precision.FP16, energy_every=50)
        st = s.new_state()
        st.p.values = p.astype(np.float16)
        init = {k: getattr(st, k).values.copy() for k in FIELDS}
        e = s.run(variant, st).energy.values
        bp = {"rho_x": np.ones((n + 1, n)), "rho_y": np.ones((n, n + 1)), "beta": np.ones((n + 1, n + 1))}
        taps = hw.StencilSpec.make(hw.Precision.FP16, h, 2).coefficients
        _, e_ref, _ = orig.run(init, {k: v.astype(np.float16) for k, v in bp.items()}, bp, taps, h, g.dt, nt,
                               variant=vname, order=2, every=50)
        np.testing.assert_allclose(e, e_ref, rtol=1e-12)
        drift[vname] = (e[-1] - e[0]) / e[0]
    assert abs(drift[None]) > 20 * abs(drift["op3"]), drift

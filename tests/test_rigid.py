"""Rigid (p = 0) walls, 2D acoustic (SURVEY §8 a', BASELINE config 1), on the CPU:
the direct image formulation (oracle/rigid.py) is pinned bit for bit to the
reference's own periodic solver run on the mirrored domain (tests/golden/rigid_*.npz,
made by tests/golden/make_rigid_golden.py), and -- for the 2nd-order stencil the
reference lacks -- to the C oracle on the mirrored domain; plus the host-side rules."""

import json
from pathlib import Path

import numpy as np
import pytest

import oracle
import oracle.rigid as orig
import paper_2310_00236_b200 as hw
from golden_cases import assert_same_bits
from paper_2310_00236_b200 import rigid

GOLD = sorted((Path(__file__).resolve().parent / "golden").glob("rigid_*.npz"))
FIELDS = ("p", "vx", "vy", "rp", "rvx", "rvy")
VAR = {"naive": None, "op3": "op3", "op6": "op6"}


def box_planes(canon, g):
    st = {"rho_x": hw.Stagger.XFACE, "rho_y": hw.Stagger.YFACE, "beta": hw.Stagger.CELL}
    return {k: hw.grids.extend_cols(hw.extend_rows(canon[k], g, st[k]), g, st[k]) for k in canon}


def load(path):
    z = np.load(path)
    d = json.loads(str(z["desc"]))
    return d, z


@pytest.mark.parametrize("path", GOLD, ids=[p.stem for p in GOLD])
def test_direct_rigid_oracle_matches_reference_mirror(path):
    d, z = load(path)
    g = hw.GridSpec(d["nx"], d["ny"], d["dx"], d["dt"], d["nt"], bc_x=hw.Boundary.RIGID, bc_y=hw.Boundary.RIGID)
    canon = {k: z[f"canon_{k}"] for k in ("rho_x", "rho_y", "beta")}
    bp = box_planes(canon, g)
    taps = hw.StencilSpec.make(hw.Precision.FP16, d["dx"], d["order"]).coefficients
    st, e, tr = orig.run({k: z[f"init_{k}"] for k in FIELDS}, {k: v.astype(np.float16) for k, v in bp.items()}, bp,
                         taps, d["dx"], d["dt"], d["nt"], variant=VAR[d["variant"]], order=d["order"],
                         every=d["every"], receivers=[tuple(r) for r in d["receivers"]])
    for k in FIELDS:
        assert_same_bits(st[k], z[f"out_{k}"], k)
    np.testing.assert_array_equal(tr, z["traces"])
    np.testing.assert_allclose(e, z["e_vals"], rtol=1e-12)
    assert np.all(st["p"][:, 0] == 0) and np.all(st["p"][0, :] == 0)  # p = 0 walls held


@pytest.mark.parametrize("order", [2, 4])
@pytest.mark.parametrize("variant", [None, hw.Variant.OP3, hw.Variant.OP6])
def test_direct_rigid_oracle_equals_mirrored_c_oracle(order, variant):
    nx, ny, nt = 20, 16, 25
    g = hw.GridSpec(nx, ny, 1.0 / nx, float(np.float16(0.3 / nx)), nt, bc_x=hw.Boundary.RIGID,
                    bc_y=hw.Boundary.RIGID, order=order)
    med = hw.build_layered_acoustic(nx, ny, [(0.5, 1.0, 1.0), (1.0, 1.3, 2.0)])
    s = hw.AcousticSolver(g, med, stencil_precision=hw.Precision.FP16, energy_every=1, receivers=((10, 8), (20, 16)))
    st = s.new_state()
    rng = np.random.default_rng(order)
    p = rng.uniform(-0.5, 0.5, st.p.values.shape)
    p[0, :] = p[-1, :] = p[:, 0] = p[:, -1] = 0
    st.p.values = p.astype(np.float16)
    vx = rng.uniform(-0.05, 0.05, st.vx.values.shape)
    vx[0, :] = vx[-1, :] = 0
    st.vx.values = vx.astype(np.float16)
    # the C oracle on the device domain the product runs (s.desc: the mirrored periodic grid)
    arrays = [s._to_device(n, getattr(st, n).values) for n in s.FIELDS]
    from paper_2310_00236_b200.efsum import variant_code

    ref = oracle.run_desc(s.desc, arrays, variant_code(variant), 0, nt, None)
    bp = box_planes(med.planes, g)
    taps = hw.StencilSpec.make(hw.Precision.FP16, g.dx, order).coefficients
    vname = {None: None, hw.Variant.OP3: "op3", hw.Variant.OP6: "op6"}[variant]
    out, e, tr = orig.run({n: getattr(st, n).values for n in FIELDS}, {k: v.astype(np.float16) for k, v in bp.items()},
                          bp, taps, g.dx, g.dt, nt, variant=vname, order=order, every=1, receivers=[(10, 8), (20, 16)])
    for j, n in enumerate(s.FIELDS):
        assert_same_bits(out[n], rigid.restrict(ref["fields"][j].astype(np.float16), getattr(st, n).values.shape), n)
    np.testing.assert_array_equal(tr, ref["traces"])
    np.testing.assert_allclose(e, ref["e_vals"] * 0.25, rtol=1e-12)


def test_rigid_grid_shapes_and_rules():
    g = hw.GridSpec(16, 12, 1 / 16, 0.01, 3, bc_x=hw.Boundary.RIGID, bc_y=hw.Boundary.RIGID)
    assert g.shape(hw.Stagger.CELL) == (13, 17) and g.shape(hw.Stagger.XFACE) == (13, 16)
    assert g.shape(hw.Stagger.YFACE) == (12, 17)
    med = hw.build_homogeneous_acoustic(16, 12, 1.0, 1.0)
    s = hw.AcousticSolver(g, med, stencil_precision=hw.Precision.FP16, receivers=((16, 12),))
    assert (s.desc.nx, s.desc.ns) == (32, 24)  # the mirrored periodic domain
    st = s.new_state()
    st.p.values[0, 3] = 1.0
    with pytest.raises(ValueError, match="zero on the walls"):
        s._field_arrays(st)
    src = hw.SourceSpec(hw.SourceKind.PRESSURE_POINT, 4, 4, hw.RickerSpec(5.0))
    with pytest.raises(ValueError, match="point sources"):
        hw.AcousticSolver(g, med, src, stencil_precision=hw.Precision.FP16)
    with pytest.raises(ValueError, match="2D acoustic"):
        hw.GridSpec(16, 12, 0.1, 0.01, 3, nz=8, bc_x=hw.Boundary.RIGID)


def test_mirror_round_trip_and_parity():
    g = hw.GridSpec(12, 10, 0.1, 0.01, 1, bc_x=hw.Boundary.RIGID, bc_y=hw.Boundary.RIGID)
    a = np.random.default_rng(0).uniform(-1, 1, g.shape(hw.Stagger.XFACE)).astype(np.float16)
    a[0, :] = a[-1, :] = 0
    d = rigid.mirror(a, hw.Stagger.XFACE, rigid.PARITY["vx"], g)
    assert d.shape == (20, 24)
    np.testing.assert_array_equal(rigid.restrict(d, a.shape), a)
    np.testing.assert_array_equal(d[:, 12:], d[:, 11::-1])        # even in x about x = nx (half sub-grid)
    np.testing.assert_array_equal(d[10 + 1:, :], -d[10 - 1:0:-1, :])  # odd in y about y = ny (integer sub-grid)

"""The decomposed path at the BASELINE configs' production shapes: each config's one-pass kernel on
an in-process slab group (the multi-GPU path's kernels, halo plan and halo recomputation, here on one
device) must reproduce the single-domain run of the same kernel bit for bit -- fields, traces -- with
the energy history within 1e-12 (bit-identical on the plane-ordered 3D paths).  The single-domain run
is pinned to the CPU oracle at these shapes by tests/test_gpu_production.py.  Rows this wide (512
threads per CTA) and slabs this thin (64 planes / 512 rows at 8 slabs) are what a real 8-GPU job runs."""

import copy

import numpy as np
import pytest

import paper_2310_00236_b200 as hw
from golden_cases import assert_same_bits

pytestmark = pytest.mark.gpu

F16 = hw.Precision.FP16


def _compare(make, variant, slabs, path, exact_energy=False):
    a, sa = make(1)
    sb = copy.deepcopy(sa)
    oa = a.run(variant, sa)
    assert a.kernel_path() == path and a.transport() == 0
    a.close()
    b, _ = make(slabs, state=False)
    ob = b.run(variant, sb)
    assert b.kernel_path() == path and b.transport() == 1
    b.close()
    for n in a.FIELDS:
        assert_same_bits(getattr(sb, n).values, getattr(sa, n).values, n)
    np.testing.assert_array_equal(np.array([t.samples for t in ob.traces]), np.array([t.samples for t in oa.traces]))
    if exact_energy:
        np.testing.assert_array_equal(ob.energy.values, oa.energy.values)
    np.testing.assert_allclose(ob.energy.values, oa.energy.values, rtol=1e-12)


def _config2(slabs, state=True):
    n = 4096
    dx = 1.0 / n
    med = hw.build_layered_acoustic(n, n, [(0.5, 1.0, 1.0), (1.0, 1.5, 2.25)])
    dt = float(np.nextafter(np.float16(0.5 * dx / med.c_max()), np.float16(0)))
    src = hw.SourceSpec(hw.SourceKind.PRESSURE_POINT, n // 2, 8, hw.RickerSpec(f_center=1 / (10 * dx), amplitude=2.0e4))
    recs = ((n // 2, 8), (0, 0), (n - 1, n - 1), (1000, 511), (3000, 512), (4095, 2048), (17, 2047), (2048, 3583))
    s = hw.AcousticSolver(hw.GridSpec(n, n, dx, dt, 7), med, src, stencil_precision=F16, receivers=recs,
                          energy_every=2, slabs=slabs)
    if not state:
        return s, None
    st = s.new_state()
    rng = np.random.default_rng(21)
    st.p.values = rng.uniform(-0.5, 0.5, (n, n)).astype(np.float16)
    st.vy.values = rng.uniform(-0.05, 0.05, (n, n)).astype(np.float16)
    st.rvy.values = rng.uniform(-1e-4, 1e-4, (n, n)).astype(np.float16)
    return s, st


@pytest.mark.parametrize("slabs", [2, 8])
def test_config2_slabs_4096(slabs):
    _compare(_config2, hw.Variant.OP3, slabs, "fused2d")


def _config4(slabs, state=True):
    n = 4096
    dx = 1.0 / n
    med = hw.build_layered_elastic(n, n, [(1.0, 1.0, 2.0, 1.0)])
    g = hw.GridSpec(n, n, dx, float(np.float16(0.4 * dx / 2)), 7, bc_y=hw.Boundary.FREE_SURFACE)
    src = hw.SourceSpec(hw.SourceKind.EXPLOSIVE, n // 2, 16, hw.RickerSpec(1 / (10 * dx), amplitude=1.0e3))
    recs = ((n // 2, 16), (0, 0), (5, 4095), (4095, 2047), (1234, 2048), (2048, 511), (7, 512))
    s = hw.ElasticSolver(g, med, src, stencil_precision=F16, receivers=recs, energy_every=2, slabs=slabs)
    if not state:
        return s, None
    st = s.new_state()
    rng = np.random.default_rng(41)
    st.sxx.values = rng.uniform(-0.05, 0.05, st.sxx.values.shape).astype(np.float16)
    st.syy.values = rng.uniform(-0.05, 0.05, st.syy.values.shape).astype(np.float16)
    st.vy.values = rng.uniform(-0.02, 0.02, st.vy.values.shape).astype(np.float16)
    st.sxy.values = rng.uniform(-0.02, 0.02, st.sxy.values.shape).astype(np.float16)
    return s, st


@pytest.mark.parametrize("slabs", [2, 8])
def test_config4_slabs_4096(slabs):
    _compare(_config4, hw.Variant.OP6, slabs, "fused2d-el")


def _config3(prec):
    def make(slabs, state=True):
        n = 512
        rng = np.random.default_rng(30)
        med = hw.build_acoustic_from_velocity(1.5 + 3.0 * rng.random((n, n, n)))
        dx = 1.0 / n
        g = hw.GridSpec(n, n, dx, float(np.float16(0.5 * dx / (med.c_max() * np.sqrt(3)))), 3, nz=n, order=2)
        recs = ((0, 0, 0), (511, 511, 511), (256, 3, 63), (17, 400, 64), (100, 200, 447), (5, 6, 448))
        s = hw.AcousticSolver(g, med, stencil_precision=prec, receivers=recs, energy_every=1, slabs=slabs)
        if not state:
            return s, None
        st = s.new_state()
        st.p.values = rng.uniform(-0.5, 0.5, (n, n, n)).astype(st.p.values.dtype)
        st.vz.values = (0.01 * rng.standard_normal((n, n, n))).astype(st.vz.values.dtype)
        return s, st

    return make


def test_config3_slabs_512():
    _compare(_config3(F16), hw.Variant.OP3, 8, "fused3d", exact_energy=True)


def test_config3_f32_slabs_512():
    _compare(_config3(hw.Precision.FP32), None, 4, "fused3d-f32", exact_energy=True)


def _config5(slabs, state=True):
    n = 512
    med = hw.build_layered_elastic(n, n, [(0.3, 1.0, 2.0, 1.0), (0.7, 1.4, 2.6, 1.3), (1.0, 1.8, 3.0, 1.6)], nz=n)
    dx = 1.0 / n
    g = hw.GridSpec(n, n, dx, float(np.float16(0.4 * dx / 3.0)), 3, nz=n, order=2)
    recs = ((0, 0, 0), (511, 511, 511), (256, 255, 63), (3, 508, 64), (9, 9, 447), (500, 1, 448))
    s = hw.ElasticSolver(g, med, stencil_precision=F16, receivers=recs, energy_every=1, slabs=slabs)
    if not state:
        return s, None
    st = s.new_state()
    rng = np.random.default_rng(50)
    for name, amp in (("vz", 0.5), ("vx", 0.1), ("sxy", 0.01), ("szz", 0.05), ("syz", 0.02), ("rsxx", 1e-4)):
        f = getattr(st, name)
        f.values = rng.uniform(-amp, amp, f.values.shape).astype(np.float16)
    return s, st


def test_config5_slabs_512():
    """Eight 64-plane slabs: the slab thickness of BASELINE's 8-GPU split of 512^3."""
    _compare(_config5, hw.Variant.OP6, 8, "fused3d-el", exact_energy=True)

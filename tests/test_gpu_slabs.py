"""Slab decomposition on the device (SURVEY §8 e): an N-slab group driven by one
process (halo slabs moved by peer copies, same exchange plan as the NCCL transport)
must reproduce the single-domain run bit for bit — fields, traces, failure step and
field — with energy within 1e-12 (per-slab partial sums)."""

import numpy as np
import pytest

import oracle
import paper_2310_00236_b200 as hw
from golden_cases import assert_same_bits

pytestmark = pytest.mark.gpu


def _pair(make, slabs):
    a, sa = make(1)
    b, sb = make(slabs)
    return a, sa, b, sb


def _compare(a, sa, oa, b, sb, ob):
    for n in a.FIELDS:
        assert_same_bits(getattr(sb, n).values, getattr(sa, n).values, n)
    np.testing.assert_array_equal(np.array([t.samples for t in ob.traces]), np.array([t.samples for t in oa.traces]))
    np.testing.assert_array_equal(ob.energy.times, oa.energy.times)
    np.testing.assert_allclose(ob.energy.values, oa.energy.values, rtol=1e-12)


def _acoustic2d(slabs, nt=40, amp=2.0):
    nx, ny = 256, 96
    dx = 1.0 / nx
    med = hw.build_layered_acoustic(nx, ny, [(0.4, 1.0, 1.0), (1.0, 1.5, 2.25)])
    g = hw.GridSpec(nx, ny, dx, float(np.float16(0.3 * dx)), nt)
    src = hw.SourceSpec(hw.SourceKind.PRESSURE_POINT, 100, 47, hw.RickerSpec(1 / (10 * dx), amplitude=amp))
    s = hw.AcousticSolver(g, med, src, stencil_precision=hw.Precision.FP16, energy_every=5, slabs=slabs,
                          receivers=((100, 47), (3, 0), (250, 95), (7, 48)))
    st = s.new_state()
    yy, xx = np.mgrid[0:ny, 0:nx] / nx
    st.p.values = np.exp(-((xx - 0.5) ** 2 + (yy - 0.2) ** 2) / 0.005).astype(np.float16)
    return s, st


@pytest.mark.parametrize("slabs", [2, 3, 4])
@pytest.mark.parametrize("variant", [None, hw.Variant.OP3])
def test_acoustic_2d_slabs_equal_single_domain(slabs, variant):
    a, sa, b, sb = _pair(_acoustic2d, slabs)
    oa = a.run(variant, sa)
    ob = b.run(variant, sb)
    _compare(a, sa, oa, b, sb, ob)


def _elastic2d(slabs, fs=True, nt=40):
    nx, ny = 96, 64
    med = hw.build_layered_elastic(nx, ny, [(0.5, 2.0, 2.0, 1.0), (1.0, 2.3, 2.8, 1.4)])
    g = hw.GridSpec(nx, ny, 0.05, 0.01, nt, bc_y=hw.Boundary.FREE_SURFACE if fs else hw.Boundary.PERIODIC)
    src = hw.SourceSpec(hw.SourceKind.VY_POINT, 40, 33, hw.RickerSpec(5.0, amplitude=20.0))
    s = hw.ElasticSolver(g, med, src, stencil_precision=hw.Precision.FP16, energy_every=4, slabs=slabs,
                         receivers=((40, 33), (10, 0), (90, 63)))
    st = s.new_state()
    rng = np.random.default_rng(3)
    st.sxx.values = rng.uniform(-0.1, 0.1, st.sxx.values.shape).astype(np.float16)
    st.vx.values = rng.uniform(-0.01, 0.01, st.vx.values.shape).astype(np.float16)
    return s, st


@pytest.mark.parametrize("slabs", [2, 3, 5])
@pytest.mark.parametrize("fs", [True, False])
def test_elastic_2d_slabs_equal_single_domain(slabs, fs):
    a, sa, b, sb = _pair(lambda k: _elastic2d(k, fs), slabs)
    oa = a.run(hw.Variant.OP6, sa)
    ob = b.run(hw.Variant.OP6, sb)
    _compare(a, sa, oa, b, sb, ob)


def _acoustic3d(slabs, order=2):
    nz, ny, nx = 32, 16, 24
    g = hw.GridSpec(nx, ny, 0.05, 0.01, 20, nz=nz, order=order)
    s = hw.AcousticSolver(g, hw.build_homogeneous_acoustic(nx, ny, 1.0, 1.0, nz=nz), stencil_precision=hw.Precision.FP16,
                          slabs=slabs, receivers=((5, 5, 30), (12, 8, 2)), energy_every=5)
    st = s.new_state()
    z, y, x = np.mgrid[0:nz, 0:ny, 0:nx]
    st.p.values = np.exp(-((x - 12) ** 2 + (y - 8) ** 2 + (z - 3) ** 2) / 10.0).astype(np.float16)
    return s, st


@pytest.mark.parametrize("slabs", [2, 4])
@pytest.mark.parametrize("order", [2, 4])
def test_acoustic_3d_slabs_equal_single_domain(slabs, order):
    a, sa, b, sb = _pair(lambda k: _acoustic3d(k, order), slabs)
    oa = a.run(hw.Variant.OP3, sa)
    ob = b.run(hw.Variant.OP3, sb)
    _compare(a, sa, oa, b, sb, ob)


def _elastic3d(slabs):
    nz, ny, nx = 32, 12, 16
    med = hw.build_layered_elastic(nx, ny, [(0.5, 1.0, 2.0, 1.0), (1.0, 1.5, 2.6, 1.3)], nz=nz)
    g = hw.GridSpec(nx, ny, 0.05, 0.004, 20, nz=nz, order=2)
    src = hw.SourceSpec(hw.SourceKind.EXPLOSIVE, 8, 6, hw.RickerSpec(10.0, amplitude=50.0), iz=15)
    s = hw.ElasticSolver(g, med, src, stencil_precision=hw.Precision.FP16, slabs=slabs,
                         receivers=((8, 6, 16), (1, 1, 31)), energy_every=5)
    st = s.new_state()
    st.vz.values = np.random.default_rng(4).uniform(-0.05, 0.05, st.vz.values.shape).astype(np.float16)
    return s, st


@pytest.mark.parametrize("slabs", [2, 4])
def test_elastic_3d_slabs_equal_single_domain(slabs):
    a, sa, b, sb = _pair(_elastic3d, slabs)
    oa = a.run(hw.Variant.OP6, sa)
    ob = b.run(hw.Variant.OP6, sb)
    _compare(a, sa, oa, b, sb, ob)


def test_slabs_range_failure_semantics_match_single_domain():
    a, sa, b, sb = _pair(lambda k: _acoustic2d(k, nt=400, amp=1e9), 3)
    ref = oracle.run_solver(a, None, sa)
    assert ref["fail"] is not None
    with pytest.raises(hw.RangeFailureError) as e1:
        a.run(None, sa)
    with pytest.raises(hw.RangeFailureError) as e2:
        b.run(None, sb)
    assert (e1.value.step, e1.value.field_name) == (e2.value.step, e2.value.field_name)
    assert sa.step == sb.step == ref["fail"][0] + 1
    for j, n in enumerate(a.FIELDS):
        assert_same_bits(getattr(sb, n).values, ref["fields"][j], n)


def test_slab_group_single_steps():
    a, sa, b, sb = _pair(lambda k: _elastic2d(k, True, nt=1), 2)
    for _ in range(3):
        a.step_compensated(sa)
        b.step_compensated(sb)
    for n in a.FIELDS:
        assert_same_bits(getattr(sb, n).values, getattr(sa, n).values, n)


@pytest.mark.parametrize("slabs", [2, 5])
def test_fused_2d_slabs_receivers_on_slab_edges(slabs):
    """The fused single-pass kernel on slabs (ghost rows exchanged once per step; its
    redundant vy halo rows read the padded medium planes) equals the single domain."""
    nx, ny = 512, 200

    def make(k):
        dx = 1.0 / nx
        med = hw.build_layered_acoustic(nx, ny, [(0.3, 1.0, 1.0), (0.55, 1.3, 2.0), (1.0, 1.5, 2.25)])
        g = hw.GridSpec(nx, ny, dx, float(np.float16(0.3 * dx)), 33)
        src = hw.SourceSpec(hw.SourceKind.PRESSURE_POINT, 200, 80, hw.RickerSpec(1 / (10 * dx), amplitude=2.0))
        edges = sorted({r * ny // slabs + d for r in range(slabs) for d in (-1, 0)} - {-1})
        s = hw.AcousticSolver(g, med, src, stencil_precision=hw.Precision.FP16, energy_every=1, slabs=k,
                              receivers=tuple((7 * j % nx, e) for j, e in enumerate(edges)) + ((0, ny - 1),))
        st = s.new_state()
        yy, xx = np.mgrid[0:ny, 0:nx] / nx
        st.p.values = np.exp(-((xx - 0.5) ** 2 + (yy - 0.2) ** 2) / 0.005).astype(np.float16)
        st.vy.values = np.random.default_rng(5).uniform(-0.01, 0.01, (ny, nx)).astype(np.float16)
        return s, st

    a, sa, b, sb = _pair(make, slabs)
    oa = a.run(hw.Variant.OP6, sa)
    ob = b.run(hw.Variant.OP6, sb)
    assert a.kernel_path() == "small2d" and b.kernel_path() == "fused2d" and b.transport() == 1
    _compare(a, sa, oa, b, sb, ob)


def _acoustic3d_onepass(slabs, prec=hw.Precision.FP16, nt=13, src_z=None, ny=8, distributed=False):
    """Config 3's one-pass kernels (2nd order, nx = 512, per-cell beta) on slabs: p(-1), p(L), v_slow(-1)
    and its residual arrive by the once-per-step exchange (HW_PLAN_FUSED_AC3)."""
    nz, nx = 40, 512
    rng = np.random.default_rng(9)
    med = hw.build_acoustic_from_velocity(1.5 + 3.0 * rng.random((nz, ny, nx)))
    dx = 1.0 / nx
    g = hw.GridSpec(nx, ny, dx, float(np.float16(0.5 * dx / (med.c_max() * np.sqrt(3)))), nt, nz=nz, order=2)
    src = None if src_z is None else hw.SourceSpec(hw.SourceKind.PRESSURE_POINT, 300, 3, hw.RickerSpec(1 / (10 * dx), amplitude=5.0), iz=src_z)
    s = hw.AcousticSolver(g, med, src, stencil_precision=prec, slabs=slabs, energy_every=3, distributed=distributed,
                          receivers=((5, 5, 30), (511, ny - 1, 0), (300, 3, 19), (17, 2, 39), (100, ny // 2, 1)))
    st = s.new_state()
    z, y, x = np.mgrid[0:nz, 0:ny, 0:nx]
    st.p.values = np.exp(-((x - 256) ** 2 / 2000.0 + (y - ny // 2) ** 2 / 4.0 + (z - 19) ** 2 / 10.0)).astype(st.p.values.dtype)
    st.vz.values = (0.01 * rng.standard_normal((nz, ny, nx))).astype(st.vz.values.dtype)
    return s, st


@pytest.mark.parametrize("slabs", [2, 3, 5, 8])
@pytest.mark.parametrize("prec,variant", [(hw.Precision.FP16, hw.Variant.OP3), (hw.Precision.FP32, None)])
def test_acoustic_3d_onepass_slabs_equal_single_domain(slabs, prec, variant):
    a, sa, b, sb = _pair(lambda k: _acoustic3d_onepass(k, prec, src_z=20), slabs)
    ref = oracle.run_solver(a, variant, sa)
    oa = a.run(variant, sa)
    ob = b.run(variant, sb)
    want = "fused3d" if prec == hw.Precision.FP16 else "fused3d-f32"
    assert a.kernel_path() == b.kernel_path() == want and b.transport() == 1
    for j, n in enumerate(a.FIELDS):
        assert_same_bits(getattr(sa, n).values, ref["fields"][j], n)
    _compare(a, sa, oa, b, sb, ob)
    np.testing.assert_allclose(oa.energy.values, ref["e_vals"], rtol=1e-12)
    np.testing.assert_array_equal(ob.energy.values, oa.energy.values)  # plane-ordered: bit-identical for any slabs


def _elastic2d_onepass(slabs, fs=True, nt=23, kind=hw.SourceKind.VY_POINT, src_y=45, nx=256, ny=120):
    """Config 4's one-pass kernel on slabs (HW_PLAN_FUSED_EL2: five fields + velocity residuals, 3 rows):
    the CTAs at a slab edge recompute the halo velocity rows from the ghosts; free-surface images only at
    the global ends."""
    med = hw.build_layered_elastic(nx, ny, [(0.4, 2.0, 2.0, 1.0), (1.0, 2.3, 2.8, 1.4)])
    g = hw.GridSpec(nx, ny, 1.0 / nx, float(np.float16(0.3 / nx / med.c_max())), nt,
                    bc_y=hw.Boundary.FREE_SURFACE if fs else hw.Boundary.PERIODIC)
    src = hw.SourceSpec(kind, 100, src_y, hw.RickerSpec(1 / (10 / nx), amplitude=20.0))
    s = hw.ElasticSolver(g, med, src, stencil_precision=hw.Precision.FP16, energy_every=4, slabs=slabs,
                         receivers=((100, src_y), (10, 0), (250, ny - 1), (7, 44), (8, 46), (9, 15)))
    st = s.new_state()
    rng = np.random.default_rng(13)
    st.sxx.values = rng.uniform(-0.1, 0.1, st.sxx.values.shape).astype(np.float16)
    st.vy.values = rng.uniform(-0.01, 0.01, st.vy.values.shape).astype(np.float16)
    st.sxy.values = rng.uniform(-0.02, 0.02, st.sxy.values.shape).astype(np.float16)
    return s, st


@pytest.mark.parametrize("slabs", [2, 3, 5, 8])
@pytest.mark.parametrize("fs", [True, False])
@pytest.mark.parametrize("kind,src_y", [(hw.SourceKind.VY_POINT, 45), (hw.SourceKind.VY_POINT, 44),
                                        (hw.SourceKind.EXPLOSIVE, 46)])
def test_elastic_2d_onepass_slabs_equal_single_domain(hwopt, slabs, fs, kind, src_y):
    hwopt(small=0)
    a, sa, b, sb = _pair(lambda k: _elastic2d_onepass(k, fs, kind=kind, src_y=src_y), slabs)
    ref = oracle.run_solver(a, hw.Variant.OP6, sa)
    oa = a.run(hw.Variant.OP6, sa)
    ob = b.run(hw.Variant.OP6, sb)
    assert a.kernel_path() == b.kernel_path() == "fused2d-el" and b.transport() == 1
    for j, n in enumerate(a.FIELDS):
        assert_same_bits(getattr(sa, n).values, ref["fields"][j], n)
    _compare(a, sa, oa, b, sb, ob)


@pytest.mark.parametrize("nx,ny,slabs", [(1024, 256, 2), (2048, 96, 3), (4096, 64, 2)])
@pytest.mark.parametrize("fs", [True, False])
def test_elastic_2d_onepass_slabs_wide_rows(hwopt, nx, ny, slabs, fs):
    """Wide rows (4 to 16 warps per CTA; the narrow cases above run one warp): the top band's first
    TMA requests ask for rows -4 and -5, which must stay inside the 3 ghost rows of a slab (they ran
    off the allocation by up to 16 KB at nx = 4096 -- an illegal address in round 2's first build)."""
    hwopt(small=0)
    a, sa, b, sb = _pair(lambda k: _elastic2d_onepass(k, fs, nt=9, nx=nx, ny=ny), slabs)
    ref = oracle.run_solver(a, hw.Variant.OP6, sa)
    oa = a.run(hw.Variant.OP6, sa)
    ob = b.run(hw.Variant.OP6, sb)
    assert a.kernel_path() == b.kernel_path() == "fused2d-el" and b.transport() == 1
    for j, n in enumerate(a.FIELDS):
        assert_same_bits(getattr(sa, n).values, ref["fields"][j], n)
    _compare(a, sa, oa, b, sb, ob)

"""The streaming 3D elastic phase kernels (csrc/hw_elastic3d_stream.cu; binary16 3D
grids with nx % 256 == 0 and nm % (2048/nx) == 0) against the CPU oracle, the generic
kernels and a slab group: bit-exact fields, traces and failure steps; energy within
1e-12."""

import numpy as np
import pytest

import oracle
import paper_2310_00236_b200 as hw
from golden_cases import assert_same_bits

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True)
def _two_phase(hwopt):  # 2nd-order layered grids would otherwise take the one-pass kernel
    hwopt(fused_el3=0)

LAYERS = [(0.3, 1.0, 2.0, 1.0), (0.7, 1.4, 2.6, 1.3), (1.0, 1.8, 3.0, 0.0)]


def _case(nx, ny, nz, nt, *, order=2, kind=hw.SourceKind.EXPLOSIVE, full=False, slabs=1, amp=30.0, seed=0,
          recs=None):
    rng = np.random.default_rng(seed)
    med = hw.build_layered_elastic(nx, ny, LAYERS, nz=nz)
    if full:
        for k in med.planes:
            med.planes[k] = med.planes[k] * (1.0 + 0.05 * rng.uniform(0.0, 1.0, med.planes[k].shape))
    dx = 1.0 / nx
    dt = float(np.float16(0.3 * dx / (med.c_max() * np.sqrt(3))))
    g = hw.GridSpec(nx, ny, dx, dt, nt, nz=nz, order=order)
    src = hw.SourceSpec(kind, nx // 2 + 1, ny // 2, hw.RickerSpec(1 / (10 * dx), amplitude=amp), iz=nz // 3)
    if recs is None:
        recs = ((nx // 2 + 1, ny // 2, nz // 3), (0, 0, 0), (nx - 1, ny - 1, nz - 1), (9, 3, nz // 2))
    s = hw.ElasticSolver(g, med, src, stencil_precision=hw.Precision.FP16, receivers=recs, energy_every=3,
                         slabs=slabs)
    st = s.new_state()
    z, y, x = np.mgrid[0:nz, 0:ny, 0:nx]
    st.vz.values = (0.1 * np.exp(-((x - nx / 2) ** 2 / 300.0 + (y - ny / 3) ** 2 / 20.0 + (z - nz / 2) ** 2 / 20.0))
                    ).astype(np.float16)
    st.sxx.values = rng.uniform(-0.05, 0.05, st.sxx.values.shape).astype(np.float16)
    st.sxy.values = rng.uniform(-0.02, 0.02, st.sxy.values.shape).astype(np.float16)
    return s, st


def _check(s, st, out, ref):
    for j, n in enumerate(s.FIELDS):
        assert_same_bits(getattr(st, n).values, ref["fields"][j], n)
    np.testing.assert_array_equal(np.array([t.samples for t in out.traces]), ref["traces"])
    np.testing.assert_array_equal(out.energy.times, ref["e_times"])
    np.testing.assert_allclose(out.energy.values, ref["e_vals"], rtol=1e-12)


@pytest.mark.parametrize("variant", [None, hw.Variant.OP3, hw.Variant.OP6])
@pytest.mark.parametrize("order", [2, 4])
def test_el3d_stream_matches_oracle(variant, order):
    s, st = _case(256, 16, 14, 10, order=order)  # TM = 8: two mid tiles, wrap on both sides
    ref = oracle.run_solver(s, variant, st)
    out = s.run(variant, st)
    assert s.kernel_path() == "stream3d"
    _check(s, st, out, ref)


@pytest.mark.parametrize("ny,nz,kind", [(8, 9, hw.SourceKind.VY_POINT), (24, 20, hw.SourceKind.EXPLOSIVE)])
def test_el3d_stream_tiles_sources_full_media(ny, nz, kind):
    s, st = _case(256, ny, nz, 8, kind=kind, full=True, order=4)
    ref = oracle.run_solver(s, hw.Variant.OP6, st)
    out = s.run(hw.Variant.OP6, st)
    assert s.kernel_path() == "stream3d"
    _check(s, st, out, ref)


@pytest.mark.parametrize("nx,ny,nz,slabs", [(1024, 10, 9, 1), (1024, 8, 12, 3), (2048, 9, 8, 1)])
def test_el3d_stream_wide_rows_2nd_order(nx, ny, nz, slabs):
    """nx = 1024 (TM = 2) and 2048 (TM = 1) at 2nd order: the row width of a GPU's slab of BASELINE
    config 5's 1024^3 / 8-GPU grid (these widths fit the shared memory at 2nd order only)."""
    s, st = _case(nx, ny, nz, 7, order=2, kind=hw.SourceKind.VY_POINT, slabs=slabs)
    ref = oracle.run_solver(s, hw.Variant.OP6, st)
    out = s.run(hw.Variant.OP6, st)
    assert s.kernel_path() == "stream3d"
    _check(s, st, out, ref)


def test_el3d_nx1024_4th_order_stays_generic():
    s, st = _case(1024, 8, 9, 3, order=4)
    ref = oracle.run_solver(s, hw.Variant.OP6, st)
    out = s.run(hw.Variant.OP6, st)
    assert s.kernel_path() == "generic"
    _check(s, st, out, ref)


def test_el3d_stream_nx512_equals_generic(hwopt):
    s1, st1 = _case(512, 12, 16, 8)
    out1 = s1.run(hw.Variant.OP6, st1)
    assert s1.kernel_path() == "stream3d"
    hwopt(path=1)
    s2, st2 = _case(512, 12, 16, 8)
    out2 = s2.run(hw.Variant.OP6, st2)
    assert s2.kernel_path() == "generic"
    for n in s1.FIELDS:
        assert_same_bits(getattr(st1, n).values, getattr(st2, n).values, n)
    np.testing.assert_array_equal(np.array([t.samples for t in out1.traces]),
                                  np.array([t.samples for t in out2.traces]))
    np.testing.assert_allclose(out1.energy.values, out2.energy.values, rtol=1e-12)


def test_el3d_stream_range_failure_matches_oracle():
    s, st = _case(256, 8, 10, 100, amp=1e9)
    ref = oracle.run_solver(s, None, st)
    assert ref["fail"] is not None
    with pytest.raises(hw.RangeFailureError) as err:
        s.run(None, st)
    assert err.value.step == ref["fail"][0]
    assert err.value.field_name == s._fail_name(ref["fail"][1])
    for j, n in enumerate(s.FIELDS):
        assert_same_bits(getattr(st, n).values, ref["fields"][j], n)


@pytest.mark.parametrize("slabs", [2, 3])
def test_el3d_stream_slabs_equal_single_domain(slabs):
    a, sa = _case(256, 8, 24, 8)
    b, sb = _case(256, 8, 24, 8, slabs=slabs)
    oa = a.run(hw.Variant.OP6, sa)
    ob = b.run(hw.Variant.OP6, sb)
    for n in a.FIELDS:
        assert_same_bits(getattr(sb, n).values, getattr(sa, n).values, n)
    np.testing.assert_array_equal(np.array([t.samples for t in ob.traces]), np.array([t.samples for t in oa.traces]))
    np.testing.assert_allclose(ob.energy.values, oa.energy.values, rtol=1e-12)

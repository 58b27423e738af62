"""The streaming 2D elastic phase kernels (csrc/hw_elastic2d_stream.cu, selected for
binary16 grids with nx % 256 == 0) against the CPU oracle, against the generic phase
kernels, and inside a slab group: bit-exact fields, traces and failure steps; energy
within 1e-12 (block partials summed in a different order)."""

import numpy as np
import pytest

import oracle
import paper_2310_00236_b200 as hw
from golden_cases import assert_same_bits

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True)
def _streaming_kernels(hwopt):  # these grids would otherwise take the persistent small-grid kernel
    hwopt(small=0)  # (or, single domain, the one-pass kernel: test_gpu_elastic_fused.py)
    hwopt(fused_el=0)

LAYERS = [(0.3, 2.0, 2.0, 1.0), (0.7, 2.3, 2.8, 1.4), (1.0, 2.6, 3.2, 0.0)]


def _case(nx, ny, nt, *, fs=True, order=4, kind=hw.SourceKind.VY_POINT, amp=20.0, full=False, slabs=1,
          seed=0, every=5, src_row=6):
    rng = np.random.default_rng(seed)
    med = hw.build_layered_elastic(nx, ny, LAYERS)
    if full:  # per-cell planes: the general (non row-uniform) medium path
        for k in med.planes:
            med.planes[k] = med.planes[k] * (1.0 + 0.05 * rng.uniform(0.0, 1.0, med.planes[k].shape))
    dx = 0.05
    dt = float(np.float16(0.4 * dx / med.c_max()))
    bc = hw.Boundary.FREE_SURFACE if fs else hw.Boundary.PERIODIC
    grid = hw.GridSpec(nx, ny, dx, dt, nt, bc_y=bc, order=order)
    src = hw.SourceSpec(kind, nx // 2 + 1, src_row, hw.RickerSpec(4.0, amplitude=amp))
    recs = ((nx // 2 + 1, src_row), (0, 0), (nx - 1, ny - 1), (7, ny // 2))
    s = hw.ElasticSolver(grid, med, src, stencil_precision=hw.Precision.FP16, receivers=recs, energy_every=every,
                         slabs=slabs)
    st = s.new_state()
    st.sxx.values = rng.uniform(-0.1, 0.1, st.sxx.values.shape).astype(np.float16)
    st.vx.values = rng.uniform(-0.01, 0.01, st.vx.values.shape).astype(np.float16)
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
@pytest.mark.parametrize("fs", [True, False])
def test_stream_matches_oracle(variant, order, fs):
    s, st = _case(256, 160, 45, fs=fs, order=order)
    ref = oracle.run_solver(s, variant, st)
    out = s.run(variant, st)
    _check(s, st, out, ref)


@pytest.mark.parametrize("ny", [8, 13, 64, 600])
@pytest.mark.parametrize("fs", [True, False])
def test_stream_row_bands(ny, fs):
    s, st = _case(256, ny, 20, fs=fs, src_row=min(6, ny - 1))
    ref = oracle.run_solver(s, hw.Variant.OP6, st)
    out = s.run(hw.Variant.OP6, st)
    _check(s, st, out, ref)


def test_stream_full_medium_and_explosive_source():
    s, st = _case(512, 96, 40, full=True, kind=hw.SourceKind.EXPLOSIVE)
    ref = oracle.run_solver(s, hw.Variant.OP6, st)
    out = s.run(hw.Variant.OP6, st)
    _check(s, st, out, ref)


def test_stream_equals_generic_kernels(hwopt):
    s1, st1 = _case(1024, 300, 40, full=True)
    out1 = s1.run(hw.Variant.OP6, st1)
    assert s1.kernel_path() == "stream2d"
    hwopt(path=1)
    s2, st2 = _case(1024, 300, 40, full=True)
    out2 = s2.run(hw.Variant.OP6, st2)
    assert s2.kernel_path() == "generic"
    assert s1.last_launch_count() == 2 + 2 * 40  # E(0) kernel + finalize, then two phase kernels per step
    for n in s1.FIELDS:
        assert_same_bits(getattr(st1, n).values, getattr(st2, n).values, n)
    np.testing.assert_array_equal(np.array([t.samples for t in out1.traces]),
                                  np.array([t.samples for t in out2.traces]))
    np.testing.assert_allclose(out1.energy.values, out2.energy.values, rtol=1e-12)


def test_stream_range_failure_matches_oracle():
    s, st = _case(256, 64, 300, amp=1e8)
    ref = oracle.run_solver(s, None, st)
    assert ref["fail"] is not None
    with pytest.raises(hw.RangeFailureError) as err:
        s.run(None, st)
    assert err.value.step == ref["fail"][0]
    assert err.value.field_name == s._fail_name(ref["fail"][1])
    for j, n in enumerate(s.FIELDS):
        assert_same_bits(getattr(st, n).values, ref["fields"][j], n)


def test_stream_single_steps_and_resume():
    s, st = _case(256, 40, 3)
    ref = oracle.run_solver(s, hw.Variant.OP3, st, nt=8)
    s.step_compensated(st, hw.Variant.OP3)
    s.run(hw.Variant.OP3, st)
    s.step_compensated(st, hw.Variant.OP3)
    s.run(hw.Variant.OP3, st)
    assert st.step == 8
    for j, n in enumerate(s.FIELDS):
        assert_same_bits(getattr(st, n).values, ref["fields"][j], n)


@pytest.mark.parametrize("slabs", [2, 3])
@pytest.mark.parametrize("fs", [True, False])
def test_stream_slabs_equal_single_domain(slabs, fs):
    a, sa = _case(256, 90, 30, fs=fs)
    b, sb = _case(256, 90, 30, fs=fs, slabs=slabs)
    oa = a.run(hw.Variant.OP6, sa)
    ob = b.run(hw.Variant.OP6, sb)
    for n in a.FIELDS:
        assert_same_bits(getattr(sb, n).values, getattr(sa, n).values, n)
    np.testing.assert_array_equal(np.array([t.samples for t in ob.traces]), np.array([t.samples for t in oa.traces]))
    np.testing.assert_allclose(ob.energy.values, oa.energy.values, rtol=1e-12)


def test_stream_free_surface_syy_rows_bit_zero():
    s, st = _case(256, 48, 60)
    st.sxx.values[:] = 0
    s.run(hw.Variant.OP6, st)
    for rows in (st.syy.values, st.rsyy.values):
        assert np.all(rows[0].view(np.uint16) == 0)
        assert np.all(rows[-1].view(np.uint16) == 0)
    assert np.any(st.syy.values[1:-1] != 0.0)


@pytest.mark.parametrize("nx,lanes,path", [(4096, hw.Precision.FP16, "stream2d"), (100, hw.Precision.FP16, "generic"),
                                           (256, hw.Precision.FP32, "generic")])
def test_stream_path_selection(nx, lanes, path):
    med = hw.build_layered_elastic(nx, 16, LAYERS)
    g = hw.GridSpec(nx, 16, 0.05, 0.004, 1, bc_y=hw.Boundary.FREE_SURFACE)
    s = hw.ElasticSolver(g, med, None, stencil_precision=lanes, update_precision=lanes)
    s.run(hw.Variant.OP3, s.new_state())
    assert s.kernel_path() == path


@pytest.mark.parametrize("nx,ny,fs", [(600, 3500, True), (264, 8000, False)])
def test_stream_any_width_multiple_of_8(nx, ny, fs):
    """Large grids of any nx % 8 == 0: nx / 8 threads, partial last warp."""
    s, st = _case(nx, ny, 6, fs=fs, src_row=min(6, ny - 1))
    ref = oracle.run_solver(s, hw.Variant.OP6, st)
    out = s.run(hw.Variant.OP6, st)
    assert s.kernel_path() == "stream2d"
    _check(s, st, out, ref)

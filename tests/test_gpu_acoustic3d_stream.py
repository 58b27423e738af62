"""The streaming 3D acoustic phase kernels (csrc/hw_acoustic3d_stream.cu, selected for
binary16 3D grids with nx % 256 == 0 and nm % (4096/nx) == 0) against the CPU oracle,
the generic kernels and a slab group: bit-exact fields, traces and failure steps;
energy within 1e-12 (block partials summed in a different order)."""

import numpy as np
import pytest

import oracle
import paper_2310_00236_b200 as hw
from golden_cases import assert_same_bits

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True)
def _two_phase(hwopt):
    """2nd-order single-domain cases would take the one-pass kernel (test_gpu_acoustic3d_fused.py)."""
    hwopt(fused3=0)


def _case(nx, ny, nz, nt, *, order=2, full=True, slabs=1, amp=5.0, seed=0, recs=None):
    rng = np.random.default_rng(seed)
    if full:
        c = 1.5 + 3.0 * rng.random((nz, ny, nx))
        med = hw.build_acoustic_from_velocity(c)
    else:
        med = hw.build_layered_acoustic(nx, ny, [(0.4, 1.0, 1.5), (1.0, 1.3, 3.0)], nz=nz)
    dx = 1.0 / nx
    dt = float(np.float16(0.4 * dx / (med.c_max() * np.sqrt(3))))
    g = hw.GridSpec(nx, ny, dx, dt, nt, nz=nz, order=order)
    src = hw.SourceSpec(hw.SourceKind.PRESSURE_POINT, nx // 2 + 3, ny // 2, hw.RickerSpec(1 / (10 * dx), amplitude=amp),
                        iz=nz // 3)
    if recs is None:
        recs = ((nx // 2 + 3, ny // 2, nz // 3), (0, 0, 0), (nx - 1, ny - 1, nz - 1), (7, 1, nz // 2), (8, ny - 2, 1))
    s = hw.AcousticSolver(g, med, src, stencil_precision=hw.Precision.FP16, receivers=recs, energy_every=4,
                          slabs=slabs)
    st = s.new_state()
    z, y, x = np.mgrid[0:nz, 0:ny, 0:nx]
    st.p.values = (np.exp(-((x - nx / 2) ** 2 / 400.0 + (y - ny / 3) ** 2 / 30.0 + (z - nz / 2) ** 2 / 30.0))
                   + rng.uniform(-1e-3, 1e-3, (nz, ny, nx))).astype(np.float16)
    st.vx.values = rng.uniform(-0.01, 0.01, (nz, ny, nx)).astype(np.float16)
    return s, st


def _check(s, st, out, ref):
    for j, n in enumerate(s.FIELDS):
        assert_same_bits(getattr(st, n).values, ref["fields"][j], n)
    np.testing.assert_array_equal(np.array([t.samples for t in out.traces]), ref["traces"])
    np.testing.assert_array_equal(out.energy.times, ref["e_times"])
    np.testing.assert_allclose(out.energy.values, ref["e_vals"], rtol=1e-12)


@pytest.mark.parametrize("variant", [None, hw.Variant.OP3, hw.Variant.OP6])
@pytest.mark.parametrize("order", [2, 4])
def test_stream3d_matches_oracle(variant, order):
    s, st = _case(256, 32, 20, 14, order=order)  # TM = 16: two mid tiles, wrap on both sides
    ref = oracle.run_solver(s, variant, st)
    out = s.run(variant, st)
    assert s.kernel_path() == "stream3d"
    _check(s, st, out, ref)


@pytest.mark.parametrize("ny,nz", [(16, 9), (48, 31), (16, 64)])
def test_stream3d_tiles_and_slab_splits(ny, nz):
    s, st = _case(256, ny, nz, 10, order=4, full=False)
    ref = oracle.run_solver(s, hw.Variant.OP3, st)
    out = s.run(hw.Variant.OP3, st)
    assert s.kernel_path() == "stream3d"
    _check(s, st, out, ref)


def test_stream3d_nx512_equals_generic(hwopt):
    s1, st1 = _case(512, 16, 24, 12)
    out1 = s1.run(hw.Variant.OP3, st1)
    assert s1.kernel_path() == "stream3d"
    assert s1.last_launch_count() == 2 + 2 * 12
    hwopt(path=1)
    s2, st2 = _case(512, 16, 24, 12)
    out2 = s2.run(hw.Variant.OP3, st2)
    assert s2.kernel_path() == "generic"
    for n in s1.FIELDS:
        assert_same_bits(getattr(st1, n).values, getattr(st2, n).values, n)
    np.testing.assert_array_equal(np.array([t.samples for t in out1.traces]),
                                  np.array([t.samples for t in out2.traces]))
    np.testing.assert_allclose(out1.energy.values, out2.energy.values, rtol=1e-12)


def test_stream3d_receiver_plane():
    nx, ny, nz = 256, 16, 12
    recs = tuple((x, y, 2) for y in range(ny) for x in range(0, nx, 5)) + ((3, 3, 11),)
    s, st = _case(nx, ny, nz, 8, recs=recs)
    ref = oracle.run_solver(s, hw.Variant.OP3, st)
    out = s.run(hw.Variant.OP3, st)
    _check(s, st, out, ref)


def test_stream3d_range_failure_matches_oracle():
    s, st = _case(256, 16, 12, 200, amp=1e9)
    ref = oracle.run_solver(s, None, st)
    assert ref["fail"] is not None
    with pytest.raises(hw.RangeFailureError) as err:
        s.run(None, st)
    assert err.value.step == ref["fail"][0]
    assert err.value.field_name == s._fail_name(ref["fail"][1])
    for j, n in enumerate(s.FIELDS):
        assert_same_bits(getattr(st, n).values, ref["fields"][j], n)


@pytest.mark.parametrize("slabs", [2, 3])
def test_stream3d_slabs_equal_single_domain(slabs):
    a, sa = _case(256, 16, 30, 10)
    b, sb = _case(256, 16, 30, 10, slabs=slabs)
    oa = a.run(hw.Variant.OP6, sa)
    ob = b.run(hw.Variant.OP6, sb)
    for n in a.FIELDS:
        assert_same_bits(getattr(sb, n).values, getattr(sa, n).values, n)
    np.testing.assert_array_equal(np.array([t.samples for t in ob.traces]), np.array([t.samples for t in oa.traces]))
    np.testing.assert_allclose(ob.energy.values, oa.energy.values, rtol=1e-12)

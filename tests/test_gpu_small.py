"""The persistent small-grid 2D acoustic kernel (csrc/hw_small2d.cu: one cooperative
launch per run, bands resident in shared memory, one neighbour exchange and one grid
barrier per step) against the CPU oracle and the fused streaming kernel: bit-exact
fields, traces and failure semantics; energy within 1e-12."""

import numpy as np
import pytest

import oracle
import paper_2310_00236_b200 as hw
from golden_cases import assert_same_bits

pytestmark = pytest.mark.gpu


def _case(nx, ny, nt, *, order=4, amp=2.0, every=1, seed=0, layered=True, recs=None):
    rng = np.random.default_rng(seed)
    dx = 1.0 / nx
    med = (hw.build_layered_acoustic(nx, ny, [(0.5, 1.0, 1.0), (1.0, 1.5, 2.25)]) if layered
           else hw.build_homogeneous_acoustic(nx, ny, 1.0, 1.0))
    if not layered:
        med.planes["beta"] = med.planes["beta"] * (1.0 + 0.1 * rng.uniform(0.0, 1.0, (ny, nx)))
    dt = float(np.float16(0.45 * dx / med.c_max()))
    g = hw.GridSpec(nx, ny, dx, dt, nt, order=order)
    src = hw.SourceSpec(hw.SourceKind.PRESSURE_POINT, nx // 2 + 1, ny // 3, hw.RickerSpec(1 / (10 * dx), amplitude=amp))
    if recs is None:
        recs = ((nx // 2 + 1, ny // 3), (0, 0), (nx - 1, ny - 1), (3, ny // 2), (nx - 2, 2))
    s = hw.AcousticSolver(g, med, src, stencil_precision=hw.Precision.FP16, receivers=recs, energy_every=every)
    st = s.new_state()
    yy, xx = np.mgrid[0:ny, 0:nx] / nx
    st.p.values = (np.exp(-((xx - 0.5) ** 2 + (yy - 0.3) ** 2) / 0.01) + rng.uniform(-1e-3, 1e-3, (ny, nx))).astype(np.float16)
    st.vx.values = rng.uniform(-0.05, 0.05, (ny, nx)).astype(np.float16)
    st.vy.values = rng.uniform(-0.05, 0.05, (ny, nx)).astype(np.float16)
    return s, st


def _check(s, st, out, ref):
    for j, n in enumerate(s.FIELDS):
        assert_same_bits(getattr(st, n).values, ref["fields"][j], n)
    np.testing.assert_array_equal(np.array([t.samples for t in out.traces]), ref["traces"])
    np.testing.assert_array_equal(out.energy.times, ref["e_times"])
    np.testing.assert_allclose(out.energy.values, ref["e_vals"], rtol=1e-12)


@pytest.mark.parametrize("variant", [None, hw.Variant.OP3, hw.Variant.OP6])
@pytest.mark.parametrize("order", [2, 4])
def test_small_matches_oracle(variant, order):
    s, st = _case(600, 150, 40, order=order)
    ref = oracle.run_solver(s, variant, st)
    out = s.run(variant, st)
    assert s.kernel_path() == "small2d"
    _check(s, st, out, ref)


@pytest.mark.parametrize("nx,ny,layered", [(150, 150, True), (64, 8, True), (256, 64, False), (98, 452, True)])
def test_small_shapes_and_media(nx, ny, layered):
    s, st = _case(nx, ny, 25, every=4, layered=layered)
    ref = oracle.run_solver(s, hw.Variant.OP3, st)
    out = s.run(hw.Variant.OP3, st)
    assert s.kernel_path() == "small2d"
    _check(s, st, out, ref)


def test_small_equals_fused(hwopt):
    s1, st1 = _case(512, 256, 60, every=5)
    out1 = s1.run(hw.Variant.OP6, st1)
    assert s1.kernel_path() == "small2d" and s1.last_launch_count() == 2 + 1
    hwopt(small=0)
    s2, st2 = _case(512, 256, 60, every=5)
    out2 = s2.run(hw.Variant.OP6, st2)
    assert s2.kernel_path() == "fused2d"
    for n in s1.FIELDS:
        assert_same_bits(getattr(st1, n).values, getattr(st2, n).values, n)
    np.testing.assert_array_equal(np.array([t.samples for t in out1.traces]),
                                  np.array([t.samples for t in out2.traces]))
    np.testing.assert_allclose(out1.energy.values, out2.energy.values, rtol=1e-12)


def test_small_range_failure_matches_oracle():
    s, st = _case(200, 60, 300, amp=1e9, layered=False)
    ref = oracle.run_solver(s, None, st)
    assert ref["fail"] is not None
    with pytest.raises(hw.RangeFailureError) as err:
        s.run(None, st)
    assert err.value.step == ref["fail"][0]
    assert err.value.field_name == s._fail_name(ref["fail"][1])
    assert st.step == ref["fail"][0] + 1
    for j, n in enumerate(s.FIELDS):
        assert_same_bits(getattr(st, n).values, ref["fields"][j], n)


def test_small_single_steps_and_resume():
    s, st = _case(128, 40, 7)
    ref = oracle.run_solver(s, hw.Variant.OP6, st, nt=16)
    s.step_compensated(st, hw.Variant.OP6)
    s.run(hw.Variant.OP6, st)
    s.step_compensated(st, hw.Variant.OP6)
    s.run(hw.Variant.OP6, st)
    assert st.step == 16
    for j, n in enumerate(s.FIELDS):
        assert_same_bits(getattr(st, n).values, ref["fields"][j], n)


LAYERS_EL = [(0.3, 2.0, 2.0, 1.0), (0.7, 2.3, 2.8, 1.4), (1.0, 2.6, 3.2, 0.0)]


def _el(nx, ny, nt, *, fs=True, order=4, kind=hw.SourceKind.VY_POINT, amp=20.0, seed=0, every=3):
    rng = np.random.default_rng(seed)
    med = hw.build_layered_elastic(nx, ny, LAYERS_EL)
    dx = 0.05
    dt = float(np.float16(0.4 * dx / med.c_max()))
    bc = hw.Boundary.FREE_SURFACE if fs else hw.Boundary.PERIODIC
    g = hw.GridSpec(nx, ny, dx, dt, nt, bc_y=bc, order=order)
    src = hw.SourceSpec(kind, nx // 2 + 1, 4, hw.RickerSpec(4.0, amplitude=amp))
    recs = ((nx // 2 + 1, 4), (0, 0), (nx - 1, ny - 1), (7, ny // 2))
    s = hw.ElasticSolver(g, med, src, stencil_precision=hw.Precision.FP16, receivers=recs, energy_every=every)
    st = s.new_state()
    st.sxx.values = rng.uniform(-0.1, 0.1, st.sxx.values.shape).astype(np.float16)
    st.vx.values = rng.uniform(-0.01, 0.01, st.vx.values.shape).astype(np.float16)
    st.sxy.values = rng.uniform(-0.02, 0.02, st.sxy.values.shape).astype(np.float16)
    return s, st


@pytest.mark.parametrize("variant", [None, hw.Variant.OP3, hw.Variant.OP6])
@pytest.mark.parametrize("order", [2, 4])
@pytest.mark.parametrize("fs", [True, False])
def test_small_elastic_matches_oracle(variant, order, fs):
    s, st = _el(600, 150, 30, fs=fs, order=order)
    ref = oracle.run_solver(s, variant, st)
    out = s.run(variant, st)
    assert s.kernel_path() == "small2d"
    _check(s, st, out, ref)


@pytest.mark.parametrize("nx,ny,kind", [(150, 150, hw.SourceKind.EXPLOSIVE), (64, 9, hw.SourceKind.VY_POINT),
                                        (98, 452, hw.SourceKind.EXPLOSIVE)])
def test_small_elastic_shapes_and_sources(nx, ny, kind):
    s, st = _el(nx, ny, 24, kind=kind)
    ref = oracle.run_solver(s, hw.Variant.OP6, st)
    out = s.run(hw.Variant.OP6, st)
    assert s.kernel_path() == "small2d"
    _check(s, st, out, ref)


def test_small_elastic_equals_phase_kernels(hwopt):
    s1, st1 = _el(512, 200, 40)
    out1 = s1.run(hw.Variant.OP6, st1)
    assert s1.kernel_path() == "small2d"
    hwopt(small=0)
    s2, st2 = _el(512, 200, 40)
    out2 = s2.run(hw.Variant.OP6, st2)
    assert s2.kernel_path() == "fused2d-el"
    for n in s1.FIELDS:
        assert_same_bits(getattr(st1, n).values, getattr(st2, n).values, n)
    np.testing.assert_array_equal(np.array([t.samples for t in out1.traces]),
                                  np.array([t.samples for t in out2.traces]))
    np.testing.assert_allclose(out1.energy.values, out2.energy.values, rtol=1e-12)


def test_small_elastic_range_failure():
    s, st = _el(200, 60, 300, amp=1e8)
    ref = oracle.run_solver(s, None, st)
    assert ref["fail"] is not None
    with pytest.raises(hw.RangeFailureError) as err:
        s.run(None, st)
    assert err.value.step == ref["fail"][0]
    assert err.value.field_name == s._fail_name(ref["fail"][1])
    for j, n in enumerate(s.FIELDS):
        assert_same_bits(getattr(st, n).values, ref["fields"][j], n)

"""The fused single-pass 2D acoustic kernel (csrc/hw_fused2d.cu) against the CPU
oracle and against the two-phase kernels: bit-exact fields and traces, energy
within 1e-12 (its fixed-order block reduction differs from the phase kernels')."""

import os

import numpy as np
import pytest

import oracle
import paper_2310_00236_b200 as hw
from golden_cases import assert_same_bits

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True)
def _streaming_kernel(hwopt):  # these grids would otherwise take the persistent small-grid kernel
    hwopt(small=0)


def _case(nx, ny, nt, *, order=4, amp=2.0, every=5, seed=0, src_row=3, layered=True):
    rng = np.random.default_rng(seed)
    dx = 1.0 / nx
    med = (hw.build_layered_acoustic(nx, ny, [(0.5, 1.0, 1.0), (1.0, 1.5, 2.25)]) if layered
           else hw.build_homogeneous_acoustic(nx, ny, 1.0, 1.0))
    dt = float(np.float16(0.5 * dx / med.c_max()))
    if dt > 0.5 * dx / med.c_max():
        dt = float(np.nextafter(np.float16(dt), np.float16(0)))
    grid = hw.GridSpec(nx, ny, dx, dt, nt, order=order)
    src = hw.SourceSpec(hw.SourceKind.PRESSURE_POINT, nx // 2 + 1, src_row,
                        hw.RickerSpec(f_center=1.0 / (10 * dx), amplitude=amp))
    recs = ((nx // 2 + 1, src_row), (0, 0), (nx - 1, ny - 1), (7, ny // 2))
    s = hw.AcousticSolver(grid, med, src, stencil_precision=hw.Precision.FP16, receivers=recs,
                          energy_every=every)
    st = s.new_state()
    yy, xx = np.mgrid[0:ny, 0:nx] / nx
    p0 = np.exp(-((xx - 0.5) ** 2 + (yy - 0.3) ** 2) / 0.01) + rng.uniform(-1e-3, 1e-3, (ny, nx))
    st.p.values = p0.astype(np.float16)
    st.vx.values = rng.uniform(-0.05, 0.05, (ny, nx)).astype(np.float16)
    return s, st


def _check(s, st, out, ref):
    for j, n in enumerate(s.FIELDS):
        assert_same_bits(getattr(st, n).values, ref["fields"][j], n)
    np.testing.assert_array_equal(np.array([t.samples for t in out.traces]), ref["traces"])
    np.testing.assert_array_equal(out.energy.times, ref["e_times"])
    np.testing.assert_allclose(out.energy.values, ref["e_vals"], rtol=1e-12)


@pytest.mark.parametrize("variant", [None, hw.Variant.OP3, hw.Variant.OP6])
@pytest.mark.parametrize("order", [2, 4])
def test_fused_matches_oracle(variant, order):
    s, st = _case(512, 300, 37, order=order)  # odd nt: result copied home from the B buffer
    ref = oracle.run_solver(s, variant, st)
    out = s.run(variant, st)
    _check(s, st, out, ref)


@pytest.mark.parametrize("ny", [8, 13, 64, 600])
def test_fused_row_bands_and_wrap(ny):
    s, st = _case(256, ny, 24, layered=False, src_row=min(3, ny - 1))
    ref = oracle.run_solver(s, hw.Variant.OP3, st)
    out = s.run(hw.Variant.OP3, st)
    _check(s, st, out, ref)


def test_fused_equals_two_phase_kernels(hwopt):
    s1, st1 = _case(1024, 256, 40)
    out1 = s1.run(hw.Variant.OP3, st1)
    hwopt(path=1)
    s2, st2 = _case(1024, 256, 40)
    out2 = s2.run(hw.Variant.OP3, st2)
    for n in s1.FIELDS:
        assert_same_bits(getattr(st1, n).values, getattr(st2, n).values, n)
    np.testing.assert_array_equal(np.array([t.samples for t in out1.traces]),
                                  np.array([t.samples for t in out2.traces]))
    np.testing.assert_allclose(out1.energy.values, out2.energy.values, rtol=1e-12)


def test_fused_range_failure_matches_oracle():
    s, st = _case(256, 64, 400, amp=1e9, layered=False)
    ref = oracle.run_solver(s, None, st)
    assert ref["fail"] is not None
    with pytest.raises(hw.RangeFailureError) as err:
        s.run(None, st)
    assert err.value.step == ref["fail"][0]
    assert err.value.field_name == s._fail_name(ref["fail"][1])
    assert st.step == ref["fail"][0] + 1
    for j, n in enumerate(s.FIELDS):
        assert_same_bits(getattr(st, n).values, ref["fields"][j], n)


def test_fused_single_steps_and_resume():
    s, st = _case(256, 40, 3)
    ref = oracle.run_solver(s, hw.Variant.OP6, st, nt=8)
    s.step_compensated(st, hw.Variant.OP6)
    s.run(hw.Variant.OP6, st)
    s.step_compensated(st, hw.Variant.OP6)
    s.run(hw.Variant.OP6, st)
    assert st.step == 8
    for j, n in enumerate(s.FIELDS):
        assert_same_bits(getattr(st, n).values, ref["fields"][j], n)


def test_fused_path_is_selected():
    s, st = _case(4096, 64, 2)
    s.run(hw.Variant.OP3, st)
    assert s.kernel_path() == "fused2d"
    assert s.last_launch_count() == 2 + 2  # E0 kernel + finalize, then one fused launch per step


def test_fused_receiver_line_records_every_trace():
    """A full receiver line on one row plus a column through every row band: all traces
    recorded (the in-kernel receiver list has no per-CTA cap)."""
    nx, ny = 512, 300
    s0, _ = _case(nx, ny, 12)
    line = tuple((x, 5) for x in range(0, nx, 3)) + tuple((17, y) for y in range(0, ny, 7)) + ((nx - 1, ny - 1),)
    s = hw.AcousticSolver(s0.grid, s0.medium, s0.source, stencil_precision=hw.Precision.FP16, receivers=line,
                          energy_every=5)
    _, st = _case(nx, ny, 12)
    ref = oracle.run_solver(s, hw.Variant.OP3, st)
    out = s.run(hw.Variant.OP3, st)
    assert s.kernel_path() == "fused2d"
    np.testing.assert_array_equal(np.array([t.samples for t in out.traces]), ref["traces"])


@pytest.mark.parametrize("nx,ny", [(600, 64), (104, 40), (264, 30), (1000, 24)])
def test_fused_any_width_multiple_of_8(nx, ny):
    """The single-pass kernel takes any nx % 8 == 0 (the reference presets' 600 x 600):
    nx / 8 threads, the last warp possibly partial (collectives over existing lanes)."""
    s, st = _case(nx, ny, 18, every=1)
    ref = oracle.run_solver(s, hw.Variant.OP6, st)
    out = s.run(hw.Variant.OP6, st)
    assert s.kernel_path() == "fused2d"
    _check(s, st, out, ref)


def test_fused_range_failure_partial_warp():
    s, st = _case(600, 32, 300, amp=1e9, layered=False)
    ref = oracle.run_solver(s, None, st)
    with pytest.raises(hw.RangeFailureError) as err:
        s.run(None, st)
    assert err.value.step == ref["fail"][0]
    assert err.value.field_name == s._fail_name(ref["fail"][1])

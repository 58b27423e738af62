"""Two steps per launch (temporal blocking, csrc/hw_tb2d.cu) for the 2D acoustic
binary16 path: bit-exact against the CPU oracle and against the single-step fused
kernel (the default; the two-step kernel is opt-in, option tb=1), for odd and even step counts, several x tiles, receiver lines,
energy every step, and range failures in either step of a pair (the host replays a
failing first step alone)."""

import numpy as np
import pytest

import oracle
import paper_2310_00236_b200 as hw
from golden_cases import assert_same_bits

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True)
def _two_step(hwopt):  # the two-step kernel is opt-in
    hwopt(tb=1)
    hwopt(small=0)


def _case(nx, ny, nt, *, order=4, amp=2.0, every=5, seed=0, src_row=3, layered=True, recs=None):
    rng = np.random.default_rng(seed)
    dx = 1.0 / nx
    med = (hw.build_layered_acoustic(nx, ny, [(0.5, 1.0, 1.0), (1.0, 1.5, 2.25)]) if layered
           else hw.build_homogeneous_acoustic(nx, ny, 1.0, 1.0))
    if not layered:  # per-cell beta: the non-row-uniform medium path
        med.planes["beta"] = med.planes["beta"] * (1.0 + 0.1 * rng.uniform(0.0, 1.0, (ny, nx)))
    dt = float(np.float16(0.45 * dx / med.c_max()))
    grid = hw.GridSpec(nx, ny, dx, dt, nt, order=order)
    src = hw.SourceSpec(hw.SourceKind.PRESSURE_POINT, nx // 2 + 1, src_row,
                        hw.RickerSpec(f_center=1.0 / (10 * dx), amplitude=amp))
    if recs is None:
        recs = ((nx // 2 + 1, src_row), (0, 0), (nx - 1, ny - 1), (7, ny // 2), (1023 % nx, 5), (1024 % nx, 6))
    s = hw.AcousticSolver(grid, med, src, stencil_precision=hw.Precision.FP16, receivers=recs, energy_every=every)
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
@pytest.mark.parametrize("nt", [20, 21])
def test_tb2_matches_oracle(variant, order, nt):
    s, st = _case(1024, 160, nt, order=order)
    ref = oracle.run_solver(s, variant, st)
    out = s.run(variant, st)
    assert s.kernel_path() == "fused2d-tb2"
    _check(s, st, out, ref)


@pytest.mark.parametrize("nx,ny", [(256, 16), (512, 40), (2048, 64), (3072, 50)])
def test_tb2_tiles_bands_and_media(nx, ny):
    s, st = _case(nx, ny, 12, every=1, layered=(nx != 2048))
    ref = oracle.run_solver(s, hw.Variant.OP3, st)
    out = s.run(hw.Variant.OP3, st)
    assert s.kernel_path() == "fused2d-tb2"
    _check(s, st, out, ref)


def test_tb2_equals_single_step_kernel(hwopt):
    recs = tuple((x, 9) for x in range(0, 4096, 7)) + tuple((1000, y) for y in range(0, 256, 3))
    s1, st1 = _case(4096, 256, 26, every=1, recs=recs)
    out1 = s1.run(hw.Variant.OP6, st1)
    assert s1.kernel_path() == "fused2d-tb2"
    hwopt(tb=0)
    s2, st2 = _case(4096, 256, 26, every=1, recs=recs)
    out2 = s2.run(hw.Variant.OP6, st2)
    assert s2.kernel_path() == "fused2d"
    for n in s1.FIELDS:
        assert_same_bits(getattr(st1, n).values, getattr(st2, n).values, n)
    np.testing.assert_array_equal(np.array([t.samples for t in out1.traces]),
                                  np.array([t.samples for t in out2.traces]))
    np.testing.assert_allclose(out1.energy.values, out2.energy.values, rtol=1e-12)


def test_tb2_range_failure_either_step_of_a_pair():
    parities = set()
    for amp in (3e4, 6e4, 1.2e5, 2.5e5, 5e5, 1e6, 2e6, 4e6, 1e9):
        s, st = _case(512, 64, 60, amp=amp, layered=False)
        ref = oracle.run_solver(s, None, st)
        if ref["fail"] is None:
            continue
        with pytest.raises(hw.RangeFailureError) as err:
            s.run(None, st)
        assert err.value.step == ref["fail"][0]
        assert err.value.field_name == s._fail_name(ref["fail"][1])
        assert st.step == ref["fail"][0] + 1
        for j, n in enumerate(s.FIELDS):
            assert_same_bits(getattr(st, n).values, ref["fields"][j], n)
        parities.add(ref["fail"][0] % 2)
    assert parities == {0, 1}


def test_tb2_resume_across_calls():
    s, st = _case(1024, 64, 5)
    ref = oracle.run_solver(s, hw.Variant.OP6, st, nt=13)
    s.run(hw.Variant.OP6, st)  # 5 steps: two pairs + one single
    s.step_compensated(st, hw.Variant.OP6)
    s.run(hw.Variant.OP6, st)
    s.step_compensated(st, hw.Variant.OP6)
    s.step_compensated(st, hw.Variant.OP6)
    assert st.step == 13
    for j, n in enumerate(s.FIELDS):
        assert_same_bits(getattr(st, n).values, ref["fields"][j], n)

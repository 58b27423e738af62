"""GPU parity: the sm_100a path through the C ABI against the reference goldens
and the CPU oracle.

Bar (north_star): per-step fields bit-exact (fp16/fp32/fp64 IEEE ops, no FMA
contraction, the reference's fold order); receiver traces bit-exact; energy
within ENERGY_RTOL relative (fp64 sums, order not pinned by the reference).
"""

import numpy as np
import pytest

import oracle
import paper_2310_00236_b200 as hw
from golden_cases import Case, assert_same_bits, names

pytestmark = pytest.mark.gpu

ENERGY_RTOL = 1e-12


def _run_names():
    return [n for n in names() if not Case(n).d["steps_api"]]


@pytest.fixture(params=["auto", "fast", "ieee"])
def div_mode(request, hwopt):
    """Run under each binary16 division path: table-verified cheap (auto), branch-free exact, IEEE."""
    if request.param != "auto":
        hwopt(div={"fast": 1, "ieee": 2}[request.param])
    return request.param


@pytest.mark.parametrize("name", _run_names())
def test_gpu_run_matches_reference_golden(name, div_mode):
    case = Case(name)
    solver = case.solver()
    st = case.initial_state(solver)
    want_fail = case.d.get("fail")
    if want_fail:
        with pytest.raises(hw.RangeFailureError) as err:
            solver.run(case.variant, st)
        assert err.value.step == want_fail[0]
        assert err.value.field_name == want_fail[1]
        assert st.step == case.d["final_step"]
    else:
        out = solver.run(case.variant, st)
        got = np.array([t.samples for t in out.traces]).reshape(case.z["traces"].shape)
        np.testing.assert_array_equal(got, case.z["traces"])
        np.testing.assert_array_equal(out.energy.times, case.z["e_times"])
        np.testing.assert_allclose(out.energy.values, case.z["e_vals"], rtol=ENERGY_RTOL, atol=0)
        assert st.step == case.d["nt"]
    for n in solver.FIELDS:
        assert_same_bits(getattr(st, n).values, case.z[f"final_{n}"], f"{name}:{n}")


@pytest.mark.parametrize("name", [n for n in names() if Case(n).d["steps_api"]])
def test_gpu_single_steps_match_reference_golden(name):
    case = Case(name)
    solver = case.solver()
    st = case.initial_state(solver)
    for k in range(case.d["steps_api"]):
        if case.variant is None:
            solver.step_baseline(st)
        else:
            solver.step_compensated(st, case.variant)
        for n in solver.FIELDS:
            assert_same_bits(getattr(st, n).values, case.z[f"step{k}_{n}"], f"{name}: step {k} {n}")
    assert st.step == case.d["steps_api"]


def _acoustic(n_x, n_y, nt, prec, *, seed=0, every=7, layered=False, order=4):
    rng = np.random.default_rng(seed)
    dx = 1.0 / n_x
    if layered:
        med = hw.build_layered_acoustic(n_x, n_y, [(0.5, 1.0, 1.0), (1.0, 1.5, 2.25)])
    else:
        med = hw.build_homogeneous_acoustic(n_x, n_y, 1.0, 1.0)
    dt = float(np.float16(0.4 * dx / np.sqrt(2.25 / 1.5)))
    grid = hw.GridSpec(n_x, n_y, dx, dt, nt, order=order)
    src = hw.SourceSpec(hw.SourceKind.PRESSURE_POINT, n_x // 2, 3,
                        hw.RickerSpec(f_center=1.0 / (10 * dx), amplitude=2.0))
    s = hw.AcousticSolver(grid, med, src, stencil_precision=prec, update_precision=prec,
                          receivers=((n_x // 2, n_y // 2), (1, 1)), energy_every=every)
    st = s.new_state()
    yy, xx = np.mgrid[0:n_y, 0:n_x] / n_x
    p0 = np.exp(-((xx - 0.5) ** 2 + (yy - 0.5) ** 2) / 0.01) + rng.uniform(-1e-3, 1e-3, (n_y, n_x))
    st.p.values = p0.astype(st.p.values.dtype)
    return s, st


@pytest.mark.parametrize("variant", [None, hw.Variant.OP3, hw.Variant.OP6])
@pytest.mark.parametrize("prec", [hw.Precision.FP16, hw.Precision.FP32, hw.Precision.FP64])
def test_gpu_acoustic_layered_vs_oracle(variant, prec):
    s, st = _acoustic(256, 192, 150, prec, layered=True)
    ref = oracle.run_solver(s, variant, st)
    out = s.run(variant, st)
    for j, n in enumerate(s.FIELDS):
        assert_same_bits(getattr(st, n).values, ref["fields"][j], n)
    np.testing.assert_array_equal(np.array([t.samples for t in out.traces]), ref["traces"])
    np.testing.assert_allclose(out.energy.values, ref["e_vals"], rtol=ENERGY_RTOL)


@pytest.mark.parametrize("order", [2, 4])
def test_gpu_acoustic_order_vs_oracle(order):
    s, st = _acoustic(128, 128, 100, hw.Precision.FP16, order=order)
    ref = oracle.run_solver(s, hw.Variant.OP3, st)
    s.run(hw.Variant.OP3, st)
    for j, n in enumerate(s.FIELDS):
        assert_same_bits(getattr(st, n).values, ref["fields"][j], n)


def test_gpu_run_resumes_from_state_step():
    s, st = _acoustic(64, 64, 40, hw.Precision.FP16)
    ref = oracle.run_solver(s, hw.Variant.OP3, st, nt=80)
    s.run(hw.Variant.OP3, st)
    s.run(hw.Variant.OP3, st)
    assert st.step == 80
    for j, n in enumerate(s.FIELDS):
        assert_same_bits(getattr(st, n).values, ref["fields"][j], n)


def test_gpu_rerun_bit_identical():
    s, st = _acoustic(96, 80, 60, hw.Precision.FP16)
    st2 = s.new_state()
    for n in s.FIELDS:
        getattr(st2, n).values = getattr(st, n).values.copy()
    a = s.run(hw.Variant.OP3, st)
    b = s.run(hw.Variant.OP3, st2)
    assert a.energy.values.tobytes() == b.energy.values.tobytes()
    for ta, tb in zip(a.traces, b.traces):
        assert ta.samples.tobytes() == tb.samples.tobytes()


def test_gpu_zero_state_stays_zero():
    g = hw.GridSpec(32, 32, 0.032, 0.01, 25)
    s = hw.AcousticSolver(g, hw.build_homogeneous_acoustic(32, 32, 1.0, 1.0), None,
                          stencil_precision=hw.Precision.FP16, receivers=((3, 4),))
    out = s.run(hw.Variant.OP3)
    assert np.all(out.traces[0].samples == 0.0)
    assert np.all(out.energy.values == 0.0)


def test_gpu_nt_zero_initial_energy_only():
    g = hw.GridSpec(16, 16, 0.032, 0.01, 0)
    s = hw.AcousticSolver(g, hw.build_homogeneous_acoustic(16, 16, 1.0, 1.0), None, receivers=((1, 1),))
    out = s.run()
    assert out.traces[0].samples.shape == (0,)
    assert list(out.energy.times) == [0.0]


def _elastic(n_x, n_y, nt, prec, fs=True, seed=0, kind=hw.SourceKind.VY_POINT):
    dx = 0.05
    med = hw.build_layered_elastic(n_x, n_y, [(0.5, 2.0, 2.0, 1.0), (1.0, 2.3, 2.8, 1.4)])
    bc = hw.Boundary.FREE_SURFACE if fs else hw.Boundary.PERIODIC
    grid = hw.GridSpec(n_x, n_y, dx, 0.01, nt, bc_y=bc)
    src = hw.SourceSpec(kind, n_x // 2, 6, hw.RickerSpec(5.0, amplitude=20.0))
    s = hw.ElasticSolver(grid, med, src, stencil_precision=prec, update_precision=prec,
                         receivers=((n_x // 2, 6), (3, n_y // 2)), energy_every=5)
    st = s.new_state()
    rng = np.random.default_rng(seed)
    st.sxx.values = rng.uniform(-0.1, 0.1, st.sxx.values.shape).astype(st.sxx.values.dtype)
    return s, st


@pytest.mark.parametrize("fs", [True, False])
@pytest.mark.parametrize("variant", [None, hw.Variant.OP3, hw.Variant.OP6])
def test_gpu_elastic_vs_oracle(fs, variant):
    s, st = _elastic(192, 160, 120, hw.Precision.FP16, fs=fs)
    ref = oracle.run_solver(s, variant, st)
    out = s.run(variant, st)
    for j, n in enumerate(s.FIELDS):
        assert_same_bits(getattr(st, n).values, ref["fields"][j], n)
    np.testing.assert_array_equal(np.array([t.samples for t in out.traces]), ref["traces"])
    np.testing.assert_allclose(out.energy.values, ref["e_vals"], rtol=ENERGY_RTOL)


def test_gpu_elastic_explosive_source_vs_oracle():
    s, st = _elastic(96, 96, 80, hw.Precision.FP16, fs=True, kind=hw.SourceKind.EXPLOSIVE)
    ref = oracle.run_solver(s, hw.Variant.OP6, st)
    s.run(hw.Variant.OP6, st)
    for j, n in enumerate(s.FIELDS):
        assert_same_bits(getattr(st, n).values, ref["fields"][j], n)


def test_gpu_free_surface_syy_rows_bit_zero():
    s, st = _elastic(64, 48, 90, hw.Precision.FP16, fs=True)
    st.sxx.values[:] = 0
    s.run(hw.Variant.OP6, st)
    for rows in (st.syy.values, st.rsyy.values):
        assert np.all(rows[0].view(np.uint16) == 0)
        assert np.all(rows[-1].view(np.uint16) == 0)
    assert np.any(st.syy.values[1:-1] != 0.0)


def test_gpu_fast_fp16_division_exhaustive():
    """The branch-free binary16 division equals the IEEE path on all 2^16 x (2^16-2050) pairs."""
    import ctypes

    from paper_2310_00236_b200 import _abi

    bad, first = ctypes.c_uint64(0), ctypes.c_uint32(0)
    _abi.check(_abi.load().hw_selftest_div16(0, ctypes.byref(bad), ctypes.byref(first)), "selftest")
    assert bad.value == 0, f"{bad.value} mismatches; first a,b = {first.value >> 16:#06x},{first.value & 0xffff:#06x}"


def test_gpu_cheap_division_table_verified_on_cpu():
    """Independently re-check, with numpy on the CPU, the device's exhaustive table of
    divisors for which fl16(fl32(a * rcp(b))) is the correctly rounded quotient."""
    import ctypes

    from paper_2310_00236_b200 import _abi

    words = (ctypes.c_uint32 * 1024)()
    _abi.check(_abi.load().hw_cheap_div_table(0, words), "table")
    bits = np.array(words, dtype=np.uint32)
    member = lambda b: bool((bits[b >> 5] >> (b & 31)) & 1)
    for b in (0x3c00, 0x3e00, 0x4080):  # 1.0, 1.5, 2.25 (the layered media): must qualify
        assert member(b)
    rng = np.random.default_rng(0)
    a = np.arange(65536, dtype=np.uint16).view(np.float16)
    finite = np.isfinite(a)
    checked = {True: 0, False: 0}
    for b in rng.integers(1, 0x7c00, 120):
        hb = np.uint16(b).view(np.float16)
        rcp = np.float32(1.0) / np.float32(hb)
        with np.errstate(all="ignore"):
            cheap = (a.astype(np.float32) * rcp).astype(np.float16)
            exact = (a.astype(np.float64) / np.float64(hb)).astype(np.float16)
        same = (cheap.view(np.uint16) == exact.view(np.uint16)) | (np.isnan(cheap) & np.isnan(exact))
        assert bool(same.all()) == member(int(b)), f"table disagrees for b={int(b):#06x}"
        checked[member(int(b))] += 1
    assert checked[True] > 0


def test_gpu_layered_media_use_cheap_division():
    s, st = _acoustic(256, 64, 2, hw.Precision.FP16, layered=True)
    s.run(hw.Variant.OP3, st)
    from paper_2310_00236_b200 import _abi

    lib = _abi.load()
    for pl in (_abi.PL_RHO_X, _abi.PL_RHO_S, _abi.PL_BETA):
        assert lib.hw_plane_div_mode(s._lib_handle(), pl) == 3

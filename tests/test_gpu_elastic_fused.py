"""The one-pass 2D elastic step (csrc/hw_elastic2d_fused.cu: binary16, single domain,
ping-pong buffers, free surface or periodic) against the CPU oracle, the two-phase
streaming kernels and the generic kernels: bit-exact fields, traces and failure steps;
energy within 1e-12 (block partials summed in a different order)."""

import numpy as np
import pytest

import oracle
import paper_2310_00236_b200 as hw
from golden_cases import assert_same_bits
from test_gpu_elastic_stream import _case, _check

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True)
def _no_small(hwopt):  # these grids would otherwise take the persistent small-grid kernel
    hwopt(small=0)


def _same(s1, st1, o1, s2, st2, o2):
    for n in s1.FIELDS:
        assert_same_bits(getattr(st1, n).values, getattr(st2, n).values, n)
    np.testing.assert_array_equal(np.array([t.samples for t in o1.traces]), np.array([t.samples for t in o2.traces]))
    np.testing.assert_array_equal(o1.energy.times, o2.energy.times)
    np.testing.assert_allclose(o1.energy.values, o2.energy.values, rtol=1e-12)


@pytest.mark.parametrize("variant", [None, hw.Variant.OP3, hw.Variant.OP6])
@pytest.mark.parametrize("order", [2, 4])
@pytest.mark.parametrize("fs", [True, False])
def test_fused_el_matches_oracle(variant, order, fs):
    s, st = _case(256, 160, 45, fs=fs, order=order)
    ref = oracle.run_solver(s, variant, st)
    out = s.run(variant, st)
    assert s.kernel_path() == "fused2d-el"
    assert s.last_launch_count() == 2 + 45
    _check(s, st, out, ref)


@pytest.mark.parametrize("ny", [8, 9, 13, 64, 600])
@pytest.mark.parametrize("fs", [True, False])
@pytest.mark.parametrize("order", [2, 4])
def test_fused_el_row_bands(ny, fs, order):
    """Row bands of 1..5 rows per CTA (every CTA touches a surface / wrap halo) to 4+."""
    s, st = _case(256, ny, 20, fs=fs, order=order, src_row=min(6, ny - 1))
    ref = oracle.run_solver(s, hw.Variant.OP6, st)
    out = s.run(hw.Variant.OP6, st)
    assert s.kernel_path() == "fused2d-el"
    _check(s, st, out, ref)


@pytest.mark.parametrize("fs", [True, False])
def test_fused_el_full_medium_and_explosive_source(fs):
    s, st = _case(512, 96, 41, fs=fs, full=True, kind=hw.SourceKind.EXPLOSIVE)
    ref = oracle.run_solver(s, hw.Variant.OP6, st)
    out = s.run(hw.Variant.OP6, st)
    assert s.kernel_path() == "fused2d-el"
    _check(s, st, out, ref)


@pytest.mark.parametrize("nt", [39, 40])
def test_fused_el_equals_stream_and_generic(hwopt, nt):
    s1, st1 = _case(1024, 300, nt, full=True)
    o1 = s1.run(hw.Variant.OP6, st1)
    assert s1.kernel_path() == "fused2d-el"
    hwopt(fused_el=0)
    s2, st2 = _case(1024, 300, nt, full=True)
    o2 = s2.run(hw.Variant.OP6, st2)
    assert s2.kernel_path() == "stream2d"
    _same(s1, st1, o1, s2, st2, o2)
    hwopt(path=1)
    s3, st3 = _case(1024, 300, nt, full=True)
    o3 = s3.run(hw.Variant.OP6, st3)
    assert s3.kernel_path() == "generic"
    _same(s1, st1, o1, s3, st3, o3)


@pytest.mark.parametrize("variant", [None, hw.Variant.OP6])
def test_fused_el_range_failure_matches_oracle(variant):
    s, st = _case(256, 64, 300, amp=1e8)
    assert s.kernel_path() == "fused2d-el"
    ref = oracle.run_solver(s, variant, st)
    assert ref["fail"] is not None
    with pytest.raises(hw.RangeFailureError) as err:
        s.run(variant, st)
    assert err.value.step == ref["fail"][0]
    assert err.value.field_name == s._fail_name(ref["fail"][1])
    for j, n in enumerate(s.FIELDS):
        assert_same_bits(getattr(st, n).values, ref["fields"][j], n)


def test_fused_el_single_steps_and_resume():
    s, st = _case(256, 40, 3)
    ref = oracle.run_solver(s, hw.Variant.OP3, st, nt=8)
    s.step_compensated(st, hw.Variant.OP3)
    s.run(hw.Variant.OP3, st)
    s.step_compensated(st, hw.Variant.OP3)
    s.run(hw.Variant.OP3, st)
    assert st.step == 8 and s.kernel_path() == "fused2d-el"
    for j, n in enumerate(s.FIELDS):
        assert_same_bits(getattr(st, n).values, ref["fields"][j], n)


def test_fused_el_receivers_on_every_row():
    nx, ny = 256, 40
    s0, _ = _case(nx, ny, 1)
    recs = tuple((x, y) for y in range(ny) for x in range(0, nx, 9))
    s, st = _case(nx, ny, 12)
    s = hw.ElasticSolver(s.grid, s.medium, s.source, stencil_precision=hw.Precision.FP16, receivers=recs,
                         energy_every=3)
    ref = oracle.run_solver(s, hw.Variant.OP6, st)
    out = s.run(hw.Variant.OP6, st)
    assert s.kernel_path() == "fused2d-el"
    _check(s, st, out, ref)


def test_fused_el_free_surface_syy_rows_bit_zero():
    s, st = _case(256, 48, 60)
    st.sxx.values[:] = 0
    s.run(hw.Variant.OP6, st)
    assert s.kernel_path() == "fused2d-el"
    for rows in (st.syy.values, st.rsyy.values):
        assert np.all(rows[0].view(np.uint16) == 0)
        assert np.all(rows[-1].view(np.uint16) == 0)
    assert np.any(st.syy.values[1:-1] != 0.0)


@pytest.mark.parametrize("fs", [True, False])
def test_fused_el_width_not_multiple_of_256(fs):
    """nx = 1000: 125 threads per CTA (a partial last warp) on a grid large enough for the one-pass path."""
    s, st = _case(1000, 2100, 6, fs=fs, src_row=700, every=3)
    assert s.kernel_path() == "fused2d-el"
    ref = oracle.run_solver(s, hw.Variant.OP6, st)
    out = s.run(hw.Variant.OP6, st)
    _check(s, st, out, ref)

"""The one-pass 3D acoustic step (csrc/hw_acoustic3d_fused.cu: 2nd order, binary16,
single domain, ping-pong buffers) against the CPU oracle, the two-phase streaming
kernels and the generic kernels: bit-exact fields, traces and failure steps; energy
within 1e-12 (block partials summed in a different order)."""

import numpy as np
import pytest

import oracle
import paper_2310_00236_b200 as hw
from golden_cases import assert_same_bits
from test_gpu_acoustic3d_stream import _case, _check

pytestmark = pytest.mark.gpu


def _same(s1, st1, o1, s2, st2, o2):
    for n in s1.FIELDS:
        assert_same_bits(getattr(st1, n).values, getattr(st2, n).values, n)
    np.testing.assert_array_equal(np.array([t.samples for t in o1.traces]), np.array([t.samples for t in o2.traces]))
    np.testing.assert_array_equal(o1.energy.times, o2.energy.times)
    np.testing.assert_allclose(o1.energy.values, o2.energy.values, rtol=1e-12)


@pytest.mark.parametrize("variant", [None, hw.Variant.OP3, hw.Variant.OP6])
@pytest.mark.parametrize("full", [True, False])
def test_fused3d_matches_oracle(variant, full):
    s, st = _case(256, 32, 20, 13, full=full)  # TM = 16: two mid tiles, wrap on both sides; odd nt
    ref = oracle.run_solver(s, variant, st)
    out = s.run(variant, st)
    assert s.kernel_path() == "fused3d"
    assert s.last_launch_count() == 2 + 13
    _check(s, st, out, ref)


@pytest.mark.parametrize("nx,ny", [(512, 16), (1024, 8), (256, 16)])
@pytest.mark.parametrize("nz", [9, 31, 64])
def test_fused3d_tiles_and_slab_splits(nx, ny, nz):
    s, st = _case(nx, ny, nz, 6, full=False)
    ref = oracle.run_solver(s, hw.Variant.OP3, st)
    out = s.run(hw.Variant.OP3, st)
    assert s.kernel_path() == "fused3d"
    _check(s, st, out, ref)


@pytest.mark.parametrize("nt", [11, 12])
def test_fused3d_equals_two_phase_and_generic(hwopt, nt):
    s1, st1 = _case(512, 16, 24, nt)
    o1 = s1.run(hw.Variant.OP3, st1)
    assert s1.kernel_path() == "fused3d"
    hwopt(fused3=0)
    s2, st2 = _case(512, 16, 24, nt)
    o2 = s2.run(hw.Variant.OP3, st2)
    assert s2.kernel_path() == "stream3d"
    _same(s1, st1, o1, s2, st2, o2)
    hwopt(path=1)
    s3, st3 = _case(512, 16, 24, nt)
    o3 = s3.run(hw.Variant.OP3, st3)
    assert s3.kernel_path() == "generic"
    _same(s1, st1, o1, s3, st3, o3)


def test_fused3d_resume_and_step_api():
    """Two runs of 5 steps (buffer A current between calls, odd launch count) == the
    oracle's 10; three single steps == the oracle's 3."""
    a, sa = _case(256, 16, 12, 5)
    ref = oracle.run_solver(a, hw.Variant.OP6, sa, nt=10)
    a.run(hw.Variant.OP6, sa)
    a.run(hw.Variant.OP6, sa)
    assert a.kernel_path() == "fused3d" and sa.step == 10
    for j, n in enumerate(a.FIELDS):
        assert_same_bits(getattr(sa, n).values, ref["fields"][j], n)
    c, sc = _case(256, 16, 12, 9)
    r3 = oracle.run_solver(c, hw.Variant.OP6, sc, nt=3)
    for _ in range(3):
        c.step_compensated(sc, hw.Variant.OP6)
    for j, n in enumerate(c.FIELDS):
        assert_same_bits(getattr(sc, n).values, r3["fields"][j], n)


def test_fused3d_receivers_everywhere():
    nx, ny, nz = 256, 16, 12
    recs = tuple((x, y, z) for z in (0, 5, 11) for y in range(ny) for x in range(0, nx, 7))
    s, st = _case(nx, ny, nz, 7, recs=recs)
    ref = oracle.run_solver(s, hw.Variant.OP3, st)
    out = s.run(hw.Variant.OP3, st)
    assert s.kernel_path() == "fused3d"
    _check(s, st, out, ref)


@pytest.mark.parametrize("variant", [None, hw.Variant.OP3])
def test_fused3d_range_failure_matches_oracle(variant):
    s, st = _case(256, 16, 12, 200, amp=1e9)
    assert s.kernel_path() == "fused3d"
    ref = oracle.run_solver(s, variant, st)
    assert ref["fail"] is not None
    with pytest.raises(hw.RangeFailureError) as err:
        s.run(variant, st)
    assert err.value.step == ref["fail"][0]
    assert err.value.field_name == s._fail_name(ref["fail"][1])
    for j, n in enumerate(s.FIELDS):
        assert_same_bits(getattr(st, n).values, ref["fields"][j], n)


def test_fused3d_zero_steps_and_zero_state():
    s, st = _case(256, 16, 12, 0)
    before = [getattr(st, n).values.copy() for n in s.FIELDS]
    s.run(hw.Variant.OP3, st)
    for b, n in zip(before, s.FIELDS):
        assert_same_bits(getattr(st, n).values, b, n)
    z, sz = _case(256, 16, 12, 5, amp=0.0)
    for n in z.FIELDS:
        getattr(sz, n).values = np.zeros_like(getattr(sz, n).values)
    z.run(hw.Variant.OP3, sz)
    for n in z.FIELDS:
        assert not np.any(getattr(sz, n).values.view(np.uint16)), n


def test_fused3d_source_on_tile_and_slab_edges():
    """Pressure source on a mid-tile edge row and a slab-segment boundary (the halo rows and the
    warm-up slab recompute neighbours' values: the source must be injected exactly once)."""
    for iz, iy in ((0, 7), (5, 8), (11, 15)):
        s, st = _case(256, 16, 12, 9)
        src = hw.SourceSpec(hw.SourceKind.PRESSURE_POINT, 17, iy, hw.RickerSpec(1 / (10 * s.grid.dx), amplitude=5.0),
                            iz=iz)
        s = hw.AcousticSolver(s.grid, s.medium, src, stencil_precision=hw.Precision.FP16,
                              receivers=((17, iy, iz), (3, 0, 0)), energy_every=4)
        ref = oracle.run_solver(s, hw.Variant.OP3, st)
        out = s.run(hw.Variant.OP3, st)
        assert s.kernel_path() == "fused3d"
        _check(s, st, out, ref)

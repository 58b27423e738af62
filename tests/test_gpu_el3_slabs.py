"""The one-pass 3D elastic kernel (config 5's path) on slabs of a decomposed domain: one halo
exchange per step (HW_PLAN_FUSED_EL3: stress rows -2 .. L, old velocities of rows -1 and L),
the halo velocities recomputed from them.  Slab groups of 1..8 slabs on one GPU (the same plan
and kernel as the NCCL transport) must reproduce the single domain and the CPU oracle bit for
bit -- fields, traces, failure step and field -- and the energy history must be BIT-IDENTICAL
for every slab count (per-plane partials summed in global plane order, SURVEY §8 e), within
1e-12 of the oracle's."""

import numpy as np
import pytest

import oracle
import paper_2310_00236_b200 as hw
from golden_cases import assert_same_bits

pytestmark = pytest.mark.gpu


def _el3(slabs, *, kind=hw.SourceKind.VY_POINT, src_z=17, nt=14, amp=30.0, nz=48, distributed=False):
    nx, ny = 256, 16  # TM = 8: two mid tiles
    med = hw.build_layered_elastic(nx, ny, [(0.3, 1.0, 2.0, 1.0), (0.7, 1.4, 2.6, 1.3), (1.0, 1.8, 3.0, 1.6)], nz=nz)
    dx = 1.0 / nx
    g = hw.GridSpec(nx, ny, dx, float(np.float16(0.3 * dx / (med.c_max() * np.sqrt(3)))), nt, nz=nz, order=2)
    src = hw.SourceSpec(kind, 101, 9, hw.RickerSpec(1 / (10 * dx), amplitude=amp), iz=src_z)
    kw = dict(distributed=True) if distributed else dict(slabs=slabs)
    s = hw.ElasticSolver(g, med, src, stencil_precision=hw.Precision.FP16, energy_every=2,
                         receivers=((101, 9, src_z), (0, 0, 0), (255, 15, nz - 1), (7, 3, nz // 2), (9, 9, 23)), **kw)
    st = s.new_state()
    rng = np.random.default_rng(11)
    z, y, x = np.mgrid[0:nz, 0:ny, 0:nx]
    st.vz.values = (0.1 * np.exp(-((x - 128) ** 2 / 300.0 + (y - 8) ** 2 / 20.0 + (z - 20) ** 2 / 20.0))).astype(np.float16)
    st.sxx.values = rng.uniform(-0.05, 0.05, st.sxx.values.shape).astype(np.float16)
    st.syz.values = rng.uniform(-0.02, 0.02, st.syz.values.shape).astype(np.float16)
    st.rvx.values = rng.uniform(-1e-4, 1e-4, st.rvx.values.shape).astype(np.float16)
    return s, st


def _run(s, st, variant=hw.Variant.OP6):
    out = s.run(variant, st)
    assert s.kernel_path() == "fused3d-el", s.kernel_path()
    return out


@pytest.mark.parametrize("kind,src_z", [(hw.SourceKind.VY_POINT, 17), (hw.SourceKind.VY_POINT, 23),
                                        (hw.SourceKind.VY_POINT, 24), (hw.SourceKind.EXPLOSIVE, 24)])
def test_el3_slabs_1_to_8_bit_identical(kind, src_z):
    """Sources on slab boundary rows (z = 17, 23, 24 sit next to / on the edges of 2, 3, 4, 6 and 8
    slabs): the neighbour slab's recomputed halo velocity must include a v_slow source."""
    s1, st1 = _el3(1, kind=kind, src_z=src_z)
    ref = oracle.run_solver(s1, hw.Variant.OP6, st1)
    o1 = _run(s1, st1)
    for j, n in enumerate(s1.FIELDS):
        assert_same_bits(getattr(st1, n).values, ref["fields"][j], n)
    np.testing.assert_array_equal(np.array([t.samples for t in o1.traces]), ref["traces"])
    np.testing.assert_allclose(o1.energy.values, ref["e_vals"], rtol=1e-12)
    for k in (2, 3, 4, 5, 6, 7, 8):
        sk, stk = _el3(k, kind=kind, src_z=src_z)
        ok = _run(sk, stk)
        assert sk.transport() == 1
        for n in s1.FIELDS:
            assert_same_bits(getattr(stk, n).values, getattr(st1, n).values, n)
        np.testing.assert_array_equal(np.array([t.samples for t in ok.traces]),
                                      np.array([t.samples for t in o1.traces]))
        np.testing.assert_array_equal(ok.energy.times, o1.energy.times)
        np.testing.assert_array_equal(ok.energy.values, o1.energy.values)  # bit-identical for any slab count
        sk.close()


@pytest.mark.parametrize("variant", [None, hw.Variant.OP3])
def test_el3_slabs_variants(variant):
    s1, st1 = _el3(1, nt=9)
    o1 = _run(s1, st1, variant)
    s4, st4 = _el3(4, nt=9)
    o4 = _run(s4, st4, variant)
    for n in s1.FIELDS:
        assert_same_bits(getattr(st4, n).values, getattr(st1, n).values, n)
    np.testing.assert_array_equal(o4.energy.values, o1.energy.values)


def test_el3_slabs_range_failure():
    s1, st1 = _el3(1, nt=200, amp=1e9)
    ref = oracle.run_solver(s1, None, st1)
    assert ref["fail"] is not None
    with pytest.raises(hw.RangeFailureError) as e1:
        _run(s1, st1, None)
    s3, st3 = _el3(3, nt=200, amp=1e9)
    with pytest.raises(hw.RangeFailureError) as e3:
        s3.run(None, st3)
    assert (e1.value.step, e1.value.field_name) == (e3.value.step, e3.value.field_name) == \
        (ref["fail"][0], s1._fail_name(ref["fail"][1]))
    for j, n in enumerate(s1.FIELDS):
        assert_same_bits(getattr(st3, n).values, ref["fields"][j], n)

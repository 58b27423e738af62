"""The one-pass 3D elastic step (csrc/hw_elastic3d_fused.cu: 2nd order, binary16, single
periodic domain or a slab, ping-pong buffers, nx 256, 512 or 1024, media constant along x) against the CPU
oracle and the two-phase streaming kernels: bit-exact fields, traces and failure steps;
energy within 1e-12."""

import numpy as np
import pytest

import oracle
import paper_2310_00236_b200 as hw
from golden_cases import assert_same_bits
from test_gpu_elastic3d_stream import _case, _check

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True)
def _fused(hwopt):
    hwopt(fused_el3=1)


@pytest.mark.parametrize("variant", [None, hw.Variant.OP3, hw.Variant.OP6])
@pytest.mark.parametrize("kind", [hw.SourceKind.EXPLOSIVE, hw.SourceKind.VY_POINT])
def test_el3d_fused_matches_oracle(variant, kind):
    s, st = _case(256, 16, 14, 9, kind=kind)  # TM = 8: two mid tiles, wrap on both sides; odd nt
    ref = oracle.run_solver(s, variant, st)
    out = s.run(variant, st)
    assert s.kernel_path() == "fused3d-el"
    _check(s, st, out, ref)


@pytest.mark.parametrize("nx,ny,nz", [(512, 8, 9), (512, 16, 31), (256, 24, 20), (512, 12, 64)])
def test_el3d_fused_tiles_and_slab_splits(nx, ny, nz):
    s, st = _case(nx, ny, nz, 6, full=(nz == 20))
    ref = oracle.run_solver(s, hw.Variant.OP6, st)
    out = s.run(hw.Variant.OP6, st)
    # media varying along x (full planes) take the streaming kernels
    assert s.kernel_path() == ("stream3d" if nz == 20 else "fused3d-el")
    _check(s, st, out, ref)


@pytest.mark.parametrize("variant", [None, hw.Variant.OP3, hw.Variant.OP6])
@pytest.mark.parametrize("ny,nz", [(8, 9), (10, 33)])
def test_el3d_fused_nx1024(variant, ny, nz):
    """Rows of 1024 cells (the per-GPU slab width of BASELINE config 5's 1024^3 / 8-GPU grid): tiles of
    TM = 2 rows, a 3-slot tap ring with the slab-(F-2) values carried in registers, thread row 1 taking
    both upper halo rows."""
    s, st = _case(1024, ny, nz, 7, kind=hw.SourceKind.VY_POINT if nz == 9 else hw.SourceKind.EXPLOSIVE)
    ref = oracle.run_solver(s, variant, st)
    out = s.run(variant, st)
    assert s.kernel_path() == "fused3d-el"
    _check(s, st, out, ref)


def test_el3d_fused_nx1024_sources_on_tile_edges_and_slabs():
    for iy, iz, kind, slabs in ((1, 0, hw.SourceKind.VY_POINT, 1), (2, 5, hw.SourceKind.VY_POINT, 2),
                                (0, 11, hw.SourceKind.EXPLOSIVE, 3), (7, 6, hw.SourceKind.VY_POINT, 4)):
        s, st = _case(1024, 8, 24, 7)
        src = hw.SourceSpec(kind, 1023 if iy == 1 else 37, iy, hw.RickerSpec(1 / (10 * s.grid.dx), amplitude=30.0), iz=iz)
        s = hw.ElasticSolver(s.grid, s.medium, src, stencil_precision=hw.Precision.FP16, slabs=slabs,
                             receivers=((37, iy, iz), (1, 2, 3), (1023, 7, 23), (0, 0, 12)), energy_every=2)
        ref = oracle.run_solver(s, hw.Variant.OP6, st)
        out = s.run(hw.Variant.OP6, st)
        assert s.kernel_path() == "fused3d-el" and s.transport() == (0 if slabs == 1 else 1)
        _check(s, st, out, ref)


def test_el3d_fused_sources_on_tile_edges():
    for iy, iz, kind in ((7, 0, hw.SourceKind.VY_POINT), (8, 5, hw.SourceKind.VY_POINT), (0, 13, hw.SourceKind.EXPLOSIVE),
                         (15, 6, hw.SourceKind.VY_POINT)):
        s, st = _case(256, 16, 14, 7)
        src = hw.SourceSpec(kind, 37, iy, hw.RickerSpec(1 / (10 * s.grid.dx), amplitude=30.0), iz=iz)
        s = hw.ElasticSolver(s.grid, s.medium, src, stencil_precision=hw.Precision.FP16,
                             receivers=((37, iy, iz), (1, 2, 3)), energy_every=2)
        ref = oracle.run_solver(s, hw.Variant.OP6, st)
        out = s.run(hw.Variant.OP6, st)
        assert s.kernel_path() == "fused3d-el"
        _check(s, st, out, ref)


@pytest.mark.parametrize("nt", [7, 8])
def test_el3d_fused_equals_two_phase(hwopt, nt):
    s1, st1 = _case(512, 16, 24, nt)
    o1 = s1.run(hw.Variant.OP6, st1)
    assert s1.kernel_path() == "fused3d-el"
    hwopt(fused_el3=0)
    s2, st2 = _case(512, 16, 24, nt)
    o2 = s2.run(hw.Variant.OP6, st2)
    assert s2.kernel_path() == "stream3d"
    for n in s1.FIELDS:
        assert_same_bits(getattr(st1, n).values, getattr(st2, n).values, n)
    np.testing.assert_array_equal(np.array([t.samples for t in o1.traces]), np.array([t.samples for t in o2.traces]))
    np.testing.assert_allclose(o1.energy.values, o2.energy.values, rtol=1e-12)


def test_el3d_fused_range_failure_and_resume():
    s, st = _case(256, 16, 12, 200, amp=1e9)
    ref = oracle.run_solver(s, None, st)
    assert ref["fail"] is not None
    with pytest.raises(hw.RangeFailureError) as err:
        s.run(None, st)
    assert s.kernel_path() == "fused3d-el"
    assert err.value.step == ref["fail"][0]
    assert err.value.field_name == s._fail_name(ref["fail"][1])
    for j, n in enumerate(s.FIELDS):
        assert_same_bits(getattr(st, n).values, ref["fields"][j], n)
    a, sa = _case(256, 16, 12, 3)
    ref = oracle.run_solver(a, hw.Variant.OP3, sa, nt=7)
    a.run(hw.Variant.OP3, sa)
    a.step_compensated(sa, hw.Variant.OP3)
    a.run(hw.Variant.OP3, sa)
    for j, n in enumerate(a.FIELDS):
        assert_same_bits(getattr(sa, n).values, ref["fields"][j], n)


@pytest.mark.parametrize("rho", [1.0, 1.37, 0.61])
def test_el3d_fused_every_division_mode(rho):
    """Densities whose binary16 divisors take the verified-reciprocal, the fast exact and the IEEE
    paths: the kernel picks the mode per plane (hw_plane_div_mode) and stays bit-exact."""
    nx, ny, nz = 256, 16, 10
    med = hw.build_layered_elastic(nx, ny, [(0.5, rho, 2.0, 1.0), (1.0, 1.7 * rho, 2.6, 1.2)], nz=nz)
    dx = 1.0 / nx
    g = hw.GridSpec(nx, ny, dx, float(np.float16(0.3 * dx / (med.c_max() * np.sqrt(3)))), 5, nz=nz, order=2)
    s = hw.ElasticSolver(g, med, None, stencil_precision=hw.Precision.FP16, receivers=((3, 4, 5),), energy_every=2)
    st = s.new_state()
    rng = np.random.default_rng(7)
    for name in ("vx", "vy", "vz", "sxx", "syz"):
        getattr(st, name).values = rng.uniform(-0.1, 0.1, getattr(st, name).values.shape).astype(np.float16)
    ref = oracle.run_solver(s, hw.Variant.OP6, st)
    out = s.run(hw.Variant.OP6, st)
    assert s.kernel_path() == "fused3d-el"
    _check(s, st, out, ref)

"""The one-pass 3D acoustic step in binary32 lanes (csrc/hw_acoustic3d_fused32.cu: 2nd order,
S = U = fp32, single domain, ping-pong buffers; BASELINE config 3's "fp32 naive" arm) against
the CPU oracle and the generic fp32 kernels: bit-exact fields, traces and failure steps;
energy within 1e-12 (block partials summed in a different order)."""

import numpy as np
import pytest

import oracle
import paper_2310_00236_b200 as hw
from golden_cases import assert_same_bits

pytestmark = pytest.mark.gpu
F32 = hw.Precision.FP32


def _case(nx, ny, nz, nt, *, full=True, layers=((0.4, 1.0, 1.5), (1.0, 1.3, 3.0)), amp=5.0, seed=0, recs=None,
          every=4):
    rng = np.random.default_rng(seed)
    if full:
        med = hw.build_acoustic_from_velocity(1.5 + 3.0 * rng.random((nz, ny, nx)))
    else:
        med = hw.build_layered_acoustic(nx, ny, list(layers), nz=nz)
    dx = 1.0 / nx
    dt = float(np.float16(0.4 * dx / (med.c_max() * np.sqrt(3))))
    g = hw.GridSpec(nx, ny, dx, dt, nt, nz=nz, order=2)
    src = hw.SourceSpec(hw.SourceKind.PRESSURE_POINT, nx // 2 + 3, ny // 2, hw.RickerSpec(1 / (10 * dx), amplitude=amp),
                        iz=nz // 3)
    if recs is None:
        recs = ((nx // 2 + 3, ny // 2, nz // 3), (0, 0, 0), (nx - 1, ny - 1, nz - 1), (7, 1, nz // 2), (8, ny - 2, 1))
    s = hw.AcousticSolver(g, med, src, stencil_precision=F32, receivers=recs, energy_every=every)
    st = s.new_state()
    z, y, x = np.mgrid[0:nz, 0:ny, 0:nx]
    st.p.values = (np.exp(-((x - nx / 2) ** 2 / 400.0 + (y - ny / 3) ** 2 / 30.0 + (z - nz / 2) ** 2 / 30.0))
                   + rng.uniform(-1e-3, 1e-3, (nz, ny, nx))).astype(np.float32)
    st.vx.values = rng.uniform(-0.01, 0.01, (nz, ny, nx)).astype(np.float32)
    return s, st


def _check(s, st, out, ref):
    for j, n in enumerate(s.FIELDS):
        assert_same_bits(getattr(st, n).values, ref["fields"][j], n)
    np.testing.assert_array_equal(np.array([t.samples for t in out.traces]), ref["traces"])
    np.testing.assert_array_equal(out.energy.times, ref["e_times"])
    np.testing.assert_allclose(out.energy.values, ref["e_vals"], rtol=1e-12)


@pytest.mark.parametrize("variant", [None, hw.Variant.OP3, hw.Variant.OP6])
@pytest.mark.parametrize("full", [True, False])
def test_fused3d_f32_matches_oracle(variant, full):
    s, st = _case(256, 32, 20, 13, full=full)  # TM = 8: four mid tiles, wrap on both sides; odd nt
    assert getattr(st, "p").values.dtype == np.float32
    ref = oracle.run_solver(s, variant, st)
    out = s.run(variant, st)
    assert s.kernel_path() == "fused3d-f32"
    assert s.last_launch_count() == 2 + 13
    _check(s, st, out, ref)


@pytest.mark.parametrize("nx,ny", [(512, 8), (128, 32), (256, 16)])
@pytest.mark.parametrize("nz", [9, 31, 64])
def test_fused3d_f32_tiles_and_slab_splits(nx, ny, nz):
    s, st = _case(nx, ny, nz, 6, full=False)
    ref = oracle.run_solver(s, None, st)
    out = s.run(None, st)
    assert s.kernel_path() == "fused3d-f32"
    _check(s, st, out, ref)


@pytest.mark.parametrize("layers", [((0.5, 1.0, 1.0), (1.0, 2.0, 4.0)),        # power-of-two rho and beta rows
                                    ((0.3, 0.5, 0.25), (0.7, 1.7, 2.3), (1.0, 2.0, 9.0))])
def test_fused3d_f32_row_divisors(layers):
    """Row-uniform divisors: powers of two take the exact-reciprocal multiply, others __fdiv_rn."""
    s, st = _case(256, 16, 24, 9, full=False, layers=layers)
    ref = oracle.run_solver(s, hw.Variant.OP3, st)
    out = s.run(hw.Variant.OP3, st)
    assert s.kernel_path() == "fused3d-f32"
    _check(s, st, out, ref)


@pytest.mark.parametrize("nt", [11, 12])
def test_fused3d_f32_equals_generic(hwopt, nt):
    s1, st1 = _case(512, 16, 24, nt)
    o1 = s1.run(None, st1)
    assert s1.kernel_path() == "fused3d-f32"
    hwopt(path=1)
    s2, st2 = _case(512, 16, 24, nt)
    o2 = s2.run(None, st2)
    assert s2.kernel_path() == "generic"
    for n in s1.FIELDS:
        assert_same_bits(getattr(st1, n).values, getattr(st2, n).values, n)
    np.testing.assert_array_equal(np.array([t.samples for t in o1.traces]), np.array([t.samples for t in o2.traces]))
    np.testing.assert_allclose(o1.energy.values, o2.energy.values, rtol=1e-12)


def test_fused3d_f32_resume_and_step_api():
    a, sa = _case(256, 16, 12, 5)
    ref = oracle.run_solver(a, None, sa, nt=10)
    a.run(None, sa)
    a.run(None, sa)
    assert a.kernel_path() == "fused3d-f32" and sa.step == 10
    for j, n in enumerate(a.FIELDS):
        assert_same_bits(getattr(sa, n).values, ref["fields"][j], n)
    c, sc = _case(256, 16, 12, 9)
    r3 = oracle.run_solver(c, hw.Variant.OP6, sc, nt=3)
    for _ in range(3):
        c.step_compensated(sc, hw.Variant.OP6)
    for j, n in enumerate(c.FIELDS):
        assert_same_bits(getattr(sc, n).values, r3["fields"][j], n)


def test_fused3d_f32_receivers_everywhere():
    nx, ny, nz = 256, 16, 12
    recs = tuple((x, y, z) for z in (0, 5, 11) for y in range(ny) for x in range(0, nx, 7))
    s, st = _case(nx, ny, nz, 7, recs=recs)
    ref = oracle.run_solver(s, None, st)
    out = s.run(None, st)
    assert s.kernel_path() == "fused3d-f32"
    _check(s, st, out, ref)


@pytest.mark.parametrize("variant", [None, hw.Variant.OP3])
def test_fused3d_f32_range_failure_matches_oracle(variant):
    s, st = _case(256, 16, 12, 400, amp=3.0e38)
    # p near 1.33e36, where the tap products c p (c = 1/dx = 256) leave binary32: overflow at step 200
    st.p.values = (st.p.values.astype(np.float64) * 1.25e36).astype(np.float32)
    assert s.kernel_path() == "fused3d-f32"
    ref = oracle.run_solver(s, variant, st)
    assert ref["fail"] is not None
    with pytest.raises(hw.RangeFailureError) as err:
        s.run(variant, st)
    assert err.value.step == ref["fail"][0]
    assert err.value.field_name == s._fail_name(ref["fail"][1])
    for j, n in enumerate(s.FIELDS):
        assert_same_bits(getattr(st, n).values, ref["fields"][j], n)


def test_fused3d_f32_source_on_tile_and_slab_edges():
    for iz, iy in ((0, 7), (5, 8), (11, 15)):
        s, st = _case(256, 16, 12, 9)
        src = hw.SourceSpec(hw.SourceKind.PRESSURE_POINT, 17, iy, hw.RickerSpec(1 / (10 * s.grid.dx), amplitude=5.0),
                            iz=iz)
        s = hw.AcousticSolver(s.grid, s.medium, src, stencil_precision=F32, receivers=((17, iy, iz), (3, 0, 0)),
                              energy_every=4)
        ref = oracle.run_solver(s, None, st)
        out = s.run(None, st)
        assert s.kernel_path() == "fused3d-f32"
        _check(s, st, out, ref)


@pytest.mark.parametrize("variant", [None, hw.Variant.OP3])
def test_fused3d_f32_per_cell_density(variant):
    """Density planes that vary along x take the per-cell division path (the other kernel
    instantiation); beta per cell as well."""
    nx, ny, nz = 256, 16, 12
    rng = np.random.default_rng(3)
    planes = {n: 1.0 + rng.random((nz, ny, nx)) for n in ("rho_x", "rho_y", "rho_z")}
    planes["beta"] = 0.2 + 0.3 * rng.random((nz, ny, nx))
    med = hw.Medium(hw.MediumKind.ACOUSTIC, nx, ny, planes, nz)
    s0, st = _case(nx, ny, nz, 7)
    s = hw.AcousticSolver(hw.GridSpec(nx, ny, 1.0 / nx, s0.grid.dt, 7, nz=nz, order=2), med, s0.source,
                          stencil_precision=F32, receivers=((5, 3, 2),), energy_every=3)
    ref = oracle.run_solver(s, variant, st)
    out = s.run(variant, st)
    assert s.kernel_path() == "fused3d-f32"
    _check(s, st, out, ref)

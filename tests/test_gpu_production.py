"""Oracle parity at the BASELINE configs' production shapes: short windows of the exact
benchmarked grids through the product kernels (the (tile, slab) work split, the CTA row
bands, shared-memory layouts and wrap-around indices of a real run), against the CPU oracle
(oracle/halfwave_oracle.c, all host threads).  Fields and receiver traces bit-exact, energy
within 1e-12, and the kernel family asserted (reference: acoustic.py:185-236,
elastic.py:242-296)."""

import numpy as np
import pytest

import oracle
import paper_2310_00236_b200 as hw
from golden_cases import assert_same_bits

pytestmark = pytest.mark.gpu

F16 = hw.Precision.FP16


def _check(s, st, out, ref, path):
    assert s.kernel_path() == path, s.kernel_path()
    for j, n in enumerate(s.FIELDS):
        assert_same_bits(getattr(st, n).values, ref["fields"][j], n)
    np.testing.assert_array_equal(np.array([t.samples for t in out.traces]).reshape(ref["traces"].shape),
                                  ref["traces"])
    np.testing.assert_array_equal(out.energy.times, ref["e_times"])
    np.testing.assert_allclose(out.energy.values, ref["e_vals"], rtol=1e-12)


def _run_both(s, variant, st, path):
    ref = oracle.run_solver(s, variant, st)
    out = s.run(variant, st)
    _check(s, st, out, ref, path)
    s.close()


def test_config2_fused2d_4096():
    """Config 2: 4096^2, 4th order, two-layer medium, Ricker at the top centre, fp16 op3 --
    the bench kernel at the bench width (512 threads x 8 cells, 148 row bands)."""
    n = 4096
    dx = 1.0 / n
    med = hw.build_layered_acoustic(n, n, [(0.5, 1.0, 1.0), (1.0, 1.5, 2.25)])
    dt = float(np.float16(0.5 * dx / med.c_max()))
    if dt > 0.5 * dx / med.c_max():
        dt = float(np.nextafter(np.float16(dt), np.float16(0)))
    src = hw.SourceSpec(hw.SourceKind.PRESSURE_POINT, n // 2, 8, hw.RickerSpec(f_center=1 / (10 * dx), amplitude=2.0e4))
    recs = ((n // 2, 8), (0, 0), (n - 1, n - 1), (1000, 1500), (3000, 2047), (4095, 2048), (17, 4000), (2048, 27))
    s = hw.AcousticSolver(hw.GridSpec(n, n, dx, dt, 12), med, src, stencil_precision=F16, receivers=recs,
                          energy_every=2)
    st = s.new_state()
    rng = np.random.default_rng(20)
    yy, xx = np.mgrid[0:n, 0:n] / n
    st.p.values = (np.exp(-((xx - 0.4) ** 2 + (yy - 0.6) ** 2) / 0.01) + rng.uniform(-1e-3, 1e-3, (n, n))).astype(np.float16)
    st.vx.values = rng.uniform(-0.05, 0.05, (n, n)).astype(np.float16)
    st.rp.values = rng.uniform(-1e-4, 1e-4, (n, n)).astype(np.float16)
    _run_both(s, hw.Variant.OP3, st, "fused2d")


@pytest.mark.parametrize("variant", [None, hw.Variant.OP6])
def test_config4_fused2d_el_4096(variant):
    """Config 4: 4096^2 elastic, free surface, explosive source, fp16 naive and op6."""
    n = 4096
    dx = 1.0 / n
    med = hw.build_layered_elastic(n, n, [(1.0, 1.0, 2.0, 1.0)])
    g = hw.GridSpec(n, n, dx, float(np.float16(0.4 * dx / 2)), 8, bc_y=hw.Boundary.FREE_SURFACE)
    src = hw.SourceSpec(hw.SourceKind.EXPLOSIVE, n // 2, 16, hw.RickerSpec(1 / (10 * dx), amplitude=1.0e3))
    recs = ((n // 2, 16), (0, 0), (5, 4095), (4095, 2000), (1234, 3000), (2048, 4095))
    s = hw.ElasticSolver(g, med, src, stencil_precision=F16, receivers=recs, energy_every=2)
    st = s.new_state()
    rng = np.random.default_rng(40)
    st.sxx.values = rng.uniform(-0.05, 0.05, st.sxx.values.shape).astype(np.float16)
    st.vy.values = rng.uniform(-0.02, 0.02, st.vy.values.shape).astype(np.float16)
    st.sxy.values = rng.uniform(-0.02, 0.02, st.sxy.values.shape).astype(np.float16)
    _run_both(s, variant, st, "fused2d-el")


def _config3(prec):
    n = 512
    rng = np.random.default_rng(30)
    med = hw.build_acoustic_from_velocity(1.5 + 3.0 * rng.random((n, n, n)))
    dx = 1.0 / n
    g = hw.GridSpec(n, n, dx, float(np.float16(0.5 * dx / (med.c_max() * np.sqrt(3)))), 3, nz=n, order=2)
    recs = ((0, 0, 0), (511, 511, 511), (256, 3, 100), (17, 400, 255))
    s = hw.AcousticSolver(g, med, stencil_precision=prec, receivers=recs, energy_every=1)
    st = s.new_state()
    a = np.arange(n) / n - 0.5
    p0 = np.exp(-(a[:, None, None] ** 2 + a[None, :, None] ** 2 + a[None, None, :] ** 2) / 0.01)
    st.p.values = p0.astype(st.p.values.dtype)
    st.vz.values = (0.01 * rng.standard_normal((n, n, n))).astype(st.vz.values.dtype)
    return s, st


def test_config3_fused3d_512():
    """Config 3: 512^3 acoustic, 2nd order, per-cell beta, Gaussian p0, fp16 op3."""
    s, st = _config3(F16)
    _run_both(s, hw.Variant.OP3, st, "fused3d")


def test_config3_fused3d_f32_512():
    """Config 3's fp32 naive arm at 512^3 (binary32 one-pass kernel)."""
    s, st = _config3(hw.Precision.FP32)
    _run_both(s, None, st, "fused3d-f32")


@pytest.mark.parametrize("path", ["fused3d-el", "stream3d"])
def test_config5_512(hwopt, path):
    """Config 5 on one GPU: 512^3 elastic, 2nd order, seeded layered lambda/mu/rho, Gaussian vz,
    fp16 op6 -- the one-pass kernel and the two-phase streaming kernels."""
    hwopt(fused_el3=1 if path == "fused3d-el" else 0)
    n = 512
    med = hw.build_layered_elastic(n, n, [(0.3, 1.0, 2.0, 1.0), (0.7, 1.4, 2.6, 1.3), (1.0, 1.8, 3.0, 1.6)], nz=n)
    dx = 1.0 / n
    g = hw.GridSpec(n, n, dx, float(np.float16(0.4 * dx / 3.0)), 2, nz=n, order=2)
    recs = ((0, 0, 0), (511, 511, 511), (256, 255, 154), (3, 508, 358))
    s = hw.ElasticSolver(g, med, stencil_precision=F16, receivers=recs, energy_every=1)
    st = s.new_state()
    a = np.arange(n) / n - 0.5
    st.vz.values = np.exp(-(a[:, None, None] ** 2 + a[None, :, None] ** 2 + a[None, None, :] ** 2) / 0.01).astype(np.float16)
    rng = np.random.default_rng(50)
    st.sxy.values = rng.uniform(-0.01, 0.01, st.sxy.values.shape).astype(np.float16)
    st.rsxx.values = rng.uniform(-1e-4, 1e-4, st.rsxx.values.shape).astype(np.float16)
    _run_both(s, hw.Variant.OP6, st, path)

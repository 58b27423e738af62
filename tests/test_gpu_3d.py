"""3D acoustic and elastic (SURVEY §8 a' extensions, BASELINE configs 3 and 5) on the
GPU against the CPU oracle: bit-exact fields and traces, energy within 1e-12."""

import numpy as np
import pytest

import oracle
import paper_2310_00236_b200 as hw
from golden_cases import assert_same_bits

pytestmark = pytest.mark.gpu


def _smooth_c(shape, seed=0):
    rng = np.random.default_rng(seed)
    f = rng.standard_normal(shape)
    k = [np.fft.fftfreq(n) for n in shape]
    kk = sum(np.meshgrid(*[ki ** 2 for ki in k], indexing="ij"))
    f = np.real(np.fft.ifftn(np.fft.fftn(f) * np.exp(-kk * 200.0)))
    f = (f - f.min()) / (f.max() - f.min())
    return 1.5 + 3.0 * f  # c in [1.5, 4.5] (BASELINE config 3)


def _check(s, st, out, ref):
    for j, n in enumerate(s.FIELDS):
        assert_same_bits(getattr(st, n).values, ref["fields"][j], n)
    np.testing.assert_array_equal(np.array([t.samples for t in out.traces]).reshape(ref["traces"].shape), ref["traces"])
    np.testing.assert_allclose(out.energy.values, ref["e_vals"], rtol=1e-12)


@pytest.mark.parametrize("order", [2, 4])
@pytest.mark.parametrize("variant", [None, hw.Variant.OP3])
def test_3d_acoustic_velocity_model_vs_oracle(order, variant):
    nz, ny, nx = 40, 24, 32
    c = _smooth_c((nz, ny, nx))
    med = hw.build_acoustic_from_velocity(c)
    dx = 1.0 / nx
    dt = float(np.float16(0.4 * dx / 4.5 / np.sqrt(3)))
    g = hw.GridSpec(nx, ny, dx, dt, 30, nz=nz, order=order)
    s = hw.AcousticSolver(g, med, stencil_precision=hw.Precision.FP16, receivers=((3, 4, 5), (16, 12, 20)),
                          energy_every=5)
    st = s.new_state()
    z, y, x = np.mgrid[0:nz, 0:ny, 0:nx]
    st.p.values = np.exp(-((x - 16) ** 2 + (y - 12) ** 2 + (z - 20) ** 2) / 20.0).astype(np.float16)
    ref = oracle.run_solver(s, variant, st)
    out = s.run(variant, st)
    _check(s, st, out, ref)


@pytest.mark.parametrize("variant", [hw.Variant.OP6, hw.Variant.OP3, None])
def test_3d_elastic_layered_vs_oracle(variant):
    nz, ny, nx = 32, 16, 24
    med = hw.build_layered_elastic(nx, ny, [(0.3, 1.0, 2.0, 1.0), (0.7, 1.4, 2.6, 1.3), (1.0, 1.8, 3.0, 1.6)], nz=nz)
    g = hw.GridSpec(nx, ny, 0.05, 0.004, 25, nz=nz, order=2)
    src = hw.SourceSpec(hw.SourceKind.EXPLOSIVE, 12, 8, hw.RickerSpec(10.0, amplitude=50.0), iz=10)
    s = hw.ElasticSolver(g, med, src, stencil_precision=hw.Precision.FP16, receivers=((12, 8, 14),), energy_every=5)
    st = s.new_state()
    z, y, x = np.mgrid[0:nz, 0:ny, 0:nx]
    st.vz.values = (0.1 * np.exp(-((x - 12) ** 2 + (y - 8) ** 2 + (z - 16) ** 2) / 12.0)).astype(np.float16)
    ref = oracle.run_solver(s, variant, st)
    out = s.run(variant, st)
    _check(s, st, out, ref)


def test_3d_mixed_lanes_vs_oracle():
    nz, ny, nx = 16, 12, 20
    g = hw.GridSpec(nx, ny, 0.05, 0.01, 12, nz=nz)
    s = hw.AcousticSolver(g, hw.build_homogeneous_acoustic(nx, ny, 1.0, 1.0, nz=nz),
                          stencil_precision=hw.Precision.FP32, update_precision=hw.Precision.FP16)
    st = s.new_state()
    st.p.values = np.random.default_rng(1).uniform(-1, 1, (nz, ny, nx)).astype(np.float16)
    ref = oracle.run_solver(s, hw.Variant.OP3, st)
    out = s.run(hw.Variant.OP3, st)
    _check(s, st, out, ref)


def test_3d_mu_zero_elastic_equals_acoustic_on_gpu():
    n, nt = 16, 30
    g = hw.GridSpec(n, n, 0.05, 0.01, nt, nz=n)
    ac = hw.AcousticSolver(g, hw.build_homogeneous_acoustic(n, n, 1.0, 2.0, nz=n), stencil_precision=hw.Precision.FP16)
    el = hw.ElasticSolver(g, hw.build_layered_elastic(n, n, [(1.0, 1.0, 2.0, 0.0)], nz=n),
                          stencil_precision=hw.Precision.FP16)
    sa, se = ac.new_state(), el.new_state()
    z, y, x = np.mgrid[0:n, 0:n, 0:n]
    blob = (0.5 * np.exp(-((x - 7) ** 2 + (y - 8) ** 2 + (z - 6) ** 2) / 8.0)).astype(np.float16)
    sa.p.values = blob.copy()
    for nm in ("sxx", "syy", "szz"):
        getattr(se, nm).values = blob.copy()
    ac.run(None, sa)
    el.run(None, se)
    for nm in ("sxx", "syy", "szz"):
        np.testing.assert_array_equal(getattr(se, nm).values, sa.p.values)
    for v in ("vx", "vy", "vz"):
        np.testing.assert_array_equal(getattr(se, v).values, getattr(sa, v).values)

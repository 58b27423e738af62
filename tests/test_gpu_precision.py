"""The paper's precision result on the B200 path, at reduced size (tools/precision_study.py runs
the full-size BASELINE configs): binary16 state with the compensated update (op3 / op6) keeps the
discrete energy (diagnostics.energy_drift, the reference's acceptance metric) far flatter than the
naive binary16 update, and binary32 naive is flatter still; fp64 is the reference arm.  The runs go
through the product kernels (fused3d, fused3d-f32, stream3d, fused2d) via solver.run()."""
import sys
from pathlib import Path

import numpy as np
import pytest

import paper_2310_00236_b200 as hw
from paper_2310_00236_b200.diagnostics import energy_drift

sys.path.insert(0, str(Path(__file__).resolve().parents[1] / "tools"))
import precision_study as ps  # noqa: E402

pytestmark = pytest.mark.gpu
F16, F32, F64 = hw.Precision.FP16, hw.Precision.FP32, hw.Precision.FP64


def _ac3(prec, n=256, nt=400):
    rng = np.random.default_rng(3)
    from scipy.ndimage import gaussian_filter

    c = gaussian_filter(rng.standard_normal((n, n, n)), sigma=4.0, mode="wrap")
    c = 1.5 + 3.0 * (c - c.min()) / (c.max() - c.min())
    med = hw.build_acoustic_from_velocity(c)
    dx = 1.0 / n
    g = hw.GridSpec(n, n, dx, ps.dt_below(0.5 * dx / (4.5 * np.sqrt(3))), nt, nz=n, order=2)
    s = hw.AcousticSolver(g, med, stencil_precision=prec, receivers=((n // 4, n // 2, n // 2),), energy_every=10)
    st = s.new_state()
    st.p.values = ps.gauss((n, n, n)).astype(st.p.values.dtype)
    return s, st


def _el3(prec, n=256, nt=300):
    layers = [(0.25, 1.2, 2.2, 1.1), (0.5, 1.5, 2.6, 1.3), (0.75, 1.8, 3.0, 1.5), (1.0, 2.0, 3.2, 1.6)]
    med = hw.build_layered_elastic(n, n, layers, nz=n)
    dx = 1.0 / n
    g = hw.GridSpec(n, n, dx, ps.dt_below(0.4 * dx / (3.2 * np.sqrt(3))), nt, nz=n, order=2)
    s = hw.ElasticSolver(g, med, stencil_precision=prec, receivers=((n // 2, n // 4, n // 2),), energy_every=10)
    st = s.new_state()
    st.vy.values = ps.gauss((n, n, n)).astype(st.vy.values.dtype)
    return s, st


def _drift(build, prec, variant):
    s, st = build(prec)
    out = s.run(variant, st)
    return energy_drift(out.energy, -1.0)["rel_deviation"], float(out.energy.values[-1]), s.kernel_path()


def test_gpu_3d_acoustic_compensation_recovers_energy():
    d64, e64, _ = _drift(_ac3, F64, None)
    d32, e32, p32 = _drift(_ac3, F32, None)
    dn, en, pn = _drift(_ac3, F16, None)
    dc, ec, pc = _drift(_ac3, F16, hw.Variant.OP3)
    assert (p32, pn, pc) == ("fused3d-f32", "fused3d", "fused3d")
    assert d64 < 1e-13
    assert d32 < 1e-6 and dc < dn / 10.0, (d32, dn, dc)
    assert abs(ec - e64) / e64 < abs(en - e64) / e64 / 10.0


def test_gpu_3d_elastic_compensation_recovers_energy():
    d64, e64, _ = _drift(_el3, F64, None)
    dn, en, pn = _drift(_el3, F16, None)
    dc, ec, pc = _drift(_el3, F16, hw.Variant.OP6)
    assert pn == pc and pn in ("fused3d-el", "stream3d"), (pn, pc)
    assert d64 < 1e-13
    assert dc < dn / 5.0, (dn, dc)
    assert abs(ec - e64) / e64 < abs(en - e64) / e64 / 5.0


def _ac2(prec, upd=None, n=1024, ny=1040, nt=1500):
    """Config 2 at 1024 x 1040 (above the persistent small-grid kernel's 2^20 cells): two-layer medium, 4th order, Ricker at the top centre (amplitude scaled
    with the grid so the field sits in binary16's normal range), energy every 10 steps."""
    dx = 1.0 / n
    med = hw.build_layered_acoustic(n, ny, [(0.5, 1.0, 1.0), (1.0, 1.5, 2.25)])
    g = hw.GridSpec(n, ny, dx, ps.dt_below(0.5 * dx / med.c_max()), nt)
    src = hw.SourceSpec(hw.SourceKind.PRESSURE_POINT, n // 2, 8, hw.RickerSpec(1.0 / (10 * dx), amplitude=5.0e3))
    s = hw.AcousticSolver(g, med, src, stencil_precision=prec, update_precision=upd, receivers=((n // 2, n // 4),),
                          energy_every=10)
    return s, s.new_state(), 2.0 * src.wavelet.delay


def test_gpu_2d_acoustic_compensation_recovers_energy():
    res = {}
    for name, prec, var in (("fp64", F64, None), ("naive", F16, None), ("op3", F16, hw.Variant.OP3)):
        s, st, t_off = _ac2(prec)
        out = s.run(var, st)
        res[name] = (energy_drift(out.energy, t_off)["rel_deviation"], float(out.energy.values[-1]), s.kernel_path())
    assert res["naive"][2] == res["op3"][2] == "fused2d"
    e64 = res["fp64"][1]
    assert res["fp64"][0] < 1e-13, res
    assert res["op3"][0] < res["naive"][0] / 5.0, res
    assert abs(res["op3"][1] - e64) / e64 < abs(res["naive"][1] - e64) / e64 / 5.0, res

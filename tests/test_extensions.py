"""Extensions the BASELINE configs need beyond the reference (SURVEY §8 a'), pinned on
the CPU oracle by their reductions to reference-native bits:

* a 3D field invariant along the new (mid) axis evolves exactly like the 2D run;
* mu = 0 elastic reproduces acoustic bits (the reference's own test_elastic.py:151-188,
  here also in 3D and for the explosive source's isotropy);
* the second-order stencil keeps constants exactly stationary and propagates like the
  fourth-order one at low wavenumber.
"""

import numpy as np
import pytest

import oracle
import paper_2310_00236_b200 as hw
from golden_cases import assert_same_bits

F16 = hw.Precision.FP16


def _gauss2d(ns, nx, cy, cx, w, amp=0.5):
    yy, xx = np.mgrid[0:ns, 0:nx].astype(np.float64)
    return amp * np.exp(-((xx - cx) ** 2 + (yy - cy) ** 2) / w)


@pytest.mark.parametrize("order", [2, 4])
@pytest.mark.parametrize("variant", [None, hw.Variant.OP3])
def test_y_invariant_3d_acoustic_equals_2d(order, variant):
    nx, nz, ny3, nt = 20, 24, 8, 30
    dx, dt = 0.05, 0.01
    p2 = _gauss2d(nz, nx, 11, 9, 9.0).astype(np.float16)
    g2 = hw.GridSpec(nx, nz, dx, dt, nt, order=order)
    s2 = hw.AcousticSolver(g2, hw.build_homogeneous_acoustic(nx, nz, 1.0, 1.0), stencil_precision=F16)
    st2 = s2.new_state()
    st2.p.values = p2
    r2 = oracle.run_solver(s2, variant, st2)
    g3 = hw.GridSpec(nx, ny3, dx, dt, nt, nz=nz, order=order)
    s3 = hw.AcousticSolver(g3, hw.build_homogeneous_acoustic(nx, ny3, 1.0, 1.0, nz=nz), stencil_precision=F16)
    st3 = s3.new_state()
    st3.p.values = np.ascontiguousarray(np.broadcast_to(p2[:, None, :], (nz, ny3, nx)))
    r3 = oracle.run_solver(s3, variant, st3)
    f2, f3 = dict(zip(s2.FIELDS, r2["fields"])), dict(zip(s3.FIELDS, r3["fields"]))
    for n2, n3 in (("p", "p"), ("vx", "vx"), ("vy", "vz"), ("rp", "rp"), ("rvx", "rvx"), ("rvy", "rvz")):
        for m in range(ny3):
            np.testing.assert_array_equal(f3[n3][:, m, :], f2[n2], err_msg=f"{n3} at y={m}")
    assert np.all(f3["vy"] == 0)
    assert np.any(f2["p"] != p2)


def _mu0_pair(ndim, nt=40, n=16):
    dx, dt = 0.05, 0.01
    kw = {} if ndim == 2 else {"nz": n}
    g = hw.GridSpec(n, n, dx, dt, nt, **kw)
    ac = hw.AcousticSolver(g, hw.build_homogeneous_acoustic(n, n, 1.0, 2.0, **kw), stencil_precision=F16)
    el = hw.ElasticSolver(g, hw.build_layered_elastic(n, n, [(1.0, 1.0, 2.0, 0.0)], **kw), stencil_precision=F16)
    sa, se = ac.new_state(), el.new_state()
    blob = _gauss2d(n, n, 7, 8, 6.0)
    if ndim == 3:
        zz = np.exp(-((np.arange(n) - 6.0) ** 2) / 8.0)
        blob = blob[None, :, :] * zz[:, None, None]
    blob = blob.astype(np.float16)
    sa.p.values = blob.copy()
    names = ("sxx", "syy") if ndim == 2 else ("sxx", "syy", "szz")
    for nm in names:
        getattr(se, nm).values = blob.copy()
    return ac, el, sa, se, names


@pytest.mark.parametrize("ndim", [2, 3])
def test_mu_zero_elastic_reproduces_acoustic_bits(ndim):
    ac, el, sa, se, names = _mu0_pair(ndim)
    ra = dict(zip(ac.FIELDS, oracle.run_solver(ac, None, sa)["fields"]))
    re_ = dict(zip(el.FIELDS, oracle.run_solver(el, None, se)["fields"]))
    for nm in names:
        np.testing.assert_array_equal(re_[nm], ra["p"], err_msg=nm)
    vel = ("vx", "vy") if ndim == 2 else ("vx", "vy", "vz")
    for v in vel:
        np.testing.assert_array_equal(re_[v], ra[v], err_msg=v)
    shear = ("sxy",) if ndim == 2 else ("sxy", "sxz", "syz")
    for s in shear:
        assert np.all(re_[s] == 0)
    assert np.any(ra["p"] != sa.p.values)


def test_explosive_source_first_step_is_isotropic_scalar_chain():
    n = 16
    g = hw.GridSpec(n, n, 0.05, 0.01, 1)
    src = hw.SourceSpec(hw.SourceKind.EXPLOSIVE, 8, 7, hw.RickerSpec(5.0, amplitude=1e3))
    el = hw.ElasticSolver(g, hw.build_layered_elastic(n, n, [(1.0, 1.0, 2.0, 1.0)]), src, stencil_precision=F16)
    out = dict(zip(el.FIELDS, oracle.run_solver(el, None)["fields"]))
    s = hw.sample_source(src, 0.5 * g.dt)
    want = np.float16(np.float16(s) * np.float16(g.dt))  # fl(round(s) * dt), no divisor for stresses
    for nm in ("sxx", "syy"):
        a = out[nm]
        assert a[7, 8] == want
        a = a.copy()
        a[7, 8] = 0
        assert np.all(a == 0)
    assert np.all(out["vx"] == 0) and np.all(out["vy"] == 0)


def test_second_order_constant_field_is_stationary():
    n = 24
    g = hw.GridSpec(n, n, 0.05, 0.02, 30, order=2)
    s = hw.AcousticSolver(g, hw.build_homogeneous_acoustic(n, n, 1.0, 1.0), stencil_precision=F16)
    st = s.new_state()
    st.p.values[:] = np.float16(0.7)
    out = dict(zip(s.FIELDS, oracle.run_solver(s, hw.Variant.OP3, st)["fields"]))
    assert np.all(out["p"] == np.float16(0.7))
    assert np.all(out["vx"] == 0) and np.all(out["vy"] == 0)


def test_second_order_matches_fourth_order_on_smooth_waves():
    n, nt = 64, 60
    res = {}
    for order in (2, 4):
        g = hw.GridSpec(n, n, 1.0 / n, 0.25 / n, nt, order=order)
        s = hw.AcousticSolver(g, hw.build_homogeneous_acoustic(n, n, 1.0, 1.0), stencil_precision=hw.Precision.FP64)
        st = s.new_state()
        yy, xx = np.mgrid[0:n, 0:n] / n
        st.p.values = np.exp(-((xx - 0.5) ** 2 + (yy - 0.5) ** 2) / 0.02)
        res[order] = oracle.run_solver(s, None, st)["fields"][0]
    rel = np.linalg.norm(res[2] - res[4]) / np.linalg.norm(res[4])
    assert 1e-6 < rel < 2e-2


def test_cfl_limits_per_order_and_dimension():
    assert hw.cfl_limit(2, 4) == pytest.approx(6.0 / (7.0 * np.sqrt(2.0)))
    assert hw.cfl_limit(2, 2) == pytest.approx(1.0 / np.sqrt(2.0))
    assert hw.cfl_limit(3, 2) == pytest.approx(1.0 / np.sqrt(3.0))
    with pytest.raises(ValueError, match="CFL"):
        hw.AcousticSolver(hw.GridSpec(16, 16, 1.0, 0.6, 1, nz=16, order=2),
                          hw.build_homogeneous_acoustic(16, 16, 1.0, 1.0, nz=16))

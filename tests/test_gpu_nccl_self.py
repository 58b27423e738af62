"""The NCCL transport (one process per GPU) on real hardware: with the option nccl_self=1 a
one-rank torch.distributed job takes the NCCL path — libnccl dlopen'ed, communicator
from hw_nccl_unique_id, periodic ghosts exchanged by grouped ncclSend/ncclRecv to itself
after every phase, control blocks all-gathered, energy all-reduced, traces broadcast —
and must reproduce the single-process run bit for bit (energy within 1e-12)."""

import socket

import numpy as np
import pytest

import paper_2310_00236_b200 as hw
from golden_cases import assert_same_bits

pytestmark = pytest.mark.gpu


@pytest.fixture
def one_rank_job(hwopt):
    import torch.distributed as dist

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1)
    hwopt(nccl_self=1)
    yield
    dist.destroy_process_group()


def _acoustic(**kw):
    nx, ny = 256, 96
    dx = 1.0 / nx
    g = hw.GridSpec(nx, ny, dx, float(np.float16(0.3 * dx)), 30)
    src = hw.SourceSpec(hw.SourceKind.PRESSURE_POINT, 100, 47, hw.RickerSpec(1 / (10 * dx), amplitude=2.0))
    s = hw.AcousticSolver(g, hw.build_layered_acoustic(nx, ny, [(0.4, 1.0, 1.0), (1.0, 1.5, 2.25)]), src,
                          stencil_precision=hw.Precision.FP16, energy_every=5, receivers=((100, 47), (3, 0), (250, 95)),
                          **kw)
    st = s.new_state()
    yy, xx = np.mgrid[0:ny, 0:nx] / nx
    st.p.values = np.exp(-((xx - 0.5) ** 2 + (yy - 0.2) ** 2) / 0.005).astype(np.float16)
    return s, st


def _elastic(**kw):
    nx, ny = 256, 64
    g = hw.GridSpec(nx, ny, 0.05, 0.004, 30, bc_y=hw.Boundary.PERIODIC)
    src = hw.SourceSpec(hw.SourceKind.VY_POINT, 40, 33, hw.RickerSpec(5.0, amplitude=20.0))
    s = hw.ElasticSolver(g, hw.build_layered_elastic(nx, ny, [(0.5, 2.0, 2.0, 1.0), (1.0, 2.3, 2.8, 1.4)]), src,
                         stencil_precision=hw.Precision.FP16, energy_every=4, receivers=((40, 33), (10, 0)), **kw)
    st = s.new_state()
    st.sxx.values = np.random.default_rng(3).uniform(-0.1, 0.1, st.sxx.values.shape).astype(np.float16)
    return s, st


def _acoustic3d(**kw):
    nz, ny, nx = 24, 16, 256
    g = hw.GridSpec(nx, ny, 1.0 / nx, float(np.float16(0.2 / nx)), 12, nz=nz, order=2)
    s = hw.AcousticSolver(g, hw.build_homogeneous_acoustic(nx, ny, 1.0, 1.0, nz=nz), stencil_precision=hw.Precision.FP16,
                          receivers=((5, 5, 20), (12, 8, 2)), energy_every=3, **kw)
    st = s.new_state()
    z, y, x = np.mgrid[0:nz, 0:ny, 0:nx]
    st.p.values = np.exp(-((x - 120) ** 2 / 200.0 + (y - 8) ** 2 / 10.0 + (z - 3) ** 2 / 10.0)).astype(np.float16)
    return s, st


def _elastic3d_onepass(**kw):  # config 5's one-pass kernel on the NCCL transport (HW_PLAN_FUSED_EL3)
    from test_gpu_el3_slabs import _el3

    return _el3(1, distributed=bool(kw.get("distributed")))


def _acoustic3d_onepass(**kw):  # config 3's one-pass kernel on the NCCL transport (HW_PLAN_FUSED_AC3)
    from test_gpu_slabs import _acoustic3d_onepass as mk

    s, st = mk(1)
    if kw.get("distributed"):
        s = hw.AcousticSolver(s.grid, s.medium, s.source, stencil_precision=s.stencil_precision,
                              receivers=s.receivers, energy_every=s.energy_every, distributed=True)
    return s, st


def _elastic2d_onepass(fs=True, **kw):  # config 4's one-pass kernel on the NCCL transport (HW_PLAN_FUSED_EL2)
    from test_gpu_slabs import _elastic2d_onepass as mk

    s, st = mk(1, fs)
    if kw.get("distributed"):
        s = hw.ElasticSolver(s.grid, s.medium, s.source, stencil_precision=s.stencil_precision,
                             receivers=s.receivers, energy_every=s.energy_every, distributed=True)
    return s, st


@pytest.mark.parametrize("make,variant", [(_acoustic, hw.Variant.OP3), (_elastic, hw.Variant.OP6),
                                          (_elastic2d_onepass, hw.Variant.OP6),
                                          (lambda **kw: _elastic2d_onepass(False, **kw), hw.Variant.OP6),
                                          (_acoustic3d, hw.Variant.OP3), (_elastic3d_onepass, hw.Variant.OP6),
                                          (_acoustic3d_onepass, hw.Variant.OP3)])
def test_nccl_transport_equals_single_process(one_rank_job, make, variant):
    a, sa = make()
    oa = a.run(variant, sa)
    b, sb = make(distributed=True)
    ob = b.run(variant, sb)
    assert a.transport() == 0 and b.transport() == 2
    for n in a.FIELDS:
        assert_same_bits(getattr(sb, n).values, getattr(sa, n).values, n)
    np.testing.assert_array_equal(np.array([t.samples for t in ob.traces]), np.array([t.samples for t in oa.traces]))
    if a.kernel_path() == b.kernel_path() and a.kernel_path() in ("fused3d-el", "fused3d"):  # plane-ordered energy
        np.testing.assert_array_equal(ob.energy.values, oa.energy.values)
    np.testing.assert_allclose(ob.energy.values, oa.energy.values, rtol=1e-12)


def test_nccl_transport_range_failure(one_rank_job):
    a, sa = _acoustic()
    sa.p.values = (sa.p.values.astype(np.float32) * 3e4).astype(np.float16)
    with pytest.raises(hw.RangeFailureError) as ea:
        a.run(None, sa)
    b, sb = _acoustic(distributed=True)
    sb.p.values = (sb.p.values.astype(np.float32) * 3e4).astype(np.float16)
    with pytest.raises(hw.RangeFailureError) as eb:
        b.run(None, sb)
    assert (eb.value.step, eb.value.field_name) == (ea.value.step, ea.value.field_name)
    for n in a.FIELDS:
        assert_same_bits(getattr(sb, n).values, getattr(sa, n).values, n)


def test_nccl_transport_device_resident_run(one_rank_job):
    """The bench's decomposed path: upload -> run_device (overlapped edge/interior bands,
    NCCL exchange every step) -> download equals the single-process run."""
    a, sa = _acoustic()
    a.run(hw.Variant.OP3, sa)
    b, sb = _acoustic(distributed=True)
    b.upload(sb)
    ms = b.run_device(hw.Variant.OP3, 0, b.grid.nt)
    b.download(sb)
    assert ms > 0 and b.transport() == 2 and b.kernel_path() == "fused2d"
    for n in a.FIELDS:
        assert_same_bits(getattr(sb, n).values, getattr(sa, n).values, n)


def test_nccl_el3_overlapped_device_resident_run(one_rank_job):
    """Config 5's one-pass kernel on the NCCL transport, overlapped: per step the edge slabs and the
    exchange on one stream, the interior slabs on another (run_device), equals the single process."""
    from test_gpu_el3_slabs import _el3

    a, sa = _el3(1, nt=11)
    a.run(hw.Variant.OP6, sa)
    b, sb = _el3(1, nt=11, distributed=True)
    b.upload(sb)
    ms = b.run_device(hw.Variant.OP6, 0, b.grid.nt)
    b.download(sb)
    assert ms > 0 and b.transport() == 2 and b.kernel_path() == "fused3d-el"
    for n in a.FIELDS:
        assert_same_bits(getattr(sb, n).values, getattr(sa, n).values, n)


@pytest.mark.parametrize("fs", [True, False])
@pytest.mark.parametrize("variant", [None, hw.Variant.OP6])
def test_nccl_el2_overlapped_device_resident_run(one_rank_job, fs, variant):
    """Config 4's one-pass kernel on the NCCL transport, overlapped: per step the two 8-row edge bands
    and the exchange on one stream, the interior bands on another (two launches per step), equals the
    single process (free surface: images at the global ends, no exchange; periodic: self exchange)."""
    a, sa = _elastic2d_onepass(fs)
    oa = a.run(variant, sa)
    b, sb = _elastic2d_onepass(fs, distributed=True)
    b.upload(sb)
    ms = b.run_device(variant, 0, b.grid.nt)
    b.download(sb)
    assert ms > 0 and b.transport() == 2 and b.kernel_path() == "fused2d-el"
    assert b.last_launch_count() >= 2 * b.grid.nt
    for n in a.FIELDS:
        assert_same_bits(getattr(sb, n).values, getattr(sa, n).values, n)
    _, sc = _elastic2d_onepass(fs)  # the host path (traces, energy) through the same overlapped loop
    oc = b.run(variant, sc)
    np.testing.assert_array_equal(np.array([t.samples for t in oc.traces]), np.array([t.samples for t in oa.traces]))
    np.testing.assert_allclose(oc.energy.values, oa.energy.values, rtol=1e-12)


@pytest.mark.parametrize("prec,variant,ny", [(hw.Precision.FP16, hw.Variant.OP3, 8), (hw.Precision.FP16, hw.Variant.OP3, 64),
                                             (hw.Precision.FP32, None, 8), (hw.Precision.FP32, hw.Variant.OP3, 32)])
def test_nccl_ac3_overlapped(one_rank_job, prec, variant, ny):
    """Config 3's one-pass kernels on the NCCL transport, overlapped: per step the edge slabs 0 and L-1
    and the exchange on one stream, the interior slabs on another (two launches per step; 1 to 8 tiles,
    CTA groups of 1 and 4), equal the single process -- fields, traces, energy bit for bit (plane order)."""
    from test_gpu_slabs import _acoustic3d_onepass as mk

    a, sa = mk(1, prec, src_z=0, ny=ny)
    oa = a.run(variant, sa)
    b, sb = mk(1, prec, src_z=0, ny=ny, distributed=True)
    ob = b.run(variant, sb)
    assert b.transport() == 2 and b.kernel_path() == a.kernel_path() == ("fused3d" if prec == hw.Precision.FP16 else "fused3d-f32")
    assert b.last_launch_count() >= 2 * b.grid.nt
    for n in a.FIELDS:
        assert_same_bits(getattr(sb, n).values, getattr(sa, n).values, n)
    np.testing.assert_array_equal(np.array([t.samples for t in ob.traces]), np.array([t.samples for t in oa.traces]))
    np.testing.assert_array_equal(ob.energy.values, oa.energy.values)

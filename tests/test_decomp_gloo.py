"""Multi-rank host logic on the CPU: world_size 2, 3 and 8 torch.distributed gloo jobs
execute the library's own halo plan (hw_exchange_plan -- the list both device transports
run) on host arrays and check every rank's ghost rows against the global arrays: periodic
wrap, free-surface ends untouched, the stencil reach of every ghosted field covered (1 row at
2nd order, 2 at 4th, 3 for the fused 2D kernel), the right fields per exchange kind, own
rows unchanged; plus the slab ownership bookkeeping."""

import ctypes
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import paper_2310_00236_b200 as hw
from paper_2310_00236_b200 import _abi, decomp

# exchange kind -> the external fields it must move (SURVEY §8 e: velocities with slow-axis
# derivatives after the velocity phase, the slow-derivative stresses / pressure after the other)
EXPECT = {
    ("ac", 2): {_abi.PLAN_VEL: {"vy"}, _abi.PLAN_STRESS: {"p"}, _abi.PLAN_FUSED: {"p", "vy", "rvy"}},
    ("ac", 3): {_abi.PLAN_VEL: {"vz"}, _abi.PLAN_STRESS: {"p"}, _abi.PLAN_FUSED_AC3: {"p", "vz", "rvz"}},
    ("el", 2): {_abi.PLAN_VEL: {"vx", "vy"}, _abi.PLAN_STRESS: {"syy", "sxy"},
                _abi.PLAN_FUSED_EL2: {"vx", "vy", "sxx", "syy", "sxy", "rvx", "rvy"}},
    ("el", 3): {_abi.PLAN_VEL: {"vx", "vy", "vz"}, _abi.PLAN_STRESS: {"szz", "sxz", "syz"},
                _abi.PLAN_FUSED_EL3: {"vx", "vy", "vz", "sxx", "syy", "szz", "sxy", "sxz", "syz", "rvx", "rvy", "rvz"}},
}


def _cases():
    F16 = hw.Precision.FP16
    ac2 = hw.AcousticSolver(hw.GridSpec(16, 37, 1 / 16, 0.01, 1), hw.build_homogeneous_acoustic(16, 37, 1.0, 1.0),
                            stencil_precision=F16)
    ac3 = hw.AcousticSolver(hw.GridSpec(8, 8, 1 / 8, 0.01, 1, nz=33, order=2),
                            hw.build_homogeneous_acoustic(8, 8, 1.0, 1.0, nz=33), stencil_precision=F16)
    el2fs = hw.ElasticSolver(hw.GridSpec(16, 35, 1 / 16, 0.005, 1, bc_y=hw.Boundary.FREE_SURFACE),
                             hw.build_layered_elastic(16, 35, [(1.0, 1.0, 2.0, 1.0)]), stencil_precision=F16)
    el2p = hw.ElasticSolver(hw.GridSpec(16, 26, 1 / 16, 0.005, 1, order=2),
                            hw.build_layered_elastic(16, 26, [(1.0, 1.0, 2.0, 1.0)]), stencil_precision=F16)
    el3 = hw.ElasticSolver(hw.GridSpec(8, 8, 1 / 8, 0.004, 1, nz=40, order=2),
                           hw.build_layered_elastic(8, 8, [(1.0, 1.0, 2.0, 1.0)], nz=40), stencil_precision=F16)
    return [("ac", 2, ac2), ("ac", 3, ac3), ("el", 2, el2fs), ("el", 2, el2p), ("el", 3, el3)]


def _shape(desc, j):
    shp = (ctypes.c_int64 * 3)()
    _abi.check(_abi.load().hw_field_shape(ctypes.byref(desc), j, shp), "hw_field_shape")
    return tuple(shp)


def _check_case(eq, ndim, s, world, rank):
    desc = s.desc
    ns, periodic = desc.ns, desc.bc_slow == _abi.BC_PERIODIC
    r0, _ = decomp.slab_range(ns, world, rank)
    for kind, want_fields in EXPECT[(eq, ndim)].items():
        if kind == _abi.PLAN_FUSED and not periodic:
            continue
        rng = np.random.default_rng(100 * kind + ndim)
        glob, fields = {}, {}
        for j in range(len(s.FIELDS)):
            gl = rng.standard_normal(_shape(desc, j)).astype(np.float32)  # same on every rank
            n_loc = decomp.local_rows(ns, world, rank, extra_row=gl.shape[0] > ns)
            glob[j] = gl
            fields[j] = decomp.with_ghosts(gl[r0:r0 + n_loc], fill=np.nan)
        p = decomp.exchange_host(desc, fields, world, rank, kind)
        assert {s.FIELDS[x["field"]] for x in p} == want_fields, (kind, p)
        depth_of = lambda j: (3 if kind in (_abi.PLAN_FUSED, _abi.PLAN_FUSED_EL2) else (2 if s.FIELDS[j].startswith("s") else 1)
                              if kind == _abi.PLAN_FUSED_EL3 else (1 if desc.order == 2 else 2))
        got = {}
        for x in p:
            assert x["nrows"] == depth_of(x["field"])
            if x["send"]:
                continue
            a, gl = fields[x["field"]], glob[x["field"]]
            for r in range(x["row0"], x["row0"] + x["nrows"]):
                g = r0 + r
                g = g % gl.shape[0] if periodic else g
                assert 0 <= g < gl.shape[0], (x, r)
                np.testing.assert_array_equal(a[r + decomp.G], gl[g])
                got.setdefault(x["field"], set()).add(r)
        for j in {x["field"] for x in p}:
            depth = depth_of(j)
            n = fields[j].shape[0] - 2 * decomp.G
            want = set()
            if periodic or rank > 0:
                want |= set(range(-depth, 0))
            if periodic or rank < world - 1:
                want |= set(range(n, n + depth))
            assert got.get(j, set()) == want, (s.FIELDS[j], kind, sorted(got.get(j, set())), sorted(want))
            np.testing.assert_array_equal(fields[j][decomp.G:decomp.G + n], glob[j][r0:r0 + n])  # own rows untouched


def _worker(rank, world, port, errq):
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        for eq, ndim, s in _cases():
            _check_case(eq, ndim, s, world, rank)
        dist.barrier()
        dist.destroy_process_group()
    except Exception as e:  # pragma: no cover - reported to the parent
        errq.put(f"rank {rank}: {e!r}")
        raise


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("world", [2, 3, 8])
def test_library_halo_plan_gloo(world):
    ctx = mp.get_context("spawn")
    errq = ctx.SimpleQueue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, errq)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(300)
    assert all(p.exitcode == 0 for p in procs), errq.get() if not errq.empty() else "worker failed"


def test_plan_pairs_match_across_ranks():
    """Every receive has its matching send (k-th receive of b from a <-> k-th send of a to b) with
    the same field and row count, for every kind and world size 1..8 (1: NCCL self exchange)."""
    for eq, ndim, s in _cases():
        for world in range(1, 9):
            kinds = list(EXPECT[(eq, ndim)])
            for kind in kinds:
                plans = [decomp.plan(s.desc, world, r, kind) for r in range(world)]
                for b in range(world):
                    for a in range(world):
                        recv = [x for x in plans[b] if not x["send"] and x["peer"] == a]
                        send = [x for x in plans[a] if x["send"] and x["peer"] == b]
                        assert [(x["field"], x["nrows"]) for x in recv] == [(x["field"], x["nrows"]) for x in send]


def test_slab_plan_covers_every_row_once():
    for ns in (8, 13, 100, 4096):
        for world in (1, 2, 3, 8):
            if ns // world < 4:
                continue
            rows = []
            for r in range(world):
                r0, r1 = decomp.slab_range(ns, world, r)
                rows.extend(range(r0, r1))
                assert decomp.local_rows(ns, world, r, extra_row=True) == (r1 - r0) + (r == world - 1)
            assert rows == list(range(ns))
            for row in (0, ns // 2, ns - 1, ns):
                r = decomp.owner_of_row(ns, world, row)
                r0, r1 = decomp.slab_range(ns, world, r)
                assert r0 <= row < r1 or (row == ns and r == world - 1)

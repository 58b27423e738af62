"""Multi-rank host logic on the CPU: world_size-2 (and 3) torch.distributed gloo jobs
run the slab plan of paper_2310_00236_b200.decomp — slab ranges, neighbours, the
canonical send/recv order — and check every rank's ghost slabs against the global
array's periodic wrap; plus source / receiver ownership bookkeeping."""

import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2310_00236_b200 import decomp


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, ns, periodic, errq):
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        rng = np.random.default_rng(7)
        glob = [rng.standard_normal((ns, 3, 5)).astype(np.float32) for _ in range(2)]  # same on every rank
        r0, r1 = decomp.slab_range(ns, world, rank)
        fields = [decomp.with_ghosts(g[r0:r1]) for g in glob]
        decomp.exchange_halos(fields, world, rank, periodic)
        prev, nxt = decomp.neighbours(world, rank, periodic)
        for g, f in zip(glob, fields):
            if prev >= 0:  # top ghosts = the G global rows just above the slab (wrapped)
                want = g[[(r0 - decomp.G + k) % ns for k in range(decomp.G)]]
                np.testing.assert_array_equal(f[:decomp.G], want)
            if nxt >= 0:
                want = g[[(r1 + k) % ns for k in range(decomp.G)]]
                np.testing.assert_array_equal(f[-decomp.G:], want)
            np.testing.assert_array_equal(f[decomp.G:-decomp.G], g[r0:r1])
        dist.barrier()
        dist.destroy_process_group()
    except Exception as e:  # pragma: no cover - reported to the parent
        errq.put(f"rank {rank}: {e!r}")
        raise


@pytest.mark.parametrize("world,ns,periodic", [(2, 16, True), (2, 17, False), (3, 20, True)])
def test_halo_exchange_gloo(world, ns, periodic):
    ctx = mp.get_context("spawn")
    errq = ctx.SimpleQueue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, ns, periodic, errq)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
    assert all(p.exitcode == 0 for p in procs), errq.get() if not errq.empty() else "worker failed"


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

"""Slab decomposition of the slow axis (SURVEY §8 e) on host arrays.

The library computes its halo plan on the host from the slab geometry alone
(`hw_exchange_plan`, include/halfwave_b200.h; csrc/hw_api.cu `halo_plan`) and both of its
transports execute exactly that list: NCCL send/recv in issue order (one process per GPU)
and peer copies inside a slab group (the k-th receive of rank b from rank a takes the k-th
send of a to b).  `exchange_host` executes the same list over torch.distributed on host
arrays, so a CPU job (gloo) can check the plan the device runs against the global array
(tests/test_decomp_gloo.py).

Rank r of N owns global slow rows [r*ns//N, (r+1)*ns//N) (the extra free-surface row of
integer sub-grids goes to the last rank) and keeps G = 3 ghost slabs on each side.
"""

from __future__ import annotations

import numpy as np

from . import _abi

G = 3  # ghost slabs per side (csrc/hw_common.cuh)


def slab_range(ns: int, world: int, rank: int) -> tuple:
    return (rank * ns // world, (rank + 1) * ns // world)


def local_rows(ns: int, world: int, rank: int, extra_row: bool) -> int:
    r0, r1 = slab_range(ns, world, rank)
    return (r1 - r0) + (1 if extra_row and rank == world - 1 else 0)


def owner_of_row(ns: int, world: int, row: int) -> int:
    for r in range(world):
        r0, r1 = slab_range(ns, world, r)
        if r0 <= row < r1 or (r == world - 1 and row >= r1):
            return r
    raise ValueError(f"row {row} outside 0..{ns}")


def plan(desc, world: int, rank: int, kind: int) -> list:
    """The library's halo plan (hw_exchange_plan) for slab `rank` of `world`."""
    return _abi.exchange_plan(desc, world, rank, kind)


def with_ghosts(slab: np.ndarray, fill=0.0) -> np.ndarray:
    """[rows + 2G, ...] with the slab in the middle (local row r at index r + G)."""
    out = np.full((slab.shape[0] + 2 * G,) + slab.shape[1:], fill, dtype=slab.dtype)
    out[G:G + slab.shape[0]] = slab
    return out


def exchange_host(desc, fields: dict, world: int, rank: int, kind: int) -> list:
    """Execute the library's plan on host arrays: `fields` maps external field index -> array
    from with_ghosts.  Returns the plan that ran."""
    import torch
    import torch.distributed as dist

    p = plan(desc, world, rank, kind)
    ops, recv = [], []
    for x in p:
        a = fields[x["field"]]
        sl = slice(x["row0"] + G, x["row0"] + G + x["nrows"])
        if x["send"]:
            ops.append(dist.P2POp(dist.isend, torch.from_numpy(np.ascontiguousarray(a[sl])), x["peer"]))
        else:
            buf = torch.from_numpy(np.empty_like(a[sl]))
            ops.append(dist.P2POp(dist.irecv, buf, x["peer"]))
            recv.append((a, sl, buf))
    if ops:
        for req in dist.batch_isend_irecv(ops):
            req.wait()
    for a, sl, buf in recv:
        a[sl] = buf.numpy()
    return p

"""Slab decomposition of the slow axis (SURVEY §8 e) — the host-side plan.

Mirrors the arithmetic of csrc/hw_api.cu (`setup_handle`, `xfers`,
`exchange_nccl`): rank r of N owns global slow rows [r*ns//N, (r+1)*ns//N) (the
extra free-surface row of integer sub-grids goes to the last rank), keeps G = 2
ghost slabs on each side, and after every phase sends its G boundary slabs to its
neighbours in a canonical order (bottom rows -> next / top ghosts <- previous,
then top rows -> previous / bottom ghosts <- next).  Periodic slow axes wrap rank
N-1 <-> 0; free surfaces keep image ghosts at the global ends.

`exchange_halos` runs that plan over torch.distributed on host arrays; it is the
CPU (gloo) model of the device exchange, used by tests/test_decomp_gloo.py.
"""

from __future__ import annotations

import numpy as np

G = 2


def slab_range(ns: int, world: int, rank: int) -> tuple:
    return (rank * ns // world, (rank + 1) * ns // world)


def local_rows(ns: int, world: int, rank: int, extra_row: bool) -> int:
    r0, r1 = slab_range(ns, world, rank)
    return (r1 - r0) + (1 if extra_row and rank == world - 1 else 0)


def neighbours(world: int, rank: int, periodic: bool) -> tuple:
    prev = rank - 1 if rank > 0 else (world - 1 if periodic else -1)
    nxt = rank + 1 if rank < world - 1 else (0 if periodic else -1)
    return prev, nxt


def owner_of_row(ns: int, world: int, row: int) -> int:
    for r in range(world):
        r0, r1 = slab_range(ns, world, r)
        if r0 <= row < r1 or (r == world - 1 and row >= r1):
            return r
    raise ValueError(f"row {row} outside 0..{ns}")


def with_ghosts(slab: np.ndarray) -> np.ndarray:
    """Allocate [rows + 2G, ...] with the slab in the middle (ghosts zero)."""
    out = np.zeros((slab.shape[0] + 2 * G,) + slab.shape[1:], dtype=slab.dtype)
    out[G:-G] = slab
    return out


def exchange_halos(fields: list, world: int, rank: int, periodic: bool) -> None:
    """Fill the inter-rank ghost slabs of `fields` (arrays from with_ghosts) in place
    with torch.distributed point-to-point messages, in the library's order."""
    import torch
    import torch.distributed as dist

    prev, nxt = neighbours(world, rank, periodic)
    ops = []
    recv = []
    for f in fields:  # phase A: bottom rows -> next, top ghosts <- prev
        if nxt >= 0:
            ops.append(dist.P2POp(dist.isend, torch.from_numpy(np.ascontiguousarray(f[-2 * G:-G])), nxt))
        if prev >= 0:
            buf = torch.empty(f[:G].shape, dtype=torch.from_numpy(f[:1]).dtype)
            ops.append(dist.P2POp(dist.irecv, buf, prev))
            recv.append((f, slice(0, G), buf))
    for f in fields:  # phase B: top rows -> prev, bottom ghosts <- next
        if prev >= 0:
            ops.append(dist.P2POp(dist.isend, torch.from_numpy(np.ascontiguousarray(f[G:2 * G])), prev))
        if nxt >= 0:
            buf = torch.empty(f[-G:].shape, dtype=torch.from_numpy(f[:1]).dtype)
            ops.append(dist.P2POp(dist.irecv, buf, nxt))
            recv.append((f, slice(f.shape[0] - G, f.shape[0]), buf))
    if ops:
        for req in dist.batch_isend_irecv(ops):
            req.wait()
    for f, sl, buf in recv:
        f[sl] = buf.numpy()

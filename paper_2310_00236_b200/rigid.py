"""Rigid (p = 0) walls for the 2D acoustic solver (BASELINE config 1; SURVEY §8 a').

The reference is periodic-only (acoustic.py:67-68).  Walls where p = 0 are the odd
reflection of the reference's own image machinery (stencil.py:121-159: images of the
integer and half sub-grids, parity signs): about a wall, p and the tangential velocity
are odd, the normal velocity is even.  That makes a rigid box exactly the periodic
problem on the mirrored domain (2 nx along a rigid x, 2 ny along a rigid y) with
odd / even extended state and even extended medium:

* every tap the rigid discretisation reads through an image is, in the mirrored
  domain, the plain periodic neighbour holding the same value;
* at a wall node the taps of the normal velocity pair up as c * a and -c * a (the
  binary16 tap coefficients are antisymmetric, c0 = -c3, c1 = -c2), whose rounded
  products sum to exactly +0, and the tangential velocity there is zero, so the
  increment is +0 and p stays 0: the zero-increment wall rule, bit for bit.

So the device runs the unchanged periodic kernels on the mirrored domain (the fused
single-pass kernel where eligible) and the host mirrors the state in and restricts it
out; the energy of the mirrored domain counts every interior cell 2^k times (k rigid
axes) and wall rows / columns half as often, i.e. it is 2^k times the trapezoid-weighted
energy of the box (weights 1/2 on wall rows / columns).  The direct image formulation
(oracle/rigid.py) and the reference's periodic solver on the mirrored domain pin it.
Requirements: no point source (a source would need its odd images), and the state must
vanish where odd symmetry forces zero (p on every wall, the tangential velocity on its
walls); ValueError otherwise.
"""

from __future__ import annotations

import numpy as np

from .grids import Boundary, GridSpec, Stagger

# parities (x, y) of the fields under reflection about a wall
PARITY = {"p": (-1, -1), "vx": (+1, -1), "vy": (-1, +1)}


def axes(grid) -> tuple:
    return (getattr(grid, "bc_x", None) is Boundary.RIGID, getattr(grid, "bc_y", None) is Boundary.RIGID)


def is_rigid(grid) -> bool:
    return any(axes(grid))


def device_grid(grid) -> GridSpec:
    """The periodic grid the device runs: doubled along every rigid axis."""
    mx, my = axes(grid)
    return GridSpec(grid.nx * (2 if mx else 1), grid.ny * (2 if my else 1), grid.dx, grid.dt, grid.nt,
                    order=getattr(grid, "order", 4))


def energy_scale(grid) -> float:
    mx, my = axes(grid)
    return 1.0 / (2 ** (int(mx) + int(my)))


def _mirror_axis(a: np.ndarray, axis: int, half: bool, sign: int) -> np.ndarray:
    """Extend along `axis` to 2n points.  Integer sub-grid (n+1 points, walls at 0 and
    n): D[n+k] = sign * A[n-k], k = 1 .. n-1.  Half sub-grid (n points at k+1/2):
    D[n+k] = sign * A[n-1-k], k = 0 .. n-1.  Periodicity supplies the wall at 0."""
    a = np.moveaxis(a, axis, 0)
    tail = a[::-1] if half else a[-2:0:-1]
    out = np.concatenate([a, (tail if sign > 0 else -tail).astype(a.dtype)], axis=0)
    return np.ascontiguousarray(np.moveaxis(out, 0, axis))


def mirror(a: np.ndarray, stagger: Stagger, parity, grid) -> np.ndarray:
    """Box array (rigid shape) -> mirrored periodic array.  Negation is exact."""
    mx, my = axes(grid)
    out = a
    if my:
        out = _mirror_axis(out, 0, stagger.half_y, parity[1])
    if mx:
        out = _mirror_axis(out, 1, stagger.half_x, parity[0])
    return out


def restrict(d: np.ndarray, shape) -> np.ndarray:
    return np.ascontiguousarray(d[: shape[0], : shape[1]])


def check_walls(a: np.ndarray, name: str, stagger: Stagger, parity, grid) -> None:
    """Odd symmetry forces zeros on the wall lines of an integer sub-grid."""
    mx, my = axes(grid)
    bad = False
    if mx and parity[0] < 0 and not stagger.half_x:
        bad |= bool(np.any(a[:, 0] != 0) or np.any(a[:, -1] != 0))
    if my and parity[1] < 0 and not stagger.half_y:
        bad |= bool(np.any(a[0, :] != 0) or np.any(a[-1, :] != 0))
    if bad:
        raise ValueError(f"rigid walls: {name} must be zero on the walls (p = 0 there; the tangential "
                         "velocity is odd about a wall)")

"""Golden vectors for the rigid-wall (p = 0) 2D acoustic extension, made by the
UNMODIFIED reference's periodic solver on the mirrored domain.

Run in the build container (the reference is not on the GPU box):

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba \
        python tests/golden/make_rigid_golden.py

The box (nx x ny cells, p on (ny+1, nx+1) nodes, vx on (ny+1, nx), vy on (ny, nx+1))
is extended to the 2nx x 2ny periodic domain with p odd about every wall, vx even in x
/ odd in y, vy odd in x / even in y, and the medium even; the reference runs that
periodic problem; the box part of its result is the rigid-wall solution and its energy
/ 4 the box's trapezoid-weighted energy.  This script builds the mirror with its own
numpy code (independent of paper_2310_00236_b200/rigid.py).  Each case writes
tests/golden/rigid_<name>.npz: the case description (JSON), the canonical fp64 planes,
the initial box state and the reference's box results (bit patterns), traces and energy.
These fixtures pin oracle/rigid.py (the direct image formulation, tests/test_rigid.py)
and the GPU path (tests/test_gpu_rigid.py).
"""

from __future__ import annotations

import json
from pathlib import Path

import numpy as np

from halfwave.acoustic import AcousticSolver
from halfwave.efsum import Variant
from halfwave.grids import GridSpec, Medium, MediumKind
from halfwave.precision import Precision

OUT = Path(__file__).resolve().parent
V = {"naive": None, "op3": Variant.OP3, "op6": Variant.OP6}


def mirror_axis(a, axis, half, sign):
    a = np.moveaxis(a, axis, 0)
    n = a.shape[0] if half else a.shape[0] - 1
    full = np.empty((2 * n,) + a.shape[1:], dtype=a.dtype)
    full[: a.shape[0]] = a
    for k in range(1 if not half else 0, n):  # D[n+k] = sign A[n-k] (integer) / sign A[n-1-k] (half)
        src = a[n - k] if not half else a[n - 1 - k]
        full[n + k] = src if sign > 0 else -src
    return np.moveaxis(full, 0, axis)


def mirror(a, half_x, half_y, px, py):
    return mirror_axis(mirror_axis(a, 0, half_y, py), 1, half_x, px)


def box_plane(canon, int_x, int_y):
    out = canon
    if int_y:
        out = np.concatenate([out, out[-1:]], axis=0)
    if int_x:
        out = np.concatenate([out, out[:, -1:]], axis=1)
    return out


def make_case(name, nx, ny, nt, *, order=4, variant="op3", cfl=0.5, every=1, receivers=(), seed=0):
    h = 1.0 / nx
    rng = np.random.default_rng(seed)
    yc = (np.arange(ny) + 0.0) * h
    # layered canonical planes (ny, nx): kappa / rho vary with depth
    rho_c = np.where(yc < 0.45 * ny * h, 1.0, 1.5)[:, None] * np.ones((1, nx))
    kappa_c = np.where(yc < 0.6 * ny * h, 1.0, 2.25)[:, None] * np.ones((1, nx))
    canon = {"rho_x": rho_c, "rho_y": rho_c.copy(), "beta": 1.0 / kappa_c}
    c_max = float(np.sqrt(np.max(kappa_c) / np.min(rho_c)))
    dt = float(np.float16(cfl * h / c_max))
    if dt > cfl * h / c_max:
        dt = float(np.nextafter(np.float16(dt), np.float16(0)))
    # box planes on the wall sub-grids, then the even mirror
    boxp = {"rho_x": box_plane(canon["rho_x"], False, True), "rho_y": box_plane(canon["rho_y"], True, False),
            "beta": box_plane(canon["beta"], True, True)}
    mir = {"rho_x": mirror(boxp["rho_x"], True, False, 1, 1), "rho_y": mirror(boxp["rho_y"], False, True, 1, 1),
           "beta": mirror(boxp["beta"], False, False, 1, 1)}
    # box state: Gaussian bump + noise with p = 0 on the walls, small velocities
    yy, xx = np.mgrid[0: ny + 1, 0: nx + 1] * h
    p = np.exp(-((xx - 0.5 * nx * h) ** 2 + (yy - 0.5 * ny * h) ** 2) / (0.01 * (nx * h) ** 2))
    p = p + rng.uniform(-1e-3, 1e-3, p.shape)
    p[0, :] = p[-1, :] = p[:, 0] = p[:, -1] = 0.0
    vx = rng.uniform(-0.02, 0.02, (ny + 1, nx))
    vx[0, :] = vx[-1, :] = 0.0  # tangential on the y walls: odd
    vy = rng.uniform(-0.02, 0.02, (ny, nx + 1))
    vy[:, 0] = vy[:, -1] = 0.0  # tangential on the x walls: odd
    box = {"p": p.astype(np.float16), "vx": vx.astype(np.float16), "vy": vy.astype(np.float16)}
    for k in ("p", "vx", "vy"):
        box["r" + k] = np.zeros_like(box[k])
    par = {"p": (False, False, -1, -1), "vx": (True, False, 1, -1), "vy": (False, True, -1, 1)}
    # the reference on the mirrored periodic domain
    grid = GridSpec(nx=2 * nx, ny=2 * ny, dx=h, dt=dt, nt=nt)
    med = Medium(MediumKind.ACOUSTIC, 2 * nx, 2 * ny, {k: np.ascontiguousarray(v) for k, v in mir.items()})
    kw = {}
    if order != 4:
        raise SystemExit("the reference is 4th-order only; 2nd-order rigid cases are pinned by oracle/rigid.py")
    solver = AcousticSolver(grid, med, None, stencil_precision=Precision.FP16, update_precision=Precision.FP16,
                            receivers=tuple(receivers), energy_every=every, **kw)
    st = solver.new_state()
    for k in ("p", "vx", "vy", "rp", "rvx", "rvy"):
        hx, hy, px, py = par[k.lstrip("r")] if k.startswith("r") else par[k]
        getattr(st, k).values = mirror(box[k], hx, hy, px, py).astype(np.float16)
    out = solver.run(V[variant], st)
    res = {}
    for k in ("p", "vx", "vy", "rp", "rvx", "rvy"):
        shp = box[k].shape
        res["out_" + k] = getattr(st, k).values[: shp[0], : shp[1]].copy()
    desc = dict(name=name, nx=nx, ny=ny, dx=h, dt=dt, nt=nt, order=order, variant=variant, every=every,
                receivers=[list(r) for r in receivers], energy_scale=0.25)
    np.savez_compressed(
        OUT / f"rigid_{name}.npz", desc=json.dumps(desc),
        **{f"canon_{k}": v for k, v in canon.items()}, **{f"init_{k}": v for k, v in box.items()}, **res,
        traces=np.array([t.samples for t in out.traces]).reshape(len(receivers), nt),
        e_times=np.asarray(out.energy.times), e_vals=0.25 * np.asarray(out.energy.values))
    print("wrote", f"rigid_{name}.npz")


if __name__ == "__main__":
    make_case("box32_op3", 32, 24, 40, variant="op3", receivers=((16, 12), (0, 5), (31, 23), (32, 24)))
    make_case("box32_op6", 32, 24, 40, variant="op6", every=3, receivers=((5, 1),))
    make_case("box40_naive", 40, 32, 30, variant="naive", cfl=0.3, every=5, receivers=((20, 16),), seed=2)

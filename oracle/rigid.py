"""Direct rigid-wall (p = 0) 2D acoustic stepper -- TEST INFRASTRUCTURE ONLY.

Only tests/ may import this module (never the product path).  It restates the
reference's acoustic step (acoustic.py:162-181) on a box with
p = 0 walls WITHOUT the mirrored-domain trick the product uses (paper_2310_00236_b200/
rigid.py): derivatives read image values at the walls, built the way the reference
pads a free surface (stencil.py:121-144: integer sub-grid ghost[-k] = sign * a[k], half
sub-grid ghost[-k] = sign * a[k-1]) with p odd and the normal velocity even about each
wall, and the wall nodes of p take a zero increment (the reference's syy surface rule,
elastic.py:224-228).  Arithmetic: numpy in the lane dtype, one op at a time (binary16
ops are computed in binary32 and rounded once -- exact by the double-rounding theorem),
the reference's tap fold order and increment / advance sequence (stepping.py:58-98,
efsum.py:100-121).  Energy: the box's trapezoid-weighted acoustic energy
(diagnostics.py:76-87 with weights 1/2 on wall rows / columns), fp64.  Stencil and
update lane must agree (S = U).  Small grids only.
"""

from __future__ import annotations

import numpy as np

DT = {16: np.float16, 32: np.float32, 64: np.float64}


def _pad(a: np.ndarray, axis: int, half: bool, rigid: bool, parity: int) -> np.ndarray:
    """Two ghost entries on each side along `axis`: periodic wrap, or wall images."""
    a = np.moveaxis(a, axis, 0)
    if not rigid:
        lo, hi = a[-2:], a[:2]
    elif half:  # half sub-grid: ghost[-k] = sign a[k-1]
        lo, hi = parity * a[1::-1], parity * a[:-3:-1]
    else:  # integer sub-grid (walls at 0 and n): ghost[-k] = sign a[k]
        lo, hi = parity * a[2:0:-1], parity * a[-2:-4:-1]
    out = np.concatenate([lo.astype(a.dtype), a, hi.astype(a.dtype)], axis=0)
    return np.moveaxis(out, 0, axis)


def _deriv(c, a, axis, half_in, rigid, parity, order):
    """Fold (stencil.py:72-79) of the 4 taps landing on the other sub-grid.  half_in:
    output on the integer sub-grid, shifts (-2..1); else on the half sub-grid (-1..2)."""
    p = np.moveaxis(_pad(a, axis, half_in, rigid, parity), axis, 0)
    n_in = a.shape[axis]
    if rigid:
        n_out = n_in + 1 if half_in else n_in - 1
    else:
        n_out = n_in
    base = 0 if half_in else 1  # padded index of the first tap
    t = [p[base + j: base + j + n_out] for j in range(4)]
    inner = c[1] * t[1] + c[2] * t[2]  # fl(fl(c1 t1) + fl(c2 t2)): one rounding per op
    if order == 2:
        out = inner
    else:
        outer = c[0] * t[0] + c[3] * t[3]
        out = inner + outer
    return np.moveaxis(out, 0, axis)


def _advance(u, t, x, variant):
    if variant is None:
        return u + x, t
    r = t + x
    s = u + r
    if variant == "op3":
        return s, r - (s - u)
    pa = s - r
    pb = s - pa
    return s, (u - pa) + (r - pb)


def _weights(n_int: int, rigid: bool) -> np.ndarray:
    w = np.ones(n_int)
    if rigid:
        w[0] = w[-1] = 0.5
    return w


def run(state: dict, planes: dict, planes64: dict, taps, dx: float, dt: float, nt: int, *, lane: int = 16,
        variant=None, order: int = 4, rigid_x: bool = True, rigid_y: bool = True, every: int = 1,
        receivers=()):
    """state: p (ny', nx'), vx (ny', nx), vy (ny, nx'), rp, rvx, rvy in the lane dtype
    (primes: +1 on rigid axes); planes: lane-rounded rho_x / rho_y / beta on those
    shapes; planes64: the same in fp64 for the energy.  Returns (state, e_vals, traces)."""
    L = DT[lane]
    c = [L(v) for v in taps]
    dtl = L(dt)
    st = {k: np.array(v, dtype=L) for k, v in state.items()}
    wx_i = _weights(st["p"].shape[1], rigid_x)  # integer-x columns
    wy_i = _weights(st["p"].shape[0], rigid_y)  # integer-y rows

    def energy(p_old, p_new, vx, vy):
        wp = np.outer(wy_i, wx_i)
        a = np.sum(wp * planes64["beta"] * (p_old.astype(np.float64) * p_new.astype(np.float64)))
        b = np.sum(wy_i[:, None] * planes64["rho_x"] * vx.astype(np.float64) ** 2)
        d = np.sum(wx_i[None, :] * planes64["rho_y"] * vy.astype(np.float64) ** 2)
        return 0.5 * dx * dx * (a + b + d)

    e_vals = [energy(st["p"], st["p"], st["vx"], st["vy"])]
    traces = np.zeros((len(receivers), nt))
    for n in range(nt):
        p_old = st["p"].copy()
        # velocity phase from p^n (p odd about every wall)
        dxp = _deriv(c, st["p"], 1, False, rigid_x, -1, order)
        st["vx"], st["rvx"] = _advance(st["vx"], st["rvx"], (dxp / planes["rho_x"]) * dtl, variant)
        dyp = _deriv(c, st["p"], 0, False, rigid_y, -1, order)
        st["vy"], st["rvy"] = _advance(st["vy"], st["rvy"], (dyp / planes["rho_y"]) * dtl, variant)
        # pressure phase: fl(ddx vx + ddy vy) (normal velocity even about its walls)
        rhs = _deriv(c, st["vx"], 1, True, rigid_x, +1, order) + _deriv(c, st["vy"], 0, True, rigid_y, +1, order)
        if rigid_x:
            rhs[:, 0] = rhs[:, -1] = L(0)
        if rigid_y:
            rhs[0, :] = rhs[-1, :] = L(0)
        st["p"], st["rp"] = _advance(st["p"], st["rp"], (rhs / planes["beta"]) * dtl, variant)
        for j, (ix, iy) in enumerate(receivers):
            traces[j, n] = float(st["p"][iy, ix])
        if (n + 1) % every == 0:
            e_vals.append(energy(p_old, st["p"], st["vx"], st["vy"]))
    return st, np.array(e_vals), traces

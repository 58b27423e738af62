"""Grid geometry, staggering, field storage and media (reference: grids.py).

Host-side mirror of the reference types with the same names, arguments and
validation errors, extended for the BASELINE configs the reference lacks
(SURVEY §8 a'):

* ``GridSpec(..., nz=None, order=4)``: ``nz`` makes the grid 3D with arrays
  indexed ``[iz, iy, ix]`` (z is the slab axis); ``order=2`` selects the
  second-order staggered stencil (inner tap pair only).
* media may be 3D (``Medium(..., nz=...)``) and acoustic media may be layered
  or built from a velocity field.

Arrays are row-major with x fastest (grids.py:3).  With free surfaces (2D
elastic, y only) the integer-y sub-grids carry one extra row (grids.py:93-96).
"""

from __future__ import annotations

import enum
import math
from dataclasses import dataclass, field

import numpy as np

from .precision import DTYPES, as_precision


def cfl_limit(ndim: int = 2, order: int = 4) -> float:
    """Leapfrog stability bound on c dt / dx.

    The staggered spatial symbol peaks at 2*(9/8 + 1/24) = 7/3 (4th order) or 2
    (2nd order) per axis, times sqrt(ndim); leapfrog needs |omega dt| <= 2.
    ndim=2, order=4 gives the reference's 6/(7 sqrt 2) (grids.py:32-35).
    """
    peak = 7.0 / 3.0 if order == 4 else 2.0
    return 2.0 / (peak * math.sqrt(ndim))


CFL_LIMIT = cfl_limit(2, 4)


class Stagger(enum.Enum):
    """Half-cell offsets (x, y[, z]).  2D members match the reference."""

    CELL = (0, 0)
    XFACE = (1, 0)
    YFACE = (0, 1)
    NODE = (1, 1)          # 2D shear node; the xy edge in 3D
    ZFACE = (0, 0, 1)      # 3D only
    XZEDGE = (1, 0, 1)     # 3D only
    YZEDGE = (0, 1, 1)     # 3D only

    @property
    def half_x(self) -> bool:
        return bool(self.value[0])

    @property
    def half_y(self) -> bool:
        return bool(self.value[1])

    @property
    def half_z(self) -> bool:
        return len(self.value) > 2 and bool(self.value[2])

    def coords(self, n: int, dx: float, axis: int) -> np.ndarray:
        off = 0.5 * (self.value[axis] if axis < len(self.value) else 0)
        return (np.arange(n) + off) * dx


class Boundary(enum.Enum):
    PERIODIC = "periodic"
    FREE_SURFACE = "free-surface"
    RIGID = "rigid"  # extension (BASELINE config 1): p = 0 walls, 2D acoustic only

    def __str__(self):
        return self.value


@dataclass(frozen=True)
class GridSpec:
    """Uniform 2D (or, with nz, 3D) grid with its time axis and boundaries."""

    nx: int
    ny: int
    dx: float
    dt: float
    nt: int
    bc_x: Boundary = Boundary.PERIODIC
    bc_y: Boundary = Boundary.PERIODIC
    nz: int | None = None
    order: int = 4

    def __post_init__(self):
        if self.nx < 8 or self.ny < 8 or (self.nz is not None and self.nz < 8):
            dims = f"{self.nx}x{self.ny}" + (f"x{self.nz}" if self.nz is not None else "")
            raise ValueError(f"grid must be at least 8 cells per axis, got {dims}")
        if not (self.dx > 0.0 and self.dt > 0.0):
            raise ValueError("dx and dt must be positive")
        if self.nt < 0:
            raise ValueError("nt must be nonnegative")
        if self.bc_x is Boundary.FREE_SURFACE:
            raise ValueError("x boundary must be periodic (or rigid); free surfaces are y-only")
        if Boundary.RIGID in (self.bc_x, self.bc_y) and self.nz is not None:
            raise ValueError("rigid walls are a 2D acoustic extension")
        if self.order not in (2, 4):
            raise ValueError(f"order must be 2 or 4, got {self.order}")
        if self.nz is not None and self.bc_y is not Boundary.PERIODIC:
            raise ValueError("3D grids are periodic on every axis")

    @property
    def ndim(self) -> int:
        return 2 if self.nz is None else 3

    @property
    def free_surface_y(self) -> bool:
        return self.bc_y is Boundary.FREE_SURFACE

    @property
    def rigid_x(self) -> bool:
        return self.bc_x is Boundary.RIGID

    @property
    def rigid_y(self) -> bool:
        return self.bc_y is Boundary.RIGID

    def rows(self, stagger: Stagger) -> int:
        """Extent along the slow axis (y in 2D, z in 3D): integer-y sub-grids carry
        the wall / surface row too (ny + 1) with free surfaces and rigid walls."""
        if self.nz is not None:
            return self.nz
        if (self.free_surface_y or self.rigid_y) and not stagger.half_y:
            return self.ny + 1
        return self.ny

    def cols(self, stagger: Stagger) -> int:
        """Extent along x: integer-x sub-grids carry both rigid walls (nx + 1)."""
        if self.nz is None and self.rigid_x and not stagger.half_x:
            return self.nx + 1
        return self.nx

    def shape(self, stagger: Stagger) -> tuple:
        if self.nz is not None:
            return (self.nz, self.ny, self.nx)
        return (self.rows(stagger), self.cols(stagger))

    def cfl(self, c_max: float) -> float:
        return c_max * self.dt / self.dx

    def cfl_limit(self) -> float:
        return cfl_limit(self.ndim, self.order)

    def check_cfl(self, c_max: float) -> None:
        got, lim = self.cfl(c_max), self.cfl_limit()
        if got > lim:
            raise ValueError(
                f"CFL number {got:.6g} exceeds the stability bound {lim:.6g} "
                f"(c_max={c_max:.6g}, dt={self.dt:.6g}, dx={self.dx:.6g})"
            )


@dataclass
class Field2D:
    """One staggered field in its storage precision (2D or 3D values)."""

    values: np.ndarray
    stagger: Stagger

    @classmethod
    def zeros(cls, grid: GridSpec, stagger: Stagger, precision) -> "Field2D":
        return cls(np.zeros(grid.shape(stagger), dtype=DTYPES[as_precision(precision)]), stagger)


Field = Field2D


class MediumKind(enum.Enum):
    ACOUSTIC = 0
    ELASTIC = 1


def plane_order(kind: MediumKind, ndim: int = 2) -> tuple:
    if kind is MediumKind.ACOUSTIC:
        return ("rho_x", "rho_y", "beta") if ndim == 2 else ("rho_x", "rho_y", "rho_z", "beta")
    return ("rho_x", "rho_y", "lam", "mu") if ndim == 2 else ("rho_x", "rho_y", "rho_z", "lam", "mu")


PLANE_ORDER = {MediumKind.ACOUSTIC: plane_order(MediumKind.ACOUSTIC), MediumKind.ELASTIC: plane_order(MediumKind.ELASTIC)}


@dataclass(frozen=True)
class Medium:
    """Material parameters as binary64 planes of shape (ny, nx) or (nz, ny, nx)."""

    kind: MediumKind
    nx: int
    ny: int
    planes: dict = field(repr=False)
    nz: int | None = None

    @property
    def ndim(self) -> int:
        return 2 if self.nz is None else 3

    @property
    def shape(self) -> tuple:
        return (self.ny, self.nx) if self.nz is None else (self.nz, self.ny, self.nx)

    def __post_init__(self):
        want = plane_order(self.kind, self.ndim)
        if tuple(self.planes) != want:
            raise ValueError(f"expected planes {want}, got {tuple(self.planes)}")
        for name, plane in self.planes.items():
            if plane.shape != self.shape or plane.dtype != np.float64:
                raise ValueError(f"plane {name} must be float64 of shape {self.shape}")

    def _where(self, name: str, bad: np.ndarray) -> str:
        idx = tuple(int(i) for i in np.argwhere(bad)[0])
        labels = ("iy", "ix") if len(idx) == 2 else ("iz", "iy", "ix")
        loc = ", ".join(f"{k}={v}" for k, v in reversed(list(zip(labels, idx))))
        return f"{name}[{loc}] = {self.planes[name][idx]!r}"

    def validate(self) -> None:
        for name, plane in self.planes.items():
            bad = ~np.isfinite(plane)
            if bad.any():
                raise ValueError(f"non-finite medium entry at {self._where(name, bad)}")
        rhos = [n for n in self.planes if n.startswith("rho_")]
        positive = rhos + (["beta"] if self.kind is MediumKind.ACOUSTIC else [])
        for name in positive:
            bad = self.planes[name] <= 0.0
            if bad.any():
                raise ValueError(f"nonpositive medium entry at {self._where(name, bad)}")
        if self.kind is MediumKind.ELASTIC:
            bad = self.planes["mu"] < 0.0
            if bad.any():
                raise ValueError(f"negative shear modulus at {self._where('mu', bad)}")
            stiff = self.planes["lam"] + 2.0 * self.planes["mu"]
            if (stiff <= 0.0).any():
                idx = tuple(int(i) for i in np.argwhere(stiff <= 0.0)[0])
                raise ValueError(f"lam + 2 mu must be positive, got {stiff[idx]!r} at {idx}")

    def c_max(self) -> float:
        rho_min = min(self.planes[n].min() for n in self.planes if n.startswith("rho_"))
        if self.kind is MediumKind.ACOUSTIC:
            return float(1.0 / math.sqrt(rho_min * self.planes["beta"].min()))
        stiff = self.planes["lam"] + 2.0 * self.planes["mu"]
        return float(math.sqrt(stiff.max() / rho_min))


def build_homogeneous_acoustic(nx: int, ny: int, rho: float, c: float, nz: int | None = None) -> Medium:
    """Constant acoustic medium, beta = 1/(rho c^2) (grids.py:199-210)."""
    if not (rho > 0.0 and c > 0.0):
        raise ValueError("rho and c must be positive")
    beta = 1.0 / (rho * c * c)
    shape = (ny, nx) if nz is None else (nz, ny, nx)
    planes = {name: np.full(shape, beta if name == "beta" else rho, dtype=np.float64)
              for name in plane_order(MediumKind.ACOUSTIC, 2 if nz is None else 3)}
    return Medium(MediumKind.ACOUSTIC, nx, ny, planes, nz)


def _layer_column(n_slow: int, half: bool, layers, pick) -> np.ndarray:
    """Sample a depth-layered profile at one sub-grid's slow-axis coordinates."""
    ys = (np.arange(n_slow) + (0.5 if half else 0.0)) / float(n_slow)
    out = np.empty(n_slow, dtype=np.float64)
    for j, y in enumerate(ys):
        for lay in layers:
            if y < lay[0]:
                out[j] = pick(*lay[1:])
                break
        else:
            out[j] = pick(*layers[-1][1:])
    return out


def _check_layers(layers, nparams: int) -> list:
    layers = [tuple(l) for l in layers]
    if not layers:
        raise ValueError("at least one layer is required")
    prev = 0.0
    for lay in layers:
        if len(lay) != nparams + 1:
            raise ValueError(f"each layer needs {nparams + 1} entries")
        if not lay[0] > prev:
            raise ValueError("layer depth fractions must be strictly increasing")
        prev = lay[0]
    if layers[-1][0] < 1.0:
        raise ValueError("layers must cover the full depth (last fraction >= 1)")
    return layers


def _layered_planes(nx, ny, nz, names_halfs, layers, picks) -> dict:
    n_slow = ny if nz is None else nz
    planes = {}
    for name, half in names_halfs:
        col = _layer_column(n_slow, half, layers, picks[name])
        if nz is None:
            planes[name] = np.repeat(col[:, None], nx, axis=1)
        else:
            planes[name] = np.ascontiguousarray(np.broadcast_to(col[:, None, None], (nz, ny, nx)))
    return planes


def build_layered_elastic(nx: int, ny: int, layers, nz: int | None = None) -> Medium:
    """Depth-layered elastic medium (grids.py:213-269): layers of
    (depth_fraction, rho, cp, cs); lam = rho (cp^2 - 2 cs^2), mu = rho cs^2, each
    plane sampled at its own staggered slow-axis coordinate."""
    layers = _check_layers(layers, 3)
    for _, rho, cp, cs in layers:
        if not (rho > 0.0 and cp > 0.0 and cs >= 0.0):
            raise ValueError("layer parameters must be positive (cs may be zero)")
        if cs >= cp:
            raise ValueError(f"shear speed {cs} must be below pressure speed {cp}")
    rho_of = lambda rho, cp, cs: rho
    picks = {
        "rho_x": rho_of, "rho_y": rho_of, "rho_z": rho_of,
        "lam": lambda rho, cp, cs: rho * (cp * cp - 2.0 * cs * cs),
        "mu": lambda rho, cp, cs: rho * cs * cs,
    }
    if nz is None:
        nh = [("rho_x", False), ("rho_y", True), ("lam", False), ("mu", False)]
    else:
        nh = [("rho_x", False), ("rho_y", False), ("rho_z", True), ("lam", False), ("mu", False)]
    m = Medium(MediumKind.ELASTIC, nx, ny, _layered_planes(nx, ny, nz, nh, layers, picks), nz)
    m.validate()
    return m


def build_layered_acoustic(nx: int, ny: int, layers, nz: int | None = None) -> Medium:
    """Depth-layered acoustic medium (extension, BASELINE config 2): layers of
    (depth_fraction, rho, kappa) with beta = 1/kappa, sampled per stagger like
    build_layered_elastic."""
    layers = _check_layers(layers, 2)
    for _, rho, kappa in layers:
        if not (rho > 0.0 and kappa > 0.0):
            raise ValueError("layer rho and kappa must be positive")
    rho_of = lambda rho, kappa: rho
    picks = {"rho_x": rho_of, "rho_y": rho_of, "rho_z": rho_of, "beta": lambda rho, kappa: 1.0 / kappa}
    if nz is None:
        nh = [("rho_x", False), ("rho_y", True), ("beta", False)]
    else:
        nh = [("rho_x", False), ("rho_y", False), ("rho_z", True), ("beta", False)]
    m = Medium(MediumKind.ACOUSTIC, nx, ny, _layered_planes(nx, ny, nz, nh, layers, picks), nz)
    m.validate()
    return m


def build_acoustic_from_velocity(c: np.ndarray, rho: float = 1.0) -> Medium:
    """Acoustic medium from a cell-centred velocity field (extension, config 3):
    constant rho, beta = 1/(rho c^2) per cell."""
    c = np.asarray(c, dtype=np.float64)
    if c.ndim not in (2, 3) or not (rho > 0.0) or not (c > 0.0).all():
        raise ValueError("c must be a positive 2D/3D field and rho positive")
    beta = 1.0 / (rho * c * c)
    names = plane_order(MediumKind.ACOUSTIC, c.ndim)
    planes = {n: (beta if n == "beta" else np.full(c.shape, rho)) for n in names}
    if c.ndim == 2:
        return Medium(MediumKind.ACOUSTIC, c.shape[1], c.shape[0], planes)
    return Medium(MediumKind.ACOUSTIC, c.shape[2], c.shape[1], planes, c.shape[0])


def extend_rows(plane: np.ndarray, grid, stagger: Stagger) -> np.ndarray:
    """Canonical plane onto a free-surface sub-grid's ny+1 rows by repeating the
    last row (grids.py:321-331)."""
    rows = grid.rows(stagger)
    if rows == plane.shape[0]:
        return plane
    return np.concatenate([plane, plane[-1:, :]], axis=0)


def extend_cols(plane: np.ndarray, grid, stagger: Stagger) -> np.ndarray:
    """Canonical plane onto a rigid-x sub-grid's nx+1 columns by repeating the last
    column (the column analogue of extend_rows)."""
    if grid.cols(stagger) == plane.shape[1]:
        return plane
    return np.concatenate([plane, plane[:, -1:]], axis=1)


# --- WMED medium files (reference grids.py:272-318): little-endian header
# b"WMED", u32 version 1, u32 kind, u32 nx, u32 ny; then the canonical planes of
# the kind, each ny*nx binary64 row-major.  2D media only (the reference format).

import struct as _struct

_WMED = _struct.Struct("<4s4I")


def save_medium(path, medium: Medium) -> None:
    if medium.ndim != 2:
        raise ValueError("the WMED format stores 2D media only")
    with open(path, "wb") as f:
        f.write(_WMED.pack(b"WMED", 1, medium.kind.value, medium.nx, medium.ny))
        for name in plane_order(medium.kind, 2):
            f.write(np.ascontiguousarray(medium.planes[name], dtype="<f8").tobytes())


def load_medium(path) -> Medium:
    raw = open(path, "rb").read()
    if len(raw) < _WMED.size:
        raise ValueError(f"{path}: truncated header")
    magic, version, kind_code, nx, ny = _WMED.unpack_from(raw)
    if magic != b"WMED":
        raise ValueError(f"{path}: bad magic {magic!r}, expected b'WMED'")
    if version != 1:
        raise ValueError(f"{path}: unsupported version {version}")
    try:
        kind = MediumKind(kind_code)
    except ValueError:
        raise ValueError(f"{path}: unknown medium kind {kind_code}") from None
    names = plane_order(kind, 2)
    need = _WMED.size + len(names) * nx * ny * 8
    if len(raw) != need:
        raise ValueError(f"{path}: size mismatch, got {len(raw)} bytes, need {need} "
                         f"for {len(names)} planes of {nx}x{ny}")
    planes = {}
    for k, name in enumerate(names):
        off = _WMED.size + k * nx * ny * 8
        planes[name] = np.frombuffer(raw, dtype="<f8", count=nx * ny, offset=off).reshape(ny, nx).astype(np.float64)
    m = Medium(kind, nx, ny, planes)
    m.validate()
    return m

"""Acoustic p-v leapfrog solver on the B200 (reference: acoustic.py).

Same entry points and arguments as ``halfwave.AcousticSolver``
(acoustic.py:56-236); every step runs in the sm_100a kernels of
csrc/hw_acoustic.cu through the C ABI.  Extensions (SURVEY §8 a'): 3D grids
(``GridSpec(nz=...)``, fields p, vx, vy, vz), the second-order stencil, and rigid
p = 0 walls (``bc_x`` / ``bc_y`` = ``Boundary.RIGID``; p on (ny+1, nx+1) nodes, run
as the mirrored periodic problem, see rigid.py).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _abi, rigid
from .efsum import Variant
from .grids import Field2D, Stagger, extend_cols, extend_rows
from .solver import DEFAULT_ENERGY_EVERY, _DeviceSolver, _grid_nz, _is_free_surface, _kind_name


@dataclass
class AcousticState:
    """Solution fields plus one residual per field (acoustic.py:35-50); 3D adds vz, rvz."""

    p: Field2D
    vx: Field2D
    vy: Field2D
    rp: Field2D
    rvx: Field2D
    rvy: Field2D
    step: int = 0
    vz: Field2D | None = None
    rvz: Field2D | None = None


class AcousticSolver(_DeviceSolver):
    EQUATION = _abi.EQ_ACOUSTIC
    DEFAULT_VARIANT = Variant.OP3
    TRACE_FIELD = "p"
    STATE_CLS = AcousticState

    def __init__(self, grid, medium, source=None, **kw):
        nz = _grid_nz(grid)
        if nz is None:
            self.FIELDS = ("p", "vx", "vy", "rp", "rvx", "rvy")
            self.STAGGERS = {"p": Stagger.CELL, "vx": Stagger.XFACE, "vy": Stagger.YFACE}
        else:
            self.FIELDS = ("p", "vx", "vy", "vz", "rp", "rvx", "rvy", "rvz")
            self.STAGGERS = {"p": Stagger.CELL, "vx": Stagger.XFACE, "vy": Stagger.YFACE, "vz": Stagger.ZFACE}
        super().__init__(grid, medium, source, **kw)

    def _validate(self, grid, medium, source, receivers, energy_every):
        if _is_free_surface(grid):
            raise ValueError("the acoustic solver supports periodic boundaries (and the rigid-wall extension) only")
        if rigid.is_rigid(grid) and source is not None:
            raise ValueError("rigid walls: point sources are not supported (they would need odd images)")
        if _kind_name(medium) != "ACOUSTIC":
            raise ValueError("acoustic solver needs an acoustic medium")
        if source is not None and getattr(source.kind, "value", source.kind) != "pressure-point":
            raise ValueError("acoustic runs drive a pressure point source")
        self._validate_common(grid, medium, source, receivers, energy_every)

    # rigid walls: the device runs the mirrored periodic domain (rigid.py)
    def _device_grid(self):
        return rigid.device_grid(self.grid) if rigid.is_rigid(self.grid) else self.grid

    def _to_device(self, name, arr):
        if not rigid.is_rigid(self.grid):
            return arr
        base = name[1:] if name.startswith("r") and name[1:] in rigid.PARITY else name
        st, par = self._stagger_of(name), rigid.PARITY[base]
        rigid.check_walls(arr, name, st, par, self.grid)
        return rigid.mirror(arr, st, par, self.grid)

    def _to_user(self, name, arr):
        if not rigid.is_rigid(self.grid):
            return arr
        return rigid.restrict(arr, self.grid.shape(self._stagger_of(name)))

    def _energy_scale(self) -> float:
        return rigid.energy_scale(self.grid)

    def _planes(self) -> dict:
        pl = self.medium.planes
        if rigid.is_rigid(self.grid):  # canonical planes -> wall sub-grids -> even mirror
            g = self.grid

            def dev(plane, st):
                box = extend_cols(extend_rows(plane, g, st), g, st)
                return rigid.mirror(box, st, (1, 1), g)

            return {_abi.PL_RHO_X: dev(pl["rho_x"], Stagger.XFACE), _abi.PL_RHO_S: dev(pl["rho_y"], Stagger.YFACE),
                    _abi.PL_BETA: dev(pl["beta"], Stagger.CELL)}
        out = {_abi.PL_RHO_X: pl["rho_x"], _abi.PL_BETA: pl["beta"]}
        if self.ndim == 2:
            out[_abi.PL_RHO_S] = pl["rho_y"]
        else:
            out[_abi.PL_RHO_M] = pl["rho_y"]
            out[_abi.PL_RHO_S] = pl["rho_z"]
        return out

    def _source_code(self) -> int:
        return _abi.SRC_PRESSURE

    def _source_time(self, step: int) -> float:
        return (step + 0.5) * self.grid.dt  # acoustic.py:177

    def new_state(self) -> AcousticState:
        return super().new_state()

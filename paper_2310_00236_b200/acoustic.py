"""Acoustic p-v leapfrog solver on the B200 (reference: acoustic.py).

Same entry points and arguments as ``halfwave.AcousticSolver``
(acoustic.py:56-236); every step runs in the sm_100a kernels of
csrc/hw_acoustic.cu through the C ABI.  Extensions (SURVEY §8 a'): 3D grids
(``GridSpec(nz=...)``, fields p, vx, vy, vz) and the second-order stencil.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _abi
from .efsum import Variant
from .grids import Field2D, Stagger
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
            raise ValueError("the acoustic solver supports periodic boundaries only")
        if _kind_name(medium) != "ACOUSTIC":
            raise ValueError("acoustic solver needs an acoustic medium")
        if source is not None and getattr(source.kind, "value", source.kind) != "pressure-point":
            raise ValueError("acoustic runs drive a pressure point source")
        self._validate_common(grid, medium, source, receivers, energy_every)

    def _planes(self) -> dict:
        pl = self.medium.planes
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

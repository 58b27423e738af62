"""Elastic velocity-stress leapfrog solver on the B200 (reference: elastic.py).

Same entry points and arguments as ``halfwave.ElasticSolver``
(elastic.py:63-296): periodic x, periodic or free-surface y, vy point source;
every step runs in csrc/hw_elastic.cu.  Extensions (SURVEY §8 a'): 3D grids
(9 fields, periodic), the second-order stencil and an explosive source
(``SourceKind.EXPLOSIVE``, injected into every normal-stress increment at
t = (n + 1/2) dt).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _abi
from .efsum import Variant
from .grids import Field2D, Stagger, extend_rows
from .solver import DEFAULT_ENERGY_EVERY, _DeviceSolver, _grid_nz, _is_free_surface, _kind_name


@dataclass
class ElasticState:
    """Five fields plus residuals (elastic.py:43-57); 3D adds vz, szz, sxz, syz."""

    vx: Field2D
    vy: Field2D
    sxx: Field2D
    syy: Field2D
    sxy: Field2D
    rvx: Field2D
    rvy: Field2D
    rsxx: Field2D
    rsyy: Field2D
    rsxy: Field2D
    step: int = 0
    vz: Field2D | None = None
    szz: Field2D | None = None
    sxz: Field2D | None = None
    syz: Field2D | None = None
    rvz: Field2D | None = None
    rszz: Field2D | None = None
    rsxz: Field2D | None = None
    rsyz: Field2D | None = None


class ElasticSolver(_DeviceSolver):
    EQUATION = _abi.EQ_ELASTIC
    DEFAULT_VARIANT = Variant.OP6
    STATE_CLS = ElasticState

    def __init__(self, grid, medium, source=None, **kw):
        if _grid_nz(grid) is None:
            self.FIELDS = ("vx", "vy", "sxx", "syy", "sxy", "rvx", "rvy", "rsxx", "rsyy", "rsxy")
            self.STAGGERS = {"vx": Stagger.XFACE, "vy": Stagger.YFACE, "sxx": Stagger.CELL,
                             "syy": Stagger.CELL, "sxy": Stagger.NODE}
            self.TRACE_FIELD = "vy"
        else:
            sol = ("vx", "vy", "vz", "sxx", "syy", "szz", "sxy", "sxz", "syz")
            self.FIELDS = sol + tuple("r" + n for n in sol)
            self.STAGGERS = {"vx": Stagger.XFACE, "vy": Stagger.YFACE, "vz": Stagger.ZFACE,
                             "sxx": Stagger.CELL, "syy": Stagger.CELL, "szz": Stagger.CELL,
                             "sxy": Stagger.NODE, "sxz": Stagger.XZEDGE, "syz": Stagger.YZEDGE}
            self.TRACE_FIELD = "vz"
        super().__init__(grid, medium, source, **kw)

    def _validate(self, grid, medium, source, receivers, energy_every):
        if _kind_name(medium) != "ELASTIC":
            raise ValueError("elastic solver needs an elastic medium")
        if source is not None:
            kind = getattr(source.kind, "value", source.kind)
            if kind not in ("vy-point", "explosive"):
                raise ValueError("elastic runs drive a vertical-velocity point source")
            if kind == "explosive" and _is_free_surface(grid) and source.iy in (0, grid.ny):
                raise ValueError("an explosive source cannot sit on a free-surface row")
        self._validate_common(grid, medium, source, receivers, energy_every)

    def _planes(self) -> dict:
        g, pl = self.grid, self.medium.planes
        lam, mu = pl["lam"], pl["mu"]
        if self.ndim == 3:
            return {_abi.PL_RHO_X: pl["rho_x"], _abi.PL_RHO_M: pl["rho_y"], _abi.PL_RHO_S: pl["rho_z"],
                    _abi.PL_LAM: lam, _abi.PL_MU: mu, _abi.PL_STIFF: lam + 2.0 * mu, _abi.PL_MU_N: mu}
        out = {
            # elastic.py:101-109 and diagnostics.py:127-131
            _abi.PL_RHO_X: extend_rows(pl["rho_x"], g, Stagger.XFACE),
            _abi.PL_RHO_S: pl["rho_y"],
            _abi.PL_LAM: extend_rows(lam, g, Stagger.CELL),
            _abi.PL_MU: extend_rows(mu, g, Stagger.CELL),
            _abi.PL_STIFF: extend_rows(lam + 2.0 * mu, g, Stagger.CELL),
            _abi.PL_MU_N: mu,
        }
        if _is_free_surface(g):  # plane-stress modulus rows (elastic.py:110-113)
            ep = extend_rows(4.0 * mu * (lam + mu) / (lam + 2.0 * mu), g, Stagger.CELL)
            out[_abi.PL_EP] = np.stack([ep[0], ep[-1]])
        return out

    def _source_code(self) -> int:
        kind = getattr(self.source.kind, "value", self.source.kind)
        return _abi.SRC_EXPLOSIVE if kind == "explosive" else _abi.SRC_VSLOW

    def _source_time(self, step: int) -> float:
        if self._source_code() == _abi.SRC_EXPLOSIVE:
            return (step + 0.5) * self.grid.dt  # stresses live on integer levels
        return step * self.grid.dt  # elastic.py:198

    def new_state(self) -> ElasticState:
        return super().new_state()

"""paper_2310_00236_b200 — B200-native (sm_100a) compensated-fp16 staggered leapfrog.

Drop-in for the hot path of the reference ``halfwave`` package: the acoustic and
elastic solvers (``AcousticSolver`` / ``ElasticSolver``) with the same
constructors, ``run`` / ``step_baseline`` / ``step_compensated`` and outputs,
executing every time step in hand-written CUDA kernels behind a C ABI
(include/halfwave_b200.h).  No CPU fallback.
"""

from ._abi import get_option, options, set_option
from .acoustic import AcousticSolver, AcousticState
from .diagnostics import EnergySeries, RangeFailureError, RunOutput, TraceSeries, compare_traces, energy_drift
from .efsum import Variant
from .elastic import ElasticSolver, ElasticState
from .grids import (
    CFL_LIMIT,
    Boundary,
    Field2D,
    GridSpec,
    Medium,
    MediumKind,
    Stagger,
    build_acoustic_from_velocity,
    build_homogeneous_acoustic,
    build_layered_acoustic,
    build_layered_elastic,
    cfl_limit,
    extend_rows,
    load_medium,
    save_medium,
)
from .config import DT16, PRESETS, ConfigError, SimConfig, parse_config
from .precision import FORMATS, Precision, round_fraction, round_to
from .sources import RickerSpec, SourceKind, SourceSpec, ricker, sample_source
from .stencil import StencilSpec

__all__ = [
    "AcousticSolver", "AcousticState", "Boundary", "CFL_LIMIT", "ElasticSolver", "ElasticState",
    "EnergySeries", "FORMATS", "Field2D", "GridSpec", "Medium", "MediumKind", "Precision",
    "RangeFailureError", "RickerSpec", "RunOutput", "SourceKind", "SourceSpec", "Stagger",
    "StencilSpec", "TraceSeries", "Variant", "build_acoustic_from_velocity",
    "build_homogeneous_acoustic", "build_layered_acoustic", "build_layered_elastic", "cfl_limit",
    "compare_traces", "energy_drift", "extend_rows", "ricker", "round_fraction", "round_to",
    "sample_source", "load_medium", "save_medium", "DT16", "PRESETS", "ConfigError", "SimConfig",
    "parse_config", "set_option", "get_option", "options",
]

__version__ = "0.1.0"

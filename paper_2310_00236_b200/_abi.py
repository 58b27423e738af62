"""ctypes binding of the C ABI in include/halfwave_b200.h.

The shared library is built in-tree (``make`` or ``__graft_entry__.build()``) to
``paper_2310_00236_b200/lib/libhalfwave_b200.so`` for sm_100a.  There is no CPU
fallback: if the library is missing, or no CUDA device is usable, every solver
call raises.
"""

from __future__ import annotations

import ctypes
from pathlib import Path

import os

LIB_PATH = Path(__file__).resolve().parent / "lib" / "libhalfwave_b200.so"


def set_library_path(path) -> None:
    """Load an alternative build of the library (A/B measurements); before the first call only."""
    global LIB_PATH
    if _lib is not None:
        raise RuntimeError("the library is already loaded")
    LIB_PATH = Path(path)

ABI_VERSION = 1

# hw_status
OK, RANGE_FAILURE, EINVAL, ECUDA, ENCCL = 0, 1, 2, 3, 4
# hw_equation
EQ_ACOUSTIC, EQ_ELASTIC = 0, 1
# hw_variant
NAIVE, OP3, OP6 = 0, 3, 6
# hw_bc
BC_PERIODIC, BC_FREE_SURFACE = 0, 1
# hw_source
SRC_NONE, SRC_PRESSURE, SRC_VSLOW, SRC_EXPLOSIVE = 0, 1, 2, 3
# hw_plane
PL_RHO_X, PL_RHO_S, PL_RHO_M, PL_BETA, PL_LAM, PL_MU, PL_STIFF, PL_MU_N, PL_EP = range(9)
NPLANES = 9

EXPORTED = (
    "hw_num_fields", "hw_field_shape", "hw_create", "hw_destroy", "hw_set_state",
    "hw_get_state", "hw_run", "hw_run_device", "hw_last_launch_count", "hw_kernel_path", "hw_transport",
    "hw_last_kernel_ms", "hw_last_error", "hw_version", "hw_selftest_div16",
    "hw_cheap_div_table", "hw_plane_div_mode", "hw_nccl_unique_id", "hw_create_group", "hw_run_group",
    "hw_set_option", "hw_get_option", "hw_exchange_plan", "hw_selftest_guard",
)

# hw_plan_kind
PLAN_VEL, PLAN_STRESS, PLAN_FUSED, PLAN_FUSED_EL3, PLAN_FUSED_AC3, PLAN_FUSED_EL2 = 0, 1, 2, 3, 4, 5


class Xfer(ctypes.Structure):
    """Mirror of ``hw_xfer``."""

    _fields_ = [("field", ctypes.c_int32), ("peer", ctypes.c_int32), ("send", ctypes.c_int32), ("pad", ctypes.c_int32),
                ("row0", ctypes.c_int64), ("nrows", ctypes.c_int64)]


class Desc(ctypes.Structure):
    """Mirror of ``hw_desc``; field order and types must match the header."""

    _fields_ = [
        ("abi_version", ctypes.c_int32),
        ("equation", ctypes.c_int32),
        ("ndim", ctypes.c_int32),
        ("order", ctypes.c_int32),
        ("bc_slow", ctypes.c_int32),
        ("lane_s", ctypes.c_int32),
        ("lane_u", ctypes.c_int32),
        ("src_kind", ctypes.c_int32),
        ("nx", ctypes.c_int64),
        ("nm", ctypes.c_int64),
        ("ns", ctypes.c_int64),
        ("dx", ctypes.c_double),
        ("dt", ctypes.c_double),
        ("taps", ctypes.c_double * 4),
        ("plane", ctypes.POINTER(ctypes.c_double) * NPLANES),
        ("src_x", ctypes.c_int64),
        ("src_m", ctypes.c_int64),
        ("src_s", ctypes.c_int64),
        ("receivers", ctypes.POINTER(ctypes.c_int64)),
        ("n_receivers", ctypes.c_int32),
        ("world_size", ctypes.c_int32),
        ("rank", ctypes.c_int32),
        ("device", ctypes.c_int32),
        ("nccl_unique_id", ctypes.c_void_p),
        ("energy_every", ctypes.c_int64),
    ]


_lib = None


def load() -> ctypes.CDLL:
    """Load the sm_100a library once; raise loudly if it is not built."""
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        raise RuntimeError(
            f"{LIB_PATH} is missing: build the CUDA library first "
            "(`make` or `python -c 'import __graft_entry__ as g; g.build()'`); "
            "there is no CPU fallback"
        )
    lib = ctypes.CDLL(str(LIB_PATH))
    P = ctypes.POINTER
    vp = ctypes.c_void_p
    i32, i64, dbl = ctypes.c_int32, ctypes.c_int64, ctypes.c_double
    lib.hw_num_fields.argtypes = [i32, i32]
    lib.hw_num_fields.restype = ctypes.c_int
    lib.hw_field_shape.argtypes = [P(Desc), i32, P(i64)]
    lib.hw_create.argtypes = [P(Desc), P(vp)]
    lib.hw_destroy.argtypes = [vp]
    lib.hw_set_state.argtypes = [vp, P(vp)]
    lib.hw_get_state.argtypes = [vp, P(vp)]
    lib.hw_run.argtypes = [vp, i32, i64, i64, P(dbl), P(dbl), P(dbl), P(dbl), P(i64), P(i64), P(i32)]
    lib.hw_run_device.argtypes = [vp, i32, i64, i64, P(dbl), P(ctypes.c_float)]
    lib.hw_last_launch_count.argtypes = [vp]
    lib.hw_last_launch_count.restype = i64
    lib.hw_kernel_path.argtypes = [vp]
    lib.hw_transport.argtypes = [vp]
    lib.hw_transport.restype = i32
    lib.hw_kernel_path.restype = ctypes.c_char_p
    lib.hw_last_kernel_ms.argtypes = [vp]
    lib.hw_last_kernel_ms.restype = dbl
    lib.hw_last_error.argtypes = []
    lib.hw_last_error.restype = ctypes.c_char_p
    lib.hw_selftest_div16.argtypes = [i32, P(ctypes.c_uint64), P(ctypes.c_uint32)]
    lib.hw_selftest_div16.restype = ctypes.c_int
    lib.hw_selftest_guard.argtypes = [i32, ctypes.c_int64]
    lib.hw_selftest_guard.restype = ctypes.c_int
    lib.hw_cheap_div_table.argtypes = [i32, P(ctypes.c_uint32)]
    lib.hw_cheap_div_table.restype = ctypes.c_int
    lib.hw_plane_div_mode.argtypes = [vp, i32]
    lib.hw_plane_div_mode.restype = ctypes.c_int
    if hasattr(lib, "hw_create_group"):  # absent only in older A/B builds
        lib.hw_nccl_unique_id.argtypes = [vp]
        lib.hw_nccl_unique_id.restype = ctypes.c_int
        lib.hw_create_group.argtypes = [P(Desc), i32, P(i32), P(vp)]
        lib.hw_create_group.restype = ctypes.c_int
        lib.hw_run_group.argtypes = [P(vp), i32, i32, i64, i64, P(dbl), P(dbl), P(dbl), P(dbl), P(i64), P(i64), P(i32)]
        lib.hw_run_group.restype = ctypes.c_int
    lib.hw_exchange_plan.argtypes = [P(Desc), i32, i32, i32, P(Xfer), i32, P(i32)]
    lib.hw_exchange_plan.restype = ctypes.c_int
    lib.hw_set_option.argtypes = [ctypes.c_char_p, i64]
    lib.hw_set_option.restype = ctypes.c_int
    lib.hw_get_option.argtypes = [ctypes.c_char_p, P(i64)]
    lib.hw_get_option.restype = ctypes.c_int
    lib.hw_version.argtypes = []
    lib.hw_version.restype = ctypes.c_char_p
    for name in ("hw_create", "hw_destroy", "hw_set_state", "hw_get_state", "hw_run", "hw_run_device"):
        getattr(lib, name).restype = ctypes.c_int
    _lib = lib
    return lib


def last_error() -> str:
    return load().hw_last_error().decode()


def check(status: int, what: str) -> None:
    if status != OK:
        raise RuntimeError(f"{what} failed (status {status}): {last_error()}")


def set_option(name: str, value: int) -> None:
    """Process-wide kernel-path option (include/halfwave_b200.h hw_set_option); applies to
    solvers whose device handle is created afterwards."""
    check(load().hw_set_option(name.encode(), int(value)), f"hw_set_option({name})")


def get_option(name: str) -> int:
    v = ctypes.c_int64(0)
    check(load().hw_get_option(name.encode(), ctypes.byref(v)), f"hw_get_option({name})")
    return int(v.value)


class options:
    """Context manager: ``with options(path=1): ...`` sets options and restores them on exit."""

    def __init__(self, **kw):
        self.kw = kw
        self.saved = {}

    def __enter__(self):
        for k, v in self.kw.items():
            self.saved[k] = get_option(k)
            set_option(k, v)
        return self

    def __exit__(self, *exc):
        for k, v in self.saved.items():
            set_option(k, v)
        return False


def exchange_plan(desc, world: int, rank: int, kind: int) -> list:
    """The library's halo plan for one slab (hw_exchange_plan): a list of dicts
    (field, peer, send, row0, nrows) in issue order.  No CUDA device needed."""
    lib = load()
    n = ctypes.c_int32(0)
    check(lib.hw_exchange_plan(ctypes.byref(desc), world, rank, kind, None, 0, ctypes.byref(n)), "hw_exchange_plan")
    buf = (Xfer * max(n.value, 1))()
    check(lib.hw_exchange_plan(ctypes.byref(desc), world, rank, kind, buf, n.value, ctypes.byref(n)), "hw_exchange_plan")
    return [dict(field=x.field, peer=x.peer, send=bool(x.send), row0=x.row0, nrows=x.nrows) for x in buf[:n.value]]

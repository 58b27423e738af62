"""CPU ORACLE — TEST INFRASTRUCTURE ONLY.

ctypes wrapper of oracle/halfwave_oracle.c, the plain-C restatement of the
reference leapfrog hot path (/root/reference/pkg/src/halfwave: acoustic.py,
elastic.py, stepping.py, stencil.py, efsum.py, diagnostics.py).  Only tests/,
__graft_entry__.smoke() and bench.py (cpu_baseline and --impl reference) may
import this package; the product never does.

Pinned against golden vectors produced by the unmodified reference
(tests/golden/make_golden.py -> tests/golden/*.npz, checked by
tests/test_oracle_golden.py).
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB = HERE / "_build" / "liboracle.so"

_lib = None


def build(force: bool = False) -> Path:
    if force or not LIB.exists() or LIB.stat().st_mtime < (HERE / "halfwave_oracle.c").stat().st_mtime:
        subprocess.run(["make", "-C", str(HERE)], check=True, capture_output=True)
    return LIB


def load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(str(LIB))
        P = ctypes.POINTER
        d = ctypes.c_double
        lib.hwo_run.argtypes = [ctypes.c_void_p, P(P(d)), ctypes.c_int, ctypes.c_int64, ctypes.c_int64,
                                P(d), P(d), P(d), P(d), P(ctypes.c_int64), P(ctypes.c_int64),
                                P(ctypes.c_int32), ctypes.c_int]
        lib.hwo_run.restype = ctypes.c_int
        lib.hwo_round.argtypes = [ctypes.c_int, P(d), P(d), ctypes.c_int64]
        lib.hwo_round.restype = None
        _lib = lib
    return _lib


def round_lane(lane: int, x: np.ndarray) -> np.ndarray:
    """Round binary64 values once into lane 16/32/64 (returned as binary64)."""
    x = np.ascontiguousarray(x, dtype=np.float64)
    out = np.empty_like(x)
    P = ctypes.POINTER(ctypes.c_double)
    load().hwo_round(lane, x.ctypes.data_as(P), out.ctypes.data_as(P), x.size)
    return out


def run_desc(desc, arrays, variant: int, step0: int, nt: int, src=None, energy: bool = True,
             nthreads: int = 0) -> dict:
    """Run the oracle on an hw_desc (paper_2310_00236_b200._abi.Desc).

    arrays: state fields in external order (update-lane numpy arrays).
    Returns dict(fields=[...same dtypes...], traces, e_times, e_vals, fail=(step, field) | None).
    """
    lib = load()
    dtype = arrays[0].dtype
    work = [np.ascontiguousarray(a, dtype=np.float64).copy() for a in arrays]
    P = ctypes.POINTER(ctypes.c_double)
    ptrs = (P * len(work))(*[w.ctypes.data_as(P) for w in work])
    nrec = desc.n_receivers
    traces = np.zeros((max(nrec, 1), max(nt, 1)), dtype=np.float64)
    cap = 1 + nt // desc.energy_every
    e_times = np.zeros(cap)
    e_vals = np.zeros(cap)
    ne = ctypes.c_int64(0)
    fs, ff = ctypes.c_int64(-1), ctypes.c_int32(-1)
    srcp = None
    if src is not None:
        src = np.ascontiguousarray(src, dtype=np.float64)
        srcp = src.ctypes.data_as(P)
    rc = lib.hwo_run(ctypes.addressof(desc), ptrs, variant, step0, nt, srcp, traces.ctypes.data_as(P),
                     e_times.ctypes.data_as(P) if energy else None,
                     e_vals.ctypes.data_as(P) if energy else None, ctypes.byref(ne), ctypes.byref(fs),
                     ctypes.byref(ff), nthreads)
    with np.errstate(over="ignore", invalid="ignore"):
        fields = [w.astype(dtype) for w in work]
    k = ne.value
    return {
        "fields": fields,
        "traces": traces[:nrec, :nt],
        "e_times": e_times[:k],
        "e_vals": e_vals[:k],
        "fail": (int(fs.value), int(ff.value)) if rc == 1 else None,
    }


def solver_arrays(solver, state) -> list:
    return [np.ascontiguousarray(getattr(state, n).values) for n in solver.FIELDS]


def run_solver(solver, variant, state=None, nt=None, energy=True, nthreads=0) -> dict:
    """The oracle twin of solver.run(variant, state): same desc, same source samples.

    Does not modify `state`; returns run_desc's dict plus `step0`.
    """
    from paper_2310_00236_b200.efsum import variant_code

    state = state if state is not None else solver.new_state()
    nt = solver.grid.nt if nt is None else nt
    src = solver.source_samples(state.step, nt)
    out = run_desc(solver.desc, solver_arrays(solver, state), variant_code(variant), state.step, nt, src,
                   energy=energy, nthreads=nthreads)
    out["step0"] = state.step
    return out


def timed_steps(desc, arrays64, variant: int, step0: int, nt: int, src=None, nthreads: int = 0,
                energy: bool = False) -> float:
    """Advance binary64-container state arrays in place by nt steps; return the wall
    seconds of the C call alone (CPU-baseline timing, no Python conversions)."""
    import time

    lib = load()
    P = ctypes.POINTER(ctypes.c_double)
    ptrs = (P * len(arrays64))(*[a.ctypes.data_as(P) for a in arrays64])
    srcp = None
    if src is not None:
        src = np.ascontiguousarray(src, dtype=np.float64)
        srcp = src.ctypes.data_as(P)
    cap = 1 + nt // desc.energy_every
    e = np.zeros(cap) if energy else None
    t0 = time.perf_counter()
    lib.hwo_run(ctypes.addressof(desc), ptrs, variant, step0, nt, srcp, None,
                e.ctypes.data_as(P) if energy else None, None, None, None, None, nthreads)
    return time.perf_counter() - t0

"""Shared solver plumbing over the C ABI (reference: acoustic.py / elastic.py).

``_DeviceSolver`` mirrors the reference solvers' constructor, state handling,
single-step API and ``run`` loop.  It validates exactly like the reference
(ValueError messages included), materialises the binary64 medium planes with
the reference's own expressions, builds one ``hw_desc`` and then hands every
step to the sm_100a library: state lives in HBM inside the handle for the whole
``run``; the host crosses the boundary once per call.

Reference objects (``halfwave.GridSpec``, ``Medium``, ``SourceSpec``,
``Precision``, ``Variant``) are accepted as well as this package's mirrors.
"""

from __future__ import annotations

import ctypes
from dataclasses import fields as dc_fields

import numpy as np

from . import _abi
from .diagnostics import EnergySeries, RangeFailureError, RunOutput, TraceSeries
from .efsum import variant_code
from .grids import Field2D, Stagger, extend_rows
from .precision import DTYPES, LANE_BITS, Precision, as_precision
from .sources import sample_source
from .stencil import StencilSpec

_PINNED = None  # torch's caching pinned-host allocator (None: not probed yet, False: unavailable)


def _host_empty(shape, dtype) -> np.ndarray:
    """A new host array for downloaded state.  Page-locked when torch + CUDA are present:
    the arrays come from torch's caching pinned allocator (returned to its pool when the
    numpy array is freed), so device<->host copies of the state run at pinned bandwidth
    without a cudaHostAlloc per call; plain numpy memory otherwise."""
    global _PINNED
    if _PINNED is None:
        try:
            import torch
            _PINNED = torch if torch.cuda.is_available() else False
        except Exception:  # noqa: BLE001 - torch is optional plumbing here
            _PINNED = False
    if _PINNED is not False:
        tdt = {np.dtype(np.float16): _PINNED.float16, np.dtype(np.float32): _PINNED.float32,
               np.dtype(np.float64): _PINNED.float64}.get(np.dtype(dtype))
        if tdt is not None:
            return _PINNED.empty(tuple(shape), dtype=tdt, pin_memory=True).numpy()
    return np.empty(shape, dtype=dtype)

DEFAULT_ENERGY_EVERY = 10


def _enum_value(x):
    return getattr(x, "value", x)


def _kind_name(medium) -> str:
    return getattr(medium.kind, "name", str(medium.kind))


def _grid_nz(grid):
    return getattr(grid, "nz", None)


def _is_free_surface(grid) -> bool:
    return _enum_value(grid.bc_y) == "free-surface"


class _DeviceSolver:
    """Common constructor / state / run machinery; subclasses define the fields."""

    EQUATION = None          # _abi.EQ_ACOUSTIC / EQ_ELASTIC
    DEFAULT_VARIANT = None   # step_compensated default
    TRACE_FIELD = None

    def __init__(self, grid, medium, source=None, *, stencil_precision=Precision.FP64,
                 update_precision=None, receivers=(), energy_every=DEFAULT_ENERGY_EVERY,
                 device: int = 0, slabs: int = 1, devices=None, distributed: bool = False):
        """Extra keywords (not in the reference): `device` (CUDA ordinal); `slabs=N`
        decomposes the slow axis into N slabs driven by this process (on `devices`,
        default all on `device`); `distributed=True` makes this process one rank of a
        torch.distributed job (one process per GPU, NCCL halo exchange)."""
        self._handle = None
        self._group = None
        self.slabs = int(slabs)
        self.devices = list(devices) if devices is not None else None
        self.distributed = bool(distributed)
        if self.slabs > 1 and self.distributed:
            raise ValueError("use either slabs= (one process) or distributed=True (one process per GPU)")
        self._validate(grid, medium, source, receivers, energy_every)
        self.grid = grid
        self.medium = medium
        self.source = source
        self.receivers = tuple(tuple(r) for r in receivers)
        self.energy_every = energy_every
        self.device = device
        sp = as_precision(stencil_precision)
        up = as_precision(update_precision) if update_precision is not None else sp
        self.stencil_precision = sp
        self.update_precision = up
        self.ndim = 2 if _grid_nz(grid) is None else 3
        self.order = getattr(grid, "order", 4)
        self.stencil = StencilSpec.make(sp, grid.dx, self.order)
        self._dgrid = self._device_grid()
        self._build_desc()

    # ------------------------------------------------------------ validation
    @staticmethod
    def _check_index(what, idx, grid, ext=None):
        ix, iy = idx[0], idx[1]
        nz = _grid_nz(grid)
        nx_, ny_ = ext if ext is not None else (grid.nx, grid.ny)
        ok = 0 <= ix < nx_ and 0 <= iy < ny_
        if nz is not None:
            iz = idx[2] if len(idx) > 2 and idx[2] is not None else -1
            ok = ok and 0 <= iz < nz
        if not ok:
            raise ValueError(f"{what} index {tuple(i for i in idx if i is not None)} is outside the grid")

    def _validate_common(self, grid, medium, source, receivers, energy_every):
        nz_m = getattr(medium, "nz", None)
        if (medium.ny, medium.nx) != (grid.ny, grid.nx) or nz_m != _grid_nz(grid):
            raise ValueError(f"medium is {medium.nx}x{medium.ny}, grid is {grid.nx}x{grid.ny}")
        medium.validate()
        grid.check_cfl(medium.c_max())
        if source is not None:
            self._check_index("source", (source.ix, source.iy, getattr(source, "iz", None)), grid)
        ext = None
        if hasattr(grid, "cols") and _grid_nz(grid) is None and self.TRACE_FIELD in self.STAGGERS:
            st = self.STAGGERS[self.TRACE_FIELD]  # receivers index the trace field's own sub-grid
            ext = (grid.cols(st), grid.ny if _is_free_surface(grid) else grid.rows(st))
        for r in receivers:
            self._check_index("receiver", tuple(r), grid, ext)
        if energy_every < 1:
            raise ValueError("energy_every must be at least 1")

    # ------------------------------------------------------------ descriptor
    def _planes(self) -> dict:
        raise NotImplementedError

    def _source_code(self) -> int:
        raise NotImplementedError

    # ------------------------------------------------------------ device domain hooks
    def _device_grid(self):
        """The grid the device runs (the mirrored periodic grid for rigid walls)."""
        return self.grid

    def _to_device(self, name, arr):
        """User state array -> device-domain array (identity unless mirrored)."""
        return arr

    def _to_user(self, name, arr):
        return arr

    def _energy_scale(self) -> float:
        return 1.0

    def _build_desc(self):
        g = self._dgrid
        nz = _grid_nz(g)
        d = _abi.Desc()
        d.abi_version = _abi.ABI_VERSION
        d.equation = self.EQUATION
        d.ndim = self.ndim
        d.order = self.order
        d.bc_slow = _abi.BC_FREE_SURFACE if _is_free_surface(g) else _abi.BC_PERIODIC
        d.lane_s = LANE_BITS[self.stencil_precision]
        d.lane_u = LANE_BITS[self.update_precision]
        d.nx = g.nx
        d.nm = 1 if nz is None else g.ny
        d.ns = g.ny if nz is None else nz
        d.dx = g.dx
        d.dt = g.dt
        for j, c in enumerate(self.stencil.coefficients):
            d.taps[j] = c
        self._keep = {}
        for pid, arr in self._planes().items():
            arr = np.ascontiguousarray(arr, dtype=np.float64)
            self._keep[pid] = arr
            d.plane[pid] = arr.ctypes.data_as(ctypes.POINTER(ctypes.c_double))
        src = self.source
        d.src_kind = _abi.SRC_NONE if src is None else self._source_code()
        if src is not None:
            d.src_x, d.src_m, d.src_s = self._to_xms((src.ix, src.iy, getattr(src, "iz", None)))
        rec = np.array([self._to_xms(r) for r in self.receivers], dtype=np.int64).reshape(-1, 3)
        self._keep["rec"] = rec
        d.receivers = rec.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)) if len(rec) else None
        d.n_receivers = len(rec)
        d.world_size = 1
        d.rank = 0
        d.device = self.device
        d.nccl_unique_id = None
        if self.distributed:
            import torch.distributed as dist

            d.world_size = dist.get_world_size()
            d.rank = dist.get_rank()
            box = [None]
            if d.rank == 0:
                uid = ctypes.create_string_buffer(128)
                _abi.check(_abi.load().hw_nccl_unique_id(uid), "hw_nccl_unique_id")
                box[0] = uid.raw
            dist.broadcast_object_list(box, src=0)
            self._uid = ctypes.create_string_buffer(box[0], 128)
            d.nccl_unique_id = ctypes.cast(self._uid, ctypes.c_void_p)
        d.energy_every = self.energy_every
        self._desc = d

    def _to_xms(self, idx):
        if self.ndim == 2:
            return (int(idx[0]), 0, int(idx[1]))
        return (int(idx[0]), int(idx[1]), int(idx[2]))

    @property
    def desc(self) -> _abi.Desc:
        """The hw_desc handed to the library (also what tests hand the CPU oracle)."""
        return self._desc

    def _lib_handle(self):
        if self._handle is None:
            lib = _abi.load()
            if self.slabs > 1:
                hs = (ctypes.c_void_p * self.slabs)()
                devs = None
                if self.devices is not None:
                    devs = (ctypes.c_int32 * self.slabs)(*[self.devices[r % len(self.devices)] for r in range(self.slabs)])
                _abi.check(lib.hw_create_group(ctypes.byref(self._desc), self.slabs, devs, hs), "hw_create_group")
                self._group = hs
                self._handle = ctypes.c_void_p(hs[0])
            else:
                h = ctypes.c_void_p()
                _abi.check(lib.hw_create(ctypes.byref(self._desc), ctypes.byref(h)), "hw_create")
                self._handle = h
        return self._handle

    def _handles(self):
        self._lib_handle()
        if self._group is not None:
            return [ctypes.c_void_p(h) for h in self._group]
        return [self._handle]

    def close(self):
        if self._handle is not None:
            _abi.load().hw_destroy(self._handle)  # releases every slab of a group
            self._handle = None
            self._group = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ------------------------------------------------------------ state
    FIELDS = ()   # external order: solution fields, then residuals
    STAGGERS = {}

    def new_state(self):
        f = lambda st: Field2D.zeros(self.grid, st, self.update_precision)
        kw = {name: f(self._stagger_of(name)) for name in self.FIELDS}
        return self.STATE_CLS(**kw)

    def _field_arrays(self, state) -> list:
        dtype = DTYPES[self.update_precision]
        out = []
        for j, name in enumerate(self.FIELDS):
            arr = np.ascontiguousarray(getattr(state, name).values, dtype=dtype)
            want = self.grid.shape(self._stagger_of(name))
            if arr.shape != tuple(want):
                raise ValueError(f"state field {name} has shape {arr.shape}, expected {tuple(want)}")
            out.append(self._to_device(name, arr))
        return out

    def _stagger_of(self, name):
        return self.STAGGERS[name] if name in self.STAGGERS else self.STAGGERS[name[1:]]

    def _upload(self, state):
        arrs = self._field_arrays(state)
        ptrs = (ctypes.c_void_p * len(arrs))(*[a.ctypes.data for a in arrs])
        for h in self._handles():  # every slab takes its rows of the global arrays
            _abi.check(_abi.load().hw_set_state(h, ptrs), "hw_set_state")
        self._uploaded = arrs

    def _download(self, state):
        dtype = DTYPES[self.update_precision]
        if self.distributed:  # rows of other ranks keep their uploaded values (own rows overwritten below)
            # a caller array that went up unconverted is updated in place (its own rows only): no full
            # global-size copy per run on every rank; converted / mirrored inputs get a fresh array
            arrs = []
            for name, u in zip(self.FIELDS, self._uploaded):
                if getattr(state, name).values is u and u.flags.writeable:
                    arrs.append(u)
                else:
                    a = _host_empty(u.shape, u.dtype)
                    np.copyto(a, u)
                    arrs.append(a)
        else:  # fresh arrays, as the reference returns (acoustic.py:147-152), in pinned memory
            arrs = [_host_empty(self._dgrid.shape(self._stagger_of(n)), dtype) for n in self.FIELDS]
        ptrs = (ctypes.c_void_p * len(arrs))(*[a.ctypes.data for a in arrs])
        for h in self._handles():
            _abi.check(_abi.load().hw_get_state(h, ptrs), "hw_get_state")
        for name, a in zip(self.FIELDS, arrs):
            getattr(state, name).values = self._to_user(name, a)

    def _hw_run(self, *args):
        lib = _abi.load()
        if self._group is not None:
            return lib.hw_run_group(self._group, self.slabs, *args)
        return lib.hw_run(self._lib_handle(), *args)

    def _fail_name(self, j: int) -> str:
        name = self.FIELDS[j]
        return name[0].upper() + name[1:]

    # ------------------------------------------------------------ sources
    def _source_time(self, step: int) -> float:
        raise NotImplementedError

    def source_samples(self, step0: int, nt: int):
        if self.source is None:
            return None
        return np.array([sample_source(self.source, self._source_time(step0 + n)) for n in range(nt)],
                        dtype=np.float64)

    # ------------------------------------------------------------ stepping
    def step_baseline(self, state):
        return self._step(state, None)

    def step_compensated(self, state, variant=None):
        return self._step(state, self.DEFAULT_VARIANT if variant is None else variant)

    def _step(self, state, variant):
        lib = _abi.load()
        h = self._lib_handle()
        self._upload(state)
        src = self.source_samples(state.step, 1)
        fs, ff = ctypes.c_int64(-1), ctypes.c_int32(-1)
        P = ctypes.POINTER(ctypes.c_double)
        rc = self._hw_run(variant_code(variant), state.step, 1,
                          src.ctypes.data_as(P) if src is not None else None,
                          None, None, None, None, ctypes.byref(fs), ctypes.byref(ff))
        if rc not in (_abi.OK, _abi.RANGE_FAILURE):
            _abi.check(rc, "hw_run")
        self._download(state)
        state.step += 1
        if rc == _abi.RANGE_FAILURE:
            raise RangeFailureError(state.step - 1, self._fail_name(ff.value))
        return state

    def run(self, variant=None, state=None) -> RunOutput:
        """March grid.nt steps; traces and energy history as the reference's run()."""
        lib = _abi.load()
        h = self._lib_handle()
        state = state if state is not None else self.new_state()
        nt, every = self.grid.nt, self.energy_every
        step0 = state.step
        self._upload(state)
        src = self.source_samples(step0, nt)
        nrec = len(self.receivers)
        traces = np.zeros((nrec, nt), dtype=np.float64)
        cap = 1 + nt // every
        e_times = np.zeros(cap, dtype=np.float64)
        e_vals = np.zeros(cap, dtype=np.float64)
        ne = ctypes.c_int64(0)
        fs, ff = ctypes.c_int64(-1), ctypes.c_int32(-1)
        P = ctypes.POINTER(ctypes.c_double)
        rc = self._hw_run(variant_code(variant), step0, nt,
                          src.ctypes.data_as(P) if src is not None else None,
                          traces.ctypes.data_as(P), e_times.ctypes.data_as(P), e_vals.ctypes.data_as(P),
                          ctypes.byref(ne), ctypes.byref(fs), ctypes.byref(ff))
        if rc not in (_abi.OK, _abi.RANGE_FAILURE):
            _abi.check(rc, "hw_run")
        self._download(state)
        if rc == _abi.RANGE_FAILURE:
            state.step = fs.value + 1
            raise RangeFailureError(fs.value, self._fail_name(ff.value))
        state.step = step0 + nt
        out_traces = []
        for j, r in enumerate(self.receivers):
            ts = TraceSeries(self.TRACE_FIELD, int(r[0]), int(r[1]), traces[j].copy())
            if self.ndim == 3:
                ts.iz = int(r[2])
            out_traces.append(ts)
        k = ne.value
        energy = EnergySeries(e_times[:k].copy(), e_vals[:k] * self._energy_scale())
        return RunOutput(out_traces, energy, {"range_failure": None})

    # ------------------------------------------------------------ bench hooks
    def run_device(self, variant, step0: int, nt: int) -> float:
        """March nt steps on the device-resident state; returns device ms (CUDA events)."""
        lib = _abi.load()
        h = self._lib_handle()
        src = self.source_samples(step0, nt)
        ms = ctypes.c_float(0.0)
        P = ctypes.POINTER(ctypes.c_double)
        _abi.check(lib.hw_run_device(h, variant_code(variant), step0, nt,
                                     src.ctypes.data_as(P) if src is not None else None,
                                     ctypes.byref(ms)), "hw_run_device")
        return ms.value

    def upload(self, state):
        self._upload(state)

    def download(self, state):
        self._download(state)

    def kernel_path(self) -> str:
        """Kernel family of the device steps: "fused2d", "stream2d" or "generic"."""
        return _abi.load().hw_kernel_path(self._lib_handle()).decode()

    def transport(self) -> int:
        """Halo transport: 0 single domain, 1 in-process slab group, 2 NCCL."""
        return int(_abi.load().hw_transport(self._lib_handle()))

    def last_launch_count(self) -> int:
        return int(_abi.load().hw_last_launch_count(self._lib_handle()))

"""Generate golden vectors by running the UNMODIFIED reference solver.

Run in the build container (the reference is not on the GPU box):

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba \
        python tests/golden/make_golden.py

Each case writes tests/golden/<name>.npz holding the case description (JSON),
the binary64 medium planes, the initial state, and the reference's outputs:
final state (bit patterns), receiver traces, energy history, or the
RangeFailureError (step, field).  Single-step cases also store the state after
every step.  The fixtures pin the CPU oracle (tests/test_oracle_golden.py) and
the GPU path (tests/test_gpu_parity.py) to the reference's own results.
"""

from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np

from halfwave.acoustic import AcousticSolver
from halfwave.diagnostics import RangeFailureError
from halfwave.efsum import Variant
from halfwave.elastic import ElasticSolver
from halfwave.grids import Boundary, GridSpec, Medium, MediumKind, build_homogeneous_acoustic, build_layered_elastic
from halfwave.precision import Precision
from halfwave.sources import RickerSpec, SourceKind, SourceSpec

OUT = Path(__file__).resolve().parent
P = {"fp16": Precision.FP16, "fp32": Precision.FP32, "fp64": Precision.FP64}
V = {"naive": None, "op3": Variant.OP3, "op6": Variant.OP6}


def gaussian(shape, cy, cx, width, amp):
    yy, xx = np.mgrid[0:shape[0], 0:shape[1]].astype(np.float64)
    return amp * np.exp(-((xx - cx) ** 2 + (yy - cy) ** 2) / width)


def make_case(name, eq, nx, ny, dx, dt, nt, *, bc="periodic", medium, source=None, receivers=(),
              stencil="fp16", update=None, variant="op3", energy_every=5, init=None, steps_api=0, seed=0):
    update = update or stencil
    grid = GridSpec(nx=nx, ny=ny, dx=dx, dt=dt, nt=nt,
                    bc_y=Boundary.FREE_SURFACE if bc == "free-surface" else Boundary.PERIODIC)
    src = None
    if source is not None:
        kind = SourceKind.PRESSURE_POINT if eq == "acoustic" else SourceKind.VY_POINT
        src = SourceSpec(kind, source["ix"], source["iy"],
                         RickerSpec(source["f_center"], source.get("delay"), source["amplitude"]))
    cls = AcousticSolver if eq == "acoustic" else ElasticSolver
    solver = cls(grid, medium, src, stencil_precision=P[stencil], update_precision=P[update],
                 receivers=tuple(receivers), energy_every=energy_every)
    state = solver.new_state()
    rng = np.random.default_rng(seed)
    names = (["p", "vx", "vy", "rp", "rvx", "rvy"] if eq == "acoustic" else
             ["vx", "vy", "sxx", "syy", "sxy", "rvx", "rvy", "rsxx", "rsyy", "rsxy"])
    if init is not None:
        for fname, fn in init.items():
            f = getattr(state, fname)
            f.values = fn(f.values.shape, rng).astype(f.values.dtype)
    init_arrays = {f"init_{n}": getattr(state, n).values.copy() for n in names}
    out = {}
    desc = dict(name=name, eq=eq, nx=nx, ny=ny, dx=dx, dt=dt, nt=nt, bc=bc, source=source,
                receivers=[list(r) for r in receivers], stencil=stencil, update=update, variant=variant,
                energy_every=energy_every, steps_api=steps_api, medium_kind=eq,
                plane_names=list(medium.planes))
    if steps_api:
        for k in range(steps_api):
            try:
                if V[variant] is None:
                    solver.step_baseline(state)
                else:
                    solver.step_compensated(state, V[variant])
            except RangeFailureError as e:
                desc["fail"] = [e.step, e.field_name]
                for n in names:
                    out[f"step{k}_{n}"] = getattr(state, n).values.copy()
                break
            for n in names:
                out[f"step{k}_{n}"] = getattr(state, n).values.copy()
    else:
        try:
            res = solver.run(V[variant], state)
            out["traces"] = np.array([t.samples for t in res.traces]).reshape(len(receivers), nt)
            out["e_times"] = res.energy.times
            out["e_vals"] = res.energy.values
        except RangeFailureError as e:
            desc["fail"] = [e.step, e.field_name]
        desc["final_step"] = state.step
        for n in names:
            out[f"final_{n}"] = getattr(state, n).values.copy()
    planes = {f"plane_{k}": v for k, v in medium.planes.items()}
    np.savez_compressed(OUT / f"{name}.npz", desc=json.dumps(desc), **planes, **init_arrays, **out)
    print(f"{name}: {desc.get('fail', 'ok')}", file=sys.stderr)


def main():
    DT16 = float(np.float16(4e-4))
    n = 40
    unit = build_homogeneous_acoustic(n, 32, rho=1.0, c=1.0)
    bump = {"p": lambda sh, rng: gaussian(sh, 14, 19, 20.0, 0.8) + rng.uniform(-1e-3, 1e-3, sh)}
    src = {"ix": 20, "iy": 15, "f_center": 5.0, "amplitude": 50.0}
    rec = ((5, 7), (20, 15), (33, 25))
    # 2D acoustic, reference-native 4th-order periodic; every precision mode
    for mode, (s, u, v) in {
        "fp16_op3": ("fp16", "fp16", "op3"), "fp16_naive": ("fp16", "fp16", "naive"),
        "fp16_op6": ("fp16", "fp16", "op6"), "fp32_naive": ("fp32", "fp32", "naive"),
        "fp32_op3": ("fp32", "fp32", "op3"), "fp64_naive": ("fp64", "fp64", "naive"),
        "fp64_op3": ("fp64", "fp64", "op3"), "mixed64_16_op3": ("fp64", "fp16", "op3"),
        "mixed64_16_naive": ("fp64", "fp16", "naive"), "mixed32_16_op6": ("fp32", "fp16", "op6"),
        "mixed16_32_op3": ("fp16", "fp32", "op3"),
    }.items():
        make_case(f"ac2d_{mode}", "acoustic", n, 32, 0.032, 0.01, 120, medium=unit, source=src,
                  receivers=rec, stencil=s, update=u, variant=v, init=bump, seed=1)
    # heterogeneous planes (Medium accepts arbitrary positive planes)
    rng = np.random.default_rng(7)
    het = Medium(MediumKind.ACOUSTIC, 36, 28, {
        "rho_x": rng.uniform(0.8, 1.6, (28, 36)), "rho_y": rng.uniform(0.8, 1.6, (28, 36)),
        "beta": rng.uniform(0.5, 1.2, (28, 36))})
    make_case("ac2d_het_fp16_op3", "acoustic", 36, 28, 0.05, 0.01, 100, medium=het, source=None,
              receivers=((3, 3), (30, 20)), init={"p": lambda sh, r: gaussian(sh, 10, 12, 9.0, 1.5),
                                                  "vx": lambda sh, r: r.uniform(-0.1, 0.1, sh)}, seed=2)
    # odd nx (scalar W=1 path), non-square, fp32 op6
    make_case("ac2d_odd_fp16_op3", "acoustic", 27, 19, 0.032, 0.01, 80,
              medium=build_homogeneous_acoustic(27, 19, rho=1.0, c=1.0),
              source={"ix": 13, "iy": 9, "f_center": 6.0, "amplitude": 20.0}, receivers=((13, 9),),
              init={"p": lambda sh, r: r.uniform(-0.5, 0.5, sh)}, seed=3)
    # per-step states through the single-step API (first 6 steps)
    make_case("ac2d_steps_fp16_op3", "acoustic", 24, 24, 0.032, 0.01, 6, medium=build_homogeneous_acoustic(24, 24, 1.0, 1.0),
              source={"ix": 12, "iy": 12, "f_center": 5.0, "amplitude": 1000.0},
              init={"p": lambda sh, r: r.uniform(-1, 1, sh), "rp": lambda sh, r: r.uniform(-1e-4, 1e-4, sh)},
              steps_api=6, seed=4)
    # range failure (test_acoustic.py:233-245)
    make_case("ac2d_overflow_fp16", "acoustic", 16, 16, 0.032, DT16, 400,
              medium=build_homogeneous_acoustic(16, 16, 1.0, 1.0),
              source={"ix": 8, "iy": 8, "f_center": 5.0, "amplitude": 1e9}, variant="naive")
    make_case("ac2d_overflow_fp16_op3", "acoustic", 16, 16, 0.032, DT16, 400,
              medium=build_homogeneous_acoustic(16, 16, 1.0, 1.0),
              source={"ix": 8, "iy": 8, "f_center": 5.0, "amplitude": 1e9}, variant="op3")

    # 2D elastic: free surface (reference-native) and periodic
    two = [(0.5, 2.0, 2.0, 1.0), (1.0, 2.3, 2.8, 1.4)]
    med = build_layered_elastic(n, 32, two)
    esrc = {"ix": 20, "iy": 6, "f_center": 5.0, "amplitude": 20.0}
    einit = {"sxx": lambda sh, r: gaussian(sh, 12, 18, 16.0, 0.5),
             "syy": lambda sh, r: gaussian(sh, 12, 18, 16.0, 0.3) + r.uniform(-1e-3, 1e-3, sh),
             "vx": lambda sh, r: r.uniform(-1e-2, 1e-2, sh)}
    for bc in ("free-surface", "periodic"):
        tag = "fs" if bc == "free-surface" else "per"
        for mode, (s, u, v) in {"fp16_op6": ("fp16", "fp16", "op6"), "fp16_op3": ("fp16", "fp16", "op3"),
                                "fp16_naive": ("fp16", "fp16", "naive"), "fp64_naive": ("fp64", "fp64", "naive"),
                                "fp32_op6": ("fp32", "fp32", "op6"),
                                "mixed64_16_op6": ("fp64", "fp16", "op6")}.items():
            make_case(f"el2d_{tag}_{mode}", "elastic", n, 32, 0.05, 0.01, 120, bc=bc, medium=med, source=esrc,
                      receivers=((20, 6), (10, 20), (35, 2)), stencil=s, update=u, variant=v, init=einit, seed=5)
    # mu = 0 layer (pressure-like cells), steps API, elastic overflow
    make_case("el2d_fs_mu0_fp16_op6", "elastic", 24, 24, 0.05, 0.008, 60, bc="free-surface",
              medium=build_layered_elastic(24, 24, [(0.5, 1.0, 2.0, 0.0), (1.0, 2.0, 2.5, 1.2)]),
              source={"ix": 12, "iy": 5, "f_center": 4.0, "amplitude": 10.0}, receivers=((12, 5),),
              init=einit, seed=6)
    make_case("el2d_steps_fs_fp16_op6", "elastic", 20, 20, 0.032, DT16, 5, bc="free-surface",
              medium=build_layered_elastic(20, 20, [(1.0, 1.0, 2.0, 1.0)]), variant="op6",
              source={"ix": 10, "iy": 5, "f_center": 8.0, "amplitude": 500.0},
              init={"syy": lambda sh, r: r.uniform(-1, 1, sh), "sxy": lambda sh, r: r.uniform(-1, 1, sh)},
              steps_api=5, seed=8)
    make_case("el2d_overflow_fp16", "elastic", 16, 16, 0.032, DT16, 10,
              medium=build_layered_elastic(16, 16, [(1.0, 1.0, 2.0, 1.0)]), variant="naive",
              source={"ix": 8, "iy": 8, "f_center": 5.0, "amplitude": 1e12})


if __name__ == "__main__":
    main()

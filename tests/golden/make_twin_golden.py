"""Golden runs of BASELINE config 1's reference-native twins, made by the UNMODIFIED reference.

Run in the build container (the reference is not on the GPU box):

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba \
        python tests/golden/make_twin_golden.py

BASELINE config 1 (256^2, rho = kappa = 1, Gaussian bump + seeded noise, 2000 steps, energy
every step) asks for 2nd order and p = 0 walls, which the reference does not have (the rigid
mirror fixtures of make_rigid_golden.py cover that).  BASELINE.md and SURVEY 8(d) also name
the twins the reference CAN run: the same state on the 4th-order periodic solver at CFL 0.5
(as configured: compensation does not help there), 0.05 and 0.0125 (the paper's regime, where
it does).  This script runs those twins -- fp16 naive and fp16 op3 at the three CFL numbers,
fp64 at CFL 0.5 -- at full size and full length and keeps, per run, the energy history
(2001 samples), two receiver traces and the SHA-256 of every final field's bit pattern, plus
the shared initial pressure (tests/golden/twin/).  tests/test_twin_golden.py pins the C
oracle to them; tests/test_gpu_twins.py the B200 path.
"""

from __future__ import annotations

import hashlib
import json
import sys
from pathlib import Path

import numpy as np

from halfwave.acoustic import AcousticSolver
from halfwave.efsum import Variant
from halfwave.grids import GridSpec, build_homogeneous_acoustic
from halfwave.precision import Precision

OUT = Path(__file__).resolve().parent / "twin"
N = 256
NT = 2000
SEED = 1
RECEIVERS = ((128, 128), (40, 200))
FIELDS = ["p", "vx", "vy", "rp", "rvx", "rvy"]
RUNS = [("fp16", "naive", 0.5), ("fp16", "op3", 0.5), ("fp64", "naive", 0.5),
        ("fp16", "naive", 0.05), ("fp16", "op3", 0.05),
        ("fp16", "naive", 0.0125), ("fp16", "op3", 0.0125)]


def initial_pressure():
    """exp(-((x-1/2)^2 + (z-1/2)^2) / 0.01) + U(-1e-3, 1e-3), CELL coordinates x = ix h (fp64)."""
    h = 1.0 / N
    x = np.arange(N) * h
    g = np.exp(-((x[None, :] - 0.5) ** 2 + (x[:, None] - 0.5) ** 2) / 0.01)
    return g + np.random.default_rng(SEED).uniform(-1e-3, 1e-3, (N, N))


def digest(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def main():
    OUT.mkdir(exist_ok=True)
    p0 = initial_pressure()
    np.savez_compressed(OUT / "twin_init.npz", p0_fp64=p0)
    h = 1.0 / N
    medium = build_homogeneous_acoustic(N, N, rho=1.0, c=1.0)
    for prec, variant, cfl in RUNS:
        dt = cfl * h  # 2^-9, 0.05 / 256, 2^-14.68...: the solver rounds dt into the update lane
        grid = GridSpec(nx=N, ny=N, dx=h, dt=dt, nt=NT)
        P = Precision.FP16 if prec == "fp16" else Precision.FP64
        solver = AcousticSolver(grid, medium, None, stencil_precision=P, update_precision=P,
                                receivers=RECEIVERS, energy_every=1)
        st = solver.new_state()
        st.p.values = p0.astype(st.p.values.dtype)  # a single cast to the update lane
        res = solver.run(None if variant == "naive" else Variant.OP3, st)
        name = f"twin_cfl{str(cfl).replace('.', 'p')}_{prec}_{variant}"
        desc = dict(name=name, n=N, nt=NT, dx=h, dt=dt, cfl=cfl, precision=prec, variant=variant,
                    receivers=[list(r) for r in RECEIVERS], seed=SEED,
                    sha256={f: digest(getattr(st, f).values) for f in FIELDS},
                    dtype=str(st.p.values.dtype))
        np.savez_compressed(OUT / f"{name}.npz", desc=json.dumps(desc),
                            traces=np.array([t.samples for t in res.traces]),
                            e_times=res.energy.times, e_vals=res.energy.values)
        e = res.energy.values
        print(f"{name}: E0 {e[0]:.9e} E_end {e[-1]:.9e} rel {(e[-1] - e[0]) / e[0]:+.3e}", file=sys.stderr)


if __name__ == "__main__":
    main()

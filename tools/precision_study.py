"""The BASELINE configs' own precision comparisons, at full size, on one B200.

Each BASELINE config names the precision arms it compares (config 1: fp16 naive vs fp16
compensated vs fp64; config 2: fp16 compensated, fp64 for the energy comparison; config 3: fp16
compensated vs fp32 naive; config 4: fp16 naive vs compensated; config 5: fp16 compensated).
This runs every arm (plus an fp64 reference where the config has none, and fp16 naive where it
shows the effect of the compensation) through the public API `solver.run(variant, state)` on
the full-size grid and step count, and reports per arm: the energy history's relative deviation
and trend after the source is off (diagnostics.energy_drift, the reference's acceptance metric),
the final energy relative to the fp64 arm, the receiver traces' relative L2 distance to the fp64
arm (diagnostics.compare_traces), and the device throughput.  Synthetic seeded inputs of the
BASELINE shapes stand in for any dataset.

    python tools/precision_study.py [configs, default 1,2,3,4,5] > profiles/r2_precision_study.jsonl
"""
import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import paper_2310_00236_b200 as hw  # noqa: E402
from paper_2310_00236_b200.diagnostics import compare_traces, energy_drift  # noqa: E402

F16, F32, F64 = hw.Precision.FP16, hw.Precision.FP32, hw.Precision.FP64
OP3, OP6 = hw.Variant.OP3, hw.Variant.OP6


def dt_below(x):
    """Largest binary16 value <= x (a binary16-exact step, as bench.py)."""
    d = float(np.float16(x))
    return float(np.nextafter(np.float16(d), np.float16(0))) if d > x else d


def gauss(shape, sigma2=0.01):
    """exp(-|x - c|^2 / sigma2) at cell coordinates of the unit box (fp64)."""
    axes = [np.arange(n) / n - 0.5 for n in shape]
    r2 = sum(a.reshape([-1 if i == k else 1 for i in range(len(shape))]) ** 2 for k, a in enumerate(axes))
    return np.exp(-r2 / sigma2)


def config1(prec, upd=None):
    n = 256
    dx = 1.0 / n
    g = hw.GridSpec(n, n, dx, 0.5 * dx, 2000, order=2, bc_x=hw.Boundary.RIGID, bc_y=hw.Boundary.RIGID)
    s = hw.AcousticSolver(g, hw.build_homogeneous_acoustic(n, n, 1.0, 1.0), stencil_precision=prec, update_precision=upd,
                          receivers=((n // 4, n // 3), (n // 2 + 7, n // 2 - 5)), energy_every=1)

    def init(st):  # p on the (n+1)^2 integer nodes, zero on the walls (tests/test_gpu_rigid.py)
        yy, xx = np.mgrid[0:n + 1, 0:n + 1] * dx
        p0 = np.exp(-((xx - 0.5) ** 2 + (yy - 0.5) ** 2) / 0.01) + np.random.default_rng(1).uniform(-1e-3, 1e-3, xx.shape)
        p0[0, :] = p0[-1, :] = p0[:, 0] = p0[:, -1] = 0.0
        st.p.values = p0.astype(st.p.values.dtype)
    return s, init, -1.0, n * n


def config2(prec, upd=None):
    import bench

    n = 4096
    s0 = bench.make_config2(hw, nt=5000)
    s = hw.AcousticSolver(s0.grid, s0.medium, s0.source, stencil_precision=prec, update_precision=upd,
                          receivers=((n // 2, 600), (n // 2 + 400, 400)), energy_every=10)  # source at (n/2, 8)
    return s, None, 2.0 * s0.source.wavelet.delay, n * n


def config3(prec, upd=None):
    from scipy.ndimage import gaussian_filter

    n = 512
    rng = np.random.default_rng(3)
    c = gaussian_filter(rng.standard_normal((n, n, n)), sigma=8.0, mode="wrap")
    c = 1.5 + 3.0 * (c - c.min()) / (c.max() - c.min())
    med = hw.build_acoustic_from_velocity(c)
    dx = 1.0 / n
    g = hw.GridSpec(n, n, dx, dt_below(0.5 * dx / (4.5 * np.sqrt(3))), 1000, nz=n, order=2)
    s = hw.AcousticSolver(g, med, stencil_precision=prec, update_precision=upd, receivers=((n // 4, n // 2, n // 2), (n // 2, n // 4, n // 3)),
                          energy_every=10)

    def init(st):
        st.p.values = gauss((n, n, n)).astype(st.p.values.dtype)
    return s, init, -1.0, n ** 3


def config4(prec, upd=None):
    n = 4096
    med = hw.build_layered_elastic(n, n, [(1.0, 1.0, 2.0, 1.0)])  # rho 1, cp 2, cs 1: lambda 2, mu 1
    dx = 1.0 / n
    g = hw.GridSpec(n, n, dx, dt_below(0.4 * dx / 2.0), 5000, bc_y=hw.Boundary.FREE_SURFACE)
    # amplitude: fields O(0.1-1) (a unit amplitude leaves them ~1e-7, in binary16's subnormal range; the source
    # sample itself must stay below binary16's 65504, and |field| < 14.2 keeps the tap products finite)
    src = hw.SourceSpec(hw.SourceKind.EXPLOSIVE, n // 2, n // 2, hw.RickerSpec(1 / (10 * dx), amplitude=3.0e4))
    s = hw.ElasticSolver(g, med, src, stencil_precision=prec, update_precision=upd, receivers=((n // 2, n // 2 + 400), (n // 2 + 283, n // 2 + 283)),  # vy off the source row
                         energy_every=10)
    return s, None, 2.0 * src.wavelet.delay, n * (n + 1)


def config5(prec, upd=None):
    n = 512
    rng = np.random.default_rng(5)
    layers, depth = [], 0.0
    for k in range(4):  # seeded random layers, cs < cp / sqrt(2) so lambda > 0
        depth = 1.0 if k == 3 else depth + 0.25
        cs = rng.uniform(0.8, 1.4)
        layers.append((depth, rng.uniform(1.0, 2.0), cs * rng.uniform(1.6, 2.0), cs))
    med = hw.build_layered_elastic(n, n, layers, nz=n)
    cmax = max(cp for _, _, cp, _ in layers)
    dx = 1.0 / n
    g = hw.GridSpec(n, n, dx, dt_below(0.4 * dx / (cmax * np.sqrt(3))), 500, nz=n, order=2)
    s = hw.ElasticSolver(g, med, stencil_precision=prec, update_precision=upd, receivers=((n // 2, n // 4, n // 2), (n // 4, n // 2, n // 3)),
                         energy_every=10)

    def init(st):
        st.vy.values = gauss((n, n, n)).astype(st.vy.values.dtype)  # Gaussian initial vz (the slow-axis velocity)
    return s, init, -1.0, n ** 3


# (name, precision, variant) per config; the fp64 arm is the reference the others are measured against
# (stencil lane, update lane) = (S, U); U None = S.  The "fp64-stencil" arms are the reference's
# update-precision ablation (test_acceptance.py:210-229): binary16 state, exact stencil.
ARMS = {
    "1": (config1, [("fp64", F64, None, None), ("fp16 naive", F16, None, None), ("fp16 op3", F16, None, OP3)]),
    "2": (config2, [("fp64", F64, None, None), ("fp16 naive", F16, None, None), ("fp16 op3", F16, None, OP3),
                    ("fp64-stencil fp16 naive", F64, F16, None), ("fp64-stencil fp16 op3", F64, F16, OP3)]),
    "3": (config3, [("fp64", F64, None, None), ("fp32 naive", F32, None, None), ("fp16 naive", F16, None, None),
                    ("fp16 op3", F16, None, OP3)]),
    "4": (config4, [("fp64", F64, None, None), ("fp16 naive", F16, None, None), ("fp16 op6", F16, None, OP6),
                    ("fp64-stencil fp16 naive", F64, F16, None), ("fp64-stencil fp16 op6", F64, F16, OP6)]),
    "5": (config5, [("fp64", F64, None, None), ("fp16 naive", F16, None, None), ("fp16 op6", F16, None, OP6)]),
}


def main():
    which = sys.argv[1].split(",") if len(sys.argv) > 1 else list(ARMS)
    for key in which:
        build, arms = ARMS[key]
        ref = None
        for name, prec, upd, variant in arms:
            s, init, t_off, cells = build(prec, upd)
            st = s.new_state()
            if init is not None:
                init(st)
            t0 = time.perf_counter()
            out = s.run(variant, st)
            wall = time.perf_counter() - t0
            d = energy_drift(out.energy, t_off)
            line = {"config": key, "arm": name, "path": s.kernel_path(), "steps": s.grid.nt,
                    "energy_rel_deviation": d["rel_deviation"], "energy_trend_slope": d["trend_slope"],
                    "energy_final": float(out.energy.values[-1]), "energy_initial": float(out.energy.values[0]),
                    "wall_s": wall, "cell_steps_per_s_wall": cells * s.grid.nt / wall}
            if ref is None:
                ref = out
            else:
                e_ref = float(ref.energy.values[-1])
                line["energy_final_rel_to_fp64"] = abs(line["energy_final"] - e_ref) / abs(e_ref)
                line["trace_l2_rel_to_fp64"] = [compare_traces(a, b)["l2_rel"] for a, b in zip(out.traces, ref.traces)]
            print(json.dumps(line), flush=True)
            del s, st, out


if __name__ == "__main__":
    main()

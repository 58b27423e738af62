"""Device-resident throughput of the BASELINE configs on one GPU (short runs):
python tools/measure_configs.py [nt] [configs] [--cpu] -> one JSON line per config.
--cpu adds the CPU oracle port (oracle/halfwave_oracle.c, all host threads) on a bounded
sample of the same config (steady state: setup timed with nt = 0 and subtracted)."""
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import paper_2310_00236_b200 as hw  # noqa: E402

CPU = "--cpu" in sys.argv
# --opt name=value: library kernel-path options (hw_set_option), e.g. --opt fused_el3=0
ARGS = []
if "--lib" in sys.argv:  # an A/B build of the library (tools/build_variant.sh); before any library call
    hw._abi.set_library_path(sys.argv[sys.argv.index("--lib") + 1])
_it = iter(sys.argv[1:])
for a in _it:
    if a == "--cpu":
        continue
    if a == "--lib":
        next(_it)
        continue
    if a == "--opt":
        k, v = next(_it).split("=")
        hw.set_option(k, int(v))
        continue
    ARGS.append(a)
NT = int(ARGS[0]) if ARGS and ARGS[0].isdigit() else 50
F16 = hw.Precision.FP16
_PEAKS = ROOT / "MEASURED_PEAKS.json"
PEAK_GBS = json.loads(_PEAKS.read_text())["hbm_gbs"] if _PEAKS.exists() else 6551.7  # measured copy GB/s


def cpu_rate(s, variant, cells, steps):
    """The oracle port on `steps` steps of the same solver description (the mirrored
    domain for rigid walls: the cells it advances are what the device advances)."""
    import os

    import oracle
    from paper_2310_00236_b200.efsum import variant_code

    st = s.new_state()
    arrays = [np.ascontiguousarray(s._to_device(n, getattr(st, n).values), dtype=np.float64) for n in s.FIELDS]
    v = variant_code(variant)
    cores = os.cpu_count() or 1
    t0 = oracle.timed_steps(s.desc, arrays, v, 0, 0, None, cores, energy=True)
    t1 = oracle.timed_steps(s.desc, arrays, v, 0, steps, s.source_samples(0, steps), cores, energy=True)
    return cells * steps / max(t1 - t0, 1e-9), cores, steps


def timed(name, s, variant, bytes_per_cell, cells, nt=NT, cpu_steps=2, init=None):
    st = s.new_state()
    if init is not None:
        init(st)
    s.upload(st)
    s.run_device(variant, 0, 3)
    ms = s.run_device(variant, 3, nt)
    rate = cells * nt / (ms / 1e3)
    line = {"config": name, "cell_steps_per_s": rate, "us_per_step": 1e3 * ms / nt,
            "B_alg": bytes_per_cell, "GBps": rate * bytes_per_cell / 1e9,
            "frac_of_peak": rate * bytes_per_cell / (PEAK_GBS * 1e9), "peak_GBps": PEAK_GBS,
            "path": s.kernel_path(), "launches": s.last_launch_count()}
    if CPU:
        cr, cores, steps = cpu_rate(s, variant, cells, cpu_steps)
        line["cpu_port_cell_steps_per_s"] = cr
        line["cpu_port"] = f"oracle port, {cores} threads, {steps} steps"
        line["gpu_over_cpu"] = rate / cr
    print(json.dumps(line), flush=True)


def cfg1(order=2, prec=F16):
    """BASELINE config 1: 256^2 cells, h = 1/256, 2nd order, dt = 0.5 h, rigid p = 0 walls
    (mirrored periodic 512^2 on the device), constant rho = kappa = 1, energy every step."""
    n = 256
    dx = 1.0 / n
    g = hw.GridSpec(n, n, dx, 0.5 * dx, NT, order=order, bc_x=hw.Boundary.RIGID, bc_y=hw.Boundary.RIGID)
    return hw.AcousticSolver(g, hw.build_homogeneous_acoustic(n, n, 1.0, 1.0), stencil_precision=prec, energy_every=1)


def gauss1(st):
    """Config 1's initial state: Gaussian bump + seeded U(-1e-3, 1e-3) noise on the (n+1)^2 pressure nodes,
    zero on the rigid walls, v = 0 (the arms' division paths see the real data, not a zero state)."""
    n = st.p.values.shape[0] - 1
    yy, xx = np.mgrid[0:n + 1, 0:n + 1] / n
    p = np.exp(-((xx - 0.5) ** 2 + (yy - 0.5) ** 2) / 0.01) + np.random.default_rng(1).uniform(-1e-3, 1e-3, xx.shape)
    p[0, :] = p[-1, :] = p[:, 0] = p[:, -1] = 0.0
    st.p.values = p.astype(st.p.values.dtype)


def cfg3(prec=F16):  # 3D acoustic 512^3, 2nd order, full beta plane (fp16 op3 vs the fp32 naive arm)
    n = 512
    rng = np.random.default_rng(0)
    c = 1.5 + 3.0 * rng.random((n, n, n))
    med = hw.build_acoustic_from_velocity(c)
    dx = 1.0 / n
    g = hw.GridSpec(n, n, dx, float(np.float16(0.5 * dx / (med.c_max() * np.sqrt(3)))), NT, nz=n, order=2)
    return hw.AcousticSolver(g, med, stencil_precision=prec, energy_every=10)


def gauss3(st):
    """Config 3's initial state: Gaussian pressure exp(-|x - c|^2 / 0.01) at cell coordinates, v = 0
    (fp64, one cast to the state's type)."""
    v = st.p.values
    n = v.shape[0]
    a = np.arange(n) / n - 0.5
    g = np.exp(-(a[:, None, None] ** 2 + a[None, :, None] ** 2 + a[None, None, :] ** 2) / 0.01)
    st.p.values = g.astype(v.dtype)


def cfg4(every=10):  # 2D elastic 4096^2, free surface
    n = 4096
    med = hw.build_layered_elastic(n, n, [(1.0, 1.0, 2.0, 1.0)])
    dx = 1.0 / n
    g = hw.GridSpec(n, n, dx, float(np.float16(0.4 * dx / 2)), NT, bc_y=hw.Boundary.FREE_SURFACE)
    src = hw.SourceSpec(hw.SourceKind.EXPLOSIVE, n // 2, 16, hw.RickerSpec(1 / (10 * dx), amplitude=1.0))
    return hw.ElasticSolver(g, med, src, stencil_precision=F16, energy_every=every)


def cfg5():  # 3D elastic 512^3 per GPU, 2nd order, layered
    n = 512
    med = hw.build_layered_elastic(n, n, [(0.3, 1.0, 2.0, 1.0), (0.7, 1.4, 2.6, 1.3), (1.0, 1.8, 3.0, 1.6)], nz=n)
    dx = 1.0 / n
    g = hw.GridSpec(n, n, dx, float(np.float16(0.4 * dx / 3.0)), NT, nz=n, order=2)
    return hw.ElasticSolver(g, med, stencil_precision=F16, energy_every=10)


if __name__ == "__main__":
    which = ARGS[1].split(",") if len(ARGS) > 1 else ["1", "3", "4", "5"]
    if "1" in which:
        for name, prec, var in (("fp16 naive", F16, None), ("fp16 op3", F16, hw.Variant.OP3),
                                ("fp64", hw.Precision.FP64, None)):
            timed(f"1: 2D acoustic 256^2 2nd order rigid walls {name}, energy every step", cfg1(2, prec), var, 24,
                  256 * 256, cpu_steps=200, init=gauss1)
    if "3" in which:
        timed("3: 3D acoustic 512^3 2nd order fp16 op3 (beta plane, Gaussian p0)", cfg3(), hw.Variant.OP3, 34,
              512 ** 3, cpu_steps=1, init=gauss3)
    if "3f32" in which:  # p, vx, vy, vz binary32 read + written, beta binary32 read
        timed("3: 3D acoustic 512^3 2nd order fp32 naive (beta plane, Gaussian p0)", cfg3(hw.Precision.FP32), None, 36,
              512 ** 3, cpu_steps=1, init=gauss3)
    if "4" in which:
        timed("4: 2D elastic 4096^2 free surface fp16 op6", cfg4(), hw.Variant.OP6, 40, 4096 * 4097, cpu_steps=5)
    if "5" in which:
        timed("5: 3D elastic 512^3 2nd order fp16 op6", cfg5(), hw.Variant.OP6, 72, 512 ** 3, cpu_steps=1)

"""Benchmark: BASELINE config 5 on B200 -- 3D isotropic elastic velocity-stress leapfrog
(9 fields + 9 Kahan residuals, binary16), 512^3 cells per GPU at N = 1, 2nd-order staggered
FD, seeded random layered lambda/mu/rho, Gaussian initial vz, 500 steps, fp16 compensated
(op6), energy every 10 steps.  The metric's "at 1/2/4/8 B200" clause is config 5's strong
scaling: at N > 1 the same 512^3 grid is split into N z-slabs (one per rank, NCCL halo
exchange), and at N = 8 the 1024^3 global grid of the config is measured as an extra key.

One bench "step" = one full config-5 run (500 leapfrog steps on the whole grid).
  value : device-resident throughput (state already in HBM), cell-steps/s, timed with CUDA
          events on the library's stream, max over ranks.
  e2e   : the same run through the public API ElasticSolver.run(OP6, state) with the state
          in pinned host memory: host -> HBM -> host inside the timed region every step.
  configs: BASELINE configs 1-4 on the same GPU in the same process (one sub-object each,
          with its own roofline and CPU baseline), so all of them fall under the same clocks.
The reference arm (--impl reference) is the CPU oracle port (oracle/halfwave_oracle.c, all
host threads) on a bounded sample of the same workload.

python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference] [--no-configs]
--gpus N > 1 without torchrun re-launches this script under torch.distributed.run.
"""

from __future__ import annotations

import argparse
import json
import os
import platform
import socket
import statistics
import subprocess
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "grid-point updates/sec (compensated fp16) at 1/2/4/8 B200; % of HBM roofline"
UNIT = "grid-point updates/s"
N5 = 512
NT5 = 500
EVERY = 10
NOMINAL_GBS = 8000.0  # the north star's nominal HBM3e figure; `peak` is the measured copy rate
B_ALG5 = 72  # bytes per cell-step: 18 binary16 arrays (9 fields + 9 residuals) read + written once
WORKLOAD = ("config5: 3D isotropic elastic velocity-stress, 512^3 cells per GPU at N=1 (z-slabs of the same grid "
            "at N>1), 2nd-order staggered FD, seeded random layered lambda/mu/rho, Gaussian initial vz, 500 steps per "
            "bench step, fp16 compensated (op6), energy every 10")


# ------------------------------------------------------------------ workloads
def layers5(seed=5, n=6):
    """Seeded random layered elastic medium: (depth fraction, rho, cp, cs) per layer, cs < cp / sqrt(2)."""
    rng = np.random.default_rng(seed)
    ends = np.sort(rng.uniform(0.05, 0.95, n - 1)).tolist() + [1.0]
    out = []
    for e in ends:
        cs = float(rng.uniform(0.6, 1.5))
        out.append((float(e), float(rng.uniform(1.0, 2.5)), cs * float(rng.uniform(1.8, 2.2)), cs))
    return out


def make_config5(hw, n=N5, nz=None, nt=NT5, distributed=False, device=0):
    nz = n if nz is None else nz
    med = hw.build_layered_elastic(n, n, layers5(), nz=nz)
    dx = 1.0 / n
    dt = float(np.float16(0.4 * dx / (med.c_max() * np.sqrt(3))))
    g = hw.GridSpec(n, n, dx, dt, nt, nz=nz, order=2)
    return hw.ElasticSolver(g, med, stencil_precision=hw.Precision.FP16, energy_every=EVERY, device=device,
                            distributed=distributed)


def init_config5(st):
    """Gaussian initial vz (fp64, one cast), everything else zero."""
    nz, ny, nx = st.vz.values.shape
    z = (np.arange(nz) + 0.5) / nz - 0.5
    y = np.arange(ny) / ny - 0.5
    x = np.arange(nx) / nx - 0.5
    st.vz.values = np.exp(-(z[:, None, None] ** 2 + y[None, :, None] ** 2 + x[None, None, :] ** 2) / 0.01).astype(
        np.float16)


def make_config2(hw, nt=5000, distributed=False):
    n = 4096
    dx = 1.0 / n
    med = hw.build_layered_acoustic(n, n, [(0.5, 1.0, 1.0), (1.0, 1.5, 2.25)])
    c_bound = med.c_max()  # 1/sqrt(min rho * min beta) = 1.5 (grids.py:186-190)
    dt = float(np.float16(0.5 * dx / c_bound))
    if dt > 0.5 * dx / c_bound:
        dt = float(np.nextafter(np.float16(dt), np.float16(0)))
    src = hw.SourceSpec(hw.SourceKind.PRESSURE_POINT, n // 2, 8, hw.RickerSpec(f_center=1 / (10 * dx), amplitude=2.0e4))
    return hw.AcousticSolver(hw.GridSpec(n, n, dx, dt, nt), med, src, stencil_precision=hw.Precision.FP16,
                             receivers=((n // 2, n // 4),), energy_every=10, distributed=distributed)


def smooth_velocity(n, seed=3, sigma=8.0):
    """Seeded Gaussian-filtered random field (periodic, FFT, binary32), min-max scaled to [1.5, 4.5]."""
    import scipy.fft as sf

    f = np.random.default_rng(seed).standard_normal((n, n, n)).astype(np.float32)
    F = sf.rfftn(f, workers=-1)
    k = np.fft.fftfreq(n).astype(np.float32)
    kr = np.fft.rfftfreq(n).astype(np.float32)
    g = lambda kk: np.exp(-2.0 * (np.pi * sigma * kk) ** 2).astype(np.float32)
    F *= g(k)[:, None, None]
    F *= g(k)[None, :, None]
    F *= g(kr)[None, None, :]
    f = sf.irfftn(F, s=(n, n, n), workers=-1)
    del F
    lo, hi = float(f.min()), float(f.max())
    return 1.5 + 3.0 * (f.astype(np.float64) - lo) / (hi - lo)


def make_config3(hw, prec, nt=1000, c=None, **kw):
    n = 512
    c = smooth_velocity(n) if c is None else c
    med = hw.build_acoustic_from_velocity(c)
    dx = 1.0 / n
    dt = float(np.float16(0.5 * dx / (4.5 * np.sqrt(3))))  # CFL <= 1/sqrt(3) at the config's c_max 4.5
    g = hw.GridSpec(n, n, dx, dt, nt, nz=c.shape[0], order=2)
    return hw.AcousticSolver(g, med, stencil_precision=prec, energy_every=10, **kw)


def init_config3(st):
    """Gaussian initial pressure at cell coordinates (fp64, one cast), v = 0."""
    nz, ny, nx = st.p.values.shape
    z, y, x = (np.arange(nz) / nz - 0.5, np.arange(ny) / ny - 0.5, np.arange(nx) / nx - 0.5)
    st.p.values = np.exp(-(z[:, None, None] ** 2 + y[None, :, None] ** 2 + x[None, None, :] ** 2) / 0.01).astype(
        st.p.values.dtype)


def make_config4(hw, nt=5000, periodic=False, **kw):
    n = 4096
    dx = 1.0 / n
    med = hw.build_layered_elastic(n, n, [(1.0, 1.0, 2.0, 1.0)])  # lambda = 2, mu = 1, rho = 1
    g = hw.GridSpec(n, n, dx, float(np.float16(0.4 * dx / 2)), nt,
                    bc_y=hw.Boundary.PERIODIC if periodic else hw.Boundary.FREE_SURFACE)
    src = hw.SourceSpec(hw.SourceKind.EXPLOSIVE, n // 2, 16, hw.RickerSpec(1 / (10 * dx), amplitude=3.0e4))
    return hw.ElasticSolver(g, med, src, stencil_precision=hw.Precision.FP16, energy_every=10, **kw)


def make_config1(hw, prec, nt=2000):
    n = 256
    dx = 1.0 / n
    g = hw.GridSpec(n, n, dx, 0.5 * dx, nt, order=2, bc_x=hw.Boundary.RIGID, bc_y=hw.Boundary.RIGID)
    return hw.AcousticSolver(g, hw.build_homogeneous_acoustic(n, n, 1.0, 1.0), stencil_precision=prec, energy_every=1)


def init_config1(st):
    n = st.p.values.shape[0] - 1
    yy, xx = np.mgrid[0:n + 1, 0:n + 1] / n
    p = np.exp(-((xx - 0.5) ** 2 + (yy - 0.5) ** 2) / 0.01) + np.random.default_rng(1).uniform(-1e-3, 1e-3, xx.shape)
    p[0, :] = p[-1, :] = p[:, 0] = p[:, -1] = 0.0
    st.p.values = p.astype(st.p.values.dtype)


# ------------------------------------------------------------------ plumbing
def peak_hbm():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        return float(json.loads(p.read_text())["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md)"


def traffic_of(key):
    """Steady-state DRAM bytes per launch of a config's step kernel from the committed ncu
    window (profiles/traffic.json, tools/traffic_window.py)."""
    tf = ROOT / "profiles" / "traffic.json"
    if not tf.exists():
        return None, None
    tj = json.loads(tf.read_text()).get(key)
    if not tj:
        return None, None
    return float(tj["dram_bytes_per_launch"]), tj["source"]


def cpu_model():
    try:
        for line in subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout.splitlines():
            if line.startswith("Model name:"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return platform.processor() or "unknown"


class Clocks:
    """nvidia-smi sampling during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        if self.proc is not None:
            self.proc.terminate()
            try:
                out, _ = self.proc.communicate(timeout=5)
            except Exception:
                self.proc.kill()
                out = ""
            self.lines = [l for l in out.splitlines() if l.strip()]

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for l in self.lines:
            parts = [x.strip() for x in l.split(",")]
            try:
                sm.append(float(parts[0]))
                mx = max(mx, float(parts[1]))
            except (ValueError, IndexError):
                continue
            for name, v in zip(names, parts[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm)}


def dist_env():
    return int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")), int(os.environ.get("LOCAL_RANK", "0"))


def spawn_ranks(n):
    """--gpus N without torchrun: re-launch this script as N ranks (one process per GPU)."""
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), str(Path(__file__).resolve()), *sys.argv[1:]]
    sys.exit(subprocess.run(cmd).returncode)


def config_dict(ws):
    """The `config` object of both arms (identical, so the driver can pair them)."""
    return {"workload": WORKLOAD, "grid": [N5, N5, N5], "leapfrog_steps_per_bench_step": NT5, "variant": "op6",
            "order": 2, "medium": "seeded random layered (6 layers, seed 5)",
            "parallelism": "single" if ws == 1 else f"z-slabs x{ws} (strong scaling), NCCL halo exchange",
            "l2": "inputs larger than L2 (state 4.8 GB > 126 MB L2)"}


def oracle_rate(desc_solver, variant, cells, steps, init=None):
    """CPU oracle (oracle/halfwave_oracle.c) on `steps` steps of a solver description, all host
    threads; steady state (the one-off setup is timed with nt = 0 and subtracted)."""
    import oracle
    from paper_2310_00236_b200.efsum import variant_code

    st = desc_solver.new_state()
    if init is not None:
        init(st)
    arrays = [np.ascontiguousarray(desc_solver._to_device(n, getattr(st, n).values), dtype=np.float64)
              for n in desc_solver.FIELDS]
    v = variant_code(variant)
    cores = os.cpu_count() or 1
    t0 = oracle.timed_steps(desc_solver.desc, arrays, v, 0, 0, None, cores, energy=True)
    t1 = oracle.timed_steps(desc_solver.desc, arrays, v, 0, steps, desc_solver.source_samples(0, steps), cores,
                            energy=True)
    el = max(t1 - t0, 1e-9)
    return cells * steps / el, cores, el


# ------------------------------------------------------------------ reference arm
SAMPLE_NZ, SAMPLE_STEPS = 64, 2


def run_reference(args):
    """--impl reference: the CPU implementation of the path (the C oracle port of the reference's
    solver; the Python reference cannot travel to the box) on the host cores, each bench step a
    bounded sample of the config-5 workload: SAMPLE_STEPS leapfrog steps on a 512 x 512 x 64
    z-window of the same medium law and initial state (the same per-cell work)."""
    ws, rank, _ = dist_env()
    if rank != 0:
        return
    import oracle
    import paper_2310_00236_b200 as hw
    from paper_2310_00236_b200.efsum import variant_code

    s = make_config5(hw, nz=SAMPLE_NZ, nt=1)
    st = s.new_state()
    init_config5(st)
    cores = os.cpu_count() or 1
    arrays = [np.ascontiguousarray(getattr(st, n).values, dtype=np.float64) for n in s.FIELDS]
    v = variant_code(hw.Variant.OP6)
    t_setup = oracle.timed_steps(s.desc, arrays, v, 0, 0, None, cores, energy=True)
    step_idx = 0

    def one():
        nonlocal step_idx
        t = oracle.timed_steps(s.desc, arrays, v, step_idx, SAMPLE_STEPS, None, cores, energy=True)
        step_idx += SAMPLE_STEPS
        return max(t - t_setup, 1e-9)

    for _ in range(args.warmup):
        one()
    el = sum(one() for _ in range(args.steps))
    cells = N5 * N5 * SAMPLE_NZ
    val = cells * SAMPLE_STEPS * args.steps / el
    cb = {"value": val, "unit": UNIT, "cores": cores, "kind": "port", "cpu": cpu_model(),
          "sample": f"{SAMPLE_STEPS} leapfrog steps of config 5 on a 512x512x{SAMPLE_NZ} z-window per bench step "
                    f"(fp16 op6, energy every 10), oracle/halfwave_oracle.c, {cores} OpenMP threads, setup excluded"}
    line = {"impl": "reference", "metric": METRIC, "value": val, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * el / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "fp16",
            "data": "synthetic", "config": config_dict(args.gpus), "cpu_baseline": cb,
            "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ B200 arm
def pinned_state(s, st):
    import torch

    for n in s.FIELDS:
        a = getattr(st, n).values
        buf = torch.empty(a.shape, dtype={2: torch.float16, 4: torch.float32, 8: torch.float64}[a.itemsize],
                          pin_memory=True).numpy()
        buf[...] = a
        getattr(st, n).values = buf


def sub_config(hw, name, make, variant, b_alg, cells, nt, path_note, init=None, cpu=None, traffic_key=None,
               repeats=2):
    """Device-resident throughput of one BASELINE config (one full run per repeat), with roofline
    and a bounded CPU-oracle sample."""
    import torch

    s = make()
    st = s.new_state()
    if init is not None:
        init(st)
    s.upload(st)
    s.run_device(variant, 0, nt)  # warm
    ms = []
    for r in range(repeats):
        ms.append(s.run_device(variant, (r + 1) * nt, nt))
    launches = s.last_launch_count()
    best = min(ms)
    torch.cuda.synchronize()
    rate = cells * nt / (best / 1e3)
    peak, _ = peak_hbm()
    achieved = b_alg * cells / (best / nt / 1e3) / 1e9
    traffic, tsrc = traffic_of(traffic_key) if traffic_key else (None, None)
    out = {"value": rate, "unit": UNIT, "leapfrog_steps": nt, "ms_per_run": best, "us_per_leapfrog_step": 1e3 * best / nt,
           "path": s.kernel_path(), "launches_per_run": launches,
           "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                        "frac_of_nominal_8000": achieved / NOMINAL_GBS,
                        "algorithmic_bytes_per_cell_step": b_alg, "traffic": traffic, "traffic_source": tsrc,
                        "note": path_note}}
    s.close()
    if cpu is not None:
        csolver, cvariant, ccells, csteps, cinit, csample = cpu()
        v, cores, el = oracle_rate(csolver, cvariant, ccells, csteps, cinit)
        out["cpu_baseline"] = {"value": v, "unit": UNIT, "cores": cores, "kind": "port", "cpu": cpu_model(),
                               "sample": f"{csample}, oracle/halfwave_oracle.c, {cores} OpenMP threads, {el:.2f} s"}
    print(f"[bench] {name}: {rate / 1e9:.1f} G cell-steps/s ({out['path']}, frac {achieved / peak:.3f})",
          file=sys.stderr, flush=True)
    return out


def extra_configs(hw, with_cpu):
    F16, F32, F64 = hw.Precision.FP16, hw.Precision.FP32, hw.Precision.FP64
    res = {}
    cpu2 = (lambda: (make_config2(hw, nt=1), hw.Variant.OP3, 4096 * 4096, 10, None,
                     "10 leapfrog steps at 4096^2 (fp16 op3)")) if with_cpu else None
    res["config2"] = sub_config(hw, "config2", lambda: make_config2(hw), hw.Variant.OP3, 24, 4096 * 4096, 5000,
                                "k_ac2d_fused, one launch per leapfrog step; layered medium per row (24 B/cell-step)",
                                cpu=cpu2, traffic_key="config2")
    c = smooth_velocity(512)
    cpu3 = (lambda: (make_config3(hw, F16, nt=1, c=c[:64]), hw.Variant.OP3, 512 * 512 * 64, 4, init_config3,
                     "4 leapfrog steps on a 512x512x64 z-window (fp16 op3)")) if with_cpu else None
    res["config3"] = sub_config(hw, "config3", lambda: make_config3(hw, F16, c=c), hw.Variant.OP3, 34, 512 ** 3, 1000,
                                "k_ac3d_fused, per-cell beta plane (34 B/cell-step)", init=init_config3, cpu=cpu3,
                                traffic_key="config3")
    res["config3_fp32_naive"] = sub_config(hw, "config3 fp32", lambda: make_config3(hw, F32, c=c), None, 36, 512 ** 3,
                                           1000, "k_ac3d_fused32, binary32 lanes (36 B/cell-step)", init=init_config3,
                                           traffic_key="config3_fp32")
    del c
    cpu4 = (lambda: (make_config4(hw, nt=1), hw.Variant.OP6, 4096 * 4097, 4, None,
                     "4 leapfrog steps at 4096^2 (fp16 op6)")) if with_cpu else None
    res["config4"] = sub_config(hw, "config4", lambda: make_config4(hw), hw.Variant.OP6, 40, 4096 * 4097, 5000,
                                "k_el2d_fused, free surface (40 B/cell-step)", cpu=cpu4, traffic_key="config4")
    # the per-GPU slab of config 5's 8-GPU grid (1024^3 over 8 z-slabs), run here as a periodic domain of
    # that shape: the rate of one GPU's kernels on its slab, without the exchange
    res["config5_slab_of_1024cubed_over_8"] = sub_config(
        hw, "config5 1024x1024x128", lambda: make_config5(hw, n=1024, nz=128, nt=200), hw.Variant.OP6, B_ALG5,
        1024 * 1024 * 128, 200, "k_el3d_fused at nx = 1024 (tiles of 2 rows): one GPU's slab of the 1024^3 / 8-GPU "
        "grid as a periodic single domain (72 B/cell-step)", init=init_config5)
    res["config1"] = sub_config(hw, "config1", lambda: make_config1(hw, F16), hw.Variant.OP3, 24, 256 * 256, 2000,
                                "persistent small-grid kernel on the mirrored 512^2 domain (cells counted: the 256^2 "
                                "box), energy every step: latency-bound, not an HBM roofline config", init=init_config1, repeats=3)
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-configs", action="store_true", help="skip the configs 1-4 sub-objects")
    ap.add_argument("--nt", type=int, default=NT5, help="leapfrog steps per bench step")
    ap.add_argument("--with-1024cubed", action="store_true",
                    help="at --gpus 8 also time config 5's 1024^3 global grid (every rank builds ~80 GB of global "
                         "host arrays first: minutes of host time; off by default so the scaling runs stay short -- "
                         "the N=1 line carries one GPU's slab of that grid as a sub-config)")
    ap.add_argument("--rank-probe", action="store_true", help=argparse.SUPPRESS)  # spawn test: print rank, exit
    args = ap.parse_args()
    ws, rank, local = dist_env()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        spawn_ranks(args.gpus)
    if ws != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={ws}: launch with torchrun --nproc-per-node {args.gpus}")
    if args.rank_probe:
        print(json.dumps({"rank": rank, "world_size": ws, "local_rank": local}), flush=True)
        return
    if args.impl == "reference":
        return run_reference(args)

    import torch

    import paper_2310_00236_b200 as hw

    torch.cuda.set_device(local)
    dist = None
    if ws > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl")
    nt = args.nt
    cells = N5 ** 3  # global grid (strong scaling: every rank owns ns / N z-slabs)
    s = make_config5(hw, nt=nt, distributed=ws > 1, device=local)
    st = s.new_state()
    init_config5(st)
    s.upload(st)

    # ---------------------------------------------------------- device-resident value
    step0 = 0
    for _ in range(args.warmup):
        s.run_device(hw.Variant.OP6, step0, nt)
        step0 += nt
    launches, ms_total = 0, 0.0
    if ws > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with Clocks(local) as clk:
        w0 = time.perf_counter()
        for _ in range(args.steps):
            ms_total += s.run_device(hw.Variant.OP6, step0, nt)
            launches += s.last_launch_count()
            step0 += nt
        torch.cuda.synchronize()
        wall = time.perf_counter() - w0
    if ws > 1:
        t = torch.tensor([ms_total], device=f"cuda:{local}", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_total = float(t.item())
        dist.barrier()
    ms_step = ms_total / args.steps
    value = cells * nt * args.steps / (ms_total / 1e3)

    # ---------------------------------------------------------- roofline of the step kernel (per GPU)
    peak, peak_src = peak_hbm()
    per_leap_ms = ms_total / (args.steps * nt)
    achieved = B_ALG5 * (cells / ws) / (per_leap_ms / 1e3) / 1e9
    traffic, traffic_src = traffic_of("config5")
    roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                "frac_of_nominal_8000": achieved / NOMINAL_GBS, "traffic": traffic, "traffic_source": traffic_src,
                "traffic_bytes_per_cell_step": traffic / cells if traffic else None, "peak_source": peak_src,
                "algorithmic_bytes_per_cell_step": B_ALG5,
                "kernel": f"{s.kernel_path()}: one launch per leapfrog step at N=1 (k_el3d_fused); achieved = "
                          f"72 B x cells per GPU / CUDA-event time per leapfrog step (launch gaps included)"}

    # ---------------------------------------------------------- end to end through the public API
    st2 = s.new_state()
    init_config5(st2)
    pinned_state(s, st2)
    s.run(hw.Variant.OP6, st2)  # warm (allocations)
    init_config5(st2)
    pinned_state(s, st2)
    share = ws if s.distributed else 1  # a rank copies only its own slab's rows
    h2d = sum(getattr(st2, n).values.nbytes for n in s.FIELDS) // share
    d2h = h2d + 8 * (1 + nt // EVERY)
    if ws > 1:
        dist.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        out = s.run(hw.Variant.OP6, st2)
        _ = float(out.energy.values[-1])
    e2e_wall = time.perf_counter() - t0
    if ws > 1:
        t = torch.tensor([e2e_wall], device=f"cuda:{local}", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_wall = float(t.item())
    e2e = {"value": cells * nt * args.steps / e2e_wall, "unit": UNIT, "h2d_bytes_per_step": int(h2d),
           "d2h_bytes_per_step": int(d2h)}
    path, transport = s.kernel_path(), s.transport()
    s.close()
    del st, st2

    # ---------------------------------------------------------- 1024^3 over 8 GPUs (the config's global grid)
    extra = {}
    if ws == 8 and args.with_1024cubed:
        # every rank builds the global host arrays (medium planes in fp64 + state): ~80 GB per rank at
        # 1024^3; measured only when the host has room for all eight ranks, reported either way
        import psutil

        need = 8 * (5 * 8 + 18 * 2 + 4) * 1024 ** 3
        ok = psutil.virtual_memory().available > need
        flag = torch.tensor([1.0 if ok else 0.0], device=f"cuda:{local}")
        dist.all_reduce(flag, op=dist.ReduceOp.MIN)
        if flag.item() > 0:
            s8 = make_config5(hw, n=1024, nt=100, distributed=True, device=local)
            s8.upload(s8.new_state())
            s8.run_device(hw.Variant.OP6, 0, 20)
            dist.barrier()
            ms8 = s8.run_device(hw.Variant.OP6, 20, 100)
            t = torch.tensor([ms8], device=f"cuda:{local}", dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            extra["config5_1024cubed_8gpu"] = {"value": 1024 ** 3 * 100 / (float(t.item()) / 1e3), "unit": UNIT,
                                              "leapfrog_steps": 100, "path": s8.kernel_path()}
            s8.close()
        else:
            extra["config5_1024cubed_8gpu"] = {"skipped": f"host memory: {need / 2**30:.0f} GiB needed for 8 ranks' "
                                                          "global host arrays"}

    if rank == 0:
        cb = None
        if not args.no_cpu_baseline and ws == 1:
            samp = make_config5(hw, nz=SAMPLE_NZ, nt=1)
            v, cores, el = oracle_rate(samp, hw.Variant.OP6, N5 * N5 * SAMPLE_NZ, 4, init_config5)
            cb = {"value": v, "unit": UNIT, "cores": cores, "kind": "port", "cpu": cpu_model(),
                  "sample": f"4 leapfrog steps of config 5 on a 512x512x{SAMPLE_NZ} z-window (fp16 op6), "
                            f"oracle/halfwave_oracle.c, {cores} OpenMP threads, {el:.2f} s"}
        configs = {}
        if not args.no_configs and ws == 1:
            with Clocks(local) as clk2:
                configs = extra_configs(hw, with_cpu=not args.no_cpu_baseline)
            configs["clocks"] = clk2.summary()
        cfg = config_dict(ws)
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "fp16", "data": "synthetic", "config": cfg,
            "roofline": roofline, "cpu_baseline": cb, "e2e": e2e, "gpu_launches": launches,
            "clocks": clk.summary(), "wall_s_timed_region": wall, "kernel_path": path, "transport": transport,
            **extra, "configs": configs,
        }
        print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()

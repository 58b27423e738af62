"""Benchmark: BASELINE config 2 on B200 — 2D acoustic 4096x4096, 4th-order staggered
FD, two-layer medium (kappa 1.0/2.25, rho 1.0/1.5, interface at mid-depth), Ricker
source at the top centre (10 points per wavelength), 5000 leapfrog steps, fp16
compensated (op3), energy logged every 10 steps.

One bench "step" = one full config-2 run (5000 leapfrog steps on 4096^2 cells).
  value : device-resident throughput (state already in HBM), cell-steps/s, timed
          with CUDA events on the library's stream, max over ranks.
  e2e   : the same run through the public API AcousticSolver.run(OP3, state) with
          host state (pinned) -> HBM -> host every step, wall-clock timed.
Multi-GPU (torchrun, one process per GPU): weak scaling by slab decomposition -- the
global grid is 4096 x (4096 N), rank r owns rows [4096 r, 4096 (r+1)) (one config-2 block
per GPU), the fused kernel runs on every slab and the ghost rows (p, vy, rvy; 3 each way)
are exchanged with NCCL send/recv once per leapfrog step.  `--decomposed on` runs that
path at N = 1 (the NCCL transport exchanging with itself: HALFWAVE_NCCL_SELF=1).

python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference] [--decomposed auto|on|off]
"""

from __future__ import annotations

import argparse
import json
import os
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
N = 4096
NT = 5000
EVERY = 10
B_ALG = 24  # bytes per cell-step: 6 fp16 arrays (p, vx, vy + 3 residuals) read + written once
WORKLOAD = ("config2: 2D acoustic 4096x4096, 4th-order staggered FD, two-layer medium "
            "(kappa 1.0/2.25, rho 1.0/1.5), Ricker top-centre, 5000 steps per bench step, "
            "fp16 compensated (op3), energy every 10")


def make_solver(hw, nt=NT, device=0, n=N, ny=None, distributed=False):
    ny = n if ny is None else ny  # slow axis: n per rank in the decomposed multi-GPU run
    dx = 1.0 / n
    med = hw.build_layered_acoustic(n, ny, [(0.5, 1.0, 1.0), (1.0, 1.5, 2.25)])
    c_bound = med.c_max()  # 1/sqrt(min rho * min beta) = 1.5, the reference's CFL bound (grids.py:186-190)
    dt = float(np.float16(0.5 * dx / c_bound))
    if dt > 0.5 * dx / c_bound:
        dt = float(np.nextafter(np.float16(dt), np.float16(0)))
    grid = hw.GridSpec(n, ny, dx, dt, nt)
    f = 1.0 / (10 * dx)  # c_min / (10 h): 10 points per wavelength
    # amplitude: peak |p| ~1.2 at the source cell and ~0.03 over the wavefield after 5000 steps (binary16's
    # normal range; 100 left the field at ~1e-4, next to binary16's subnormals); the source sample stays far
    # below binary16's 65504 and the tap products c p finite (tools/precision_study.py)
    src = hw.SourceSpec(hw.SourceKind.PRESSURE_POINT, n // 2, 8, hw.RickerSpec(f_center=f, amplitude=2.0e4))
    return hw.AcousticSolver(grid, med, src, stencil_precision=hw.Precision.FP16,
                             update_precision=hw.Precision.FP16, receivers=((n // 2, n // 4),),
                             energy_every=EVERY, device=device, distributed=distributed)


def peak_hbm():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        return float(json.loads(p.read_text())["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md)"


class Clocks:
    """nvidia-smi sampling during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.proc = None

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
        else:
            self.lines = []

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


def cpu_baseline(hw, steps=40):
    """The CPU oracle port (oracle/halfwave_oracle.c, OpenMP over rows, all host
    threads) on a bounded sample of the same workload: `steps` leapfrog steps of
    config 2 at 4096^2 with energy every 10.  Steady-state rate: the one-off setup
    (lane rounding of the medium planes) is timed with nt=0 and subtracted."""
    import oracle
    from paper_2310_00236_b200.efsum import variant_code

    s = make_solver(hw, nt=1)
    st = s.new_state()
    cores = os.cpu_count() or 1
    arrays = [np.ascontiguousarray(getattr(st, n).values, dtype=np.float64) for n in s.FIELDS]
    v = variant_code(hw.Variant.OP3)
    t_setup = oracle.timed_steps(s.desc, arrays, v, 0, 0, None, cores, energy=True)
    t_run = oracle.timed_steps(s.desc, arrays, v, 0, steps, s.source_samples(0, steps), cores, energy=True)
    el = max(t_run - t_setup, 1e-9)
    return {"value": N * N * steps / el, "unit": UNIT, "cores": cores, "kind": "port",
            "sample": f"{steps} leapfrog steps of config 2 at 4096x4096 (fp16 op3, energy every 10), "
                      f"oracle/halfwave_oracle.c, {cores} OpenMP threads, {el:.1f} s"}


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def run_reference(args):
    """--impl reference: the CPU implementation of the path (oracle port; the
    Python reference cannot travel to the box) on the host cores."""
    ws, rank, _ = dist_env()
    if rank != 0:
        return
    import paper_2310_00236_b200 as hw
    import oracle
    from paper_2310_00236_b200.efsum import variant_code

    s = make_solver(hw, nt=1)
    st = s.new_state()
    cores = os.cpu_count() or 1
    arrays = [np.ascontiguousarray(getattr(st, n).values, dtype=np.float64) for n in s.FIELDS]
    per_step = 10  # leapfrog steps per bench step (a bounded sample of the 5000-step run)
    v = variant_code(hw.Variant.OP3)
    t_setup = oracle.timed_steps(s.desc, arrays, v, 0, 0, None, cores, energy=True)
    step_idx = 0

    def one():
        nonlocal step_idx
        t = oracle.timed_steps(s.desc, arrays, v, step_idx, per_step, s.source_samples(step_idx, per_step),
                               cores, energy=True)
        step_idx += per_step
        return max(t - t_setup, 1e-9)

    for _ in range(args.warmup):
        one()
    el = sum(one() for _ in range(args.steps))
    v = N * N * per_step * args.steps / el
    cb = {"value": v, "unit": UNIT, "cores": cores, "kind": "port",
          "sample": f"{per_step} leapfrog steps of config 2 at 4096x4096 per bench step (fp16 op3, energy "
                    f"every 10), oracle/halfwave_oracle.c, {cores} OpenMP threads, setup excluded"}
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * el / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "fp16",
            "data": "synthetic", "config": {"workload": WORKLOAD, "sample_steps_per_bench_step": per_step},
            "cpu_baseline": cb, "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--nt", type=int, default=NT, help="leapfrog steps per bench step")
    ap.add_argument("--decomposed", default="auto", choices=["auto", "on", "off"],
                    help="slab decomposition with NCCL halo exchange (auto: when N > 1)")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)

    import torch

    import paper_2310_00236_b200 as hw

    ws, rank, local = dist_env()
    dist = None
    decomposed = args.decomposed == "on" or (args.decomposed == "auto" and ws > 1)
    torch.cuda.set_device(local)
    if ws > 1 or decomposed:
        import torch.distributed as dist

        if ws > 1:
            dist.init_process_group("nccl")
        else:  # --decomposed on at N = 1: one-rank job on the NCCL transport (self exchange)
            import socket

            with socket.socket() as sk:
                sk.bind(("127.0.0.1", 0))
                port = sk.getsockname()[1]
            dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1)
            os.environ["HALFWAVE_NCCL_SELF"] = "1"
    dev = local
    parallelism = "single"
    s = None
    if decomposed:
        try:
            s = make_solver(hw, nt=args.nt, device=dev, ny=N * ws, distributed=True)
            s.upload(s.new_state())
            parallelism = f"slabs x{ws} (NCCL halo exchange of p, vy, rvy once per step)"
        except Exception as exc:  # keep the scaling run alive: fall back to replicas, say so
            s = None
            parallelism = f"replicas x{ws} (decomposed run failed: {type(exc).__name__}: {exc})"[:300]
    if s is None:
        s = make_solver(hw, nt=args.nt, device=dev)
        if ws > 1 and not decomposed:
            parallelism = f"replicas x{ws}"
    cells = N * N  # per rank

    # ---------------------------------------------------------- device-resident value
    st = s.new_state()
    s.upload(st)
    step0 = 0
    for _ in range(args.warmup):
        s.run_device(hw.Variant.OP3, step0, args.nt)
        step0 += args.nt
    launches = 0
    ms_total = 0.0
    if ws > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with Clocks(dev) as clk:
        w0 = time.perf_counter()
        for _ in range(args.steps):
            ms_total += s.run_device(hw.Variant.OP3, step0, args.nt)
            launches += s.last_launch_count()
            step0 += args.nt
        torch.cuda.synchronize()
        wall = time.perf_counter() - w0
    if ws > 1:
        t = torch.tensor([ms_total], device=f"cuda:{dev}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_total = float(t.item())
        dist.barrier()
    ms_step = ms_total / args.steps
    value = ws * cells * args.nt * args.steps / (ms_total / 1e3)

    # ---------------------------------------------------------- roofline of the step
    peak, peak_src = peak_hbm()
    per_leap_ms = ms_total / (args.steps * args.nt)
    achieved = B_ALG * cells / (per_leap_ms / 1e3) / 1e9
    traffic, traffic_src = None, None
    tf = ROOT / "profiles" / "traffic.json"  # dram bytes per launch from the committed ncu --set full capture
    if tf.exists():
        tj = json.loads(tf.read_text())
        traffic, traffic_src = float(tj["dram_bytes_per_launch"]), tj["source"]
    roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                "traffic": traffic, "traffic_source": traffic_src,
                "traffic_bytes_per_cell_step": traffic / cells if traffic else None, "peak_source": peak_src,
                "algorithmic_bytes_per_cell_step": B_ALG,
                "kernel": "k_ac2d_fused (one launch per leapfrog step of 4096^2 cells); achieved uses the "
                          "CUDA-event time of the whole step loop (launch gaps included)"}

    # ---------------------------------------------------------- end to end through the public API
    import torch as _t

    def pinned_like(a):
        buf = _t.empty(a.shape, dtype={2: _t.float16, 4: _t.float32, 8: _t.float64}[a.itemsize], pin_memory=True)
        out = buf.numpy()
        out[...] = a
        return out

    st2 = s.new_state()
    for n in s.FIELDS:
        getattr(st2, n).values = pinned_like(getattr(st2, n).values)
    share = ws if s.distributed else 1  # a rank copies only its own slab's rows
    h2d = sum(getattr(st2, n).values.nbytes for n in s.FIELDS) // share + 8 * args.nt
    d2h = h2d - 8 * args.nt + 8 * args.nt * len(s.receivers) + 8 * (1 + args.nt // EVERY)
    s.run(hw.Variant.OP3, st2)  # warm (allocations)
    for n in s.FIELDS:
        getattr(st2, n).values = pinned_like(getattr(st2, n).values)
    if ws > 1:
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        out = s.run(hw.Variant.OP3, st2)
        _ = float(out.energy.values[-1])
    e2e_wall = time.perf_counter() - t0
    if ws > 1:
        t = torch.tensor([e2e_wall], device=f"cuda:{dev}", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_wall = float(t.item())
    e2e = {"value": ws * cells * args.nt * args.steps / e2e_wall, "unit": UNIT,
           "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h)}

    if rank == 0:
        cb = None
        if not args.no_cpu_baseline and ws == 1:
            cb = cpu_baseline(hw)
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "fp16", "data": "synthetic",
            "config": {"workload": WORKLOAD, "grid": [N, N * ws if s.distributed else N],
                       "leapfrog_steps_per_bench_step": args.nt, "variant": "op3", "parallelism": parallelism,
                       "path": s.kernel_path(), "transport": s.transport(),
                       "l2": "inputs larger than L2 (state 192 MiB > 126 MB L2)"},
            "roofline": roofline, "cpu_baseline": cb, "e2e": e2e, "gpu_launches": launches,
            "clocks": clk.summary(), "wall_s_timed_region": wall,
        }
        print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()

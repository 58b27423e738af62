"""Decomposed-compute efficiency on one B200: BASELINE config 5 (512^3, op6), config 3 (512^3, op3; 3f32: its
fp32 naive arm), config 4 (4096^2 elastic op6, free surface) or config 2 (4096^2, op3) run as an in-process slab group of N = 1, 2, 4, 8 slabs on one GPU (the multi-GPU path's
kernels, exchange plan and halo recomputation; the exchange is a peer copy on the same device, not
overlapped) -- cell-steps/s relative to the single domain.
python tools/measure_slabs.py [5|3|3f32|4|2] [nt] -> one JSON line per N."""
import ctypes
import json
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
import paper_2310_00236_b200 as hw  # noqa: E402
from paper_2310_00236_b200.efsum import variant_code  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "5"
nt = int(sys.argv[2]) if len(sys.argv) > 2 else 100
base = None
for n in (1, 2, 4, 8):
    if cfg == "5":
        s = bench.make_config5(hw, nt=nt)
        s = hw.ElasticSolver(s.grid, s.medium, stencil_precision=hw.Precision.FP16, energy_every=bench.EVERY, slabs=n)
        st = s.new_state()
        bench.init_config5(st)
        v, cells = hw.Variant.OP6, 512 ** 3
    elif cfg in ("3", "3f32"):
        if n == 1:
            c3 = bench.smooth_velocity(512)
        prec = hw.Precision.FP16 if cfg == "3" else hw.Precision.FP32
        s = bench.make_config3(hw, prec, nt=nt, c=c3, slabs=n)
        st = s.new_state()
        bench.init_config3(st)
        v, cells = (hw.Variant.OP3 if cfg == "3" else None), 512 ** 3
    elif cfg == "4":
        s = bench.make_config4(hw, nt=nt, slabs=n)
        st = s.new_state()
        v, cells = hw.Variant.OP6, 4096 * 4097
    else:
        s0 = bench.make_config2(hw, nt=nt)
        s = hw.AcousticSolver(s0.grid, s0.medium, s0.source, stencil_precision=hw.Precision.FP16,
                              receivers=s0.receivers, energy_every=10, slabs=n)
        st = s.new_state()
        v, cells = hw.Variant.OP3, 4096 ** 2
    s.upload(st)
    P = ctypes.POINTER(ctypes.c_double)
    src = s.source_samples(0, nt)
    cap = 1 + nt // s.energy_every
    tr = np.zeros((max(len(s.receivers), 1), nt))
    et, ev, ne = np.zeros(cap), np.zeros(cap), ctypes.c_int64()
    fs, ff = ctypes.c_int64(), ctypes.c_int32()

    def go():
        t0 = time.perf_counter()
        rc = s._hw_run(variant_code(v), 0, nt, src.ctypes.data_as(P) if src is not None else None,
                       tr.ctypes.data_as(P), et.ctypes.data_as(P), ev.ctypes.data_as(P), ctypes.byref(ne),
                       ctypes.byref(fs), ctypes.byref(ff))
        assert rc == 0, rc
        return time.perf_counter() - t0

    go()
    t = min(go() for _ in range(2))
    rate = cells * nt / t
    base = base or rate
    print(json.dumps({"config": cfg, "slabs": n, "path": s.kernel_path(), "transport": s.transport(),
                      "ms_per_step": 1e3 * t / nt, "G_cell_steps_per_s": rate / 1e9, "vs_single": rate / base,
                      "energy_last": float(ev[ne.value - 1])}), flush=True)
    s.close()

"""Run the UNMODIFIED reference on the desk runs of its acceptance gate (criteria 4-8,
pkg/tests/test_acceptance.py:36-90: paper-acoustic desk in fp64 / fp16 naive / fp16 op3 /
fp64-stencil + fp16-update naive and op3; paper-elastic desk in fp64 / fp16 naive / op6 / op3)
and keep each run's traces and energy history as fixtures (tests/golden/acceptance/<kind>_<name>.npz).

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba python tests/golden/make_acceptance_golden.py
"""
import time
from pathlib import Path

import numpy as np
from halfwave.config import parse_config

OUT = Path(__file__).resolve().parent / "acceptance"

# (stencil, update, mode) per run, as test_acceptance.py:36-49
ACOUSTIC = {
    "fp64": ("fp64", "fp64", "baseline"),
    "fp16-base": ("fp16", "fp16", "baseline"),
    "fp16-op3": ("fp16", "fp16", "op3"),
    "mixed-naive": ("fp64", "fp16", "baseline"),
    "mixed-op3": ("fp64", "fp16", "op3"),
}
ELASTIC = {
    "fp64": ("fp64", "fp64", "baseline"),
    "fp16-base": ("fp16", "fp16", "baseline"),
    "fp16-op6": ("fp16", "fp16", "op6"),
    "fp16-op3": ("fp16", "fp16", "op3"),
}


def main():
    OUT.mkdir(parents=True, exist_ok=True)
    for preset, runs in (("paper-acoustic", ACOUSTIC), ("paper-elastic", ELASTIC)):
        for name, (s, u, m) in runs.items():
            cfg = parse_config(None, preset=preset, desk=True,
                               sets=[f"precision.stencil={s}", f"precision.update={u}", f"precision.mode={m}"])
            t0 = time.perf_counter()
            out = cfg.run()
            np.savez_compressed(OUT / f"{preset}_{name}.npz",
                                traces=np.array([np.asarray(t.samples, dtype=np.float64) for t in out.traces]),
                                e_times=np.asarray(out.energy.times, dtype=np.float64),
                                e_vals=np.asarray(out.energy.values, dtype=np.float64),
                                t_source_off=2.0 * cfg.source.wavelet.delay)
            print(preset, name, f"{time.perf_counter() - t0:.1f}s", flush=True)


if __name__ == "__main__":
    main()

"""bench.py keeps the driver's JSON-line contract: the reference arm (CPU oracle port, runs
here) and the B200 arm (GPU)."""

import json
import os
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
BASE_KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
             "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"}


def _run(*args, timeout=600, nlines=1):
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), *args], capture_output=True, text=True,
                         timeout=timeout, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.strip().startswith("{")]
    assert len(lines) == nlines, out.stdout
    return json.loads(lines[0]) if nlines == 1 else [json.loads(l) for l in lines]


def test_gpus_n_spawns_n_ranks():
    """--gpus 2 outside torchrun re-launches bench.py as two ranks (one process per GPU)."""
    ranks = _run("--gpus", "2", "--rank-probe", nlines=2, timeout=300)
    assert sorted(r["rank"] for r in ranks) == [0, 1] and {r["world_size"] for r in ranks} == {2}


def test_world_size_mismatch_fails_loudly():
    env = dict(os.environ, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", "2", "--rank-probe"], capture_output=True,
                         text=True, timeout=120, cwd=ROOT, env=env)
    assert out.returncode != 0 and "WORLD_SIZE" in out.stderr


def test_reference_arm_line():
    d = _run("--impl", "reference", "--steps", "1", "--warmup", "0")
    assert BASE_KEYS <= set(d) and d["impl"] == "reference"
    assert d["value"] > 0 and d["higher_is_better"] is True and d["n_gpus"] == 1
    cb = d["cpu_baseline"]
    assert cb["kind"] in ("port", "reference") and cb["cores"] >= 1 and cb["value"] == d["value"] and cb["sample"]
    assert d["e2e"] == {"value": d["value"], "unit": d["unit"], "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}


@pytest.mark.gpu
def test_b200_arm_line():
    d = _run("--steps", "1", "--warmup", "1", "--nt", "40", timeout=1200)
    ref = _run("--impl", "reference", "--steps", "1", "--warmup", "0")
    assert BASE_KEYS <= set(d) and "impl" not in d
    assert d["config"] == ref["config"]  # the driver pairs the two arms by config
    assert d["n_gpus"] == 1 and d["value"] > 1e10 and d["dtype"] == "fp16" and d["scaling"] == "strong"
    r = d["roofline"]
    assert r["bound"] == "hbm" and r["unit"] == "GB/s" and 0 < r["frac"] < 1.5
    assert abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-9
    assert d["cpu_baseline"]["kind"] == "port" and d["cpu_baseline"]["cores"] >= 1
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] == 18 * 512 ** 3 * 2 and e["d2h_bytes_per_step"] > 0
    assert d["gpu_launches"] >= 40 and d["kernel_path"] == "fused3d-el"
    assert "sm_mhz" in d["clocks"] and "reasons" in d["clocks"]
    c = d["configs"]
    for k, path in (("config1", "small2d"), ("config2", "fused2d"), ("config3", "fused3d"),
                    ("config3_fp32_naive", "fused3d-f32"), ("config4", "fused2d-el")):
        assert c[k]["path"] == path and c[k]["value"] > 1e9 and c[k]["roofline"]["frac"] > 0
    for k in ("config2", "config3", "config4"):
        assert c[k]["cpu_baseline"]["value"] > 0

"""Run the UNMODIFIED reference CLI on the desk presets and keep its traces.csv /
energy.csv / summary.json as fixtures (tests/golden/cli/<preset>/).

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba python tests/golden/make_cli_golden.py
"""
import shutil
import subprocess
import sys
import tempfile
from pathlib import Path

OUT = Path(__file__).resolve().parent / "cli"
for preset in ("paper-acoustic", "paper-elastic"):
    with tempfile.TemporaryDirectory() as tmp:
        subprocess.run([sys.executable, "-m", "halfwave.cli", "run", "--preset", preset, "--desk", "--out", tmp],
                       check=True)
        src = Path(tmp) / f"{preset}-desk"
        dst = OUT / preset
        dst.mkdir(parents=True, exist_ok=True)
        for name in ("traces.csv", "energy.csv", "summary.json"):
            shutil.copy(src / name, dst / name)
        print(preset, sorted(p.name for p in dst.iterdir()))

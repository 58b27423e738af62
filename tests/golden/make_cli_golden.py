"""Run the UNMODIFIED reference CLI on the desk presets and keep its traces.csv /
energy.csv / summary.json as fixtures (tests/golden/cli/<preset>/); and on
tests/golden/cli/range-failure/case.ini -- every parameter passes the static audit, but the light
elastic medium amplifies the injection past the binary16 range mid-wavelet -- keeping the exit code
and summary.json (the failing step and field).

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

case = OUT / "range-failure" / "case.ini"
with tempfile.TemporaryDirectory() as tmp:
    r = subprocess.run([sys.executable, "-m", "halfwave.cli", "run", "--config", str(case), "--out", tmp])
    src = Path(tmp) / "overdrive"
    shutil.copy(src / "summary.json", case.parent / "summary.json")
    (case.parent / "exit_code.txt").write_text(f"{r.returncode}\n")
    print("range-failure", r.returncode, sorted(p.name for p in src.iterdir()))

"""Short config-2 run for ncu captures: python tools/profile_step.py [nt] [variant]."""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import paper_2310_00236_b200 as hw  # noqa: E402
import bench  # noqa: E402

nt = int(sys.argv[1]) if len(sys.argv) > 1 else 20
variant = {"naive": None, "op3": hw.Variant.OP3, "op6": hw.Variant.OP6}[sys.argv[2] if len(sys.argv) > 2 else "op3"]
s = bench.make_solver(hw, nt=nt)
st = s.new_state()
s.upload(st)
ms = s.run_device(variant, 0, nt)
print(f"{nt} steps: {ms:.3f} ms, {ms / nt * 1e3:.1f} us/step, {s.last_launch_count()} launches")

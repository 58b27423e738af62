import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import bench
import paper_2310_00236_b200 as hw
nt = 60
for (n, nz) in ((1024, 128), (512, 512), (256, 2048)):
    s = bench.make_config5(hw, n=n, nz=nz, nt=nt)
    st = s.new_state()
    s.upload(st)
    s.run_device(hw.Variant.OP6, 0, 10)
    ms = s.run_device(hw.Variant.OP6, 10, nt)
    cells = n * n * nz
    print(n, nz, s.kernel_path(), f"{ms/nt:.3f} ms/step", f"{cells*nt/ms/1e6:.1f} G cell-steps/s", f"frac {72*cells*nt/ms/1e6/6545:.3f}", flush=True)
    s.close()

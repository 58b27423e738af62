import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import paper_2310_00236_b200 as hw
import argparse
ap = argparse.ArgumentParser()
ap.add_argument("--nx", type=int, default=1024); ap.add_argument("--ny", type=int, default=512)
ap.add_argument("--slabs", type=int, default=2); ap.add_argument("--nt", type=int, default=12)
ap.add_argument("--per", action="store_true"); ap.add_argument("--nosrc", action="store_true")
ap.add_argument("--layers", type=int, default=1); ap.add_argument("--variant", default="op6")
ap.add_argument("--every", type=int, default=10); ap.add_argument("--vsrc", action="store_true")
a = ap.parse_args()
nx, ny = a.nx, a.ny
dx = 1.0 / nx
lay = [(1.0, 1.0, 2.0, 1.0)] if a.layers == 1 else [(0.4, 2.0, 2.0, 1.0), (1.0, 2.3, 2.8, 1.4)]
med = hw.build_layered_elastic(nx, ny, lay)
g = hw.GridSpec(nx, ny, dx, float(np.float16(0.3 * dx / med.c_max())), a.nt, bc_y=hw.Boundary.PERIODIC if a.per else hw.Boundary.FREE_SURFACE)
src = None if a.nosrc else hw.SourceSpec(hw.SourceKind.VY_POINT if a.vsrc else hw.SourceKind.EXPLOSIVE, nx // 2, 16, hw.RickerSpec(1 / (10 * dx), amplitude=3.0e4))
s = hw.ElasticSolver(g, med, src, stencil_precision=hw.Precision.FP16, energy_every=a.every, slabs=a.slabs)
st = s.new_state()
v = {"op6": hw.Variant.OP6, "naive": None, "op3": hw.Variant.OP3}[a.variant]
try:
    out = s.run(v, st)
    print("ok", s.kernel_path(), s.transport())
except Exception as e:
    print("FAIL", str(e)[:80])

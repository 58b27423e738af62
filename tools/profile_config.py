"""Short run of one BASELINE config for ncu:
python tools/profile_config.py [--lib <variant.so>] [--opt name=value ...] <1|2|3|3f32|4|5> [nt]."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2310_00236_b200 as hw  # noqa: E402

args = sys.argv[1:]
if "--lib" in args:  # an A/B build of the library (tools/build_variant.sh); before any library call
    i = args.index("--lib")
    hw._abi.set_library_path(args[i + 1])
    del args[i:i + 2]
opts = []
while "--opt" in args:  # --opt name=value: library kernel-path options (hw_set_option)
    i = args.index("--opt")
    opts.append(args[i + 1].split("="))
    del args[i:i + 2]
sys.argv = sys.argv[:1]  # (measure_configs parses its own command line at import)
import tools.measure_configs as mc  # noqa: E402

for k, v in opts:
    hw.set_option(k, int(v))
which = args[0]
nt = int(args[1]) if len(args) > 1 else 6


def cfg2():
    import bench
    return bench.make_config2(hw, nt=nt)


s = {"1": lambda: mc.cfg1(2), "2": cfg2, "3": mc.cfg3, "3f32": lambda: mc.cfg3(hw.Precision.FP32), "4": mc.cfg4,
     "5": mc.cfg5}[which]()
st = s.new_state()
if which in ("3", "3f32"):
    mc.gauss3(st)
s.upload(st)
v = hw.Variant.OP6 if which in ("4", "5") else (None if which == "3f32" else hw.Variant.OP3)
ms = s.run_device(v, 0, nt)
print(f"config {which}: {nt} steps {ms:.3f} ms, path {s.kernel_path()}")

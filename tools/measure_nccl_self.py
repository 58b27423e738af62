"""The NCCL slab path on one B200: config 5 (512^3, op6), config 4 (4096^2 elastic op6; 4p: periodic, so the
self exchange moves rows), config 3 (512^3 op3; 3f32: fp32 naive) or config 2 (4096^2, op3) single domain vs
the same grid as a one-rank NCCL job (option nccl_self: every step's halo exchange goes through
NCCL to the rank itself, edge slabs + exchange overlapped with the interior slabs).
python tools/measure_nccl_self.py [nt] [5|4|4p|3|3f32|2] -> one JSON line."""
import json
import os
import socket
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import bench  # noqa: E402
import paper_2310_00236_b200 as hw  # noqa: E402

nt = int(sys.argv[1]) if len(sys.argv) > 1 else 50
cfg = sys.argv[2] if len(sys.argv) > 2 else "5"
with socket.socket() as sk:
    sk.bind(("127.0.0.1", 0))
    port = sk.getsockname()[1]
dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1)
out = {}
for name, kw in (("single", {}), ("nccl_self", {"distributed": True})):
    with hw.options(nccl_self=1):
        v = hw.Variant.OP6
        if cfg == "5":
            s = bench.make_config5(hw, nt=nt, **kw)
            st = s.new_state()
            bench.init_config5(st)
        elif cfg in ("4", "4p"):
            s = bench.make_config4(hw, nt=nt, periodic=cfg == "4p", **kw)
            st = s.new_state()
        elif cfg in ("3", "3f32"):
            c3 = out.get("_c3")
            if c3 is None:
                c3 = out["_c3"] = bench.smooth_velocity(512)
            s = bench.make_config3(hw, hw.Precision.FP16 if cfg == "3" else hw.Precision.FP32, nt=nt, c=c3, **kw)
            st = s.new_state()
            bench.init_config3(st)
            v = hw.Variant.OP3 if cfg == "3" else None
        else:
            s = bench.make_config2(hw, nt=nt, **kw)
            st = s.new_state()
            v = hw.Variant.OP3
        s.upload(st)
        s.run_device(v, 0, 10)
        ms = s.run_device(v, 10, nt)
    cells = 512 ** 3 if cfg in ("5", "3", "3f32") else 4096 ** 2
    out[name] = {"ms_per_step": ms / nt, "G_cell_steps_per_s": cells * nt / ms / 1e6, "path": s.kernel_path(),
                 "transport": s.transport()}
    s.close()
out.pop("_c3", None)
out["config"] = cfg
out["nccl_over_single"] = out["single"]["ms_per_step"] / out["nccl_self"]["ms_per_step"]
print(json.dumps(out))
dist.destroy_process_group()

"""Strong-scaling proxy on one B200: config 5's 512^3 grid cut into N z-slabs, ONE slab (512 x 512 x 512/N)
run as a one-rank NCCL job (option nccl_self: edge slabs + exchange to itself overlapped with the interior
slabs) -- the per-GPU step of an N-GPU run, with the self exchange standing in for NVLink -- against the
single-domain 512^3 step / N.  python tools/measure_strong_proxy.py [--opt name=value ...] [nt] [edge_ctas ...] -> one JSON line per N."""
import json
import socket
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch.distributed as dist  # noqa: E402

import bench  # noqa: E402
import paper_2310_00236_b200 as hw  # noqa: E402

args = sys.argv[1:]
while "--opt" in args:  # --opt name=value: library kernel-path options (hw_set_option)
    i = args.index("--opt")
    k, v = args[i + 1].split("=")
    hw.set_option(k, int(v))
    del args[i:i + 2]
nt = int(args[0]) if args else 200
sweep = [int(a) for a in args[1:]] or [0]
with socket.socket() as sk:
    sk.bind(("127.0.0.1", 0))
    port = sk.getsockname()[1]
dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1)


def step_us(nz, distributed, edge=0):
    with hw.options(nccl_self=1, el3_edge_ctas=edge):
        s = bench.make_config5(hw, nz=nz, nt=nt, distributed=distributed)
        st = s.new_state()
        bench.init_config5(st)
        s.upload(st)
        s.run_device(hw.Variant.OP6, 0, 20)
        ms = min(s.run_device(hw.Variant.OP6, 20, nt), s.run_device(hw.Variant.OP6, 20 + nt, nt))
        path, tr = s.kernel_path(), s.transport()
        s.close()
    return 1e3 * ms / nt, path, tr


t1, _, _ = step_us(512, False)
for n in (2, 4, 8):
    for e in sweep:
        t, path, tr = step_us(512 // n, True, e)
        print(json.dumps({"config": "5", "n_gpus_proxied": n, "slab": [512, 512, 512 // n], "edge_ctas": e or "auto",
                          "single_512cubed_us": round(t1, 1), "slab_step_us": round(t, 1), "ideal_us": round(t1 / n, 1),
                          "parallel_efficiency_proxy": round(t1 / n / t, 4), "path": path, "transport": tr}), flush=True)
dist.destroy_process_group()

#!/usr/bin/env python3
"""HBM throughput of the token-permutation kernel (bam_permute_blocks): the
fused Q/K/V/dO gather of one CP rank's blocks at config 4 (world 8) and the
inverse scatter of O.  Prints one JSON line (bytes moved = read + write)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2503_11367_b200 import cp, mask as M  # noqa: E402
from paper_2503_11367_b200.workloads import CONFIGS  # noqa: E402

cfg = CONFIGS[int(os.environ.get("CFG", "4"))]
world = int(os.environ.get("WORLD", "8"))
desc = M.build_bitfield(cfg["segments"]).device_descriptors()
plan = cp.make_cp_plan(desc, world, 0, "lpt")
lay = plan.layout
T, dev = desc.shape[0], torch.device("cuda")
Hq, Hkv = cfg["Hq"], cfg["Hkv"]
xs = [torch.randn(T, h, 128, device=dev).to(torch.bfloat16) for h in (Hq, Hkv, Hkv, Hq)]
ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
res = {}
for it in range(6):
    ev[0].record()
    outs = cp.shard_rows(*xs, layout=lay)
    ev[1].record()
    full = torch.empty_like(xs[0])
    ev[2].record()
    cp.unshard_rows(outs[0], lay, full)
    ev[3].record()
    torch.cuda.synchronize()
    if it:
        g = sum(o.numel() * o.element_size() for o in outs) * 2
        s = outs[0].numel() * outs[0].element_size() * 2
        res.setdefault("gather", []).append(g / ev[0].elapsed_time(ev[1]) / 1e6)
        res.setdefault("scatter", []).append(s / ev[2].elapsed_time(ev[3]) / 1e6)
print(json.dumps({"config": cfg["name"], "world": world, "local_blocks": lay.n_local,
                  "gather_qkvdo_GBps": max(res["gather"]), "scatter_o_GBps": max(res["scatter"])}))

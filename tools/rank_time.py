#!/usr/bin/env python3
"""Per-rank attention kernel times of a CP plan, emulated on one GPU (no
exchange): separates the kernels' own per-rank efficiency from the
communication in bench.py's N>1 fwd_ms / bwd_ms.

    python tools/rank_time.py --config 4 --world 4
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2503_11367_b200 import attention as A, cp, mask as M  # noqa: E402
from paper_2503_11367_b200.workloads import CONFIGS  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=4)
ap.add_argument("--world", type=int, default=4)
ap.add_argument("--iters", type=int, default=3)
args = ap.parse_args()
cfg = CONFIGS[args.config]
mask = M.build_bitfield(cfg["segments"])
desc = mask.device_descriptors()
T, dev = desc.shape[0], torch.device("cuda")
g = torch.Generator(device=dev).manual_seed(1234)
Hq, Hkv = cfg["Hq"], cfg["Hkv"]
q = torch.randn(T, Hq, 128, device=dev, generator=g, dtype=torch.bfloat16)
k = torch.randn(T, Hkv, 128, device=dev, generator=g, dtype=torch.bfloat16)
v = torch.randn(T, Hkv, 128, device=dev, generator=g, dtype=torch.bfloat16)
do = torch.randn(T, Hq, 128, device=dev, generator=g, dtype=torch.bfloat16)
nb = T // 128
for r in range(args.world):
    plan = cp.make_cp_plan(desc, args.world, r, "lpt")
    lay = plan.layout
    k_all = torch.zeros((args.world * lay.max_blocks * 128, Hkv, 128), dtype=k.dtype, device=dev)
    v_all = torch.zeros_like(k_all)
    cp.permute_blocks([k, v], [k_all, v_all], lay.k_row[:nb], scatter=True)
    ql, dol = cp.shard_rows(q, do, layout=lay)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    f, b = [], []
    for it in range(args.iters + 1):
        ev[0].record()
        o, lse = A.attn_forward(ql, k_all, v_all, plan.attn)
        ev[1].record()
        ws = A.BackwardWorkspace(ql, o, lse, dol, plan.attn, None)
        ws.main(k_all, v_all)
        ev[2].record()
        torch.cuda.synchronize()
        if it:
            f.append(ev[0].elapsed_time(ev[1]))
            b.append(ev[1].elapsed_time(ev[2]))
    print(json.dumps({"rank": r, "fwd_ms": round(min(f), 3), "bwd_main_ms": round(min(b), 3)}),
          flush=True)

#!/usr/bin/env python3
"""Run the single-GPU attention fwd+bwd of a BASELINE config a few times
(profiling driver for ncu: `ncu -k regex:attn_ ... python tools/run_attn.py`)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2503_11367_b200 import attention as A, mask as M  # noqa: E402
from paper_2503_11367_b200.workloads import CONFIGS  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=4)
ap.add_argument("--iters", type=int, default=2)
ap.add_argument("--tokens", type=int, default=0, help="truncate the mask to this many tokens")
args = ap.parse_args()
cfg = CONFIGS[args.config]
segs = cfg["segments"]
if args.tokens:
    out, tot = [], 0
    for m, c in segs:
        c = min(c, args.tokens - tot)
        if c <= 0:
            break
        out.append((m, c))
        tot += c
    segs = out
mask = M.build_bitfield(segs)
plan = A.plan_for_mask(mask)
T, dev = len(mask), torch.device("cuda")
g = torch.Generator(device=dev).manual_seed(1234)
q = torch.randn(T, cfg["Hq"], 128, device=dev, generator=g, dtype=torch.bfloat16)
k = torch.randn(T, cfg["Hkv"], 128, device=dev, generator=g, dtype=torch.bfloat16)
v = torch.randn(T, cfg["Hkv"], 128, device=dev, generator=g, dtype=torch.bfloat16)
do = torch.randn(T, cfg["Hq"], 128, device=dev, generator=g, dtype=torch.bfloat16)
for _ in range(args.iters):
    o, lse = A.attn_forward(q, k, v, plan)
    dq, dk, dv = A.attn_backward(q, k, v, o, lse, do, plan)
torch.cuda.synchronize()
print("ok", T)

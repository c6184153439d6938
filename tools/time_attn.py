#!/usr/bin/env python3
"""Quick CUDA-event timing of the single-GPU fwd / bwd kernels on a BASELINE
config (development aid; bench.py is the contract)."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2503_11367_b200 import attention as A, mask as M  # noqa: E402
from paper_2503_11367_b200.workloads import CONFIGS, SWEEP_128K  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="4")
ap.add_argument("--iters", type=int, default=5)
ap.add_argument("--heads", type=int, default=0, help="override Hq")
ap.add_argument("--kv-heads", type=int, default=0, help="override Hkv")
args = ap.parse_args()
out = {}
for name in args.config.split(","):
    if name.isdigit():
        cfg = CONFIGS[int(name)]
        segs, Hq, Hkv = cfg["segments"], cfg["Hq"], cfg["Hkv"]
    else:
        segs, Hq, Hkv = SWEEP_128K[name], 32, 8
    Hq, Hkv = args.heads or Hq, args.kv_heads or Hkv
    mask = M.build_bitfield(segs)
    desc = mask.device_descriptors()
    plan = A.build_plan(desc)
    n_allowed = M.count_allowed(desc)
    T, dev = len(mask), torch.device("cuda")
    g = torch.Generator(device=dev).manual_seed(1234)
    q = torch.randn(T, Hq, 128, device=dev, generator=g, dtype=torch.bfloat16)
    k = torch.randn(T, Hkv, 128, device=dev, generator=g, dtype=torch.bfloat16)
    v = torch.randn(T, Hkv, 128, device=dev, generator=g, dtype=torch.bfloat16)
    do = torch.randn(T, Hq, 128, device=dev, generator=g, dtype=torch.bfloat16)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    f_ms, b_ms = [], []
    for it in range(args.iters + 2):
        ev[0].record()
        o, lse = A.attn_forward(q, k, v, plan)
        ev[1].record()
        dq, dk, dv = A.attn_backward(q, k, v, o, lse, do, plan, dkv_fp32=True, timer=(ev[2], ev[3]))
        torch.cuda.synchronize()
        if it >= 2:
            f_ms.append(ev[0].elapsed_time(ev[1]))
            b_ms.append(ev[2].elapsed_time(ev[3]))
    f, b = min(f_ms), min(b_ms)
    ff, fb = 4 * 128 * Hq * n_allowed, 10 * 128 * Hq * n_allowed
    out[name] = {"fwd_ms": f, "bwd_main_ms": b, "fwd_tflops": ff / f / 1e9, "bwd_tflops": fb / b / 1e9,
                 "fwdbwd_tflops": (ff + fb) / (f + b) / 1e9}
    print(name, json.dumps(out[name]), flush=True)

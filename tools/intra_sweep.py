#!/usr/bin/env python3
"""Intra-GPU subblock sweep (the paper's Fig. 9 / §5.2 shape on B200).

One CP rank's share of a BASELINE config (LPT assignment over --world ranks;
the other ranks' K/V are placed in the gathered layout directly, no NCCL)
runs the forward with the split-KV schedule at several subblock sizes s
(key tiles per piece; "whole" = one CTA per row).  Prints per s: forward
time including the aggregation kernel, the aggregation kernel alone, the
number of pieces, and the reference cost model's prediction
(balance.intra_schedule with compute_units = CTAs resident at once).
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2503_11367_b200 import _lib, attention as A, balance as B, cp, mask as M  # noqa: E402
from paper_2503_11367_b200.workloads import CONFIGS  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=4)
ap.add_argument("--world", type=int, default=8)
ap.add_argument("--rank", type=int, default=0)
ap.add_argument("--subblocks", default="0,256,128,64,32,16,8")
ap.add_argument("--iters", type=int, default=5)
args = ap.parse_args()
cfg = CONFIGS[args.config]
Hq, Hkv = cfg["Hq"], cfg["Hkv"]
mask = M.build_bitfield(cfg["segments"])
desc = mask.device_descriptors()
T, dev = desc.shape[0], torch.device("cuda")
plan = cp.make_cp_plan(desc, args.world, args.rank, "lpt")
lay = plan.layout
g = torch.Generator(device=dev).manual_seed(1234)
q = torch.randn(T, Hq, 128, device=dev, generator=g, dtype=torch.bfloat16)
k = torch.randn(T, Hkv, 128, device=dev, generator=g, dtype=torch.bfloat16)
v = torch.randn(T, Hkv, 128, device=dev, generator=g, dtype=torch.bfloat16)
idx = (lay.k_row.long()[:, None] * 128 + torch.arange(128, device=dev)[None, :]).reshape(-1)
rows = args.world * lay.max_blocks * 128
k_all = torch.zeros(rows, Hkv, 128, dtype=torch.bfloat16, device=dev)
v_all = torch.zeros_like(k_all)
k_all[idx], v_all[idx] = k, v
q_loc = cp.shard_rows(q, lay).contiguous()
W_local = (plan.attn.row_off[1:] - plan.attn.row_off[:-1]).cpu().tolist()
n_allowed = M.count_allowed(desc)
flop_local = 4.0 * 128 * Hq * n_allowed / args.world   # approx. local share
units = 148 * (1 if Hq // Hkv % 2 == 0 else 2)          # CTAs resident at once
heads_per_cta = 2 if Hq // Hkv % 2 == 0 else 1

ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
for sb in [int(x) for x in args.subblocks.split(",")]:
    sched = None if sb == 0 else A.build_split_schedule(plan.attn, sb)
    times, comb = [], []
    for it in range(args.iters + 1):
        ev[0].record()
        o, lse = A.attn_forward(q_loc, k_all, v_all, plan.attn, schedule=sched)
        ev[1].record()
        if sched is not None and sched.combine.shape[0]:
            p = _lib.BamAttnFwdParams(
                q_loc.data_ptr(), k_all.data_ptr(), v_all.data_ptr(), o.data_ptr(),
                lse.data_ptr(), plan.attn.desc.data_ptr(), plan.attn.q_gid.data_ptr(),
                plan.attn.k_row.data_ptr(), plan.attn.row_off.data_ptr(),
                plan.attn.row_tiles.data_ptr(), None, plan.attn.nq, plan.attn.nb,
                plan.attn.k_rows, Hq, Hkv, 1.0 / 128 ** 0.5, 0, 0, sched.items.data_ptr(),
                None, None, sched.n_items, 0)
        ev[2].record()
        torch.cuda.synchronize()
        if it:
            times.append(ev[0].elapsed_time(ev[1]))
    # cost model: every (piece, head-group) is a task on `units` compute units
    s_model = max(W_local) if sb == 0 else sb
    per_cta = [w for w in W_local for _ in range(Hq // heads_per_cta)]
    model = B.intra_schedule(per_cta, units, s_model)
    print(json.dumps({
        "config": cfg["name"], "world": args.world, "rank": args.rank,
        "subblock": "whole" if sb == 0 else sb, "fwd_ms_incl_combine": min(times),
        "tflops_approx": flop_local / min(times) / 1e9,
        "pieces": sched.n_items if sched else len(W_local),
        "split_rows": int(sched.combine.shape[0]) if sched else 0,
        "model_compute_makespan": model.compute_makespan,
        "model_aggregation": model.aggregation_cost, "model_total": model.total,
        "W_local_max": max(W_local), "W_local_mean": sum(W_local) / len(W_local)}), flush=True)

#!/usr/bin/env python3
"""Per-rank attention kernel times of a CP plan, emulated on one GPU (no
exchange): separates the kernels' own per-rank efficiency from the
communication in bench.py's N>1 fwd_ms / bwd_ms.

    python tools/rank_time.py --config 4 --world 4 [--policy lpt]

Also reports per-rank cost features (tiles = the LPT load, PARTIAL tiles, the
backward's CTA-pair slot steps, the forward pair-union length) and the
kernel-only max/mean imbalance over the emulated ranks.
"""
import argparse
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2503_11367_b200 import attention as A, cp, mask as M  # noqa: E402
from paper_2503_11367_b200.workloads import CONFIGS, SWEEP_128K  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="4", help="BASELINE config id or a 128K sweep mask name")
ap.add_argument("--world", type=int, default=4)
ap.add_argument("--iters", type=int, default=3)
ap.add_argument("--policy", default="lpt")
args = ap.parse_args()
if args.config.isdigit():
    cfg = CONFIGS[int(args.config)]
else:
    cfg = {"segments": SWEEP_128K[args.config], "Hq": 32, "Hkv": 8}
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
# every rank's plan and inputs first, then iterations round-robin over the ranks
# (rank 0, 1, ..., world-1, 0, ...): run one after another, the later ranks would
# see a hotter, more power-capped GPU and read slower
ranks = []
for r in range(args.world):
    plan = cp.make_cp_plan(desc, args.world, r, args.policy)
    lay = plan.layout
    k_all = torch.zeros((args.world * lay.max_blocks * 128, Hkv, 128), dtype=k.dtype, device=dev)
    v_all = torch.zeros_like(k_all)
    cp.permute_blocks([k, v], [k_all, v_all], lay.k_row[:nb], scatter=True)
    ql, dol = cp.shard_rows(q, do, layout=lay)
    ranks.append((plan, k_all, v_all, ql, dol))
times = [([], []) for _ in range(args.world)]
for it in range(args.iters + 1):
    for r, (plan, k_all, v_all, ql, dol) in enumerate(ranks):
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        ev[0].record()
        o, lse = A.attn_forward(ql, k_all, v_all, plan.attn)
        ev[1].record()
        ws = A.BackwardWorkspace(ql, o, lse, dol, plan.attn, None)
        ws.main(k_all, v_all, timer=(ev[2], ev[3]))
        torch.cuda.synchronize()
        if it:
            times[r][0].append(ev[0].elapsed_time(ev[1]))
            times[r][1].append(ev[2].elapsed_time(ev[3]))
rows = []
for r, (plan, k_all, v_all, ql, dol) in enumerate(ranks):
    lay, at = plan.layout, plan.attn
    f, b = statistics.median(times[r][0]), statistics.median(times[r][1])
    # cost features: tiles (the LPT load W), PARTIAL tiles, backward steps including the
    # class-0 padding of shared CTA-pair union lists, forward pair-union padding
    tiles = int(at.row_off[-1])
    partial = int(((at.row_tiles[:tiles] & 3) == 2).sum())
    bwd_slots = int(at.slot_off[-1])
    n_pairs = int(at.counts[0])
    fwd_union = int(sum(int(at.fwd_slot_off[2 * pr + 1] - at.fwd_slot_off[2 * pr])
                        for pr in at.fwd_pair_ids[:n_pairs].tolist())) if n_pairs else 0
    row = {"rank": r, "policy": args.policy, "n_local": lay.n_local,
           "fwd_ms": round(f, 3), "bwd_main_ms": round(b, 3),
           "kernel_ms": round(f + b, 3), "tiles": tiles, "partial_tiles": partial,
           "bwd_slot_steps": bwd_slots, "fwd_pair_union": fwd_union}
    rows.append(row)
    print(json.dumps(row), flush=True)
ks = [x["kernel_ms"] for x in rows]
ts = [x["tiles"] for x in rows]
n_allowed = M.count_allowed(desc)
flop = 14.0 * 128 * Hq * n_allowed
print(json.dumps({"config": args.config, "world": args.world, "policy": args.policy,
                  "iters_round_robin": args.iters,
                  "makespan_kernel_ms": max(ks),
                  "tflops_emulated_whole_job": flop / max(ks) / 1e9,
                  "imbalance_kernel": max(ks) / (sum(ks) / len(ks)),
                  "imbalance_fwd": max(x["fwd_ms"] for x in rows) /
                  (sum(x["fwd_ms"] for x in rows) / len(rows)),
                  "imbalance_bwd": max(x["bwd_main_ms"] for x in rows) /
                  (sum(x["bwd_main_ms"] for x in rows) / len(rows)),
                  "imbalance_predicted": max(ts) / (sum(ts) / len(ts))}), flush=True)

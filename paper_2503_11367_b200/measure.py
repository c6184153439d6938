"""Measured counterpart of ``balance_report``: run every
CP rank's share of the masked attention fwd+bwd for each distribution policy
on this GPU and report the per-rank kernel times, the makespan and the
measured imbalance beside the reference's cost-model prediction
(ref: balance.py:271-311, cli.py:86-117; the paper's Table 5 shape,
PAPER.md:804-823).

Ranks are emulated one after another on one device: each rank's query blocks
run against all keys placed in the rank-major gathered layout, exactly the
kernels a CP rank launches (the collectives, which do not depend on the
policy's balance, are not timed).  The report's four policies map to:

  causal      zigzag blocks, whole rows
  inter_only  LPT blocks,    whole rows
  intra_only  zigzag blocks, forward rows split into subblocks (split-KV)
  balanced    LPT blocks,    forward rows split into subblocks (split-KV)
"""

from __future__ import annotations

import torch

from . import attention as A
from . import cp
from .mask import BitfieldMask

POLICIES = {
    "causal": ("zigzag", False),
    "inter_only": ("lpt", False),
    "intra_only": ("zigzag", True),
    "balanced": ("lpt", True),
}


def _time_rank(q, k, v, do, desc, world, rank, dist_policy, subblock, iters):
    plan = cp.make_cp_plan(desc, world, rank, dist_policy)
    lay = plan.layout
    nb = desc.shape[0] // cp.BLOCK
    k_all = torch.zeros((world * lay.max_blocks * cp.BLOCK,) + tuple(k.shape[1:]), dtype=k.dtype,
                        device=k.device)
    v_all = torch.zeros_like(k_all)
    # place every key block at its gathered row (what the all-gather produces)
    cp.permute_blocks([k, v], [k_all, v_all], lay.k_row[:nb], scatter=True)
    ql, dol = cp.shard_rows(q, do, layout=lay)
    sched = A.build_split_schedule(plan.attn, subblock) if subblock else None
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    times = []
    for it in range(iters + 1):
        ev[0].record()
        o, lse = A.attn_forward(ql, k_all, v_all, plan.attn, schedule=sched)
        A.attn_backward(ql, k_all, v_all, o, lse, dol, plan.attn, dkv_fp32=True)
        ev[1].record()
        torch.cuda.synchronize()
        if it:
            times.append(ev[0].elapsed_time(ev[1]))
    loads = plan.assignment.loads.cpu().tolist()
    return min(times), loads


def measure_policies(mask: BitfieldMask, num_gpus: int, subblock_size: int, heads: int = 32,
                     kv_heads: int = 8, head_dim: int = 128, iters: int = 2, seed: int = 1234):
    """{policy: {"ms_per_rank", "makespan_ms", "imbalance_measured",
    "imbalance_predicted"}} for the four report policies."""
    desc = mask.device_descriptors()
    T = desc.shape[0]
    if T % cp.BLOCK:
        raise ValueError(f"measured report needs T % {cp.BLOCK} == 0")
    dev = desc.device
    g = torch.Generator(device=dev).manual_seed(seed)
    q = torch.randn(T, heads, head_dim, device=dev, generator=g, dtype=torch.bfloat16)
    k = torch.randn(T, kv_heads, head_dim, device=dev, generator=g, dtype=torch.bfloat16)
    v = torch.randn(T, kv_heads, head_dim, device=dev, generator=g, dtype=torch.bfloat16)
    do = torch.randn(T, heads, head_dim, device=dev, generator=g, dtype=torch.bfloat16)
    out = {}
    for name, (dist_policy, split) in POLICIES.items():
        per_rank, loads = [], None
        for r in range(num_gpus):
            ms, loads = _time_rank(q, k, v, do, desc, num_gpus, r, dist_policy,
                                   subblock_size if split else 0, iters)
            per_rank.append(ms)
        mean = sum(per_rank) / len(per_rank)
        out[name] = {
            "distribution": dist_policy, "split_kv_subblock": subblock_size if split else None,
            "ms_per_rank": per_rank, "makespan_ms": max(per_rank),
            "imbalance_measured": max(per_rank) / mean if mean > 0 else 1.0,
            "imbalance_predicted": (max(loads) / (sum(loads) / len(loads))
                                    if sum(loads) else 1.0),
        }
    return out

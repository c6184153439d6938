#!/usr/bin/env python3
"""Config-5 sweep: mask patterns x distribution policies at 128K on N GPUs.

    torchrun --nproc-per-node N --master-addr 127.0.0.1 tools/sweep_policies.py

For each mask (causal, prefix-LM, multimodal, multi-image; BASELINE.json
config 5) and policy (lpt = the paper's workload-balanced distribution,
zigzag = the causal-CP baseline, contiguous = naive uniform token split) runs
the CP attention fwd+bwd (NCCL all-gather / reduce-scatter included), timed
with CUDA events, max over ranks.  Prints one JSON line per (mask, policy):
TFLOP/s (whole job, algorithmic masked FLOP), per-GPU, predicted imbalance
(BlockAssignment.imbalance of the device assignment) and measured imbalance
(max / mean of per-rank fwd+bwd kernel time).  This is the shape of the
paper's Table 5 measured on B200.
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2503_11367_b200 import attention as A, cp, mask as M  # noqa: E402
from paper_2503_11367_b200.workloads import SWEEP_128K  # noqa: E402

rank, world = int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))
local = int(os.environ.get("LOCAL_RANK", 0))
torch.cuda.set_device(local)
dev = torch.device("cuda", local)
if world > 1:
    dist.init_process_group("nccl", device_id=dev)
Hq, Hkv, iters = 32, 8, int(os.environ.get("SWEEP_ITERS", "3"))
masks = os.environ.get("SWEEP_MASKS", ",".join(SWEEP_128K)).split(",")
policies = os.environ.get("SWEEP_POLICIES", "lpt,zigzag,contiguous").split(",")


def barrier():
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()


for name in masks:
    mask = M.build_bitfield(SWEEP_128K[name])
    desc = mask.device_descriptors()
    T = desc.shape[0]
    n_allowed = M.count_allowed(desc)
    flop = 14.0 * 128 * Hq * n_allowed
    g = torch.Generator(device=dev).manual_seed(1234)
    q = torch.randn(T, Hq, 128, device=dev, generator=g, dtype=torch.bfloat16)
    k = torch.randn(T, Hkv, 128, device=dev, generator=g, dtype=torch.bfloat16)
    v = torch.randn(T, Hkv, 128, device=dev, generator=g, dtype=torch.bfloat16)
    do = torch.randn(T, Hq, 128, device=dev, generator=g, dtype=torch.bfloat16)
    for pol in policies:
        plan = cp.make_cp_plan(desc, world, rank, pol)
        lay = plan.layout
        ql, kl, vl, dol = cp.shard_rows(q, k, v, do, layout=lay)

        def step(ev):
            k_all, v_all = cp.gather_kv(kl, vl, lay) if world > 1 else (kl, vl)
            ev[0].record()
            o, lse = A.attn_forward(ql, k_all, v_all, plan.attn)
            dq, dka, dva = A.attn_backward(ql, k_all, v_all, o, lse, dol, plan.attn, dkv_fp32=True)
            ev[1].record()
            if world > 1:
                cp.scatter_dkv(dka, dva, lay)

        for _ in range(2):
            step([torch.cuda.Event(enable_timing=True) for _ in range(2)])
        barrier()
        evs = [[torch.cuda.Event(enable_timing=True) for _ in range(2)] for _ in range(iters)]
        s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s0.record()
        for i in range(iters):
            step(evs[i])
        s1.record()
        barrier()
        t = torch.tensor([s0.elapsed_time(s1) / iters,
                          sum(e[0].elapsed_time(e[1]) for e in evs) / iters],
                         dtype=torch.float64, device=dev)
        if world > 1:
            tmax, tsum = t.clone(), t.clone()
            dist.all_reduce(tmax, op=dist.ReduceOp.MAX)
            dist.all_reduce(tsum, op=dist.ReduceOp.SUM)
        else:
            tmax, tsum = t, t
        loads = plan.assignment.loads.cpu().tolist()
        if rank == 0:
            ms = tmax[0].item()
            print(json.dumps({
                "mask": name, "policy": pol, "n_gpus": world, "tokens": T, "ms_per_step": ms,
                "tflops": flop / ms / 1e9, "tflops_per_gpu": flop / ms / 1e9 / world,
                "imbalance_predicted": max(loads) / (sum(loads) / len(loads)),
                "imbalance_measured": tmax[1].item() / (tsum[1].item() / world),
                "n_allowed": n_allowed}), flush=True)
        del ql, kl, vl, dol
    del q, k, v, do
if world > 1:
    dist.destroy_process_group()

#!/usr/bin/env python3
"""Kernel / copy timeline of one CP step on rank 0 (torch.profiler, CUPTI):
where the time between the attention kernels goes at N>1.

    torchrun --nproc-per-node 4 --master-addr 127.0.0.1 tools/step_timeline.py [--config 4]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2503_11367_b200 import cp, mask as M  # noqa: E402
from paper_2503_11367_b200.workloads import CONFIGS  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=4)
ap.add_argument("--transport", default="auto")
ap.add_argument("--out", default="gpurun_out/step_timeline.json")
args = ap.parse_args()
local = int(os.environ.get("LOCAL_RANK", 0))
torch.cuda.set_device(local)
dev = torch.device("cuda", local)
dist.init_process_group("nccl", device_id=dev)
rank, world = dist.get_rank(), dist.get_world_size()
cfg = CONFIGS[args.config]
desc = M.build_bitfield(cfg["segments"]).device_descriptors()
T = desc.shape[0]
g = torch.Generator(device=dev).manual_seed(1234)
q, k, v, do = (torch.randn(T, h, 128, device=dev, generator=g, dtype=torch.bfloat16)
               for h in (cfg["Hq"], cfg["Hkv"], cfg["Hkv"], cfg["Hq"]))
plan = cp.make_cp_plan(desc, world, rank, "lpt")
ql, kl, vl, dol = cp.shard_rows(q, k, v, do, layout=plan.layout)


def step():
    o, lse, gathered = cp.cp_forward(ql, kl, vl, plan, transport=args.transport)
    return cp.cp_backward(ql, gathered, o, lse, dol, plan, transport=args.transport)


for _ in range(3):
    step()
torch.cuda.synchronize()
dist.barrier()
from torch.profiler import ProfilerActivity, profile  # noqa: E402
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    for _ in range(2):
        step()
    torch.cuda.synchronize()
dist.barrier()
if rank == 0:
    evs = []
    for e in prof.events():
        if e.device_type == torch.autograd.DeviceType.CUDA:
            evs.append((e.time_range.start, e.time_range.end, e.name))
    evs.sort()
    t0 = evs[0][0]
    rows = [{"start_us": round(s - t0, 1), "dur_us": round(e - s, 1), "name": n[:90]}
            for s, e, n in evs]
    os.makedirs(os.path.dirname(args.out) or ".", exist_ok=True)
    json.dump(rows, open(args.out, "w"), indent=0)
    for r in rows:
        if r["dur_us"] > 20:
            print(r)
dist.destroy_process_group()

#!/usr/bin/env python3
"""Achieved NVLink bandwidth of the CP exchange steps alone (config 4 shapes).

    torchrun --nproc-per-node N --master-addr 127.0.0.1 tools/exchange_bw.py

Times, on the current stream with CUDA events (max over ranks), the forward
K/V all-gather and the backward dK/dV reduce-scatter of the padded config-4
shards, through both transports: "nccl" (cp.gather_kv / cp.scatter_dkv) and
"ce" (cp.SymmExchange copy-engine pulls / pushes over torch symmetric
memory, its device barriers included), plus "ce_head_major" = the
gather_overlapped() pulls bench.py uses (one copy stream per peer).  Prints one JSON line per
(step, transport): peer bytes per rank (what crosses NVLink into, for the
gather, or out of, for the reduce-scatter, one GPU) and that over the time.
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2503_11367_b200 import cp, mask as M  # noqa: E402
from paper_2503_11367_b200.workloads import CONFIGS  # noqa: E402

rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
local = int(os.environ.get("LOCAL_RANK", 0))
dev = torch.device("cuda", local)
torch.cuda.set_device(dev)
dist.init_process_group("nccl", device_id=dev)
iters = int(os.environ.get("EXCHANGE_ITERS", "10"))

cfg = CONFIGS[4]
Hkv, D = cfg["Hkv"], 128
desc = M.build_bitfield(cfg["segments"]).device_descriptors()
plan = cp.make_cp_plan(desc, world, rank, "lpt")
lay = plan.layout
n_loc = lay.n_local * 128
rows = lay.max_blocks * 128
g = torch.Generator(device=dev).manual_seed(1234 + rank)
k_loc = torch.randn(n_loc, Hkv, D, device=dev, generator=g, dtype=torch.bfloat16)
v_loc = torch.randn_like(k_loc)
dk_all = torch.randn(world * rows, Hkv, D, device=dev, generator=g, dtype=torch.float32)
dv_all = torch.randn_like(dk_all)
ex = plan.exchange(Hkv, D, dev)

gather_bytes = (world - 1) * rows * Hkv * D * 2 * 2          # bf16 K and V from every peer
rs_bytes = (world - 1) * rows * Hkv * D * 4 * 2              # fp32 dK and dV to every peer

steps = {
    ("kv_all_gather", "nccl"): (lambda: cp.gather_kv(k_loc, v_loc, lay), gather_bytes),
    ("kv_all_gather", "ce"): (lambda: ex.gather(rows, 0, k_loc, v_loc), gather_bytes),
    ("kv_all_gather", "ce_head_major"): (lambda: ex.gather_overlapped(rows, k_loc, v_loc, 8),
                                         gather_bytes),
    ("kv_all_gather", "ce_head_major_2chunks"): (
        lambda: ex.gather_overlapped(rows, k_loc, v_loc, 2), gather_bytes),
    ("kv_all_gather", "ce_head_major_1chunk"): (
        lambda: ex.gather_overlapped(rows, k_loc, v_loc, 1), gather_bytes),
    ("dkv_reduce_scatter", "nccl"): (lambda: cp.scatter_dkv(dk_all, dv_all, lay), rs_bytes),
    ("dkv_reduce_scatter", "ce"): (lambda: ex.reduce_scatter(rows, 0, dk_all, dv_all, n_loc),
                                   rs_bytes),
}


def sync():
    dist.barrier()
    torch.cuda.synchronize()


for (name, transport), (fn, nbytes) in steps.items():
    for _ in range(3):
        fn()
    sync()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        fn()
    e1.record()
    sync()
    ms = torch.tensor([e0.elapsed_time(e1) / iters], device=dev)
    dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    ms = ms.item()
    if rank == 0:
        print(json.dumps({"step": name, "transport": transport, "n_gpus": world,
                          "workload": "config4_emu_multi_image_128k", "rows_per_rank": rows,
                          "peer_bytes_per_rank": nbytes, "ms": ms,
                          "nvlink_gbs_per_rank": nbytes / ms / 1e6}), flush=True)
dist.barrier()
dist.destroy_process_group()

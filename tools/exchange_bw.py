#!/usr/bin/env python3
"""Achieved NVLink bandwidth of the CP exchange steps alone (config 4 shapes).

    torchrun --nproc-per-node N --master-addr 127.0.0.1 tools/exchange_bw.py

Times, on the current stream with CUDA events (max over ranks), the forward
K/V all-gather and the backward dK/dV reduce-scatter of the padded config-4
shards, through both transports: "nccl" (cp.gather_kv / cp.scatter_dkv) and
"ce" (cp.SymmExchange copy-engine pulls / pushes over torch symmetric
memory, its device barriers included), plus "ce_overlapped_<k>streams" = the
gather_overlapped() pulls bench.py uses (peer by peer in rotation order on k
streams joined per peer, one group of KV heads and one arrival flag each;
k = 1 by default) and
"ce_peer_sequential_<k>" (the same with a join between peers).  Prints one JSON line per
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
    ("kv_all_gather", "ce_overlapped_1stream"): (
        lambda: ex.gather_overlapped(rows, k_loc, v_loc, 1), gather_bytes),   # bench.py's
    ("kv_all_gather", "ce_overlapped_2streams"): (
        lambda: ex.gather_overlapped(rows, k_loc, v_loc, 2), gather_bytes),
    ("kv_all_gather", "ce_overlapped_4streams"): (
        lambda: ex.gather_overlapped(rows, k_loc, v_loc, 4), gather_bytes),
    ("kv_all_gather", "ce_overlapped_8streams"): (
        lambda: ex.gather_overlapped(rows, k_loc, v_loc, 8), gather_bytes),
    ("kv_all_gather", "ce_peer_sequential_8"): (lambda: peer_sequential(rows, k_loc, v_loc, 8),
                                                gather_bytes),
    ("kv_all_gather", "ce_peer_sequential_4"): (lambda: peer_sequential(rows, k_loc, v_loc, 4),
                                                gather_bytes),
    ("kv_all_gather", "ce_peer_sequential_2"): (lambda: peer_sequential(rows, k_loc, v_loc, 2),
                                                gather_bytes),
    ("dkv_reduce_scatter", "nccl"): (lambda: cp.scatter_dkv(dk_all, dv_all, lay), rs_bytes),
    ("dkv_reduce_scatter", "ce"): (lambda: ex.reduce_scatter(rows, 0, dk_all, dv_all, n_loc),
                                   rs_bytes),
}


def peer_sequential(rows, k_g, v_g, streams_per_peer):
    """K/V gather into head-major buffers peer by peer (rotation order rank+1,
    rank+2, ...): each peer's rows are pulled as ``streams_per_peer`` concurrent
    head-group copies, the next peer starts when they are done (the arrival
    pattern a row list sorted by owner would want, tools/fwd_order_sim.py)."""
    from paper_2503_11367_b200 import _lib
    nkv, d = k_g.shape[1], 128
    n = k_g.shape[0]
    mine = ex.kv[:2 * rows * nkv * d].view(2, nkv, rows, d)
    k_all = torch.empty((nkv, world * rows, d), dtype=k_g.dtype, device=dev)
    v_all = torch.empty_like(k_all)
    _lib.call("bam_kv_head_major", k_g.data_ptr(), v_g.data_ptr(), n, nkv, mine[0].data_ptr(),
              mine[1].data_ptr(), rows, 0, k_all.data_ptr(), v_all.data_ptr(), world * rows,
              rank * rows)
    ex.kv_h.barrier(channel=0)
    cur = torch.cuda.current_stream()
    while len(ex.streams) < streams_per_peer:
        ex.streams.append(torch.cuda.Stream(device=dev))
    per = nkv // streams_per_peer
    row_b = rows * d * 2
    prev = torch.cuda.Event()
    prev.record(cur)
    for step in range(1, world):
        r = (rank + step) % world
        src = ex.kv_h.get_buffer(r, (2, nkv, rows, d), torch.bfloat16, 0)
        done = []
        for i in range(streams_per_peer):
            st = ex.streams[i]
            st.wait_event(prev)
            with torch.cuda.stream(st):
                for t, dst in ((0, k_all), (1, v_all)):
                    _lib.call("bam_copy_2d", dst[i * per, r * rows:].data_ptr(), world * row_b,
                              src[t, i * per].data_ptr(), row_b, row_b, per)
            e = torch.cuda.Event()
            e.record(st)
            done.append(e)
        for e in done:
            cur.wait_event(e)
        prev = torch.cuda.Event()
        prev.record(cur)
    ex.kv_h.barrier(channel=0)
    return k_all, v_all


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

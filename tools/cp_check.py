#!/usr/bin/env python3
"""NCCL parity check of the context-parallel attention (autograd API).

    torchrun --nproc-per-node N --master-addr 127.0.0.1 tools/cp_check.py [--policy lpt]

Every rank runs cp_bitfield_attention forward + backward on its LPT-assigned
query blocks (K/V all-gather and dK/dV reduce-scatter over NCCL); rank 0
gathers the outputs and gradients and checks them against the fp32 CPU
oracle on the full sequence (bf16 tolerance: max-abs 2e-2, rel-L2 1e-2).
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2503_11367_b200 import cp, mask as M  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--policy", default="lpt")
ap.add_argument("--transport", default="nccl", choices=["nccl", "ce"])
ap.add_argument("--groups", type=int, default=1)
ap.add_argument("--heads", type=int, default=8)
ap.add_argument("--kv-heads", type=int, default=2)
args = ap.parse_args()
rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
local = int(os.environ.get("LOCAL_RANK", rank))
torch.cuda.set_device(local)
dev = torch.device("cuda", local)
dist.init_process_group("nccl", device_id=dev)

segs = [("text", 512), ("img0", 1024), ("text", 640), ("img1", 512), ("text", 1408)]
mask = M.build_bitfield(segs)
T, Hq, Hkv = len(mask), args.heads, args.kv_heads
plan = cp.make_cp_plan(mask, world, rank, args.policy)
lay = plan.layout
g = torch.Generator().manual_seed(1234)
q = torch.randn(T, Hq, 128, generator=g).to(torch.bfloat16)
k = torch.randn(T, Hkv, 128, generator=g).to(torch.bfloat16)
v = torch.randn(T, Hkv, 128, generator=g).to(torch.bfloat16)
do = torch.randn(T, Hq, 128, generator=g).to(torch.bfloat16)
q_loc, k_loc, v_loc, do_loc = cp.shard_rows(*(t.to(dev) for t in (q, k, v, do)), layout=lay)
q_loc.requires_grad_(True)
k_loc.requires_grad_(True)
v_loc.requires_grad_(True)
for _ in range(2):   # twice: the second step reuses the transport's buffers
    for t in (q_loc, k_loc, v_loc):
        t.grad = None
    o = cp.cp_bitfield_attention(q_loc, k_loc, v_loc, plan, groups=args.groups,
                                 transport=args.transport)
    o.backward(do_loc)
torch.cuda.synchronize()

# gather every rank's rows (padded to max_blocks) on rank 0
def gather(x):
    pad = cp.pad_rows(x.detach(), lay)
    out = [torch.empty_like(pad) for _ in range(world)] if rank == 0 else None
    dist.gather(pad, out, dst=0)
    return out

outs = {name: gather(t) for name, t in
        (("o", o), ("dq", q_loc.grad), ("dk", k_loc.grad), ("dv", v_loc.grad))}
blocks = [None] * world
for r in range(world):
    blocks[r] = cp.cp_layout(plan.assignment.owner, world, r).local_blocks.cpu().tolist()
if rank == 0:
    from oracle import attention_ref, mask_ref
    desc = np.asarray(mask.descriptors, np.int64)
    o_ref, lse_ref = attention_ref.attention_fwd(q, k, v, desc, np.arange(T))
    dq_ref, dk_ref, dv_ref = attention_ref.attention_bwd(q, k, v, o_ref, lse_ref, do, desc,
                                                         np.arange(T))
    refs = {"o": o_ref, "dq": dq_ref, "dk": dk_ref, "dv": dv_ref}
    report = {}
    for name, parts in outs.items():
        full = torch.empty_like(refs[name])
        for r in range(world):
            for i, b in enumerate(blocks[r]):
                full[b * 128:(b + 1) * 128] = parts[r][i * 128:(i + 1) * 128].float().cpu()
        ma = (full - refs[name]).abs().max().item()
        rl = ((full - refs[name]).norm() / refs[name].norm()).item()
        report[name] = {"max_abs": ma, "rel_l2": rl, "ok": ma <= 2e-2 and rl <= 1e-2}
    ok = all(x["ok"] for x in report.values())
    print(json.dumps({"world": world, "policy": args.policy, "transport": args.transport,
                      "groups": args.groups, "ok": ok,
                      "imbalance_predicted": plan.predicted_imbalance, **report}))
    dist.destroy_process_group()
    sys.exit(0 if ok else 1)
dist.destroy_process_group()

#!/usr/bin/env python3
"""Intra-GPU tail of the attention kernels (row f1 of SURVEY.md §8(f)): per-CTA
{start, end, SM} of the forward head-pair kernel and the backward kernel from a
-DBAM_CTA_CLOCK build (%globaltimer), and the bound they put on what a
persistent LPT work-queue kernel could gain over the hardware block scheduler
walking the same heavy-first item order.

    python tools/build_variant.py attn_fwd.cu,attn_bwd.cu libbam_clk.so -DBAM_CTA_CLOCK
    BAM_LIB_PATH=paper_2503_11367_b200/libbam_clk.so python tools/cta_tail.py --config 4 --world 1
    # real CP ranks (one process per GPU, the exchange included):
    BAM_LIB_PATH=... torchrun --nproc-per-node 4 --master-addr 127.0.0.1 tools/cta_tail.py --transport ce

Per kernel and (emulated) rank it reports:
  span_ms        first CTA start -> last CTA end
  busy_frac      sum of CTA durations / (SMs x span): the SM-time the kernel used
  lpt_gain_bound span / (sum of CTA durations / SMs) - 1: the most ANY reordering
                 of the same CTAs over the SMs could save (perfect balance, zero gaps)
  tail_ms        span - the time the first SM ran out of work
  gap_us         median gap between consecutive CTAs on one SM (block launch +
                 the CTA's own prologue before its first recorded instruction)
  flag_wait_frac (real CP ranks, copy-engine transport) SM-time the forward's TMA
                 warps spent waiting on K/V arrival flags / (SMs x span): an upper
                 bound on the exchange time the forward exposes (a wait shorter
                 than the two-tile K/V ring's lead costs nothing)
"""
import argparse
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2503_11367_b200 import _lib, attention as A, cp, mask as M  # noqa: E402
from paper_2503_11367_b200.workloads import CONFIGS, SWEEP_128K  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="4", help="BASELINE config id or a 128K sweep mask name")
ap.add_argument("--world", type=int, default=1, help="emulated CP ranks (1: the whole sequence)")
ap.add_argument("--policy", default="lpt")
ap.add_argument("--out", default="gpurun_out/cta_tail.jsonl")
ap.add_argument("--transport", default="ce", help="real CP ranks (torchrun): ce | nccl")
args = ap.parse_args()
REAL = int(os.environ.get("WORLD_SIZE", "1")) > 1
if REAL:
    local = int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    args.world = dist.get_world_size()
if args.config.isdigit():
    cfg = CONFIGS[int(args.config)]
else:
    cfg = {"segments": SWEEP_128K[args.config], "Hq": 32, "Hkv": 8}
lib = _lib.load()
mask = M.build_bitfield(cfg["segments"])
desc = mask.device_descriptors()
T, dev = desc.shape[0], torch.device("cuda", torch.cuda.current_device())
g = torch.Generator(device=dev).manual_seed(1234)
Hq, Hkv = cfg["Hq"], cfg["Hkv"]
q = torch.randn(T, Hq, 128, device=dev, generator=g, dtype=torch.bfloat16)
k = torch.randn(T, Hkv, 128, device=dev, generator=g, dtype=torch.bfloat16)
v = torch.randn(T, Hkv, 128, device=dev, generator=g, dtype=torch.bfloat16)
do = torch.randn(T, Hq, 128, device=dev, generator=g, dtype=torch.bfloat16)
nb = T // 128
CAP = 1 << 20
fbuf = torch.zeros(CAP * 8, dtype=torch.int64, device=dev)
bbuf = torch.zeros(CAP * 8, dtype=torch.int64, device=dev)


def analyse(buf, kernel, rank):
    r = buf.view(CAP, 8).cpu()
    r = r[r[:, 0] > 0]
    flag_wait = int(r[:, 4].sum())
    r = r[:, :4].tolist()
    if not r:
        return None
    t0 = min(x[0] for x in r)
    span = max(x[1] for x in r) - t0
    per_sm = {}
    for s, e, sm, w in r:
        per_sm.setdefault(sm, []).append((s, e, w))
    busy = sum(e - s for s, e, _ in (y for x in per_sm.values() for y in x))
    nsm = len(per_sm)
    gaps, overlap = [], 0
    for lst in per_sm.values():
        lst.sort()
        for a, b in zip(lst, lst[1:]):
            if b[0] < a[1]:
                overlap += 1
            gaps.append(b[0] - a[1])
    first_idle = min(max(e for _, e, _ in lst) for lst in per_sm.values()) - t0
    durs = sorted(e - s for s, e, _ in (y for x in per_sm.values() for y in x))
    return {"kernel": kernel, "config": args.config, "world": args.world, "rank": rank,
            "policy": args.policy, "ctas": len(r), "sms": nsm,
            "span_ms": span / 1e6, "busy_frac": busy / (nsm * span),
            "lpt_gain_bound": span / (busy / nsm) - 1.0,
            "tail_ms": (span - first_idle) / 1e6,
            "gap_us_median": statistics.median(gaps) / 1e3 if gaps else 0.0,
            "gap_us_mean": statistics.mean(gaps) / 1e3 if gaps else 0.0,
            "cta_ms_median": statistics.median(durs) / 1e6, "cta_ms_max": durs[-1] / 1e6,
            "overlapping_ctas_on_one_sm": overlap,
            "flag_wait_frac": flag_wait / (nsm * span),
            "mode": f"real CP ({args.transport})" if REAL else "emulated ranks"}


os.makedirs(os.path.dirname(args.out) or ".", exist_ok=True)


def record(run):
    """Warm up, then one recorded run(); returns this rank's analysis rows."""
    for it in range(3):
        if it == 2:
            fbuf.zero_()
            bbuf.zero_()
            torch.cuda.synchronize()
            _lib.check(lib.bam_set_cta_clock_buffer(fbuf.data_ptr(), bbuf.data_ptr()))
        run()
        torch.cuda.synchronize()
        if REAL:
            dist.barrier()
    _lib.check(lib.bam_set_cta_clock_buffer(0, 0))
    return [x for x in (analyse(fbuf, "fwd_split", r_id), analyse(bbuf, "bwd", r_id)) if x]


rows = []
if REAL:
    r_id = dist.get_rank()
    cpp = cp.make_cp_plan(desc, args.world, r_id, args.policy)
    ql, kl, vl, dol = cp.shard_rows(q, k, v, do, layout=cpp.layout)

    def run():
        o, lse, gathered = cp.cp_forward(ql, kl, vl, cpp, transport=args.transport)
        cp.cp_backward(ql, gathered, o, lse, dol, cpp, transport=args.transport)
    mine = record(run)
    allr = [None] * args.world
    dist.all_gather_object(allr, mine)
    if r_id == 0:
        rows = [x for lst in allr for x in lst]
    dist.destroy_process_group()
else:
    for r_id in range(args.world):
        if args.world == 1:
            plan = A.build_plan(desc)
            ql, dol, k_all, v_all = q, do, k, v
        else:
            cpp = cp.make_cp_plan(desc, args.world, r_id, args.policy)
            lay = cpp.layout
            plan = cpp.attn
            k_all = torch.zeros((args.world * lay.max_blocks * 128, Hkv, 128), dtype=k.dtype,
                                device=dev)
            v_all = torch.zeros_like(k_all)
            cp.permute_blocks([k, v], [k_all, v_all], lay.k_row[:nb], scatter=True)
            ql, dol = cp.shard_rows(q, do, layout=lay)

        def run():
            o, lse = A.attn_forward(ql, k_all, v_all, plan)
            A.BackwardWorkspace(ql, o, lse, dol, plan, None).main(k_all, v_all)
        rows += record(run)
if rows:
    with open(args.out, "a") as fh:
        for row in rows:
            print(json.dumps(row), flush=True)
            fh.write(json.dumps(row) + "\n")

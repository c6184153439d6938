#!/usr/bin/env python3
"""Benchmark: bitfield-masked attention fwd+bwd (CP over N GPUs) on B200.

Metric (BASELINE.json): masked-attn fwd+bwd TFLOP/s and % of dense BF16 peak
at CP = 1/2/4/8, with the per-rank load imbalance.  A step is one forward +
backward of the context-parallel attention over the whole sequence of the
workload (default: config 4, the 128K EMU-style interleaved multi-image mask,
GQA 32q/8kv, d=128), including the K/V all-gather and the dK/dV
reduce-scatter when N > 1.  The sequence is fixed as N grows ("strong").

Algorithmic FLOP per step = 14 * d * Hq * N_allowed (fwd 4, bwd 10; the
FlashAttention convention), N_allowed = exact count of mask.py:106-112 true
pairs (bam_count_allowed, no tile padding).  value = FLOP / max-over-ranks
step time (whole job); tflops_per_gpu = value / N.

Usage:  python bench.py [--gpus N] [--steps K] [--warmup W] [--config 4]
        torchrun --nproc-per-node N bench.py --gpus N ...
        python bench.py --impl reference ...    (the CPU path, see below)

--impl reference times the reference's CPU implementation of the path: the
reference itself is pure Python with no attention code, so the
arm runs the repo's CPU oracle port (oracle/: fp32 masked attention on all
host threads, plus the C restatement of block_workloads), on rank 0 only.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

D = 128
PEAKS_FALLBACK = {"bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0, "hbm_gbs": 6650.0}
METRIC = "masked-attn fwd+bwd TFLOP/s/GPU & %BF16 peak at CP=1/2/4/8; load imbalance"


def _claim_stdout():
    """Keep stdout for the one JSON line: native libraries (NCCL prints its
    version banner on rank 0) write to fd 1 directly, so fd 1 is pointed at
    stderr and the JSON goes to a private duplicate of the original stdout."""
    global _JSON_OUT
    sys.stdout.flush()
    _JSON_OUT = os.fdopen(os.dup(1), "w")
    os.dup2(2, 1)


_JSON_OUT = None


def emit(line):
    out = _JSON_OUT if _JSON_OUT is not None else sys.stdout
    out.write(json.dumps(line) + "\n")
    out.flush()


def load_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as fh:
            p = json.load(fh)
        return p, "measured (MEASURED_PEAKS.json)"
    except Exception:
        return PEAKS_FALLBACK, "fallback (B200_PROFILING.md)"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="bam", choices=["bam", "reference"])
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--policy", default="lpt", choices=["lpt", "zigzag", "contiguous"])
    ap.add_argument("--e2e-steps", type=int, default=None)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-sample-blocks", type=int, default=2)
    ap.add_argument("--transport", default="auto", choices=["auto", "nccl", "ce"],
                    help="CP exchange (N > 1): copy-engine pulls/pushes over symmetric memory "
                         "('ce'), NCCL collectives, or 'auto' = ce when every rank can map its "
                         "peers, else NCCL (agreed collectively)")
    ap.add_argument("--groups", type=int, default=1,
                    help="KV-head groups pipelining the CP collectives with compute (N > 1); "
                         "1 measured best at N=2/4 (profiles/r01/head_group_ablation.md)")
    return ap.parse_args()


# --------------------------------------------------------------------------- clocks
class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *exc):
        self.out = ""
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.out, _ = self.proc.communicate(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        rows = []
        for line in (self.out or "").strip().splitlines():
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                rows.append((float(parts[1]), float(parts[2]), parts[5:9]))
            except ValueError:
                continue
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for _, _, r in rows for i, v in enumerate(r) if v == "Active"})
        return {"sm_mhz": statistics.median(r[0] for r in rows), "sm_max_mhz": rows[0][1],
                "reasons": reasons, "samples": len(rows)}


# --------------------------------------------------------------------------- CPU arm
def cpu_attention_sample(segments, Hq, Hkv, blocks, seed=1234):
    """fp32 oracle fwd+bwd for `blocks` query blocks (all heads), each against
    the keys of its non-skip tiles only (blockwise-sparse, PAPER.md:616-619:
    skipped tiles are never computed, as on the GPU); returns (seconds,
    masked FLOP, sample description)."""
    import numpy as np
    import torch

    from oracle import attention_ref, mask_ref

    desc, _ = mask_ref.build_bitfield(segments)
    desc = np.asarray(desc, np.int64)
    T = desc.shape[0]
    classes, _ = mask_ref.block_workloads_c(desc, 128)
    g = torch.Generator().manual_seed(seed)
    k = torch.randn(T, Hkv, D, generator=g)
    v = torch.randn(T, Hkv, D, generator=g)
    rows = np.concatenate([np.arange(b * 128, (b + 1) * 128) for b in blocks])
    q = torch.randn(len(rows), Hq, D, generator=g)
    do = torch.randn(len(rows), Hq, D, generator=g)
    n_allowed = mask_ref.count_allowed_rows(desc, rows)
    keys = [np.concatenate([np.arange(kb * 128, (kb + 1) * 128)
                            for kb in np.nonzero(classes[b])[0]]) for b in blocks]
    t0 = time.perf_counter()
    for i, b in enumerate(blocks):
        sl = slice(i * 128, (i + 1) * 128)
        kp = torch.from_numpy(keys[i])
        ks, vs = k[kp], v[kp]
        o, lse = attention_ref.attention_fwd(q[sl], ks, vs, desc, rows[sl], k_pos=keys[i])
        attention_ref.attention_bwd(q[sl], ks, vs, o, lse, do[sl], desc, rows[sl], k_pos=keys[i])
    dt = time.perf_counter() - t0
    return dt, 14.0 * D * Hq * n_allowed, (f"{len(blocks)} query block(s) {list(blocks)} x {Hq} "
                                           f"heads vs the keys of their non-skip tiles")


def sample_blocks(nb, count, step=0):
    return [int((i + 0.5 + step * 0.37) * nb / count) % nb for i in range(count)]


def run_reference(args, cfg, rank, world):
    """--impl reference: the CPU path timed on the host cores (rank 0 only)."""
    import torch

    if rank != 0:
        return
    # torchrun sets OMP_NUM_THREADS=1 per rank; rank 0 alone works here, on every core
    torch.set_num_threads(max(1, len(os.sched_getaffinity(0))))
    threads = torch.get_num_threads()
    nb = sum(c for _, c in cfg["segments"]) // 128
    for w in range(args.warmup):
        cpu_attention_sample(cfg["segments"], cfg["Hq"], cfg["Hkv"], sample_blocks(nb, 1, w))
    planning = cpu_planning_sample(cfg["segments"], max(world, cfg["cp"]))
    times, flops = [], []
    for s in range(args.steps):
        dt, fl, sample = cpu_attention_sample(cfg["segments"], cfg["Hq"], cfg["Hkv"],
                                              sample_blocks(nb, 1, s + args.warmup))
        times.append(dt)
        flops.append(fl)
    value = sum(flops) / sum(times) / 1e12
    ms = 1e3 * sum(times) / len(times)
    line = {
        "metric": METRIC, "value": value, "unit": "TFLOP/s", "impl": "reference",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic",
        "config": {"workload": cfg["name"], "tokens": nb * 128, "Hq": cfg["Hq"],
                   "Hkv": cfg["Hkv"], "head_dim": D, "cp": world},
        "cpu_baseline": {"value": value, "unit": "TFLOP/s", "cores": threads, "kind": "port",
                         "sample": "per step: 1 query block x all heads vs the keys of its "
                                   "non-skip tiles, fp32 oracle fwd+bwd (oracle/attention_ref.py; "
                                   "the reference has no attention code)",
                         "planning": planning},
        "e2e": {"value": value, "unit": "TFLOP/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    emit(line)


# --------------------------------------------------------------------------- planning
def time_planning(M, CP, B, A, cfg, world, rank, policy, plan, reps=5):
    """The planning stage on the GPU (north-star subsystem 2): K1 block
    summaries + K2 tile classes / W (classify_device), K3 the block
    assignment, and the per-rank planner (bam_plan_build), each timed with
    CUDA events on the current stream (median of ``reps``); plus the
    wall-clock of the whole public call chain build_bitfield + make_cp_plan
    (its one host sync included)."""
    import torch

    mask = M.build_bitfield(cfg["segments"])
    desc = mask.device_descriptors()
    lay = plan.layout
    n_tiles = int(plan.assignment.loads[rank].item())
    ks = {"classify_us": [], "assign_us": [], "plan_build_us": [], "mask_plan_wall_ms": []}
    for _ in range(reps):
        e = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        torch.cuda.synchronize()
        e[0].record()
        classes, W = M.classify_device(desc, 128)
        e[1].record()
        asg = B.DISTRIBUTIONS[policy](W, world)
        e[2].record()
        A.native_plan(desc, classes, W, nq=lay.n_local, n_tiles=n_tiles, owner=asg.owner,
                      world=world, rank=rank, max_blocks=lay.max_blocks)
        e[3].record()
        torch.cuda.synchronize()
        ks["classify_us"].append(1e3 * e[0].elapsed_time(e[1]))
        ks["assign_us"].append(1e3 * e[1].elapsed_time(e[2]))
        ks["plan_build_us"].append(1e3 * e[2].elapsed_time(e[3]))
        t0 = time.perf_counter()
        CP.make_cp_plan(M.build_bitfield(cfg["segments"]), world, rank, policy)
        torch.cuda.synchronize()
        ks["mask_plan_wall_ms"].append(1e3 * (time.perf_counter() - t0))
    out = {k: statistics.median(v) for k, v in ks.items()}
    nb = desc.shape[0] // 128
    out.update({"blocks": nb, "tiles_classified": nb * nb,
                "what": "K1+K2 = bam_block_summarize + bam_classify (8*T B read, nb^2 + 4 nb B "
                        "written), K3 = the policy's assignment kernel(s), plan_build = "
                        "bam_plan_build; mask_plan_wall_ms = host wall of build_bitfield + "
                        "make_cp_plan incl. its one sync"})
    return out


def cpu_planning_sample(segments, G, rows=16):
    """The reference's planning algorithm on the CPU: block_workloads
    (mask.py:168-188 -- classify every (query block, key block) pair with the
    OR short-circuit then an exact element count) + lpt_distribute
    (balance.py:58-76), as restated in oracle/ (pure Python, one core,
    pinned to the reference's outputs by tests/golden).  Rows are
    independent, so ``rows`` evenly spaced query-block rows are classified and
    the time is scaled by nb / rows; LPT runs in full on the resulting W
    (the oracle's numpy W)."""
    import numpy as np

    from oracle import balance_ref, mask_ref

    desc, _ = mask_ref.build_bitfield(segments)
    T = len(desc)
    ranges = mask_ref.block_ranges(T, 128)
    nb = len(ranges)
    pick = sorted({int((i + 0.5) * nb / rows) for i in range(rows)})
    t0 = time.perf_counter()
    for b in pick:
        for kr in ranges:
            mask_ref.classify_pair(desc, ranges[b], kr)
    dt = time.perf_counter() - t0
    W = list(mask_ref.block_workloads_c(np.asarray(desc, np.int64), 128)[1])
    t1 = time.perf_counter()
    balance_ref.lpt(W, G)
    lpt_s = time.perf_counter() - t1
    return {"block_workloads_s_extrapolated": dt * nb / len(pick), "lpt_distribute_s": lpt_s,
            "cores": 1, "kind": "port",
            "sample": f"{len(pick)} of {nb} query-block rows classified (x{nb}/{len(pick)}); "
                      f"LPT over all {nb} blocks, G={G}",
            "reference_itself_measured_in_build_container": {
                "config1_4K_block_workloads_s": 2.37, "config2_32K_block_workloads_s": 172.4,
                "t2_extrapolated_128K_s": 172.4 * 16, "cores": 1,
                "source": "tests/golden/config{1,2}_workloads.json reference_seconds "
                          "(make_golden.py ran the reference's block_workloads)"}}


# --------------------------------------------------------------------------- GPU arm
def main():
    args = parse()
    _claim_stdout()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    from paper_2503_11367_b200.workloads import CONFIGS

    cfg = CONFIGS[args.config]
    if args.impl == "reference":
        return run_reference(args, cfg, rank, world)

    import torch
    import torch.distributed as dist

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)

    from paper_2503_11367_b200 import _lib, attention as A, balance as B, cp as CP, mask as M

    Hq, Hkv = cfg["Hq"], cfg["Hkv"]
    mask = M.build_bitfield(cfg["segments"])
    desc = mask.device_descriptors()
    T = desc.shape[0]
    n_allowed = M.count_allowed(desc)
    flop_step = 14.0 * D * Hq * n_allowed

    plan = CP.make_cp_plan(desc, world, rank, args.policy)
    layout = plan.layout
    loads = plan.assignment.loads.cpu().tolist()
    imb_pred = max(loads) / (sum(loads) / len(loads)) if sum(loads) else 1.0

    # synthetic inputs: same bytes on every rank (cuda generator, seed 1234, order Q K V dO)
    gen = torch.Generator(device=dev).manual_seed(1234)
    q = torch.randn(T, Hq, D, device=dev, generator=gen, dtype=torch.bfloat16)
    k = torch.randn(T, Hkv, D, device=dev, generator=gen, dtype=torch.bfloat16)
    v = torch.randn(T, Hkv, D, device=dev, generator=gen, dtype=torch.bfloat16)
    do = torch.randn(T, Hq, D, device=dev, generator=gen, dtype=torch.bfloat16)
    q_loc, k_loc, v_loc, do_loc = CP.shard_rows(q, k, v, do, layout=layout)  # one permute launch
    del q, k, v, do
    # local share of the algorithmic FLOP (for the per-kernel roofline)
    rows_allowed = None
    flop_local_fwd = 4.0 * D * Hq * n_allowed / world
    flop_local_bwd = 10.0 * D * Hq * n_allowed / world

    n_groups = args.groups if world > 1 else 1
    # transport agreed collectively ("auto": copy engines when peer memory maps on every
    # rank, else NCCL); at N=1 there is no exchange
    transport = CP.resolve_transport(args.transport, plan, Hkv, D, dev)

    def step(ev):
        """ev: [step start, fwd end, bwd end, fwd kernels start/end, bwd main start/end...]:
        the kernel-only pairs exclude the exchange barriers and waits"""
        ev[0].record()
        o, lse, gathered = CP.cp_forward(q_loc, k_loc, v_loc, plan, groups=n_groups,
                                         transport=transport, timer=(ev[3], ev[4]))
        ev[1].record()
        timers = [(ev[5 + 2 * i], ev[6 + 2 * i]) for i in range(len(gathered))]
        dq, dk, dv = CP.cp_backward(q_loc, gathered, o, lse, do_loc, plan, timers=timers,
                                    transport=transport)
        ev[2].record()
        return dq, dk, dv

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    mk = lambda: [torch.cuda.Event(enable_timing=True)  # noqa: E731
                  for _ in range(5 + 2 * n_groups)]
    for _ in range(args.warmup):
        step(mk())
    barrier()
    evs = [mk() for _ in range(args.steps)]
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    launches0 = _lib.launch_count
    with ClockSampler(local_rank) as clk:
        barrier()
        start.record()
        for s in range(args.steps):
            step(evs[s])
        end.record()
        barrier()
    launches = _lib.launch_count - launches0
    elapsed = start.elapsed_time(end)
    fwd_ms = sum(e[0].elapsed_time(e[1]) for e in evs) / args.steps
    bwd_ms = sum(e[1].elapsed_time(e[2]) for e in evs) / args.steps
    fwd_kernel_ms = sum(e[3].elapsed_time(e[4]) for e in evs) / args.steps
    bwd_main_ms = sum(e[5 + 2 * i].elapsed_time(e[6 + 2 * i])
                      for e in evs for i in range(n_groups)) / args.steps
    # per-rank kernel-only time: the forward kernels + the backward main kernel(s); the
    # step windows (fwd_ms + bwd_ms) end at exchange barriers, i.e. with the slowest rank
    kernel_ms = fwd_kernel_ms + bwd_main_ms
    t = torch.tensor([elapsed, kernel_ms, fwd_ms + bwd_ms], dtype=torch.float64, device=dev)
    per_rank_kernel_ms = [kernel_ms]
    if world > 1:
        tmax = t.clone()
        dist.all_reduce(tmax, op=dist.ReduceOp.MAX)
        tsum = t.clone()
        dist.all_reduce(tsum, op=dist.ReduceOp.SUM)
        allk = [torch.zeros(1, dtype=torch.float64, device=dev) for _ in range(world)]
        dist.all_gather(allk, t[1:2].clone())
        per_rank_kernel_ms = [x.item() for x in allk]
        elapsed_max = tmax[0].item()
        imb_meas = tmax[1].item() / (tsum[1].item() / world)
        imb_window = tmax[2].item() / (tsum[2].item() / world)
    else:
        elapsed_max = elapsed
        imb_meas = imb_window = 1.0
    ms_step = elapsed_max / args.steps
    value = flop_step / (ms_step * 1e-3) / 1e12

    # ---------------------------------------------------------------- e2e (public API, host buffers)
    # the input pipeline's fill / drain (first H2D, last D2H: ~27 ms each over PCIe at
    # config 4) is exposed once per run, so a run of 30 steps carries 1/30 of it
    e2e_steps = args.e2e_steps if args.e2e_steps is not None else max(30, args.steps)
    h_in = [t.cpu().pin_memory() for t in (q_loc, k_loc, v_loc, do_loc)]
    h_out = [torch.empty(t.shape, dtype=torch.bfloat16).pin_memory()
             for t in (q_loc, q_loc, k_loc, v_loc)]
    h2d = sum(t.numel() * t.element_size() for t in h_in)
    d2h = sum(t.numel() * t.element_size() for t in h_out)

    # A training loop's input pipeline: step s+1's H2D copies (copy stream) and step
    # s-1's D2H read-back (second copy stream) overlap step s's kernels; every
    # step's copies still happen inside the timed region.
    cur = torch.cuda.current_stream()
    s_in, s_out = torch.cuda.Stream(device=dev), torch.cuda.Stream(device=dev)
    dev_in = [[torch.empty(t.shape, dtype=t.dtype, device=dev) for t in h_in] for _ in range(2)]
    h_outs = [h_out, [torch.empty_like(t).pin_memory() for t in h_out]]
    # q/k/v land before dO (the forward starts while dO is still copying), and o
    # is read back while the backward runs.
    ev_in = [torch.cuda.Event() for _ in range(2)]       # q, k, v copied
    ev_do = [torch.cuda.Event() for _ in range(2)]       # dO copied
    ev_fwd = [torch.cuda.Event() for _ in range(2)]
    ev_free = [torch.cuda.Event() for _ in range(2)]

    def issue_h2d(s):
        b = s % 2
        with torch.cuda.stream(s_in):
            if s >= 2:
                s_in.wait_event(ev_free[b])   # step s-2 is done with this buffer
            for i, (d, h) in enumerate(zip(dev_in[b], h_in)):
                d.copy_(h, non_blocking=True)
                if i == 2:
                    ev_in[b].record(s_in)
            ev_do[b].record(s_in)

    plan_stream = torch.cuda.Stream(device=dev, priority=-1)   # high priority: planning
    # kernels interleave with the attention CTAs instead of queueing behind them

    def e2e_run(n, fresh_plan=False):
        """fresh_plan: every step uses a plan built from a freshly built mask
        (build_bitfield + make_cp_plan, as a training loop with a new mask per
        batch), prepared one step ahead on the planning stream while the
        previous step computes; all of it inside the timed region."""
        plans, ev_plan = [plan], [None]

        def prepare(s):
            with torch.cuda.stream(plan_stream):
                plans.append(CP.make_cp_plan(M.build_bitfield(cfg["segments"]), world, rank,
                                             args.policy))
                e = torch.cuda.Event()
                e.record(plan_stream)
                ev_plan.append(e)

        issue_h2d(0)
        if fresh_plan:
            prepare(0)
        for s in range(n):
            b = s % 2
            if s + 1 < n:
                issue_h2d(s + 1)
            cur.wait_event(ev_in[b])
            pl = plan
            if fresh_plan:
                cur.wait_event(ev_plan[s + 1])
                pl = plans[s + 1]
            qd, kd, vd = (t.detach().requires_grad_(True) for t in dev_in[b][:3])
            dod = dev_in[b][3]
            if world > 1:
                o = CP.cp_bitfield_attention(qd, kd, vd, pl, groups=n_groups,
                                             transport=transport)
            else:
                o = A.bitfield_attention(qd, kd, vd, pl.attn)
            ev_fwd[b].record(cur)
            with torch.cuda.stream(s_out):
                s_out.wait_event(ev_fwd[b])
                h_outs[b][0].copy_(o.detach(), non_blocking=True)
            cur.wait_event(ev_do[b])
            o.backward(dod)
            outs = (qd.grad, kd.grad, vd.grad)
            ev_free[b].record(cur)
            with torch.cuda.stream(s_out):
                s_out.wait_event(ev_free[b])
                for dst, src in zip(h_outs[b][1:], outs):
                    dst.copy_(src, non_blocking=True)
                    src.record_stream(s_out)
                o.record_stream(s_out)
            if fresh_plan and s + 1 < n:
                # the next batch's mask + plan, once this step's backward is queued: the
                # host's one sync (plan stream only) then overlaps the backward
                prepare(s + 1)
        cur.wait_stream(s_out)
        cur.wait_stream(plan_stream)

    def e2e_time(fresh_plan):
        e2e_run(1, fresh_plan)
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        e2e_run(e2e_steps, fresh_plan)
        e1.record()
        barrier()
        ms = e0.elapsed_time(e1) / e2e_steps
        if world > 1:
            tt = torch.tensor([ms], dtype=torch.float64, device=dev)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            ms = tt.item()
        return ms

    e2e_ms = e2e_time(False)
    e2e_fresh_ms = e2e_time(True)
    planning = time_planning(M, CP, B, A, cfg, world, rank, args.policy, plan)
    e2e_value = flop_step / (e2e_ms * 1e-3) / 1e12
    e2e_fresh_value = flop_step / (e2e_fresh_ms * 1e-3) / 1e12

    peaks, peak_src = load_peaks()
    traffic = None
    try:   # DRAM bytes per launch from the committed ncu --set full capture (N=1 only)
        with open(os.path.join(ROOT, "profiles", "r02", "traffic.json")) as fh:
            tr = json.load(fh).get(cfg["name"], {}).get("attn_bwd_kernel")
        if tr and world == tr["n_gpus"]:
            traffic = tr["dram_bytes_per_launch"]
    except Exception:
        traffic = None
    # the kernels are timed inside a long fwd+bwd step (K steps back to back), so the
    # denominator is the driver's sustained bf16 figure; the burst one is reported beside it
    peak_burst = peaks["bf16_tflops"]
    peak = peaks.get("bf16_tflops_sustained", peak_burst)
    peak_kind = "bf16_tflops_sustained" if "bf16_tflops_sustained" in peaks else "bf16_tflops"
    bwd_achieved = flop_local_bwd / (bwd_main_ms * 1e-3) / 1e12
    fwd_achieved = flop_local_fwd / (fwd_kernel_ms * 1e-3) / 1e12
    fwd_kernel = ("bam attn_fwd_split_kernel (GQA head pairs)" if (Hq // Hkv) % 2 == 0 else
                  "bam attn_fwd_split_kernel (MHA query-block pairs) + attn_fwd_kernel (rest)")

    cpu_baseline = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        import torch as _t
        nb = T // 128
        dt, fl, sample = cpu_attention_sample(cfg["segments"], Hq, Hkv,
                                              sample_blocks(nb, args.cpu_sample_blocks))
        cpu_baseline = {"value": fl / dt / 1e12, "unit": "TFLOP/s", "cores": _t.get_num_threads(),
                        "kind": "port", "sample": sample + " (fp32 oracle fwd+bwd, torch CPU, "
                                                           "blockwise-sparse)",
                        "seconds": dt,
                        "planning": cpu_planning_sample(cfg["segments"], max(world, cfg["cp"]))}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic",
            "config": {"workload": cfg["name"], "tokens": T, "Hq": Hq, "Hkv": Hkv, "head_dim": D,
                       "cp": world, "policy": args.policy, "n_allowed": n_allowed,
                       "kv_head_groups": n_groups,
                       "transport": transport if world > 1 else None,
                       "flop_per_step": flop_step,
                       "l2": "inputs larger than L2 (Q alone %.2f GiB per rank)" %
                             (q_loc.numel() * 2 / 2**30)},
            "tflops_per_gpu": value / world,
            "frac_of_peak": value / world / peak,
            "frac_of_burst_peak": value / world / peak_burst,
            "fwd_ms": fwd_ms, "bwd_ms": bwd_ms, "fwd_kernel_ms": fwd_kernel_ms,
            "bwd_main_ms": bwd_main_ms,
            "imbalance_predicted": imb_pred, "imbalance_measured": imb_meas,
            "imbalance_measured_basis": "max/mean over ranks of per-rank kernel-only time "
                                        "(forward kernels + backward main kernel, CUDA events "
                                        "around the launches; no exchange barrier inside)",
            "per_rank_kernel_ms": per_rank_kernel_ms,
            "imbalance_step_window": imb_window,
            "roofline": {"bound": "tensor", "kernel": "bam attn_bwd_kernel (tcgen05)",
                         "achieved": bwd_achieved, "peak": peak, "unit": "TFLOP/s",
                         "frac": bwd_achieved / peak, "traffic": traffic,
                         "traffic_unit": "DRAM bytes per launch (the committed ncu --set full capture, profiles/r02/traffic.json)",
                         "peak_source": peak_src + " " + peak_kind +
                         " (kernel timed inside a long step)",
                         "peak_burst": peak_burst, "frac_of_burst": bwd_achieved / peak_burst,
                         "fwd": {"kernel": fwd_kernel, "achieved": fwd_achieved,
                                 "frac": fwd_achieved / peak,
                                 "frac_of_burst": fwd_achieved / peak_burst}},
            "cpu_baseline": cpu_baseline,
            "e2e": {"value": e2e_value, "unit": "TFLOP/s", "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h, "ms_per_step": e2e_ms,
                    "api": "cp_bitfield_attention" if world > 1 else "bitfield_attention",
                    "steps": e2e_steps,
                    "copies": "pinned host buffers; H2D of step s+1 and D2H of step s on two "
                              "copy streams overlap step s's kernels (double-buffered); "
                              "the forward waits for q/k/v only, the backward for dO, and o "
                              "is read back during the backward",
                    "fresh_mask_plan_per_step": {
                        "value": e2e_fresh_value, "ms_per_step": e2e_fresh_ms,
                        "what": "every step runs on a plan from a freshly built mask "
                                "(build_bitfield + make_cp_plan), prepared one step ahead on a "
                                "high-priority planning stream while the previous step's "
                                "backward runs"}},
            "planning": planning,
            "gpu_launches": launches,
            "clocks": clk.summary(),
        }
        emit(line)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()

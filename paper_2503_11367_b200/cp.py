"""Context-parallel bitfield-masked attention (one process per GPU, NCCL).

The paper's runtime: query blocks are assigned to
CP ranks by the workload-balanced LPT policy (balance.py:58-76); every rank
all-gathers K/V (Llama-3 style all-gather CP, not ring attention) and runs
the masked attention for its own query blocks against all keys; the backward
reduce-scatters the dK/dV partials back to the key owners.

Layout on rank r (``cp_layout``):
  local blocks      the global block ids owned by r, ascending
  local q/k/v/o     [n_local*128, H, 128]   (rows of those blocks, in order)
  gathered k/v      [world*max_blocks*128, Hkv, 128], rank-major; rank g's
                    local block i sits at block-row g*max_blocks + i, so the
                    kernels read global block kb at ``k_row[kb]``
Ranks own different block counts (LPT balances work, not tokens), so every
rank's K/V shard is padded to ``max_blocks`` rows for the collectives.

Exchange steps (the only cross-rank traffic): ``gather_kv`` (all-gather of
K and V) and ``scatter_dkv`` (fp32 reduce-scatter of the dK/dV partials).
Both run per KV-head group on a side stream: the forward of group g starts
when its K/V land (overlapping the gather of group g+1); the reduce-scatter
of group g overlaps the backward kernel of group g+1.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import torch
import torch.distributed as dist

from . import _lib
from . import attention as A
from . import balance as B
from .mask import BitfieldMask, classify_device

BLOCK = A.BLOCK


@dataclass
class CPLayout:
    world: int
    rank: int
    owner: torch.Tensor        # int32 [nb] rank owning each global block
    local_blocks: torch.Tensor  # int32 [n_local] ascending global ids of this rank
    k_row: torch.Tensor        # int32 [nb] block-row of each global block in gathered K/V
    counts: list               # blocks per rank
    max_blocks: int

    @property
    def n_local(self) -> int:
        return int(self.local_blocks.shape[0])


def cp_layout(owner: torch.Tensor, world: int, rank: int) -> CPLayout:
    """Index plumbing from an owner vector (device or CPU tensor)."""
    owner = owner.to(torch.int64)
    nb = owner.shape[0]
    order = torch.sort(owner, stable=True).indices          # blocks grouped by rank, ascending id
    counts_t = torch.bincount(owner, minlength=world)
    counts = [int(c) for c in counts_t.cpu().tolist()]
    max_blocks = max(max(counts), 1)
    starts = torch.cumsum(counts_t, 0) - counts_t
    pos = torch.empty(nb, dtype=torch.int64, device=owner.device)
    pos[order] = torch.arange(nb, device=owner.device)
    pos_in_owner = pos - starts[owner]
    k_row = (owner * max_blocks + pos_in_owner).to(torch.int32)
    lo = sum(counts[:rank])
    local = order[lo:lo + counts[rank]].to(torch.int32)
    return CPLayout(world=world, rank=rank, owner=owner.to(torch.int32), local_blocks=local,
                    k_row=k_row, counts=counts, max_blocks=max_blocks)


def permute_blocks(srcs, dsts, idx: torch.Tensor, scatter: bool = False) -> None:
    """Token permutation with ``bam_permute_blocks``: for
    every (src, dst) pair, gather (dst block i = src block idx[i]) or scatter
    (dst block idx[i] = src block i) 128-row blocks, all tensors in one launch.
    Tensors are contiguous CUDA tensors whose rows are 16-byte multiples."""
    srcs, dsts = list(srcs), list(dsts)
    if not 1 <= len(srcs) == len(dsts) <= 4:
        raise ValueError("permute_blocks: 1..4 (src, dst) pairs")
    _lib.require_cuda()
    for t in srcs + dsts:
        if not (t.is_cuda and t.is_contiguous()):
            raise ValueError("permute_blocks: tensors must be contiguous CUDA tensors "
                             "(no CPU fallback)")
    idx = idx.to(device=srcs[0].device, dtype=torch.int32).contiguous()
    n = len(srcs)
    row_bytes = [t[0].numel() * t.element_size() if t.shape[0] else 16 for t in srcs]
    _lib.call("bam_permute_blocks", (ctypes.c_void_p * n)(*[t.data_ptr() for t in srcs]),
              (ctypes.c_void_p * n)(*[t.data_ptr() for t in dsts]),
              (ctypes.c_int64 * n)(*row_bytes), n, idx.data_ptr(), int(idx.numel()), BLOCK,
              int(scatter))


def shard_rows(*xs: torch.Tensor, layout: CPLayout = None):
    """Rows of this rank's blocks (in ``layout.local_blocks`` order) from
    full-sequence [T, ...] CUDA tensors: one fused gather launch for all of
    them.  ``shard_rows(x, layout)`` returns one tensor, ``shard_rows(q, k,
    v, layout=layout)`` a list."""
    if layout is None and xs and isinstance(xs[-1], CPLayout):
        xs, layout = xs[:-1], xs[-1]
    xs = [x.contiguous() for x in xs]
    outs = [torch.empty((layout.n_local * BLOCK,) + tuple(x.shape[1:]), dtype=x.dtype,
                        device=x.device) for x in xs]
    for i in range(0, len(xs), 4):
        permute_blocks(xs[i:i + 4], outs[i:i + 4], layout.local_blocks)
    return outs[0] if len(outs) == 1 else outs


def unshard_rows(y_loc: torch.Tensor, layout: CPLayout, out: torch.Tensor) -> torch.Tensor:
    """Inverse of ``shard_rows``: scatter this rank's rows back to their
    sequence positions in the full [T, ...] tensor ``out`` (other rows kept)."""
    permute_blocks([y_loc.contiguous()], [out], layout.local_blocks, scatter=True)
    return out


def pad_rows(x: torch.Tensor, layout: CPLayout) -> torch.Tensor:
    rows = layout.max_blocks * BLOCK
    if x.shape[0] == rows:
        return x.contiguous()
    out = torch.zeros((rows,) + tuple(x.shape[1:]), dtype=x.dtype, device=x.device)
    out[: x.shape[0]] = x
    return out


def gather_kv(k_loc: torch.Tensor, v_loc: torch.Tensor, layout: CPLayout, group=None):
    """All-gather the padded K/V shards -> gathered [world*max_blocks*128, Hkv, d]."""
    world = layout.world
    kp, vp = pad_rows(k_loc, layout), pad_rows(v_loc, layout)
    k_all = torch.empty((world * kp.shape[0],) + tuple(kp.shape[1:]), dtype=kp.dtype,
                        device=kp.device)
    v_all = torch.empty_like(k_all)
    dist.all_gather_into_tensor(k_all, kp, group=group)
    dist.all_gather_into_tensor(v_all, vp, group=group)
    return k_all, v_all


def scatter_dkv(dk_all: torch.Tensor, dv_all: torch.Tensor, layout: CPLayout, group=None):
    """Reduce-scatter the fp32 dK/dV partials to the key owners; returns this
    rank's [n_local*128, Hkv, d] fp32 gradients."""
    rows = layout.max_blocks * BLOCK
    dk = torch.empty((rows,) + tuple(dk_all.shape[1:]), dtype=dk_all.dtype, device=dk_all.device)
    dv = torch.empty_like(dk)
    dist.reduce_scatter_tensor(dk, dk_all, op=dist.ReduceOp.SUM, group=group)
    dist.reduce_scatter_tensor(dv, dv_all, op=dist.ReduceOp.SUM, group=group)
    n = layout.n_local * BLOCK
    return dk[:n], dv[:n]


@dataclass
class CPPlan:
    layout: CPLayout
    attn: A.AttentionPlan
    assignment: B.DeviceAssignment
    policy: str

    @property
    def predicted_imbalance(self) -> float:
        return self.assignment.to_host().imbalance


def make_cp_plan(mask_or_desc, world: int, rank: int, policy: str = "lpt") -> CPPlan:
    """Classify the mask (replicated, deterministic on every rank), assign
    query blocks with ``policy`` ("lpt" | "zigzag" | "contiguous") and build
    this rank's attention plan.  Every rank computes the identical plan, so
    no plan exchange is needed."""
    desc = (mask_or_desc.device_descriptors() if isinstance(mask_or_desc, BitfieldMask)
            else mask_or_desc)
    if desc.shape[0] % BLOCK:
        raise ValueError(f"CP attention needs T % {BLOCK} == 0")
    classes, W = classify_device(desc, BLOCK)
    asg = B.DISTRIBUTIONS[policy](W, world)
    layout = cp_layout(asg.owner, world, rank)
    attn = A.build_plan(desc, q_gid=layout.local_blocks, k_row=layout.k_row,
                        k_rows=world * layout.max_blocks, classes=classes, W=W)
    return CPPlan(layout=layout, attn=attn, assignment=asg, policy=policy)


_COMM_STREAMS: dict = {}


def _comm_stream(device) -> torch.cuda.Stream:
    s = _COMM_STREAMS.get(device)
    if s is None:
        s = _COMM_STREAMS[device] = torch.cuda.Stream(device=device)
    return s


def _head_groups(Hkv: int, groups: int):
    groups = max(1, min(groups, Hkv))
    while Hkv % groups:
        groups -= 1
    per = Hkv // groups
    return [(g * per, per) for g in range(groups)]


def cp_forward(q_loc, k_loc, v_loc, plan: CPPlan, group=None, scale=None, groups: int = 1):
    """All-gather K/V per KV-head group on a side stream; the forward of group
    g starts as soon as its K/V have landed, overlapping the gather of group
    g+1 (the paper overlaps communication per head).
    Returns (o, lse, [(k_all_g, v_all_g)])."""
    Hq, Hkv = q_loc.shape[1], k_loc.shape[1]
    grp = Hq // Hkv
    cur = torch.cuda.current_stream()
    comm = _comm_stream(q_loc.device)
    o = torch.empty_like(q_loc)
    lse = torch.empty(Hq, q_loc.shape[0], dtype=torch.float32, device=q_loc.device)
    gathered, events = [], []
    comm.wait_stream(cur)
    with torch.cuda.stream(comm):
        for kv0, nkv in _head_groups(Hkv, groups):
            kg = k_loc[:, kv0:kv0 + nkv].contiguous()
            vg = v_loc[:, kv0:kv0 + nkv].contiguous()
            k_all, v_all = gather_kv(kg, vg, plan.layout, group)
            ev = torch.cuda.Event()
            ev.record(comm)
            gathered.append((k_all, v_all))
            events.append(ev)
    for (kv0, nkv), (k_all, v_all), ev in zip(_head_groups(Hkv, groups), gathered, events):
        cur.wait_event(ev)
        k_all.record_stream(cur)
        v_all.record_stream(cur)
        A.attn_forward(q_loc, k_all, v_all, plan.attn, scale, h_begin=kv0 * grp, nh=nkv * grp,
                       out=(o, lse))
    return o, lse, gathered


def cp_backward(q_loc, gathered, o, lse, do, plan: CPPlan, group=None, scale=None,
                timers=None):
    """Per KV-head group: backward kernel -> fp32 dK/dV partials of every key,
    reduce-scattered on the side stream while the next group computes."""
    Hq = q_loc.shape[1]
    Hkv = sum(k.shape[1] for k, _ in gathered)
    grp = Hq // Hkv
    cur = torch.cuda.current_stream()
    comm = _comm_stream(q_loc.device)
    ws = A.BackwardWorkspace(q_loc, o, lse, do, plan.attn, scale)
    parts, kv0 = [], 0
    for i, (k_all, v_all) in enumerate(gathered):
        nkv = k_all.shape[1]
        dk_all, dv_all = ws.main(k_all, v_all, h_begin=kv0 * grp, nh=nkv * grp,
                                 timer=None if timers is None else timers[i])
        ev = torch.cuda.Event()
        ev.record(cur)
        with torch.cuda.stream(comm):
            comm.wait_event(ev)
            dk_all.record_stream(comm)
            dv_all.record_stream(comm)
            parts.append(scatter_dkv(dk_all, dv_all, plan.layout, group))
        kv0 += nkv
    dq = ws.finalize()
    cur.wait_stream(comm)
    dk = torch.cat([p[0] for p in parts], dim=1) if len(parts) > 1 else parts[0][0]
    dv = torch.cat([p[1] for p in parts], dim=1) if len(parts) > 1 else parts[0][1]
    return dq, A.to_bf16(dk.contiguous()), A.to_bf16(dv.contiguous())


class _CPAttention(torch.autograd.Function):
    @staticmethod
    def forward(ctx, q, k, v, plan, group, scale, groups):
        o, lse, gathered = cp_forward(q, k, v, plan, group, scale, groups)
        flat = [t for kv in gathered for t in kv]
        ctx.save_for_backward(q, o, lse, *flat)
        ctx.plan, ctx.group, ctx.scale = plan, group, scale
        return o

    @staticmethod
    def backward(ctx, do):
        q, o, lse, *flat = ctx.saved_tensors
        gathered = list(zip(flat[0::2], flat[1::2]))
        dq, dk, dv = cp_backward(q, gathered, o, lse, do.contiguous(), ctx.plan, ctx.group,
                                 ctx.scale)
        return dq, dk, dv, None, None, None, None


def cp_bitfield_attention(q_loc, k_loc, v_loc, plan: CPPlan, group=None, scale=None,
                          groups: int = 1):
    """Context-parallel bitfield attention with autograd.  Inputs are this
    rank's rows (``shard_rows``) of q/k/v; returns this rank's O rows.  K/V
    travel in ``groups`` KV-head groups so communication overlaps compute."""
    return _CPAttention.apply(q_loc, k_loc, v_loc, plan, group, scale, groups)

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
K and V are gathered on a side stream, V overlapping the K-only work.
"""

from __future__ import annotations

from dataclasses import dataclass

import torch
import torch.distributed as dist

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


def shard_rows(x: torch.Tensor, layout: CPLayout) -> torch.Tensor:
    """Rows of this rank's blocks from a full-sequence [T, H, d] tensor."""
    idx = (layout.local_blocks.to(torch.int64)[:, None] * BLOCK +
           torch.arange(BLOCK, device=layout.local_blocks.device)[None, :]).reshape(-1)
    return x.index_select(0, idx.to(x.device))


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


def cp_forward(q_loc, k_loc, v_loc, plan: CPPlan, group=None, scale=None):
    k_all, v_all = gather_kv(k_loc, v_loc, plan.layout, group)
    o, lse = A.attn_forward(q_loc, k_all, v_all, plan.attn, scale)
    return o, lse, k_all, v_all


def cp_backward(q_loc, k_all, v_all, o, lse, do, plan: CPPlan, group=None, scale=None):
    dq, dk_all, dv_all = A.attn_backward(q_loc, k_all, v_all, o, lse, do, plan.attn, scale,
                                         dkv_fp32=True)
    dk, dv = scatter_dkv(dk_all, dv_all, plan.layout, group)
    return dq, A.to_bf16(dk.contiguous()), A.to_bf16(dv.contiguous())


class _CPAttention(torch.autograd.Function):
    @staticmethod
    def forward(ctx, q, k, v, plan, group, scale):
        o, lse, k_all, v_all = cp_forward(q, k, v, plan, group, scale)
        ctx.save_for_backward(q, k_all, v_all, o, lse)
        ctx.plan, ctx.group, ctx.scale = plan, group, scale
        return o

    @staticmethod
    def backward(ctx, do):
        q, k_all, v_all, o, lse = ctx.saved_tensors
        dq, dk, dv = cp_backward(q, k_all, v_all, o, lse, do.contiguous(), ctx.plan, ctx.group,
                                 ctx.scale)
        return dq, dk, dv, None, None, None


def cp_bitfield_attention(q_loc, k_loc, v_loc, plan: CPPlan, group=None, scale=None):
    """Context-parallel bitfield attention with autograd.  Inputs are this
    rank's rows (``shard_rows``) of q/k/v; returns this rank's O rows."""
    return _CPAttention.apply(q_loc, k_loc, v_loc, plan, group, scale)

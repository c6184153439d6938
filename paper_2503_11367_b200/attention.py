"""Bitfield-masked attention forward/backward on B200 (libbam tcgen05 kernels).

The reference has no attention code; the semantics are the
mask predicate of mask.py:106-112 applied to scaled dot-product attention,
computed blockwise over non-skip 128x128 tiles.

Layouts (token-major, head_dim 128, bf16):
  q, o, do      [nq*128, Hq, 128]     the local query blocks, local order
  k, v          [k_rows*128, Hkv, 128] key/value blocks; global block kb sits
                                       at block-row ``k_row[kb]``
  lse           [Hq, nq*128] fp32 (natural log)
GQA: query head h reads KV head h // (Hq // Hkv).

``AttentionPlan`` carries everything derived from the mask and the block
assignment (classes, W, tile lists, processing orders); it is built once per
mask on the device and reused by forward and backward.
"""

from __future__ import annotations

import math
import os
from dataclasses import dataclass

import torch

from . import _lib
from .mask import BitfieldMask, classify_device

BLOCK = 128
HEAD_DIM = 128


@dataclass
class AttentionPlan:
    """Everything the kernels need for one rank (``bam_plan_build``); int32
    device views into one workspace.  Forward pair / item lists are sized by
    their upper bounds; ``counts`` (device) holds the real lengths, which the
    kernels read (``BamAttnFwdParams.dev_counts``)."""
    desc: torch.Tensor        # int64 [nb*128]
    nb: int
    classes: torch.Tensor     # uint8 [nb, nb]
    W: torch.Tensor           # int32 [nb]
    q_gid: torch.Tensor       # int32 [nq] global block of each local query block
    k_row: torch.Tensor       # int32 [nb] block-row of global block kb in k/v
    k_rows: int
    row_off: torch.Tensor     # int32 [nq+1]
    row_tiles: torch.Tensor   # int32 kb << 2 | class (this rank's key blocks first under CP)
    col_off: torch.Tensor     # int32 [nb+1]
    col_tiles: torch.Tensor   # int32 j << 2 | class
    fwd_order: torch.Tensor   # int32 [nq] heavy-first local query blocks
    bwd_order: torch.Tensor   # int32 [nb] heavy-first key blocks
    # backward CTA pairs (clusters of 2 sharing the Q/dO stream), bam_build_pair_lists
    slot_kb: torch.Tensor | None = None
    slot_off: torch.Tensor | None = None
    slot_tiles: torch.Tensor | None = None
    pair_shared: torch.Tensor | None = None
    # forward query-block pairs: shared pairs (fwd_pair_ids, counts[0] of them) and
    # whole-row items (j, 0, W, -1) for the blocks of the other pairs (counts[1])
    fwd_pair_ids: torch.Tensor | None = None
    fwd_slot_q: torch.Tensor | None = None
    fwd_slot_off: torch.Tensor | None = None
    fwd_slot_tiles: torch.Tensor | None = None
    fwd_rest_items: torch.Tensor | None = None
    counts: torch.Tensor | None = None
    # geometric work classes over fwd_order: the head-pair kernel's CTA order; over
    # fwd_pair_ids (shared pairs heavy-first): the query-block-pair kernel's
    fwd_classes: torch.Tensor | None = None
    fwd_pair_classes: torch.Tensor | None = None
    row_cnt: torch.Tensor | None = None
    col_cnt: torch.Tensor | None = None

    @property
    def nq(self) -> int:
        return int(self.q_gid.shape[0])


def _plan_sizes(nb: int, nq: int, n_tiles: int) -> dict:
    """int32 element counts of bam_plan_build's buffers (include/bam.h)."""
    P, F, t = (nb + 1) // 2, (nq + 1) // 2, max(n_tiles, 1)
    return {"k_row": nb, "q_gid": nq, "row_cnt": nq, "row_off": nq + 1, "row_tiles": t,
            "col_cnt": nb, "col_off": nb + 1, "col_tiles": t,
            "fwd_order": nq, "bwd_order": nb, "slot_kb": 2 * P, "slot_cnt": 2 * P,
            "slot_off": 2 * P + 1, "slot_tiles": 2 * t, "pair_shared": P, "fwd_slot_q": 2 * F,
            "fwd_slot_cnt": 2 * F, "fwd_slot_off": 2 * F + 1, "fwd_slot_tiles": 2 * t,
            "fwd_shared": F, "fwd_pair_ids": F, "fwd_rest_items": 4 * nq, "counts": 2,
            "fwd_classes": 17, "fwd_pair_w": F, "fwd_pair_classes": 17}


def native_plan(desc: torch.Tensor, classes: torch.Tensor, W: torch.Tensor, *, nq: int,
                n_tiles: int, owner: torch.Tensor | None = None, world: int = 1,
                rank: int = 0, max_blocks: int | None = None) -> AttentionPlan:
    """One ``bam_plan_build`` call on the current stream (no host sync): the
    gathered layout (k_row, this rank's q_gid), tile lists, heavy-first
    orders, backward CTA pairs and forward query-block pairs.  ``nq``,
    ``max_blocks`` and ``n_tiles`` (sum of W over the rank's blocks) size the
    buffers; under CP they come from the assignment's one D2H."""
    nb = classes.shape[0]
    max_blocks = nq if max_blocks is None else max_blocks
    sizes = _plan_sizes(nb, nq, n_tiles)
    pad = lambda n: -(-n // 64) * 64            # noqa: E731  256-B aligned views (int4 items)
    ws = torch.empty(sum(pad(n) for n in sizes.values()), dtype=torch.int32,
                     device=classes.device)
    views, off = {}, 0
    for name, n in sizes.items():
        views[name] = ws[off:off + n]
        off += pad(n)
    bp = _lib.BamPlan(classes.data_ptr(), owner.data_ptr() if owner is not None else None, nb,
                      nq, world, rank, max_blocks, 0,
                      *[views[name].data_ptr() for name in _lib.PLAN_BUFFERS])
    _lib.call("bam_plan_build", bp)
    return AttentionPlan(
        desc=desc, nb=nb, classes=classes, W=W, q_gid=views["q_gid"], k_row=views["k_row"],
        k_rows=world * max_blocks, row_off=views["row_off"], row_tiles=views["row_tiles"],
        col_off=views["col_off"], col_tiles=views["col_tiles"], fwd_order=views["fwd_order"],
        bwd_order=views["bwd_order"], slot_kb=views["slot_kb"], slot_off=views["slot_off"],
        slot_tiles=views["slot_tiles"], pair_shared=views["pair_shared"],
        fwd_pair_ids=views["fwd_pair_ids"], fwd_slot_q=views["fwd_slot_q"],
        fwd_slot_off=views["fwd_slot_off"], fwd_slot_tiles=views["fwd_slot_tiles"],
        fwd_rest_items=views["fwd_rest_items"].view(nq, 4), counts=views["counts"],
        fwd_classes=views["fwd_classes"], fwd_pair_classes=views["fwd_pair_classes"],
        row_cnt=views["row_cnt"], col_cnt=views["col_cnt"])


def build_plan(desc: torch.Tensor, classes: torch.Tensor | None = None,
               W: torch.Tensor | None = None) -> AttentionPlan:
    """Single-GPU plan: every query block against every key block (identity
    layout).  One host sync (the tile count that sizes the lists)."""
    _lib.require_cuda()
    T = desc.shape[0]
    if T % BLOCK:
        raise ValueError(f"attention needs T % {BLOCK} == 0 (T={T})")
    nb = T // BLOCK
    if classes is None:
        classes, W = classify_device(desc, BLOCK)
    n_tiles = int(W.sum().item())
    return native_plan(desc, classes, W, nq=nb, n_tiles=n_tiles)


def plan_for_mask(mask: BitfieldMask) -> AttentionPlan:
    return build_plan(mask.device_descriptors())


def _check_qkv(q, k, v, plan: AttentionPlan):
    for name, t in (("q", q), ("k", k), ("v", v)):
        if t.dtype != torch.bfloat16 or not t.is_cuda or not t.is_contiguous():
            raise ValueError(f"{name} must be a contiguous bf16 CUDA tensor")
        if t.dim() != 3 or t.shape[2] != HEAD_DIM:
            raise ValueError(f"{name} must be [tokens, heads, {HEAD_DIM}]")
    if q.shape[0] != plan.nq * BLOCK:
        raise ValueError(f"q has {q.shape[0]} rows, plan expects {plan.nq * BLOCK}")
    if k.shape != v.shape or k.shape[0] != plan.k_rows * BLOCK:
        raise ValueError(f"k/v must be [{plan.k_rows * BLOCK}, Hkv, {HEAD_DIM}]")
    if q.shape[1] % k.shape[1]:
        raise ValueError("Hq must be a multiple of Hkv")


def _check_kv_head_major(k, v, plan: AttentionPlan):
    """Head-major K/V [Hkv, k_rows*128, 128] (the copy-engine CP gather's layout)."""
    for name, t in (("k", k), ("v", v)):
        if t.dtype != torch.bfloat16 or not t.is_cuda or not t.is_contiguous():
            raise ValueError(f"{name} must be a contiguous bf16 CUDA tensor")
    if k.shape != v.shape or k.dim() != 3 or k.shape[1:] != (plan.k_rows * BLOCK, HEAD_DIM):
        raise ValueError(f"head-major k/v must be [Hkv, {plan.k_rows * BLOCK}, {HEAD_DIM}]")
    return k.shape[0]


def _check_group(Hq, Hkv, h_begin, nh):
    nh = nh or Hq
    if h_begin < 0 or h_begin + nh > Hq or nh % Hkv:
        raise ValueError(f"head group [{h_begin}, {h_begin + nh}) of Hq={Hq} over Hkv={Hkv}")
    return nh


@dataclass
class SplitSchedule:
    """Intra-GPU split-KV schedule (the paper's subblocks, PAPER.md:564-584;
    ref balance.py:217-265): every local query-block row is cut into pieces of
    at most ``subblock`` key tiles (``split_block``), the pieces are ordered
    longest first (LPT) and the GPU's block scheduler hands them to SMs as
    they free up; rows cut into >= 2 pieces are merged by the aggregation
    kernel (``bam_attn_fwd_combine``)."""
    subblock: int
    items: torch.Tensor       # int32 [n_items, 4]: (j, first tile, end tile, slot | -1)
    combine: torch.Tensor     # int32 [n_combine, 4]: (j, first slot, n pieces, 0)
    n_slots: int

    @property
    def n_items(self) -> int:
        return int(self.items.shape[0])


def build_split_schedule(plan: AttentionPlan, subblock: int) -> SplitSchedule:
    """All on the device: bam_split_count/fill cut the rows, bam_lpt_assign
    (one unit) orders the pieces by (-size, block, index)."""
    from .balance import lpt_device

    if subblock < 1:
        raise ValueError("subblock_size must be >= 1")
    dev = plan.row_off.device
    nq = plan.nq
    cnt = (plan.row_off[1:] - plan.row_off[:-1]).to(torch.int32).contiguous()
    pcnt = torch.empty(nq, dtype=torch.int32, device=dev)
    poff = torch.empty(nq + 1, dtype=torch.int32, device=dev)
    _lib.call("bam_split_count", cnt.data_ptr(), nq, subblock, pcnt.data_ptr(), poff.data_ptr())
    n_pieces = int(poff[-1].item())
    size = torch.empty(max(n_pieces, 1), dtype=torch.int32, device=dev)
    blk, idx = torch.empty_like(size), torch.empty_like(size)
    _lib.call("bam_split_fill", cnt.data_ptr(), nq, subblock, poff.data_ptr(), size.data_ptr(),
              blk.data_ptr(), idx.data_ptr())
    size, blk, idx = size[:n_pieces], blk[:n_pieces], idx[:n_pieces]
    split = pcnt[blk.long()] >= 2
    slot = torch.where(split, torch.cumsum(split.to(torch.int32), 0) - 1,
                       torch.full_like(size, -1)).to(torch.int32)
    t0 = idx * subblock
    rec = torch.stack([blk, t0, t0 + size, slot], dim=1).to(torch.int32)
    order = lpt_device(size.contiguous(), 1).flat.long()      # LPT: (-size, block, index)
    items = rec[order].contiguous()
    first = split & (idx == 0)
    comb = torch.stack([blk[first], slot[first], pcnt[blk[first].long()],
                        torch.zeros_like(blk[first])], dim=1).to(torch.int32).contiguous()
    return SplitSchedule(subblock=subblock, items=items, combine=comb,
                         n_slots=int(split.sum().item()))


def attn_forward(q, k, v, plan: AttentionPlan, scale: float | None = None, *,
                 h_begin: int = 0, nh: int = 0, out=None, schedule: SplitSchedule | None = None,
                 kv_ready=None, kv_head_major: bool = False, timer=None):
    """Returns (o bf16 [nq*128, Hq, 128], lse fp32 [Hq, nq*128]).

    ``timer=(start, end)``: CUDA events recorded right before the first and
    after the last kernel launch (kernel-only time).

    ``kv_head_major``: k/v are [Hkv, k_rows*128, 128] instead of token-major
    (then ``kv_ready`` flags are per (rank, group of ``flag_heads`` KV heads):
    ``flags[owner*Hkv + (hkv // flag_heads) * flag_heads]``).

    ``kv_ready=(flags, epoch, rank, rows_per_rank[, flag_heads])`` (context
    parallelism with the copy-engine exchange): k/v may still be arriving; the
    forward kernels wait per tile until the flag of its owner (block-row //
    rows_per_rank) is >= epoch for tiles of other ranks and start on this
    rank's own.

    Head groups (context-parallel pipelining): with ``nh`` > 0 only query
    heads [h_begin, h_begin+nh) are computed, against the ``k.shape[1]`` KV
    heads of ``k``/``v``; ``out=(o, lse)`` receives them in place."""
    Hq, Hkv = q.shape[1], k.shape[1]
    if kv_head_major:
        Hkv = _check_kv_head_major(k, v, plan)
        if q.dtype != torch.bfloat16 or not q.is_cuda or not q.is_contiguous():
            raise ValueError("q must be a contiguous bf16 CUDA tensor")
    elif nh or h_begin:
        for name, t in (("q", q), ("k", k), ("v", v)):
            if t.dtype != torch.bfloat16 or not t.is_cuda or not t.is_contiguous():
                raise ValueError(f"{name} must be a contiguous bf16 CUDA tensor")
    else:
        _check_qkv(q, k, v, plan)
    nh = _check_group(Hq, Hkv, h_begin, nh)
    scale = 1.0 / math.sqrt(HEAD_DIM) if scale is None else float(scale)
    if out is None:
        o = torch.empty_like(q)
        lse = torch.empty(Hq, q.shape[0], dtype=torch.float32, device=q.device)
    else:
        o, lse = out
    part_o = part_ml = None
    if schedule is not None and schedule.n_slots:
        part_o = torch.empty(schedule.n_slots, Hq, 128, 128, dtype=torch.float32, device=q.device)
        part_ml = torch.empty(schedule.n_slots, Hq, 128, 2, dtype=torch.float32, device=q.device)
    p = _lib.BamAttnFwdParams(
        q.data_ptr(), k.data_ptr(), v.data_ptr(), o.data_ptr(), lse.data_ptr(),
        plan.desc.data_ptr(), plan.q_gid.data_ptr(), plan.k_row.data_ptr(),
        plan.row_off.data_ptr(), plan.row_tiles.data_ptr(), plan.fwd_order.data_ptr(),
        plan.nq, plan.nb, plan.k_rows, Hq, Hkv, scale, h_begin, nh,
        schedule.items.data_ptr() if schedule is not None else None,
        part_o.data_ptr() if part_o is not None else None,
        part_ml.data_ptr() if part_ml is not None else None,
        schedule.n_items if schedule is not None else 0, 0)
    p.kv_head_major = int(kv_head_major)
    if plan.counts is not None and schedule is None:
        p.dev_counts = plan.counts.data_ptr()
    if (plan.fwd_classes is not None and schedule is None
            and os.environ.get("BAM_FWD_CLASS_ORDER", "1") != "0"):
        p.order_classes = plan.fwd_classes.data_ptr()
    if kv_ready is not None:
        # the head-pair, query-pair and one-head kernels honour the flags (not the
        # CTA-pair kernel, nor split-KV schedules)
        if schedule is not None:
            raise ValueError("kv_ready needs whole rows")
        flags, epoch, rank, rows_per_rank, *flag_heads = kv_ready
        if rows_per_rank < 1 or plan.k_rows // rows_per_rank > 64 or not 0 <= rank < 64:
            raise ValueError("kv_ready: rows_per_rank >= 1, at most 64 ranks")
        p.kv_ready, p.kv_epoch, p.kv_rank, p.kv_rows_per_rank = (flags.data_ptr(), int(epoch),
                                                                 int(rank), int(rows_per_rank))
        p.kv_flag_heads = int(flag_heads[0]) if flag_heads else 0
    if timer is not None:
        timer[0].record()
    _launch_fwd(p, plan, schedule, (nh // Hkv) % 2 == 0, kv_ready is not None)
    if timer is not None:
        timer[1].record()
    return o, lse


def _launch_fwd(p, plan: AttentionPlan, schedule, pair_heads: bool, flagged: bool):
    """Kernel choice.  GQA (an even number of query heads per KV head): the
    split-row head-pair kernel.  MHA: shared query-block pairs in the
    split-row kernel, the other blocks as whole-row items of the one-head
    kernel.  Split-KV schedules: the one-head kernel + the combine."""
    pairs = schedule is None and plan.fwd_pair_ids is not None
    if pairs and not pair_heads and (flagged or os.environ.get("BAM_FWD_QPAIRS", "1") != "0"):
        entry = "bam_attn_fwd_qpairs"
    elif pairs and pair_heads and not flagged and os.environ.get("BAM_FWD_2CTA", "0") == "1":
        # shared query-block pairs on CTA pairs (cta_group::2).  Opt-in: measured
        # 1084-1106 vs 1137-1143 TFLOP/s for the one-CTA head-pair kernel on config 4 --
        # the forward is bound by MUFU / softmax latency, not by the K/V operand traffic
        # the CTA pair halves (profiles/r01/fwd_2cta.md)
        entry = "bam_attn_fwd_2cta"
    else:
        _lib.call("bam_attn_fwd", p)
        if schedule is not None and schedule.combine.shape[0]:
            _lib.call("bam_attn_fwd_combine", p, schedule.combine.data_ptr(),
                      int(schedule.combine.shape[0]))
        return
    if p.order_classes and plan.fwd_pair_classes is not None:
        p.order_classes = plan.fwd_pair_classes.data_ptr()
    _lib.call(entry, p, plan.fwd_pair_ids.data_ptr(), int(plan.fwd_pair_ids.shape[0]),
              plan.fwd_slot_q.data_ptr(), plan.fwd_slot_off.data_ptr(),
              plan.fwd_slot_tiles.data_ptr())
    n_rest = int(plan.fwd_rest_items.shape[0])
    if n_rest:
        p.items, p.n_items = plan.fwd_rest_items.data_ptr(), n_rest
        _lib.call("bam_attn_fwd", p)


class BackwardWorkspace:
    """Per-call backward state: the (lse*log2e, D) pairs and the fp32 dQ
    accumulator shared by every head group's main kernel."""

    def __init__(self, q, o, lse, do, plan: AttentionPlan, scale):
        for name, t in (("o", o), ("do", do)):
            if t.shape != q.shape or t.dtype != torch.bfloat16 or not t.is_contiguous():
                raise ValueError(f"{name} must be a contiguous bf16 tensor shaped like q")
        self.q, self.o, self.lse, self.do, self.plan = q, o, lse, do, plan
        self.scale = 1.0 / math.sqrt(HEAD_DIM) if scale is None else float(scale)
        Hq, dev = q.shape[1], q.device
        self.delta = torch.empty(Hq, 2, q.shape[0], dtype=torch.float32, device=dev)
        self.dq_acc = torch.empty(Hq, q.shape[0], 128, dtype=torch.float32, device=dev)
        self.dq = torch.empty_like(q)
        # preprocess and finalize only touch q-shaped buffers: k/v pointers unused there
        self._call("bam_attn_bwd_preprocess", q, q, q, q, 0, 0, 1)

    def _pairs(self) -> bool:
        return self.plan.pair_shared is not None and os.environ.get("BAM_BWD_PAIRS", "1") != "0"

    def _params(self, k, v, dk, dv, h_begin, nh, Hkv, kv_head_major=False, dkv_peers=None,
                rows_per_owner=0, dkv_bf16=False):
        pl = self.plan
        pairs = self._pairs()
        col_off, col_tiles, order = ((pl.slot_off, pl.slot_tiles, pl.slot_kb) if pairs else
                                     (pl.col_off, pl.col_tiles, pl.bwd_order))
        return _lib.BamAttnBwdParams(
            self.q.data_ptr(), k.data_ptr(), v.data_ptr(), self.o.data_ptr(), self.do.data_ptr(),
            self.lse.data_ptr(), self.delta.data_ptr(), self.dq_acc.data_ptr(),
            self.dq.data_ptr(), dk.data_ptr() if dk is not None else None,
            dv.data_ptr() if dv is not None else None, pl.desc.data_ptr(),
            pl.q_gid.data_ptr(), pl.k_row.data_ptr(), col_off.data_ptr(),
            col_tiles.data_ptr(), order.data_ptr(), pl.nq, pl.nb, pl.k_rows,
            self.q.shape[1], Hkv, self.scale, h_begin, nh,
            pl.pair_shared.data_ptr() if pairs else None,
            int(pl.slot_kb.shape[0]) if pairs else 0, 0, int(kv_head_major), int(dkv_bf16),
            dkv_peers.data_ptr() if dkv_peers is not None else None, int(rows_per_owner), 0)

    def _call(self, name, k, v, dk, dv, h_begin, nh, Hkv, **kw):
        _lib.call(name, self._params(k, v, dk, dv, h_begin, nh, Hkv, **kw))

    def main(self, k, v, *, h_begin=0, nh=0, timer=None, kv_head_major=False, dkv_peers=None,
             rows_per_owner=0, bf16=False):
        """dK/dV fp32 partials of the head group, [k_rows*128, Hkv, 128]; dQ
        accumulates.  kv_head_major: k/v are [Hkv, k_rows*128, 128].
        dkv_peers (int64 device tensor of per-rank workspace-slot addresses)
        with rows_per_owner: the partials go straight to their owners (fused
        reduce-scatter); returns (None, None).  bf16: the kernel writes the
        complete bf16 gradients (one GPU, no partial sums follow)."""
        rows = self.plan.k_rows * BLOCK
        if kv_head_major:
            Hkv = _check_kv_head_major(k, v, self.plan)
        else:
            Hkv = k.shape[1]
            if k.shape != v.shape or k.shape[0] != rows or not k.is_contiguous():
                raise ValueError(f"k/v must be contiguous [{rows}, Hkv, 128]")
        nh = _check_group(self.q.shape[1], Hkv, h_begin, nh)
        if dkv_peers is not None:
            dk = dv = None
        else:
            dt = torch.bfloat16 if bf16 else torch.float32
            dk = torch.empty((rows, Hkv, HEAD_DIM), dtype=dt, device=k.device)
            dv = torch.empty((rows, Hkv, HEAD_DIM), dtype=dt, device=k.device)
        if timer is not None:
            timer[0].record()
        self._call("bam_attn_bwd_main", k, v, dk, dv, h_begin, nh, Hkv,
                   kv_head_major=kv_head_major, dkv_peers=dkv_peers,
                   rows_per_owner=rows_per_owner, dkv_bf16=bf16 and dkv_peers is None)
        if timer is not None:
            timer[1].record()
        return dk, dv

    def finalize(self):
        self._call("bam_attn_bwd_finalize", self.q, self.q, self.q, self.q, 0, 0, 1)
        return self.dq


def attn_backward(q, k, v, o, lse, do, plan: AttentionPlan, scale: float | None = None,
                  dkv_fp32: bool = False, timer=None):
    """Returns (dq bf16, dk, dv) with dk/dv fp32 [k_rows*128, Hkv, 128]
    partials when ``dkv_fp32`` (for a CP reduce-scatter), else bf16."""
    _check_qkv(q, k, v, plan)
    ws = BackwardWorkspace(q, o, lse, do, plan, scale)
    dk, dv = ws.main(k, v, timer=timer, bf16=not dkv_fp32)
    return ws.finalize(), dk, dv


def to_bf16(x: torch.Tensor) -> torch.Tensor:
    out = torch.empty(x.shape, dtype=torch.bfloat16, device=x.device)
    _lib.call("bam_f32_to_bf16", x.data_ptr(), out.data_ptr(), x.numel())
    return out


class _BitfieldAttention(torch.autograd.Function):
    @staticmethod
    def forward(ctx, q, k, v, plan, scale):
        o, lse = attn_forward(q, k, v, plan, scale)
        ctx.save_for_backward(q, k, v, o, lse)
        ctx.plan = plan
        ctx.scale = scale
        return o

    @staticmethod
    def backward(ctx, do):
        q, k, v, o, lse = ctx.saved_tensors
        dq, dk, dv = attn_backward(q, k, v, o, lse, do.contiguous(), ctx.plan, ctx.scale)
        return dq, dk, dv, None, None


PAD_BIT = 1 << 60   # descriptor of padding tokens (a modality bit no real token uses)


def padded_descriptors(desc: torch.Tensor) -> torch.Tensor:
    """Pad a descriptor array to a multiple of 128 tokens with PAD_BIT tokens.

    A pure-modality pad token attends only other pad tokens (mask.py:110-112)
    and no real token attends it: text needs a shared bit (text descriptors
    carry registered modality bits only) and modality tokens need equality.
    Needs bit 60 to be unused, i.e. at most 59 registered modalities."""
    T = desc.shape[0]
    pad = (-T) % BLOCK
    if pad == 0:
        return desc
    if bool(((desc & PAD_BIT) != 0).any()):
        raise ValueError("cannot pad a mask that uses modality bit 60 (60 modalities)")
    return torch.cat([desc, torch.full((pad,), PAD_BIT, dtype=desc.dtype, device=desc.device)])


def bitfield_attention(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor,
                       mask_or_plan, scale: float | None = None) -> torch.Tensor:
    """Single-GPU bitfield-masked attention with autograd.

    ``mask_or_plan``: a ``BitfieldMask`` (planned here) or an ``AttentionPlan``.
    Sequences that are not a multiple of 128 tokens are padded with tokens
    that nothing attends (``padded_descriptors``); the padding is sliced off."""
    if isinstance(mask_or_plan, AttentionPlan):
        return _BitfieldAttention.apply(q, k, v, mask_or_plan, scale)
    T = q.shape[0]
    pad = (-T) % BLOCK
    if pad == 0:
        return _BitfieldAttention.apply(q, k, v, plan_for_mask(mask_or_plan), scale)
    plan = build_plan(padded_descriptors(mask_or_plan.device_descriptors()))
    zq = q.new_zeros((pad,) + tuple(q.shape[1:]))
    zk = k.new_zeros((pad,) + tuple(k.shape[1:]))
    o = _BitfieldAttention.apply(torch.cat([q, zq]), torch.cat([k, zk]), torch.cat([v, zk]),
                                 plan, scale)
    return o[:T]

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
import os
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
    """Index plumbing from an owner vector (device or CPU tensor), with torch
    ops: the host-side statement of the layout that ``make_cp_plan`` builds
    on the device (``bam_plan_build``'s layout kernel; tests compare them).
    Used by the CPU (gloo) exchange tests and tools."""
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


_EXCHANGES: dict = {}


class SymmExchange:
    """Copy-engine K/V all-gather and dK/dV reduce-scatter over NVLink peer
    memory (torch symmetric memory, CUDA IPC).  Every rank's
    K/V shard lives in a symmetric buffer that the peers PULL with
    cudaMemcpyAsync, and the dK/dV partials are PUSHED into the owners'
    symmetric workspaces (or stored there by the backward kernel's epilogue),
    so the transfers run on the copy engines and take no SMs from the
    attention kernels (NCCL's kernels do).

    The symmetric buffers are sized for a CAPACITY of ``cap_rows`` padded
    rows per rank; every call takes the plan's own ``rows`` (its
    ``max_blocks * 128`` <= capacity) and packs the data densely for that
    shape, so plans of different shapes -- a new mask every batch changes
    the LPT block counts -- reuse one exchange (``CPPlan.exchange``)."""

    def __init__(self, cap_rows: int, hkv: int, d: int, world: int, rank: int, device,
                 group=None):
        import torch.distributed._symmetric_memory as symm_mem

        pg = group if group is not None else dist.group.WORLD
        self.world, self.rank, self.d, self.hkv = world, rank, d, hkv
        self.cap_rows = cap_rows
        self.kv = symm_mem.empty((2 * cap_rows * hkv * d,), dtype=torch.bfloat16, device=device)
        self.kv_h = symm_mem.rendezvous(self.kv, pg.group_name)
        self.ws = symm_mem.empty((world * 2 * cap_rows * hkv * d,), dtype=torch.float32,
                                 device=device)
        self.ws_h = symm_mem.rendezvous(self.ws, pg.group_name)
        # one stream per peer so the copies run on several copy engines at once
        self.streams = [torch.cuda.Stream(device=device) for _ in range(self.world)]
        self.flags, self.epoch = None, 0   # gather_overlapped's arrival flags
        self.head_chunks = int(os.environ.get("BAM_CP_HEAD_CHUNKS", "1"))   # pull streams
        self._cache = {}

    def _check(self, rows: int, kv0: int, nkv: int):
        if rows > self.cap_rows or kv0 + nkv > self.hkv:
            raise ValueError(f"exchange capacity {self.cap_rows} rows x {self.hkv} KV heads "
                             f"< plan {rows} rows, heads [{kv0}, {kv0 + nkv})")

    def _fan_out(self, copies):
        """Run copies[r]() on peer stream r, joined back into the current stream."""
        cur = torch.cuda.current_stream()
        while len(self.streams) < len(copies):
            self.streams.append(torch.cuda.Stream(device=cur.device))
        start = torch.cuda.Event()
        start.record(cur)
        done = []
        for r, fn in enumerate(copies):
            st = self.streams[r]
            st.wait_event(start)
            with torch.cuda.stream(st):
                fn()
            ev = torch.cuda.Event()
            ev.record(st)
            done.append(ev)
        for ev in done:
            cur.wait_event(ev)

    def gather_overlapped(self, rows: int, k_g: torch.Tensor, v_g: torch.Tensor,
                          head_chunks: int | None = None):
        """K/V all-gather that lets the attention start early, into HEAD-MAJOR
        buffers [nkv, world*rows, d]: this rank's rows go straight into the
        gathered buffers before the barrier (event ``ev_local``, one
        ``bam_kv_head_major`` launch); the peers' shards are then pulled PEER BY
        PEER in rotation order rank+1, rank+2, ... (the order of the forward's
        tile lists, bam_plan_build), on ``head_chunks`` copy streams that each
        own a group of KV heads: per (peer, group, K|V) one strided copy-engine
        copy (``bam_copy_2d``) followed by one stream-ordered flag store per
        (peer, group) ``flags[peer*nkv + h0] = epoch`` (bam_stream_write_i32, no
        SM; ``kv_flag_heads`` = the group size) that the forward kernel waits on
        per tile.  Every rank pulls from a different peer at a time; one stream
        and one flag per peer (the default) measured 581 GB/s per rank at N=4,
        two streams joined per peer 551 (per-head copies and flags from all
        peers at once: 300-367, tools/exchange_bw.py).
        ``ev_all``: every pull landed.
        Returns (k_all, v_all, ev_local, ev_all, (flags, epoch, heads per flag))."""
        nkv, d = k_g.shape[1], self.d
        self._check(rows, 0, nkv)
        chunks = max(1, min(nkv, head_chunks or self.head_chunks))
        while nkv % chunks:
            chunks -= 1
        n = k_g.shape[0]
        mine = self.kv[:2 * rows * nkv * d].view(2, nkv, rows, d)
        k_all = torch.empty((nkv, self.world * rows, d), dtype=k_g.dtype, device=k_g.device)
        v_all = torch.empty_like(k_all)
        # this rank's rows, head-major, into its symmetric buffer and its gathered slot
        kc, vc = k_g.contiguous(), v_g.contiguous()
        _lib.call("bam_kv_head_major", kc.data_ptr(), vc.data_ptr(), n, nkv,
                  mine[0].data_ptr(), mine[1].data_ptr(), rows, 0, k_all.data_ptr(),
                  v_all.data_ptr(), self.world * rows, self.rank * rows)
        self.kv_h.barrier(channel=0)          # every rank's slice is in place
        cur = torch.cuda.current_stream()
        ev_local = torch.cuda.Event()
        ev_local.record(cur)
        if self.flags is None or self.flags.numel() < self.world * nkv:
            self.flags = torch.zeros(self.world * nkv, dtype=torch.int32, device=k_g.device)
        self.epoch += 1
        epoch = self.epoch
        per = nkv // chunks
        row_b = rows * d * 2                   # one head's rows of one rank, bytes
        dpitch = self.world * row_b

        # peer by peer: the `chunks` streams pull one peer's head groups together and
        # join before the next peer (without the join they drift onto different peers)
        while len(self.streams) < chunks:
            self.streams.append(torch.cuda.Stream(device=cur.device))
        prev = torch.cuda.Event()
        prev.record(cur)
        for step in range(1, self.world):
            r = (self.rank + step) % self.world
            src = self.kv_h.get_buffer(r, (2, nkv, rows, d), torch.bfloat16, 0)
            done = []
            for g in range(chunks):
                st = self.streams[g]
                st.wait_event(prev)
                h0 = g * per
                with torch.cuda.stream(st):
                    for t, dst in ((0, k_all), (1, v_all)):
                        _lib.call("bam_copy_2d", dst[h0, r * rows:].data_ptr(), dpitch,
                                  src[t, h0].data_ptr(), row_b, row_b, per)
                    # one flag per (peer, head group): BamAttnFwdParams.kv_flag_heads = per
                    _lib.call("bam_stream_write_i32", self.flags[r * nkv + h0:].data_ptr(), epoch)
                e = torch.cuda.Event()
                e.record(st)
                done.append(e)
            if chunks == 1:
                prev = done[0]
            else:
                prev = torch.cuda.Event()
                for e in done:
                    self.streams[0].wait_event(e)
                prev.record(self.streams[0])
        cur.wait_event(prev)
        for t in (k_all, v_all):
            for st in self.streams[:chunks]:
                t.record_stream(st)
        ev_all = torch.cuda.Event()
        ev_all.record(cur)
        self.kv_h.barrier(channel=0)          # all pulls done before anyone rewrites
        return k_all, v_all, ev_local, ev_all, (self.flags, epoch, per)

    def gather(self, rows: int, kv0: int, k_g: torch.Tensor, v_g: torch.Tensor):
        """This rank's [n_local*128, nkv, d] K/V slice of the KV heads
        [kv0, kv0+nkv) -> gathered rank-major [world*rows, nkv, d] K and V
        (the NCCL layout)."""
        nkv, d = k_g.shape[1], self.d
        self._check(rows, kv0, nkv)
        off = 2 * rows * kv0 * d
        mine = self.kv[off:off + 2 * rows * nkv * d].view(2, rows, nkv, d)
        mine[0, :k_g.shape[0]].copy_(k_g)
        mine[1, :v_g.shape[0]].copy_(v_g)
        k_all = torch.empty((self.world * rows, nkv, d), dtype=k_g.dtype, device=k_g.device)
        v_all = torch.empty_like(k_all)
        self.kv_h.barrier(channel=0)          # every rank's slice is in place

        def pull(r):
            def fn():
                src = self.kv_h.get_buffer(r, (2, rows, nkv, d), torch.bfloat16, off)
                k_all[r * rows:(r + 1) * rows].copy_(src[0])
                v_all[r * rows:(r + 1) * rows].copy_(src[1])
            return fn
        self._fan_out([pull((self.rank + step) % self.world) for step in range(self.world)])
        for t in (k_all, v_all):
            for st in self.streams:
                t.record_stream(st)
        self.kv_h.barrier(channel=0)          # all pulls done before anyone rewrites
        return k_all, v_all

    def peer_slots(self, rows: int, nkv: int) -> torch.Tensor:
        """int64 device tensor: for every rank r, the UVA address of THIS rank's
        slot [2][nkv][rows][d] fp32 in rank r's workspace, which the backward
        kernel's epilogue stores into directly (dkv_peers)."""
        self._check(rows, 0, nkv)
        key = ("slots", rows, nkv)
        t = self._cache.get(key)
        if t is None:
            per = rows * nkv * self.d
            base = self.rank * 2 * per
            ptrs = [self.ws_h.get_buffer(r, (2 * per,), torch.float32, base).data_ptr()
                    for r in range(self.world)]
            t = self._cache[key] = torch.tensor(ptrs, dtype=torch.int64, device=self.ws.device)
        return t

    def reduce_direct(self, rows: int, nkv: int, n_local: int):
        """Tail of the fused reduce-scatter: once every rank's backward kernel has
        stored its partials into the owners' workspaces (barrier), sum them into
        this rank's bf16 dK/dV."""
        per = rows * nkv * self.d
        self.ws_h.barrier(channel=0)          # every rank's kernel has finished its stores
        out = self._reduce(0, n_local, nkv, part=2 * per, comp=per, head=rows * self.d,
                           row=self.d)
        self.ws_h.barrier(channel=0)          # summed before the next kernel stores
        return out

    def _reduce(self, base, n_local, nkv, *, part, comp, head, row):
        """bf16 [n_local, nkv, d] dK and dV = sum of the world partials in the
        workspace (one bam_reduce_partials_bf16 launch)."""
        dk = torch.empty((n_local, nkv, self.d), dtype=torch.bfloat16, device=self.ws.device)
        dv = torch.empty_like(dk)
        src = self.ws[base:base + self.world * part]
        _lib.call("bam_reduce_partials_bf16", src.data_ptr(), self.world, part, comp, head, row,
                  nkv, n_local, dk.data_ptr(), dv.data_ptr())
        return dk, dv

    def reduce_scatter(self, rows: int, kv0: int, dk_all: torch.Tensor, dv_all: torch.Tensor,
                       n_local: int):
        """fp32 partials [world*rows, nkv, d] of every key (KV heads
        [kv0, kv0+nkv)) -> this rank's summed [n_local*128, nkv, d] dK and dV."""
        nkv, d = dk_all.shape[1], self.d
        self._check(rows, kv0, nkv)
        per = rows * nkv * d
        base = self.world * 2 * rows * kv0 * d

        def push(r):
            def fn():
                dst = self.ws_h.get_buffer(r, (2, rows, nkv, d), torch.float32,
                                           base + self.rank * 2 * per)
                dst[0].copy_(dk_all[r * rows:(r + 1) * rows])
                dst[1].copy_(dv_all[r * rows:(r + 1) * rows])
            return fn
        self._fan_out([push((self.rank + step) % self.world) for step in range(self.world)])
        for t in (dk_all, dv_all):
            for st in self.streams:
                t.record_stream(st)
        self.ws_h.barrier(channel=0)          # every rank's partials have landed
        out = self._reduce(base, n_local, nkv, part=2 * per, comp=per, head=d, row=nkv * d)
        self.ws_h.barrier(channel=0)          # summed before the next pushes
        return out


def exchange_capacity(rows: int, nb: int, world: int) -> int:
    """Padded rows per rank the exchange is allocated for: the plan's rows
    plus 1/8 headroom, rounded up to 1024 tokens and capped at the whole
    sequence, so the block counts of later masks (LPT moves a few blocks
    between ranks) fit without a new rendezvous."""
    cap = -(-(rows + rows // 8) // 1024) * 1024
    return max(rows, min(cap, -(-nb * BLOCK // 1024) * 1024))


@dataclass
class CPPlan:
    layout: CPLayout
    attn: A.AttentionPlan
    assignment: B.DeviceAssignment
    policy: str

    def exchange(self, hkv: int, d: int, device, group=None) -> SymmExchange:
        """The copy-engine transport for this plan.  One exchange per (world,
        rank, KV heads, d, device, group), allocated with headroom
        (``exchange_capacity``) and reused by every later plan that fits, so
        a new mask every batch does not rendezvous again; a plan that does
        not fit replaces it (the old buffers are released after a device
        sync and a barrier).  Every rank computes the identical plan, so all
        ranks take the same branch (creating one is a collective)."""
        lay = self.layout
        rows = lay.max_blocks * BLOCK
        key = (lay.world, lay.rank, hkv, d, str(device), id(group))
        ex = _EXCHANGES.get(key)
        if ex is None or ex.cap_rows < rows:
            if ex is not None:
                torch.cuda.synchronize(device)
                ex.kv_h.barrier(channel=0)
                del _EXCHANGES[key]
                del ex
            cap = exchange_capacity(rows, self.attn.nb, lay.world)
            ex = _EXCHANGES[key] = SymmExchange(cap, hkv, d, lay.world, lay.rank, device, group)
        return ex

    @property
    def predicted_imbalance(self) -> float:
        return self.assignment.to_host().imbalance


def make_cp_plan(mask_or_desc, world: int, rank: int, policy: str = "lpt") -> CPPlan:
    """Classify the mask (replicated, deterministic on every rank), assign
    query blocks with ``policy`` ("lpt" | "zigzag" | "contiguous") and build
    this rank's attention plan (``bam_plan_build``).  Every rank computes the
    identical plan, so no plan exchange is needed.

    All on the current stream with ONE host synchronisation: the D2H of the
    assignment's per-rank offsets and loads, which give the shapes (this
    rank's block count, the padded rank stride, the tile-list length).  Run it
    on a side stream to build the next batch's plan under this batch's
    attention."""
    desc = (mask_or_desc.device_descriptors() if isinstance(mask_or_desc, BitfieldMask)
            else mask_or_desc)
    if desc.shape[0] % BLOCK:
        raise ValueError(f"CP attention needs T % {BLOCK} == 0")
    classes, W = classify_device(desc, BLOCK)
    asg = B.DISTRIBUTIONS[policy](W, world)
    host = torch.cat([asg.off.to(torch.int64), asg.loads]).cpu().tolist()   # the one sync
    off, loads = host[:world + 1], host[world + 1:]
    counts = [off[g + 1] - off[g] for g in range(world)]
    if counts[rank] == 0:
        raise ValueError(f"rank {rank} owns no query block ({len(W)} blocks over {world} ranks)")
    max_blocks = max(counts)
    attn = A.native_plan(desc, classes, W, nq=counts[rank], n_tiles=loads[rank],
                         owner=asg.owner, world=world, rank=rank, max_blocks=max_blocks)
    layout = CPLayout(world=world, rank=rank, owner=asg.owner, local_blocks=attn.q_gid,
                      k_row=attn.k_row, counts=counts, max_blocks=max_blocks)
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


TRANSPORTS = ("auto", "nccl", "ce")
_TRANSPORT_CHOICE: dict = {}


def resolve_transport(transport: str, plan: "CPPlan", hkv: int, d: int, device,
                      group=None) -> str:
    """"auto" (the default) -> "ce" when the symmetric-memory exchange can be
    built on every rank, else "nccl".  The outcome is agreed collectively
    (MIN over ranks of a success flag on the process group), so the ranks
    never run different transports; it is decided once per group.  "auto"
    at world 1 needs no exchange ("local"); a forced "nccl" / "ce" runs the
    exchange even then (a one-rank process group)."""
    if transport not in TRANSPORTS and transport != "local":
        raise ValueError(f"transport must be one of {TRANSPORTS}")
    if transport != "auto":
        return transport
    if plan.layout.world == 1:
        return "local"
    key = (id(group), str(device))
    choice = _TRANSPORT_CHOICE.get(key)
    if choice is None:
        ok = 1
        try:
            plan.exchange(hkv, d, device, group)
        except Exception:   # noqa: BLE001  (no peer mapping / symmetric memory on this box)
            ok = 0
        flag = torch.tensor([ok], dtype=torch.int32, device=device)
        dist.all_reduce(flag, op=dist.ReduceOp.MIN, group=group)
        choice = _TRANSPORT_CHOICE[key] = "ce" if int(flag.item()) == 1 else "nccl"
    return choice


def cp_forward(q_loc, k_loc, v_loc, plan: CPPlan, group=None, scale=None, groups: int = 1,
               transport: str = "auto", timer=None):
    """K/V all-gather + the rank's attention forward.

    transport "ce" (what "auto" picks when peer memory works): copy-engine
    pulls from symmetric memory; with one head group the forward (GQA head
    pairs, or MHA query-block pairs + whole rows) starts on this rank's own key
    tiles at once and waits per tile on per-(rank, KV head) arrival flags for
    the rest (no SM is spent on the transfer, so the spin cannot starve it).
    Otherwise (``groups`` > 1 or "nccl") K/V travel per KV-head group on a side
    stream and the forward of group g starts when its K/V have landed,
    overlapping the gather of group g+1.

    ``timer=(start, end)`` CUDA events recorded right around the forward
    kernel launches (kernel-only time, no exchange barrier inside).
    Returns (o, lse, [(k_all_g, v_all_g)]); the overlapped path's single
    group is head-major [Hkv, rows, d] (``_kv_head_major`` tells them apart)."""
    Hq, Hkv = q_loc.shape[1], k_loc.shape[1]
    grp = Hq // Hkv
    d = k_loc.shape[2]
    transport = resolve_transport(transport, plan, Hkv, d, k_loc.device, group)
    o = torch.empty_like(q_loc)
    lse = torch.empty(Hq, q_loc.shape[0], dtype=torch.float32, device=q_loc.device)
    if transport == "local":
        A.attn_forward(q_loc, k_loc, v_loc, plan.attn, scale, out=(o, lse), timer=timer)
        return o, lse, [(k_loc, v_loc)]
    cur = torch.cuda.current_stream()
    comm = _comm_stream(q_loc.device)
    rows = plan.layout.max_blocks * BLOCK
    gathered, events = [], []
    hg = _head_groups(Hkv, groups)
    ex = plan.exchange(Hkv, d, k_loc.device, group) if transport == "ce" else None
    if ex is not None and len(hg) == 1:
        # the forward starts on this rank's key tiles while the copy engines pull the
        # peers' K/V: every tile list (CSR rows and, for MHA, the query-block pairs'
        # union lists) holds this rank's key blocks first, then each peer's in the
        # order the pulls land
        comm.wait_stream(cur)
        with torch.cuda.stream(comm):
            k_all, v_all, ev_local, ev_all, (flags, epoch, flag_heads) = ex.gather_overlapped(
                rows, k_loc, v_loc)
        cur.wait_event(ev_local)
        k_all.record_stream(cur)
        v_all.record_stream(cur)
        A.attn_forward(q_loc, k_all, v_all, plan.attn, scale, out=(o, lse),
                       kv_ready=(flags, epoch, plan.layout.rank, plan.layout.max_blocks,
                                 flag_heads),
                       kv_head_major=True, timer=timer)
        cur.wait_event(ev_all)
        return o, lse, [(k_all, v_all)]
    comm.wait_stream(cur)
    with torch.cuda.stream(comm):
        for kv0, nkv in hg:
            if ex is not None:
                k_all, v_all = ex.gather(rows, kv0, k_loc[:, kv0:kv0 + nkv],
                                         v_loc[:, kv0:kv0 + nkv])
            else:
                kg = k_loc[:, kv0:kv0 + nkv].contiguous()
                vg = v_loc[:, kv0:kv0 + nkv].contiguous()
                k_all, v_all = gather_kv(kg, vg, plan.layout, group)
            ev = torch.cuda.Event()
            ev.record(comm)
            gathered.append((k_all, v_all))
            events.append(ev)
    for i, ((kv0, nkv), (k_all, v_all), ev) in enumerate(zip(hg, gathered, events)):
        cur.wait_event(ev)
        k_all.record_stream(cur)
        v_all.record_stream(cur)
        if timer is not None and i == 0:
            timer[0].record()
        A.attn_forward(q_loc, k_all, v_all, plan.attn, scale, h_begin=kv0 * grp, nh=nkv * grp,
                       out=(o, lse))
    if timer is not None:
        timer[1].record()
    return o, lse, gathered


def _kv_head_major(k_all, plan: CPPlan) -> bool:
    """Gathered K/V are token-major [k_rows*128, nkv, d] or head-major
    [nkv, k_rows*128, d]; nkv < 128 <= k_rows*128 tells them apart."""
    return k_all.shape[0] != plan.attn.k_rows * BLOCK


def cp_backward(q_loc, gathered, o, lse, do, plan: CPPlan, group=None, scale=None,
                timers=None, transport: str = "auto"):
    """The rank's backward: dQ of its query rows and the fp32 dK/dV partials
    of every key, reduce-scattered to the key owners.

    "ce" with one head group: the reduce-scatter is fused into the backward
    kernel's epilogue (each CTA stores its partial rows straight into the
    owner's symmetric workspace), then one barrier and a local sum.
    Otherwise, per KV-head group: backward kernel, then the reduce-scatter of
    that group on the side stream while the next group computes.
    ``timers[i] = (start, end)``: events around head group i's main kernel."""
    Hq = q_loc.shape[1]
    kvh = [_kv_head_major(k, plan) for k, _ in gathered]
    if any(kvh) and len(gathered) != 1:
        raise ValueError("head-major gathered K/V come as one head group")
    Hkv = sum(k.shape[0] if h else k.shape[1] for (k, _), h in zip(gathered, kvh))
    grp = Hq // Hkv
    d = q_loc.shape[2]
    transport = resolve_transport(transport, plan, Hkv, d, q_loc.device, group)
    ws = A.BackwardWorkspace(q_loc, o, lse, do, plan.attn, scale)
    if transport == "local":
        k_all, v_all = gathered[0]
        dk, dv = ws.main(k_all, v_all, timer=None if timers is None else timers[0], bf16=True)
        return ws.finalize(), dk, dv
    cur = torch.cuda.current_stream()
    comm = _comm_stream(q_loc.device)
    rows = plan.layout.max_blocks * BLOCK
    n_loc_rows = plan.layout.n_local * BLOCK
    ex = plan.exchange(Hkv, d, q_loc.device, group) if transport == "ce" else None
    if kvh[0] and ex is None:
        raise ValueError("head-major gathered K/V need the copy-engine transport")
    if ex is not None and len(gathered) == 1:
        k_all, v_all = gathered[0]
        ws.main(k_all, v_all, kv_head_major=kvh[0], dkv_peers=ex.peer_slots(rows, Hkv),
                rows_per_owner=rows, timer=None if timers is None else timers[0])
        done = torch.cuda.Event()
        done.record(cur)
        with torch.cuda.stream(comm):
            comm.wait_event(done)
            dk, dv = ex.reduce_direct(rows, Hkv, n_loc_rows)
        dq = ws.finalize()
        cur.wait_stream(comm)
        dk.record_stream(cur)          # allocated on the comm stream
        dv.record_stream(cur)
        return dq, dk, dv
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
            parts.append(ex.reduce_scatter(rows, kv0, dk_all, dv_all, n_loc_rows)
                         if ex is not None else
                         scatter_dkv(dk_all, dv_all, plan.layout, group))
        kv0 += nkv
    dq = ws.finalize()
    cur.wait_stream(comm)
    for t in (t for pr in parts for t in pr):
        t.record_stream(cur)           # allocated on the comm stream
    dk = torch.cat([p[0] for p in parts], dim=1) if len(parts) > 1 else parts[0][0]
    dv = torch.cat([p[1] for p in parts], dim=1) if len(parts) > 1 else parts[0][1]
    if dk.dtype != torch.bfloat16:   # NCCL reduce-scatter: fp32 sums
        dk, dv = A.to_bf16(dk.contiguous()), A.to_bf16(dv.contiguous())
    return dq, dk, dv


class _CPAttention(torch.autograd.Function):
    @staticmethod
    def forward(ctx, q, k, v, plan, group, scale, groups, transport):
        o, lse, gathered = cp_forward(q, k, v, plan, group, scale, groups, transport)
        flat = [t for kv in gathered for t in kv]
        ctx.save_for_backward(q, o, lse, *flat)
        ctx.plan, ctx.group, ctx.scale, ctx.transport = plan, group, scale, transport
        return o

    @staticmethod
    def backward(ctx, do):
        q, o, lse, *flat = ctx.saved_tensors
        gathered = list(zip(flat[0::2], flat[1::2]))
        dq, dk, dv = cp_backward(q, gathered, o, lse, do.contiguous(), ctx.plan, ctx.group,
                                 ctx.scale, transport=ctx.transport)
        return dq, dk, dv, None, None, None, None, None


def cp_bitfield_attention(q_loc, k_loc, v_loc, plan: CPPlan, group=None, scale=None,
                          groups: int = 1, transport: str = "auto"):
    """Context-parallel bitfield attention with autograd.  Inputs are this
    rank's rows (``shard_rows``) of q/k/v; returns this rank's O rows.

    ``transport``: "auto" (default) uses the copy-engine exchange over
    NVLink peer memory -- the forward overlaps the K/V pulls, the
    reduce-scatter is fused into the backward -- and falls back to NCCL
    collectively when peer memory is unavailable; "nccl" / "ce" force one.
    ``groups`` > 1 pipelines the exchange per KV-head group."""
    return _CPAttention.apply(q_loc, k_loc, v_loc, plan, group, scale, groups, transport)

"""Workload-balanced context parallelism -- drop-in for ``mmplan.balance``.

Same names, dataclasses, signatures and errors as
``/root/reference/pkg/src/mmplan/balance.py``.  The assignment work runs in
libbam:

* ``lpt_distribute`` (balance.py:58-76) -> ``bam_lpt_assign`` (GPU sort by
  (-W, id) + warp argmin over (load, gpu)), bit-exact including the order of
  blocks inside each GPU's list;
* ``zigzag_distribute`` (balance.py:79-102) -> ``bam_zigzag_assign``;
* ``intra_schedule`` (balance.py:223-265) -> ``bam_split_count/fill`` +
  ``bam_lpt_assign`` over the pieces (the reference's list scheduler is LPT
  over pieces sorted by (-size, block, index));
* ``ilp_optimal`` (balance.py:124-192) -> ``bam_ilp_optimal`` (native host
  branch-and-bound; the reference's exact oracle, budget-limited).

``contiguous_distribute`` (the naive uniform split of BASELINE.json config 5)
is an addition.  ``*_device`` variants keep everything on the GPU for the
attention planner.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass
from typing import Sequence

import torch

from . import _lib

DEFAULT_ALPHA = 0.25
DEFAULT_BETA = 0.5

ILP_MAX_BLOCKS = 14
ILP_MAX_GPUS = 4


class BudgetError(ValueError):
    """Raised when an exact-search instance exceeds the oracle budget."""


@dataclass(frozen=True)
class BlockAssignment:
    """Query blocks mapped to GPUs, with per-GPU load bookkeeping."""

    gpu_blocks: tuple[tuple[int, ...], ...]
    loads: tuple[int, ...]

    @property
    def makespan(self) -> int:
        return max(self.loads)

    @property
    def imbalance(self) -> float:
        """Makespan relative to the perfectly balanced load (balance.py:42-48)."""
        total = sum(self.loads)
        if total == 0:
            return 1.0
        return self.makespan / (total / len(self.loads))


@dataclass(frozen=True)
class DeviceAssignment:
    """Device-resident assignment: owner[n], flat[n] (items grouped by unit,
    assignment order), off[G+1], loads[G] (int64)."""

    owner: torch.Tensor
    flat: torch.Tensor
    off: torch.Tensor
    loads: torch.Tensor

    def to_host(self) -> BlockAssignment:
        flat = self.flat.cpu().tolist()
        off = self.off.cpu().tolist()
        G = len(off) - 1
        return BlockAssignment(
            gpu_blocks=tuple(tuple(flat[off[g]:off[g + 1]]) for g in range(G)),
            loads=tuple(self.loads.cpu().tolist()))


def _check_inputs(workloads: Sequence[int], num_gpus: int) -> None:
    if num_gpus < 1:
        raise ValueError("num_gpus must be >= 1")
    if len(workloads) == 0:
        raise ValueError("workloads must be nonempty")


def _weights(workloads) -> torch.Tensor:
    _lib.require_cuda()
    if isinstance(workloads, torch.Tensor):
        return workloads.to(device="cuda", dtype=torch.int32).contiguous()
    ws = [int(w) for w in workloads]
    if any(w < 0 or w >= 1 << 31 for w in ws):
        raise ValueError("workloads must be integers in [0, 2^31)")
    return torch.tensor(ws, dtype=torch.int32, device="cuda")


def _outputs(n: int, G: int, dev):
    return (torch.empty(n, dtype=torch.int32, device=dev),
            torch.empty(n, dtype=torch.int32, device=dev),
            torch.empty(G + 1, dtype=torch.int32, device=dev),
            torch.empty(G, dtype=torch.int64, device=dev))


def lpt_device(w: torch.Tensor, num_units: int) -> DeviceAssignment:
    """LPT over int32 weights on the device (no host synchronisation)."""
    n = w.shape[0]
    owner, flat, off, loads = _outputs(n, num_units, w.device)
    ws = torch.empty(int(_lib.load().bam_lpt_workspace_bytes(n)), dtype=torch.uint8,
                     device=w.device)
    _lib.call("bam_lpt_assign", w.data_ptr(), n, num_units, owner.data_ptr(), flat.data_ptr(),
              off.data_ptr(), loads.data_ptr(), ws.data_ptr())
    return DeviceAssignment(owner, flat, off, loads)


def _chunk_device(fn: str, w: torch.Tensor, num_gpus: int) -> DeviceAssignment:
    n = w.shape[0]
    owner, flat, off, loads = _outputs(n, num_gpus, w.device)
    _lib.call(fn, w.data_ptr(), n, num_gpus, owner.data_ptr(), flat.data_ptr(), off.data_ptr(),
              loads.data_ptr())
    return DeviceAssignment(owner, flat, off, loads)


def zigzag_device(w: torch.Tensor, num_gpus: int) -> DeviceAssignment:
    return _chunk_device("bam_zigzag_assign", w, num_gpus)


def contiguous_device(w: torch.Tensor, num_gpus: int) -> DeviceAssignment:
    return _chunk_device("bam_contiguous_assign", w, num_gpus)


def lpt_distribute(workloads: Sequence[int], num_gpus: int) -> BlockAssignment:
    """Assign blocks to GPUs, heaviest first, each to the least-loaded GPU.

    Ties break deterministically: equal workloads by lower block id, equal
    loads by lower GPU id."""
    _check_inputs(workloads, num_gpus)
    return lpt_device(_weights(workloads), num_gpus).to_host()


def zigzag_distribute(workloads: Sequence[int], num_gpus: int) -> BlockAssignment:
    """The causal-attention baseline: GPU i gets chunks i and 2G-1-i."""
    _check_inputs(workloads, num_gpus)
    return zigzag_device(_weights(workloads), num_gpus).to_host()


def contiguous_distribute(workloads: Sequence[int], num_gpus: int) -> BlockAssignment:
    """Naive uniform token split: GPU g gets the g-th contiguous run of blocks."""
    _check_inputs(workloads, num_gpus)
    return contiguous_device(_weights(workloads), num_gpus).to_host()


DISTRIBUTIONS = {"lpt": lpt_device, "zigzag": zigzag_device, "contiguous": contiguous_device}


def ilp_optimal(workloads: Sequence[int], num_gpus: int) -> BlockAssignment:
    """Provably optimal makespan assignment (exact search, small instances),
    then the lexicographically smallest assignment vector achieving it."""
    if not workloads:
        raise ValueError("workloads must be nonempty")
    n = len(workloads)
    w = (ctypes.c_int64 * n)(*[int(x) for x in workloads])
    asg = (ctypes.c_int32 * n)()
    mk = ctypes.c_int64()
    rc = _lib.load().bam_ilp_optimal(ctypes.cast(w, ctypes.c_void_p), n, num_gpus,
                                     ctypes.cast(asg, ctypes.c_void_p),
                                     ctypes.cast(ctypes.byref(mk), ctypes.c_void_p))
    if rc == _lib.BAM_BUDGET_EXCEEDED:
        raise BudgetError(_lib.load().bam_last_error().decode())
    if rc != _lib.BAM_OK:
        raise ValueError(_lib.load().bam_last_error().decode())
    blocks: list[list[int]] = [[] for _ in range(num_gpus)]
    for b in range(n):
        blocks[asg[b]].append(b)
    return BlockAssignment(
        gpu_blocks=tuple(tuple(x) for x in blocks),
        loads=tuple(sum(int(workloads[b]) for b in x) for x in blocks))


@dataclass(frozen=True)
class Subblock:
    """A slice of one query block's key-block work, at most ``s`` blocks."""

    block: int
    index: int
    size: int


@dataclass(frozen=True)
class IntraGpuSchedule:
    """Subblocks of one GPU's query blocks scheduled onto compute units."""

    unit_tasks: tuple[tuple[Subblock, ...], ...]
    compute_makespan: int
    aggregation_cost: float

    @property
    def total(self) -> float:
        return self.compute_makespan + self.aggregation_cost


def split_block(workload: int, subblock_size: int) -> list[int]:
    """Sizes of the ceil(W/s) subblocks: all ``s`` except one remainder."""
    full, rem = divmod(workload, subblock_size)
    return [subblock_size] * full + ([rem] if rem else [])


def intra_schedule(
    workloads: Sequence[int],
    compute_units: int,
    subblock_size: int,
    alpha: float = DEFAULT_ALPHA,
    beta: float = DEFAULT_BETA,
) -> IntraGpuSchedule:
    """Split blocks into subblocks and list-schedule them onto compute units
    (balance.py:223-265): pieces by descending size to the least-loaded unit;
    a block split into k >= 2 pieces pays alpha*(k-1)+beta aggregation."""
    if compute_units < 1:
        raise ValueError("compute_units must be >= 1")
    if subblock_size < 1:
        raise ValueError("subblock_size must be >= 1")
    ws = [int(w) for w in workloads]
    aggregation = 0.0
    for w in ws:   # float accumulation in block order, exactly as the reference
        k = -(-w // subblock_size) if w > 0 else 0
        if k >= 2:
            aggregation += alpha * (k - 1) + beta
    n_pieces = sum(-(-w // subblock_size) for w in ws if w > 0)
    if n_pieces == 0:
        return IntraGpuSchedule(unit_tasks=tuple(() for _ in range(compute_units)),
                                compute_makespan=0, aggregation_cost=aggregation)
    wt = _weights(ws)
    n = len(ws)
    dev = wt.device
    cnt = torch.empty(n, dtype=torch.int32, device=dev)
    off = torch.empty(n + 1, dtype=torch.int32, device=dev)
    _lib.call("bam_split_count", wt.data_ptr(), n, subblock_size, cnt.data_ptr(), off.data_ptr())
    size = torch.empty(n_pieces, dtype=torch.int32, device=dev)
    blk = torch.empty_like(size)
    idx = torch.empty_like(size)
    _lib.call("bam_split_fill", wt.data_ptr(), n, subblock_size, off.data_ptr(), size.data_ptr(),
              blk.data_ptr(), idx.data_ptr())
    asg = lpt_device(size, compute_units)
    flat = asg.flat.cpu().tolist()
    uoff = asg.off.cpu().tolist()
    blk_h, idx_h, size_h = blk.cpu().tolist(), idx.cpu().tolist(), size.cpu().tolist()
    units = tuple(
        tuple(Subblock(block=blk_h[i], index=idx_h[i], size=size_h[i])
              for i in flat[uoff[u]:uoff[u + 1]])
        for u in range(compute_units))
    return IntraGpuSchedule(unit_tasks=units, compute_makespan=int(asg.loads.max().item()),
                            aggregation_cost=aggregation)


POLICIES = ("causal", "inter_only", "intra_only", "balanced")


def balance_report(
    workloads: Sequence[int],
    num_gpus: int,
    compute_units: int,
    subblock_size: int,
    alpha: float = DEFAULT_ALPHA,
    beta: float = DEFAULT_BETA,
) -> dict:
    """Compare the four distribution policies (balance.py:271-311): causal =
    zigzag + whole-block, inter_only = LPT + whole-block, intra_only = zigzag
    + subblocked, balanced = LPT + subblocked."""
    whole = max(workloads) if workloads else 1
    whole = max(whole, 1)
    policies = {
        "causal": (zigzag_distribute, whole),
        "inter_only": (lpt_distribute, whole),
        "intra_only": (zigzag_distribute, subblock_size),
        "balanced": (lpt_distribute, subblock_size),
    }
    report: dict[str, dict] = {}
    for name, (distribute, s) in policies.items():
        assignment = distribute(workloads, num_gpus)
        per_gpu = [
            intra_schedule([workloads[b] for b in blocks], compute_units, s, alpha, beta)
            for blocks in assignment.gpu_blocks
        ]
        report[name] = {
            "loads": list(assignment.loads),
            "makespan": assignment.makespan,
            "imbalance": assignment.imbalance,
            "compute_makespan": max(sched.compute_makespan for sched in per_gpu),
            "aggregation_cost": max(sched.aggregation_cost for sched in per_gpu),
            "total": max(sched.total for sched in per_gpu),
        }
    return report

"""CPU restatement of the reference distribution policies (TEST INFRASTRUCTURE ONLY).

Restates ``/root/reference/pkg/src/mmplan/balance.py``.  Assignments are
returned as ``(gpu_blocks: tuple[tuple[int]], loads: tuple[int])``.
"""

from __future__ import annotations

import itertools
from typing import Sequence

DEFAULT_ALPHA = 0.25   # balance.py:20
DEFAULT_BETA = 0.5     # balance.py:21


def _loads(gpu_blocks, w):
    return tuple(sum(w[b] for b in blocks) for blocks in gpu_blocks)


def imbalance(loads: Sequence[int]) -> float:
    """balance.py:42-48: makespan / (sum / G), 1.0 when the sum is zero."""
    total = sum(loads)
    if total == 0:
        return 1.0
    return max(loads) / (total / len(loads))


def lpt(w: Sequence[int], G: int):
    """balance.py:58-76 restated as an explicit argmin (the heap always holds
    one (load, gpu) entry per GPU, so popping it is argmin over (load, g))."""
    if G < 1:
        raise ValueError("num_gpus must be >= 1")
    if not w:
        raise ValueError("workloads must be nonempty")
    load = [0] * G
    blocks = [[] for _ in range(G)]
    for b in sorted(range(len(w)), key=lambda i: (-w[i], i)):
        g = min(range(G), key=lambda h: (load[h], h))
        blocks[g].append(b)
        load[g] += w[b]
    gb = tuple(tuple(x) for x in blocks)
    return gb, _loads(gb, w)


def zigzag(w: Sequence[int], G: int):
    """balance.py:79-102: 2G contiguous chunks (extras first); GPU i gets
    chunks i and 2G-1-i."""
    if G < 1:
        raise ValueError("num_gpus must be >= 1")
    if not w:
        raise ValueError("workloads must be nonempty")
    base, extra = divmod(len(w), 2 * G)
    bounds = [0]
    for i in range(2 * G):
        bounds.append(bounds[-1] + base + (i < extra))
    chunk = [list(range(bounds[i], bounds[i + 1])) for i in range(2 * G)]
    gb = tuple(tuple(chunk[i] + chunk[2 * G - 1 - i]) for i in range(G))
    return gb, _loads(gb, w)


def contiguous(w: Sequence[int], G: int):
    """Naive uniform contiguous split (BASELINE.json config 5); not in the
    reference.  Block counts as equal as possible, extras to the first GPUs."""
    if G < 1:
        raise ValueError("num_gpus must be >= 1")
    if not w:
        raise ValueError("workloads must be nonempty")
    base, extra = divmod(len(w), G)
    gb, lo = [], 0
    for g in range(G):
        n = base + (g < extra)
        gb.append(tuple(range(lo, lo + n)))
        lo += n
    gb = tuple(gb)
    return gb, _loads(gb, w)


def makespan_exhaustive(w: Sequence[int], G: int) -> int:
    """Optimal makespan by enumeration (tests/oracles.py:129-137 restated)."""
    best = sum(w)
    for assign in itertools.product(range(G), repeat=len(w)):
        load = [0] * G
        for b, g in enumerate(assign):
            load[g] += w[b]
        best = min(best, max(load))
    return best


def split_block(workload: int, s: int):
    """balance.py:217-220."""
    full, rem = divmod(workload, s)
    return [s] * full + ([rem] if rem else [])


def intra_schedule(w: Sequence[int], C: int, s: int, alpha=DEFAULT_ALPHA, beta=DEFAULT_BETA):
    """balance.py:223-265 -> (unit_tasks as tuples of (block, index, size),
    compute_makespan, aggregation_cost)."""
    if C < 1:
        raise ValueError("compute_units must be >= 1")
    if s < 1:
        raise ValueError("subblock_size must be >= 1")
    pieces, agg = [], 0.0
    for b, wb in enumerate(w):
        sizes = split_block(wb, s)
        pieces += [(b, i, sz) for i, sz in enumerate(sizes)]
        if len(sizes) >= 2:
            agg += alpha * (len(sizes) - 1) + beta
    pieces.sort(key=lambda p: (-p[2], p[0], p[1]))
    load = [0] * C
    units = [[] for _ in range(C)]
    for p in pieces:
        u = min(range(C), key=lambda h: (load[h], h))
        units[u].append(p)
        load[u] += p[2]
    return tuple(tuple(x) for x in units), max(load), agg


def balance_report(w, G, C, s, alpha=DEFAULT_ALPHA, beta=DEFAULT_BETA) -> dict:
    """balance.py:271-311."""
    whole = max(max(w) if w else 1, 1)
    policies = {
        "causal": (zigzag, whole),
        "inter_only": (lpt, whole),
        "intra_only": (zigzag, s),
        "balanced": (lpt, s),
    }
    out = {}
    for name, (dist, sub) in policies.items():
        gb, loads = dist(w, G)
        scheds = [intra_schedule([w[b] for b in blocks], C, sub, alpha, beta) for blocks in gb]
        out[name] = {
            "loads": list(loads),
            "makespan": max(loads),
            "imbalance": imbalance(loads),
            "compute_makespan": max(x[1] for x in scheds),
            "aggregation_cost": max(x[2] for x in scheds),
            "total": max(x[1] + x[2] for x in scheds),
        }
    return out

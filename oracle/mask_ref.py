"""CPU restatement of the reference bitfield mask (TEST INFRASTRUCTURE ONLY).

Restates ``/root/reference/pkg/src/mmplan/mask.py``; every function names the
lines it follows.  Descriptors are plain Python ints here (arbitrary
precision, exactly like the reference) so the range / control-bit checks see
the same values the reference sees.
"""

from __future__ import annotations

import ctypes
import os
from typing import Sequence

import numpy as np

TEXT = "text"
TEXT_BIT = 1                      # mask.py:28
MAX_MODALITIES = 60               # mask.py:29
CONTROL_MASK = 0b111 << 61        # mask.py:30
SKIP, FULL, PARTIAL = "skip", "full", "partial"   # mask.py:32-34
CLASS_CODE = {SKIP: 0, FULL: 1, PARTIAL: 2}
CODE_CLASS = {v: k for k, v in CLASS_CODE.items()}


class OracleMaskError(ValueError):
    pass


def build_bitfield(segments: Sequence[tuple[str, int]]):
    """mask.py:71-103 -> (descriptors list[int], modalities tuple)."""
    if not segments:
        raise OracleMaskError("segments must be nonempty")
    order: list[str] = []
    for name, count in segments:
        if count < 1:
            raise OracleMaskError(f"segment {name!r}: count must be >= 1")
        if name != TEXT and name not in order:
            order.append(name)
    if len(order) > MAX_MODALITIES:
        raise OracleMaskError(f"{len(order)} modalities exceed the {MAX_MODALITIES} limit")
    bits = {name: 2 << i for i, name in enumerate(order)}
    text_desc = 1 | sum(bits.values())          # mask.py:91-94: bit 0 | every modality bit
    out: list[int] = []
    for name, count in segments:
        out += [text_desc if name == TEXT else bits[name]] * count
    validate(out, len(order))
    return out, tuple(order)


def validate(descriptors: Sequence[int], n_modalities: int) -> None:
    """mask.py:53-68: first failing token, first failing check, in order."""
    if n_modalities > MAX_MODALITIES:
        raise OracleMaskError(f"{n_modalities} modalities exceed the {MAX_MODALITIES} limit")
    for t, d in enumerate(descriptors):
        if d < 0 or d >= 1 << 64:
            raise OracleMaskError(f"token {t}: descriptor out of 64-bit range")
        if d & CONTROL_MASK:
            raise OracleMaskError(f"token {t}: reserved control bits set")
        if d == 0:
            raise OracleMaskError(f"token {t}: no modality bit set")
        if not d & TEXT_BIT and bin(d).count("1") != 1:
            raise OracleMaskError(f"token {t}: pure modality token must set exactly one bit")


def materialize(descriptors: Sequence[int], q: int, k: int) -> bool:
    """mask.py:106-112, the single mask predicate."""
    dq, dk = descriptors[q], descriptors[k]
    if dq & TEXT_BIT:
        return k <= q and (dq & dk) != 0
    return dk == dq


def dense_rows(desc: np.ndarray, rows: np.ndarray, cols: np.ndarray | None = None) -> np.ndarray:
    """Vectorised mask.py:106-112 for query positions ``rows`` x key positions
    ``cols`` (default: all keys).  ``desc`` is int64 (valid masks only: bits
    61-63 clear, so int64 holds them losslessly)."""
    if cols is None:
        cols = np.arange(desc.shape[0])
    dq = desc[rows][:, None]
    dk = desc[cols][None, :]
    text = (dq & 1) != 0
    causal = cols[None, :] <= rows[:, None]
    return np.where(text, causal & ((dq & dk) != 0), dk == dq)


def block_ranges(length: int, block_size: int):
    """mask.py:128-129."""
    return [(lo, min(lo + block_size, length)) for lo in range(0, length, block_size)]


def classify_pair(descriptors: Sequence[int], qr, kr) -> str:
    """mask.py:132-165: OR short-circuit, uniform same-modality FULL, then an
    exact element count."""
    q_or = 0
    for q in range(*qr):
        q_or |= descriptors[q]
    k_or = 0
    for k in range(*kr):
        k_or |= descriptors[k]
    if q_or & k_or == 0:
        return SKIP
    q0, k0 = descriptors[qr[0]], descriptors[kr[0]]
    if (not q0 & TEXT_BIT and q0 == k0
            and all(descriptors[q] == q0 for q in range(*qr))
            and all(descriptors[k] == k0 for k in range(*kr))):
        return FULL
    allowed = sum(1 for q in range(*qr) for k in range(*kr) if materialize(descriptors, q, k))
    if allowed == 0:
        return SKIP
    if allowed == (qr[1] - qr[0]) * (kr[1] - kr[0]):
        return FULL
    return PARTIAL


def block_workloads_py(descriptors: Sequence[int], block_size: int):
    """mask.py:168-188, pure Python (small T only).  Returns (classes as
    nested tuples of strings, workloads tuple)."""
    if block_size < 1:
        raise OracleMaskError("block_size must be >= 1")
    ranges = block_ranges(len(descriptors), block_size)
    classes, work = [], []
    for qr in ranges:
        row = tuple(classify_pair(descriptors, qr, kr) for kr in ranges)
        classes.append(row)
        work.append(sum(1 for c in row if c != SKIP))
    return tuple(classes), tuple(work)


def block_workloads_np(desc: np.ndarray, block_size: int):
    """mask.py:168-188 vectorised with numpy: per query block, the dense
    predicate against all keys, then per key block all/any.  Exact (it counts
    every element).  Returns (uint8 classes [nb, nb], int64 W [nb])."""
    desc = np.asarray(desc, dtype=np.int64)
    T = desc.shape[0]
    nb = (T + block_size - 1) // block_size
    classes = np.zeros((nb, nb), dtype=np.uint8)
    pad = nb * block_size - T
    cols = np.arange(T)
    for b in range(nb):
        lo, hi = b * block_size, min((b + 1) * block_size, T)
        m = dense_rows(desc, np.arange(lo, hi), cols)
        if pad:
            m = np.concatenate([m, np.zeros((hi - lo, pad), dtype=bool)], axis=1)
        m = m.reshape(hi - lo, nb, block_size)
        cnt = m.sum(axis=(0, 2))
        sizes = np.full(nb, block_size, dtype=np.int64)
        sizes[-1] = T - (nb - 1) * block_size
        tot = sizes * (hi - lo)
        classes[b] = np.where(cnt == 0, 0, np.where(cnt == tot, 1, 2))
    return classes, (classes != 0).sum(axis=1).astype(np.int64)


# --- C restatement (fast exact counting for 32K-128K parity) -----------------

_HERE = os.path.dirname(os.path.abspath(__file__))
_C_LIB = None


def c_oracle_path() -> str:
    return os.path.join(_HERE, "_build", "libbam_oracle.so")


def _c_lib():
    global _C_LIB
    if _C_LIB is None:
        path = c_oracle_path()
        if not os.path.exists(path):
            raise RuntimeError(f"C oracle not built: {path} (run __graft_entry__.build())")
        lib = ctypes.CDLL(path)
        lib.oracle_block_workloads.argtypes = [
            ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p,
            ctypes.c_int]
        lib.oracle_block_workloads.restype = ctypes.c_int
        lib.oracle_count_allowed.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int]
        lib.oracle_count_allowed.restype = ctypes.c_int64
        lib.oracle_lpt.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32,
                                   ctypes.c_void_p, ctypes.c_void_p]
        lib.oracle_lpt.restype = ctypes.c_int
        _C_LIB = lib
    return _C_LIB


def block_workloads_c(desc: np.ndarray, block_size: int, threads: int = 0):
    """C restatement of mask.py:132-188 (exact element counts)."""
    desc = np.ascontiguousarray(desc, dtype=np.int64)
    T = desc.shape[0]
    nb = (T + block_size - 1) // block_size
    classes = np.zeros((nb, nb), dtype=np.uint8)
    W = np.zeros(nb, dtype=np.int64)
    rc = _c_lib().oracle_block_workloads(desc.ctypes.data, T, block_size, classes.ctypes.data,
                                         W.ctypes.data, threads)
    if rc != 0:
        raise RuntimeError(f"oracle_block_workloads failed: {rc}")
    return classes, W


def count_allowed_c(desc: np.ndarray, threads: int = 0) -> int:
    """Number of (q, k) pairs with materialize() true (the FLOP count basis)."""
    desc = np.ascontiguousarray(desc, dtype=np.int64)
    return int(_c_lib().oracle_count_allowed(desc.ctypes.data, desc.shape[0], threads))


def count_allowed_rows(desc: np.ndarray, rows: np.ndarray) -> int:
    return int(dense_rows(np.asarray(desc, np.int64), np.asarray(rows)).sum())

"""Bitfield attention masks -- drop-in for the reference ``mmplan.mask``.

Same names, constants, signatures, return types and error messages as
``/root/reference/pkg/src/mmplan/mask.py``; the per-token work runs on the GPU
through libbam (include/bam.h):

* ``build_bitfield`` (mask.py:71-103): the modality registry is host
  bookkeeping over the segment list; the per-token descriptors are expanded
  on the device (``bam_mask_expand``) and validated there.
* ``BitfieldMask.validate`` (mask.py:53-68): ``bam_mask_validate`` finds the
  first failing token and check; the 64-bit range check runs on the host
  while the Python ints are converted to int64.
* ``block_workloads`` (mask.py:168-188): ``bam_block_summarize`` +
  ``bam_classify`` -- bit-exact tile classes and W per query block.

Descriptors live on the device as int64 (valid masks keep bits 61-63 clear,
mask.py:30); the Python tuple view of the reference dataclass is
materialised lazily on first access.
"""

from __future__ import annotations

import json
from dataclasses import dataclass
from typing import Iterable, Sequence

import torch

from . import _lib

MASK_SCHEMA_VERSION = 1

TEXT = "text"
TEXT_BIT = 1
MAX_MODALITIES = 60
CONTROL_MASK = 0b111 << 61

SKIP = "skip"
FULL = "full"
PARTIAL = "partial"
CLASS_NAMES = (SKIP, FULL, PARTIAL)   # device class codes 0, 1, 2

DEFAULT_BLOCK_SIZE = 128

_VALIDATE_MESSAGES = {
    1: "reserved control bits set",
    2: "no modality bit set",
    3: "pure modality token must set exactly one bit",
}


class MaskError(ValueError):
    """Raised for invalid descriptors or segment specs."""


def _device() -> torch.device:
    _lib.require_cuda()
    return torch.device("cuda", torch.cuda.current_device())


def _to_int64(d: int) -> int:
    return d - (1 << 64) if d >= 1 << 63 else d


class _Lazy:
    """Data descriptor behind a frozen-dataclass field whose value may be
    derived on first access from device tensors (``build(obj)``).  The
    dataclass machinery sees a required field (``__get__`` on the class
    raises AttributeError, so there is no default); ``__init__`` and
    ``dataclasses.replace`` store through ``__set__``; assignment on an
    instance still raises ``FrozenInstanceError``."""

    def __init__(self, build):
        self.build = build

    def __set_name__(self, owner, name):
        self.slot = "_v_" + name

    def __get__(self, obj, owner=None):
        if obj is None:
            raise AttributeError(self.slot)
        d = obj.__dict__
        if self.slot not in d:
            d[self.slot] = self.build(obj)
        return d[self.slot]

    def __set__(self, obj, value):
        obj.__dict__[self.slot] = value


def _descriptors_from_device(mask) -> tuple:
    vals = mask.__dict__["_dev"].cpu().tolist()
    return tuple(v + (1 << 64) if v < 0 else v for v in vals)


@dataclass(frozen=True)
class BitfieldMask:
    """Per-token descriptors for one packed sequence (mask.py:43-68): the
    reference's frozen dataclass, same fields (``dataclasses.fields``,
    ``asdict``, ``replace`` and equality behave identically).

    ``descriptors`` (tuple of ints) and ``modalities`` (registration order;
    modality i uses bit i+1).  Masks built on the GPU keep their int64
    descriptors on the device (``device_descriptors()``, not a dataclass
    field); the tuple is materialised on first access.
    """

    descriptors: tuple = _Lazy(_descriptors_from_device)
    modalities: tuple

    @classmethod
    def _from_device(cls, desc: torch.Tensor, modalities: Sequence[str]) -> "BitfieldMask":
        obj = object.__new__(cls)
        obj.__dict__["_dev"] = desc.to(torch.int64)
        object.__setattr__(obj, "modalities", tuple(modalities))
        return obj

    def __len__(self) -> int:
        d = self.__dict__
        if "_v_descriptors" not in d and d.get("_dev") is not None:
            return int(d["_dev"].shape[0])
        return len(self.descriptors)

    def _first_out_of_range(self):
        if "_v_descriptors" not in self.__dict__:
            return None            # device-built: int64 by construction
        for t, d in enumerate(self.descriptors):
            if not 0 <= d < 1 << 64:
                return t
        return None

    def device_descriptors(self) -> torch.Tensor:
        """int64 [T] descriptors on the current CUDA device (cached; not a
        dataclass field).  Out-of-range values (rejected by ``validate``)
        are replaced by 1 here."""
        dev_t = self.__dict__.get("_dev")
        if dev_t is None:
            dev = _device()
            vals = [_to_int64(d) if 0 <= d < 1 << 64 else 1 for d in self.descriptors]
            dev_t = torch.tensor(vals, dtype=torch.int64, device=dev)
        elif dev_t.device.type != "cuda":
            dev_t = dev_t.to(_device())
        self.__dict__["_dev"] = dev_t
        return dev_t

    def validate(self) -> None:
        """mask.py:53-68 -- raises MaskError for the first failing token."""
        if len(self.modalities) > MAX_MODALITIES:
            raise MaskError(
                f"{len(self.modalities)} modalities exceed the {MAX_MODALITIES} limit")
        T = len(self)
        if T == 0:
            return
        desc = self.device_descriptors()
        err = torch.empty(1, dtype=torch.int64, device=desc.device)
        _lib.call("bam_mask_validate", desc.data_ptr(), T, err.data_ptr())
        code = int(err.item()) & 0xFFFFFFFFFFFFFFFF
        first_range = self._first_out_of_range()
        if code == 0xFFFFFFFFFFFFFFFF and first_range is None:
            return
        tok, kind = (code >> 2, code & 3) if code != 0xFFFFFFFFFFFFFFFF else (None, 0)
        if first_range is not None and (tok is None or first_range <= tok):
            raise MaskError(f"token {first_range}: descriptor out of 64-bit range")
        raise MaskError(f"token {tok}: {_VALIDATE_MESSAGES[kind]}")


def build_bitfield(segments: Sequence[tuple[str, int]]) -> BitfieldMask:
    """Descriptors for a packed sequence of (modality, token count) runs
    (mask.py:71-103).  Modalities register in order of first appearance;
    text tokens get bit 0 plus every registered modality bit."""
    if not segments:
        raise MaskError("segments must be nonempty")
    modalities: list[str] = []
    for modality, count in segments:
        if count < 1:
            raise MaskError(f"segment {modality!r}: count must be >= 1")
        if modality != TEXT and modality not in modalities:
            modalities.append(modality)
    if len(modalities) > MAX_MODALITIES:
        raise MaskError(f"{len(modalities)} modalities exceed the {MAX_MODALITIES} limit")
    bit_of = {name: 1 << (i + 1) for i, name in enumerate(modalities)}
    text_desc = TEXT_BIT
    for b in bit_of.values():
        text_desc |= b
    seg_desc, seg_end, total = [], [], 0
    for modality, count in segments:
        seg_desc.append(text_desc if modality == TEXT else bit_of[modality])
        total += int(count)
        seg_end.append(total)
    dev = _device()
    sd = torch.tensor(seg_desc, dtype=torch.int64, device=dev)
    se = torch.tensor(seg_end, dtype=torch.int64, device=dev)
    desc = torch.empty(total, dtype=torch.int64, device=dev)
    _lib.call("bam_mask_expand", sd.data_ptr(), se.data_ptr(), len(seg_desc), total, desc.data_ptr())
    mask = BitfieldMask._from_device(desc, modalities)
    mask.validate()
    return mask


def materialize(mask: BitfieldMask, q: int, k: int) -> bool:
    """Whether query token ``q`` attends key token ``k`` (mask.py:106-112)."""
    dq = mask.descriptors[q]
    dk = mask.descriptors[k]
    if dq & TEXT_BIT:
        return k <= q and (dq & dk) != 0
    return dk == dq


def _classes_from_device(work) -> tuple:
    rows = work.__dict__["class_codes"].cpu().tolist()
    return tuple(tuple(CLASS_NAMES[c] for c in row) for row in rows)


def _workloads_from_device(work) -> tuple:
    return tuple(work.__dict__["workload_tensor"].cpu().tolist())


@dataclass(frozen=True)
class BlockWorkload:
    """Blockwise classification and per-query-block work (mask.py:115-125):
    the reference's frozen dataclass with the same fields.

    ``classes`` ([query block][key block] strings) and ``workloads`` are
    materialised on first access from the device results, which stay
    available as ``class_codes`` (uint8 [nb, nb], 0 skip / 1 full /
    2 partial) and ``workload_tensor`` (int32 [nb]) -- attributes, not
    dataclass fields.
    """

    block_size: int
    classes: tuple = _Lazy(_classes_from_device)
    workloads: tuple = _Lazy(_workloads_from_device)

    @classmethod
    def _from_device(cls, block_size: int, class_codes: torch.Tensor,
                     workload_tensor: torch.Tensor) -> "BlockWorkload":
        obj = object.__new__(cls)
        object.__setattr__(obj, "block_size", block_size)
        obj.__dict__["class_codes"] = class_codes
        obj.__dict__["workload_tensor"] = workload_tensor
        return obj

    @property
    def num_blocks(self) -> int:
        wt = self.__dict__.get("workload_tensor")
        if "_v_workloads" not in self.__dict__ and wt is not None:
            return int(wt.shape[0])
        return len(self.workloads)

    @property
    def class_codes(self) -> torch.Tensor:
        t = self.__dict__.get("class_codes")
        if t is None:
            codes = [[CLASS_NAMES.index(c) for c in row] for row in self.classes]
            t = torch.tensor(codes, dtype=torch.uint8, device=_device()).reshape(
                len(codes), len(codes[0]) if codes else 0)
            self.__dict__["class_codes"] = t
        return t

    @property
    def workload_tensor(self) -> torch.Tensor:
        t = self.__dict__.get("workload_tensor")
        if t is None:
            t = torch.tensor(list(self.workloads), dtype=torch.int32, device=_device())
            self.__dict__["workload_tensor"] = t
        return t


def block_summaries(desc: torch.Tensor, block_size: int) -> torch.Tensor:
    """Per-block OR / AND / text flags (raw BamBlockSummary records, 40 B each)."""
    T = desc.shape[0]
    nb = (T + block_size - 1) // block_size
    out = torch.empty(nb * 5, dtype=torch.int64, device=desc.device)   # 5 x 8 B per record
    _lib.call("bam_block_summarize", desc.data_ptr(), T, block_size, out.data_ptr())
    return out


def classify_device(desc: torch.Tensor, block_size: int = DEFAULT_BLOCK_SIZE):
    """Device-only block classification: returns (classes uint8 [nb, nb], W int32 [nb])."""
    T = desc.shape[0]
    nb = (T + block_size - 1) // block_size
    summ = block_summaries(desc, block_size)
    classes = torch.empty(nb, nb, dtype=torch.uint8, device=desc.device)
    W = torch.empty(nb, dtype=torch.int32, device=desc.device)
    _lib.call("bam_classify", desc.data_ptr(), summ.data_ptr(), nb, classes.data_ptr(),
              W.data_ptr())
    return classes, W


def count_allowed(desc: torch.Tensor, block_size: int = DEFAULT_BLOCK_SIZE,
                  classes: torch.Tensor | None = None) -> int:
    """Exact number of (q, k) pairs with materialize() true (device count)."""
    T = desc.shape[0]
    nb = (T + block_size - 1) // block_size
    summ = block_summaries(desc, block_size)
    if classes is None:
        classes = torch.empty(nb, nb, dtype=torch.uint8, device=desc.device)
        W = torch.empty(nb, dtype=torch.int32, device=desc.device)
        _lib.call("bam_classify", desc.data_ptr(), summ.data_ptr(), nb, classes.data_ptr(),
                  W.data_ptr())
    out = torch.empty(1, dtype=torch.int64, device=desc.device)
    _lib.call("bam_count_allowed", desc.data_ptr(), summ.data_ptr(), classes.data_ptr(), nb,
              out.data_ptr())
    return int(out.item())


def block_workloads(mask: BitfieldMask, block_size: int = DEFAULT_BLOCK_SIZE) -> BlockWorkload:
    """Classify every (query block, key block) pair and count work per row
    (mask.py:168-188).  ``skip`` pairs are fully masked, ``full`` fully
    unmasked, ``partial`` otherwise; W_b counts the non-skip pairs."""
    if block_size < 1:
        raise MaskError("block_size must be >= 1")
    mask.validate()
    if len(mask) == 0:
        dev = _device()
        return BlockWorkload._from_device(block_size,
                                          torch.empty(0, 0, dtype=torch.uint8, device=dev),
                                          torch.empty(0, dtype=torch.int32, device=dev))
    classes, W = classify_device(mask.device_descriptors(), block_size)
    return BlockWorkload._from_device(block_size, classes, W)


# --- documents (mask.py:193-252) -------------------------------------------

def mask_to_doc(mask: BitfieldMask) -> dict:
    return {
        "schema_version": MASK_SCHEMA_VERSION,
        "modalities": list(mask.modalities),
        "descriptors": list(mask.descriptors),
    }


def segments_to_doc(segments: Sequence[tuple[str, int]]) -> dict:
    return {
        "schema_version": MASK_SCHEMA_VERSION,
        "segments": [{"modality": m, "count": c} for m, c in segments],
    }


def mask_from_doc(doc: dict) -> BitfieldMask:
    """Load a mask from a segments document or a raw-descriptor document."""
    if not isinstance(doc, dict):
        raise MaskError("mask document must be an object")
    if "segments" in doc:
        raw = doc["segments"]
        if not isinstance(raw, list) or not raw:
            raise MaskError("'segments' must be a non-empty list")
        segments = []
        for i, entry in enumerate(raw):
            if not isinstance(entry, dict) or "modality" not in entry or "count" not in entry:
                raise MaskError(f"segments[{i}]: needs 'modality' and 'count'")
            segments.append((str(entry["modality"]), int(entry["count"])))
        return build_bitfield(segments)
    if "descriptors" in doc:
        descriptors = tuple(int(d) for d in doc["descriptors"])
        modalities = tuple(str(m) for m in doc.get("modalities", ()))
        mask = BitfieldMask(descriptors=descriptors, modalities=modalities)
        mask.validate()
        return mask
    raise MaskError("mask document needs 'segments' or 'descriptors'")


def load_mask(path: str) -> BitfieldMask:
    with open(path, "r", encoding="utf-8") as fh:
        return mask_from_doc(json.load(fh))


def _run_length(row: Iterable[str]) -> list[list]:
    encoded: list[list] = []
    for cls in row:
        if encoded and encoded[-1][1] == cls:
            encoded[-1][0] += 1
        else:
            encoded.append([1, cls])
    return encoded


def workload_to_doc(work: BlockWorkload) -> dict:
    return {
        "schema_version": MASK_SCHEMA_VERSION,
        "block_size": work.block_size,
        "workloads": list(work.workloads),
        "classes_rle": [_run_length(row) for row in work.classes],
    }

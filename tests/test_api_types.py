"""CPU tests: the drop-in result types are the reference's frozen dataclasses
(ref mask.py:43-50, 115-125; balance.py:31-55, 195-214) -- same fields,
``asdict`` / ``replace`` / equality / hashing / immutability -- including the
objects the GPU path builds lazily from device tensors (``_from_device``)."""

import dataclasses

import pytest
import torch

from paper_2503_11367_b200 import balance as B
from paper_2503_11367_b200 import mask as M


def test_bitfield_mask_is_reference_dataclass():
    m = M.BitfieldMask(descriptors=(0b111, 0b010, 0b010, 0b100), modalities=("A", "B"))
    assert dataclasses.is_dataclass(m)
    assert [f.name for f in dataclasses.fields(m)] == ["descriptors", "modalities"]
    assert dataclasses.asdict(m) == {"descriptors": (7, 2, 2, 4), "modalities": ("A", "B")}
    assert len(m) == 4
    with pytest.raises(dataclasses.FrozenInstanceError):
        m.descriptors = (1,)
    r = dataclasses.replace(m, modalities=("A", "C"))
    assert r.modalities == ("A", "C") and r.descriptors == m.descriptors
    assert m == M.BitfieldMask((7, 2, 2, 4), ("A", "B"))
    assert hash(m) == hash(M.BitfieldMask((7, 2, 2, 4), ("A", "B")))
    with pytest.raises(TypeError):
        M.BitfieldMask((1,))          # both fields are required, as in the reference


def test_device_built_mask_materialises_lazily():
    # int64 storage of a descriptor >= 2^63 reads back as the unsigned value
    d = M.BitfieldMask._from_device(torch.tensor([7, 2, -1]), ("A",))
    assert len(d) == 3 and "_v_descriptors" not in d.__dict__
    assert d.descriptors == (7, 2, (1 << 64) - 1)
    assert d == M.BitfieldMask((7, 2, (1 << 64) - 1), ("A",))
    assert dataclasses.asdict(d) == {"descriptors": (7, 2, (1 << 64) - 1), "modalities": ("A",)}


def test_block_workload_is_reference_dataclass():
    codes = torch.tensor([[1, 0], [2, 1]], dtype=torch.uint8)
    w = M.BlockWorkload._from_device(128, codes, torch.tensor([1, 2], dtype=torch.int32))
    assert [f.name for f in dataclasses.fields(w)] == ["block_size", "classes", "workloads"]
    assert w.num_blocks == 2
    ref = M.BlockWorkload(block_size=128, classes=(("full", "skip"), ("partial", "full")),
                          workloads=(1, 2))
    assert w == ref and hash(w) == hash(ref)
    assert dataclasses.asdict(w) == dataclasses.asdict(ref)
    with pytest.raises(dataclasses.FrozenInstanceError):
        w.workloads = (0, 0)
    assert torch.equal(w.class_codes, codes)


def test_balance_types_are_frozen_dataclasses():
    a = B.BlockAssignment(gpu_blocks=((0, 2), (1,)), loads=(5, 4))
    assert [f.name for f in dataclasses.fields(a)] == ["gpu_blocks", "loads"]
    assert a.makespan == 5 and a.imbalance == 5 / 4.5
    with pytest.raises(dataclasses.FrozenInstanceError):
        a.loads = (0, 0)
    s = B.IntraGpuSchedule(unit_tasks=((B.Subblock(0, 0, 2),),), compute_makespan=2,
                           aggregation_cost=0.0)
    assert s.total == 2.0
    assert [f.name for f in dataclasses.fields(B.Subblock)] == ["block", "index", "size"]

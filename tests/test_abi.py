"""CPU tests of the C-ABI boundary: libbam.so loads and exports every entry
point declared in include/bam.h, with ctypes signatures that match; host-only
entry points (ILP, error text) work without a GPU."""

import ctypes
import os
import re

import pytest

from conftest import ROOT


def header_functions():
    text = open(os.path.join(ROOT, "include", "bam.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(bam_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_header_symbol():
    from paper_2503_11367_b200 import _lib

    lib = _lib.load()
    names = header_functions()
    assert len(names) >= 15
    for name in names:
        assert hasattr(lib, name), name
    assert set(names) == set(_lib.SIGNATURES), set(names) ^ set(_lib.SIGNATURES)


def test_struct_sizes_match_header():
    from paper_2503_11367_b200 import _lib

    lib = _lib.load()
    assert ctypes.sizeof(_lib.BamBlockSummary) == 40
    for name in ("BamBlockSummary", "BamAttnFwdParams", "BamAttnBwdParams", "BamPlan"):
        assert lib.bam_sizeof(name.encode()) == ctypes.sizeof(getattr(_lib, name)), name
    assert lib.bam_sizeof(b"nope") == -1


def test_ilp_host_entry_point():
    from paper_2503_11367_b200 import balance

    # test_balance.py:92-129 pins
    assert balance.ilp_optimal([1, 2, 2, 4, 5, 2, 2, 8], 4).makespan == 8
    assert balance.ilp_optimal([3, 3, 3], 3).makespan == 3
    got = balance.ilp_optimal([5, 5], 4)
    assert got.makespan == 5 and sorted(got.loads) == [0, 0, 5, 5]
    assert balance.ilp_optimal([3, 3, 2, 2, 2], 2).makespan == 6
    assert balance.ilp_optimal([2, 2, 2, 2], 2).gpu_blocks == ((0, 1), (2, 3))
    with pytest.raises(balance.BudgetError):
        balance.ilp_optimal([1] * 15, 2)
    with pytest.raises(balance.BudgetError):
        balance.ilp_optimal([1] * 5, 5)


def test_ilp_matches_golden(golden):
    from paper_2503_11367_b200 import balance

    for case in golden("balance_cases.json"):
        if "ilp" in case:
            got = balance.ilp_optimal(case["workloads"], case["gpus"])
            assert [list(x) for x in got.gpu_blocks] == case["ilp"]["gpu_blocks"]
            assert got.imbalance == case["ilp"]["imbalance"]


def test_product_fails_loudly_without_gpu():
    import torch

    from paper_2503_11367_b200 import balance, mask

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        mask.build_bitfield([("text", 4)])
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        balance.lpt_distribute([1, 2, 3], 2)


def test_argument_errors_match_reference():
    from paper_2503_11367_b200 import balance, mask

    with pytest.raises(ValueError, match="num_gpus must be >= 1"):
        balance.lpt_distribute([1], 0)
    with pytest.raises(ValueError, match="workloads must be nonempty"):
        balance.zigzag_distribute([], 2)
    with pytest.raises(mask.MaskError, match="segments must be nonempty"):
        mask.build_bitfield([])
    with pytest.raises(mask.MaskError, match="count must be >= 1"):
        mask.build_bitfield([("text", 0)])
    with pytest.raises(mask.MaskError, match="61 modalities"):
        mask.build_bitfield([(f"m{i}", 1) for i in range(61)])
    with pytest.raises(ValueError, match="compute_units must be >= 1"):
        balance.intra_schedule([1], 0, 1)
    assert balance.split_block(5, 2) == [2, 2, 1]
    assert balance.split_block(0, 2) == []

"""CPU tests: the oracle restatement pinned against the reference's own
outputs (golden vectors from tests/golden/make_golden.py) and the literal
pins of the reference test-suite (test_mask.py, test_balance.py)."""

import math

import numpy as np
import pytest
import torch

from conftest import load_golden, unrle
from oracle import attention_ref, balance_ref, mask_ref

PACKED = [("text", 1), ("A", 2), ("B", 2), ("text", 3)]
PACKED_DESCRIPTORS = [0b111, 0b010, 0b010, 0b100, 0b100, 0b111, 0b111, 0b111]   # test_mask.py:27-28
PACKED_DENSE = [                                                                 # test_mask.py:32-41
    [1, 0, 0, 0, 0, 0, 0, 0], [0, 1, 1, 0, 0, 0, 0, 0], [0, 1, 1, 0, 0, 0, 0, 0],
    [0, 0, 0, 1, 1, 0, 0, 0], [0, 0, 0, 1, 1, 0, 0, 0], [1, 1, 1, 1, 1, 1, 0, 0],
    [1, 1, 1, 1, 1, 1, 1, 0], [1, 1, 1, 1, 1, 1, 1, 1]]
WORKLOAD_SEGMENTS = [("text", 1), ("A", 2), ("text", 2), ("B", 2), ("text", 1)]
WORKLOAD_VECTOR = (1, 2, 2, 4, 5, 2, 2, 8)                                       # test_mask.py:44-45
PACKED_W = [1, 2, 2, 4, 5, 2, 2, 8]


def test_reference_pins_mask():
    d, mods = mask_ref.build_bitfield(PACKED)
    assert d == PACKED_DESCRIPTORS and mods == ("A", "B")
    for q in range(8):
        for k in range(8):
            assert mask_ref.materialize(d, q, k) == bool(PACKED_DENSE[q][k])
    d2, _ = mask_ref.build_bitfield(WORKLOAD_SEGMENTS)
    assert mask_ref.block_workloads_py(d2, 1)[1] == WORKLOAD_VECTOR
    d3, _ = mask_ref.build_bitfield([(m, c * 128) for m, c in WORKLOAD_SEGMENTS])
    assert tuple(mask_ref.block_workloads_np(np.array(d3), 128)[1]) == WORKLOAD_VECTOR
    dc, _ = mask_ref.build_bitfield([("text", 8)])
    assert mask_ref.block_workloads_py(dc, 1)[1] == tuple(range(1, 9))


def test_reference_pins_balance():
    assert balance_ref.lpt(PACKED_W, 4)[1] == (8, 6, 6, 6)                      # test_balance.py:24-27
    assert balance_ref.lpt([3] * 8, 4)[1] == (6, 6, 6, 6)
    assert balance_ref.lpt([2, 2, 2, 2], 2)[0] == ((0, 2), (1, 3))
    assert balance_ref.zigzag(list(range(1, 9)), 4)[1] == (9, 9, 9, 9)          # test_balance.py:69-71
    assert balance_ref.zigzag(PACKED_W, 4)[1] == (9, 4, 4, 9)
    assert balance_ref.zigzag([3, 3, 2], 2)[1] == (3, 5)
    assert balance_ref.zigzag([1, 2, 3, 4], 2)[0] == ((0, 3), (1, 2))
    assert balance_ref.lpt([3, 3, 2, 2, 2], 2)[1] and max(balance_ref.lpt([3, 3, 2, 2, 2], 2)[1]) == 7
    assert balance_ref.makespan_exhaustive([3, 3, 2, 2, 2], 2) == 6
    assert balance_ref.intra_schedule([1, 5], 2, 2)[1] == 3                      # test_balance.py:150-155
    assert balance_ref.intra_schedule([1, 5], 2, 5)[1:] == (5, 0.0)
    assert balance_ref.intra_schedule([1, 5], 2, 2)[2] == pytest.approx(1.0)
    rep = balance_ref.balance_report(PACKED_W, 4, 4, 2)                          # test_balance.py:224-229
    assert [rep[p]["makespan"] for p in ("causal", "balanced", "inter_only", "intra_only")] == [9, 8, 8, 9]


def test_oracle_mask_vs_reference_golden():
    for case in load_golden("mask_cases.json"):
        d = case["descriptors"]
        if "segments" in case:
            d2, mods = mask_ref.build_bitfield([tuple(s) for s in case["segments"]])
            assert d2 == d and list(mods) == case["modalities"]
        bs = case["block_size"]
        cls, W = mask_ref.block_workloads_np(np.asarray(d, np.int64), bs)
        assert list(W) == case["workloads"], case["tag"]
        got = tuple(tuple(mask_ref.CODE_CLASS[c] for c in row) for row in cls.tolist())
        assert got == unrle(case["classes_rle"]), case["tag"]
        if len(d) <= 96:
            assert mask_ref.block_workloads_py(d, bs) == (got, tuple(case["workloads"]))


def test_c_oracle_vs_reference_golden():
    for case in load_golden("mask_cases.json"):
        cls, W = mask_ref.block_workloads_c(np.asarray(case["descriptors"], np.int64),
                                            case["block_size"])
        assert list(W) == case["workloads"], case["tag"]
        got = tuple(tuple(mask_ref.CODE_CLASS[c] for c in row) for row in cls.tolist())
        assert got == unrle(case["classes_rle"]), case["tag"]


@pytest.mark.parametrize("name", ["config1_workloads.json", "config2_workloads.json"])
def test_c_oracle_vs_reference_configs(name):
    case = load_golden(name)
    d, _ = mask_ref.build_bitfield([tuple(s) for s in case["segments"]])
    cls, W = mask_ref.block_workloads_c(np.asarray(d, np.int64), 128)
    assert list(W) == case["workloads"]
    got = tuple(tuple(mask_ref.CODE_CLASS[c] for c in row) for row in cls.tolist())
    assert got == unrle(case["classes_rle"])


def test_validation_messages_oracle():
    for case in load_golden("validation_cases.json"):
        if "segments" in case:
            call = lambda: mask_ref.build_bitfield([tuple(s) for s in case["segments"]])  # noqa
        else:
            desc = [int(x) for x in case["descriptors"]]
            call = lambda: mask_ref.validate(desc, len(case["modalities"]))  # noqa
        if case["error"] is None:
            call()
        else:
            with pytest.raises(ValueError) as ei:
                call()
            assert str(ei.value) == case["error"]


def test_oracle_balance_vs_reference_golden():
    for case in load_golden("balance_cases.json"):
        w, G = case["workloads"], case["gpus"]
        gb, loads = balance_ref.lpt(w, G)
        assert [list(x) for x in gb] == case["lpt"]["gpu_blocks"]
        assert balance_ref.imbalance(loads) == case["lpt"]["imbalance"]
        gb, loads = balance_ref.zigzag(w, G)
        assert [list(x) for x in gb] == case["zigzag"]["gpu_blocks"]
        it = case["intra"]
        units, mk, agg = balance_ref.intra_schedule(w, it["compute_units"], it["subblock_size"])
        assert mk == it["compute_makespan"] and agg == it["aggregation_cost"]
        if "unit_tasks" in it:
            assert [[list(p) for p in u] for u in units] == it["unit_tasks"]
        assert balance_ref.balance_report(w, G, it["compute_units"], it["subblock_size"]) == case["report"]


def test_oracle_reference_cli_golden_ilp():
    # ref tests/test_cli.py:46-53: cp-distribute -g 4 -c 2 -s 2 --ilp on the reference fixture
    doc = load_golden("report_two_encoders_ilp.json")
    fx = load_golden("mask_two_encoders_fixture.json")
    d, _ = mask_ref.build_bitfield([(s["modality"], s["count"]) for s in fx["segments"]])
    _, W = mask_ref.block_workloads_np(np.asarray(d, np.int64), 128)
    assert list(W) == doc["workloads"] == [1, 2, 2, 4, 5, 2, 2, 8]
    assert (doc["gpus"], doc["compute_units"], doc["subblock_size"]) == (4, 2, 2)
    assert balance_ref.balance_report(list(W), 4, 2, 2) == doc["policies"]
    assert balance_ref.makespan_exhaustive(list(W), 4) == doc["ilp_optimal"]["makespan"] == 8


def test_attention_oracle_vs_dense_autograd():
    d, _ = mask_ref.build_bitfield([("text", 40), ("img", 50), ("text", 38)])
    T = len(d)
    g = torch.Generator().manual_seed(0)
    q = torch.randn(T, 4, 128, generator=g)
    k = torch.randn(T, 2, 128, generator=g)
    v = torch.randn(T, 2, 128, generator=g)
    do = torch.randn(T, 4, 128, generator=g)
    pos = np.arange(T)
    o, lse = attention_ref.attention_fwd(q, k, v, d, pos, chunk=37)
    dq, dk, dv = attention_ref.attention_bwd(q, k, v, o, lse, do, d, pos, chunk=37)
    o2, dq2, dk2, dv2 = attention_ref.attention_dense_autograd(q, k, v, do, d, pos)
    for a, b in ((o, o2), (dq, dq2), (dk, dk2), (dv, dv2)):
        assert torch.allclose(a, b, atol=1e-4, rtol=1e-4)


def test_attention_oracle_rows_subset():
    # CP: a rank's rows (non-contiguous positions) against all keys
    d, _ = mask_ref.build_bitfield([("text", 64), ("a", 64), ("text", 128)])
    T = len(d)
    g = torch.Generator().manual_seed(1)
    q = torch.randn(T, 2, 128, generator=g)
    k = torch.randn(T, 2, 128, generator=g)
    v = torch.randn(T, 2, 128, generator=g)
    rows = np.array(list(range(128, 192)) + list(range(0, 32)))
    o_all, lse_all = attention_ref.attention_fwd(q, k, v, d, np.arange(T))
    o, lse = attention_ref.attention_fwd(q[rows], k, v, d, rows)
    assert torch.allclose(o, o_all[rows], atol=1e-5)
    assert torch.allclose(lse, lse_all[:, rows], atol=1e-5)


def test_n_allowed_config1():
    # config 1 N_allowed = 8,783,360
    d, _ = mask_ref.build_bitfield([("text", 128), ("image", 1024), ("text", 2944)])
    assert mask_ref.count_allowed_c(np.asarray(d, np.int64)) == 8_783_360

"""Property tests of the GPU mask / balance path in the reference suite's
style (hypothesis against independent brute force; ref tests/test_mask.py:155-174,
tests/test_balance.py:47-65, 131-140), derandomized so every run draws the
same examples."""

import numpy as np
import pytest
from hypothesis import HealthCheck, given, settings
from hypothesis import strategies as st

from oracle import balance_ref, mask_ref

pytestmark = pytest.mark.gpu

SETTINGS = settings(max_examples=100, deadline=None, derandomize=True,
                    suppress_health_check=[HealthCheck.too_slow])

segments_st = st.lists(
    st.tuples(st.sampled_from(["text", "image", "audio", "video"]), st.integers(1, 80)),
    min_size=1, max_size=8).filter(lambda s: sum(c for _, c in s) <= 512)


@SETTINGS
@given(segs=segments_st, block=st.sampled_from([1, 16, 128]))
def test_classes_and_workloads_equal_brute_force(segs, block):
    """K2 bit-exact contract: GPU tile classes and W equal the element-wise
    brute force of the reference semantics (mask.py:106-188)."""
    from paper_2503_11367_b200 import mask as M

    mask = M.build_bitfield(segs)
    work = M.block_workloads(mask, block)
    classes, W = mask_ref.block_workloads_py(list(mask.descriptors), block)
    assert list(work.workloads) == list(W)
    assert [list(r) for r in work.classes] == [list(r) for r in classes]


@SETTINGS
@given(segs=segments_st)
def test_workload_sum_at_block_one_is_allowed_pairs(segs):
    """ΣW at block size 1 equals the exact allowed-pair count (test_mask.py:150-153),
    and both equal the GPU count_allowed kernel."""
    from paper_2503_11367_b200 import mask as M

    mask = M.build_bitfield(segs)
    desc = np.asarray(mask.descriptors, np.int64)
    dense = mask_ref.dense_rows(desc, np.arange(desc.shape[0]))
    assert sum(M.block_workloads(mask, 1).workloads) == int(dense.sum())
    assert M.count_allowed(mask.device_descriptors()) == int(dense.sum())


@SETTINGS
@given(w=st.lists(st.integers(0, 300), min_size=1, max_size=400), G=st.integers(1, 16))
def test_lpt_bound_and_zigzag_comparison(w, G):
    """LPT bound makespan * G <= sum W + max W * G (test_balance.py:47-55), the
    GPU assignment equals the restatement, and LPT <= zigzag when n <= 2G."""
    from paper_2503_11367_b200 import balance as B

    a = B.lpt_distribute(w, G)
    assert a.makespan * G <= sum(w) + max(w) * G
    gb, loads = balance_ref.lpt(w, G)
    assert a.gpu_blocks == gb and a.loads == loads
    if len(w) <= 2 * G:
        assert a.makespan <= B.zigzag_distribute(w, G).makespan


@SETTINGS
@given(w=st.lists(st.integers(1, 40), min_size=1, max_size=9), G=st.integers(1, 3))
def test_graham_bound_against_exact(w, G):
    """3G * LPT <= (4G - 1) * OPT with OPT from the GPU-side exact search
    (bam_ilp_optimal), itself equal to exhaustive search (test_balance.py:131-140)."""
    from paper_2503_11367_b200 import balance as B

    opt = B.ilp_optimal(w, G)
    assert opt.makespan == balance_ref.makespan_exhaustive(w, G)
    assert 3 * G * B.lpt_distribute(w, G).makespan <= (4 * G - 1) * opt.makespan

"""GPU parity: tcgen05 attention forward/backward vs the fp32 CPU oracle.

Tolerance (BASELINE.json north star): bf16 kernel vs fp32 oracle,
max-abs <= 2e-2 and relative-L2 <= 1e-2 on O, dQ, dK, dV; LSE max-abs 2e-3.
"""

import math

import numpy as np
import pytest
import torch

from oracle import attention_ref, mask_ref

pytestmark = pytest.mark.gpu

MAX_ABS = 2e-2
REL_L2 = 1e-2


def rel_l2(a, b):
    a, b = a.float().cpu(), b.float().cpu()
    return ((a - b).norm() / b.norm().clamp_min(1e-12)).item()


def max_abs(a, b):
    return (a.float().cpu() - b.float().cpu()).abs().max().item()


def inputs(T, Hq, Hkv, seed=1234):
    g = torch.Generator().manual_seed(seed)
    q = torch.randn(T, Hq, 128, generator=g).to(torch.bfloat16)
    k = torch.randn(T, Hkv, 128, generator=g).to(torch.bfloat16)
    v = torch.randn(T, Hkv, 128, generator=g).to(torch.bfloat16)
    do = torch.randn(T, Hq, 128, generator=g).to(torch.bfloat16)
    return q, k, v, do


def assert_close(name, got, ref):
    ma, rl = max_abs(got, ref), rel_l2(got, ref)
    assert ma <= MAX_ABS and rl <= REL_L2, f"{name}: max-abs {ma:.3e} rel-L2 {rl:.3e}"


def run_case(desc_list, Hq, Hkv, seed=1234, check_bwd=True):
    from paper_2503_11367_b200 import attention as A

    desc = np.asarray(desc_list, dtype=np.int64)
    T = desc.shape[0]
    q, k, v, do = inputs(T, Hq, Hkv, seed)
    dev = torch.device("cuda")
    plan = A.build_plan(torch.from_numpy(desc).to(dev))
    # plan tile lists must equal the oracle's classification
    ref_cls, ref_w = mask_ref.block_workloads_np(desc, 128)
    assert np.array_equal(plan.classes.cpu().numpy(), ref_cls)
    assert np.array_equal(plan.W.cpu().numpy(), ref_w)
    qd, kd, vd, dod = (t.to(dev) for t in (q, k, v, do))
    o, lse = A.attn_forward(qd, kd, vd, plan)
    torch.cuda.synchronize()
    pos = np.arange(T)
    o_ref, lse_ref = attention_ref.attention_fwd(q, k, v, desc, pos)
    assert_close("O", o, o_ref)
    assert max_abs(lse, lse_ref) <= 2e-3, f"LSE max-abs {max_abs(lse, lse_ref):.3e}"
    if not check_bwd:
        return
    dq, dk, dv = A.attn_backward(qd, kd, vd, o, lse, dod, plan, dkv_fp32=True)
    torch.cuda.synchronize()
    dq_ref, dk_ref, dv_ref = attention_ref.attention_bwd(q, k, v, o_ref, lse_ref, do, desc, pos)
    assert_close("dQ", dq, dq_ref)
    assert_close("dK", dk, dk_ref)
    assert_close("dV", dv, dv_ref)


def test_selftest_umma():
    from paper_2503_11367_b200 import _lib

    g = torch.Generator().manual_seed(7)
    a, b, v, x = (torch.randn(128, 128, generator=g).to(torch.bfloat16) for _ in range(4))
    dev = torch.device("cuda")
    out = torch.empty(3, 128, 128, dtype=torch.float32, device=dev)
    ad, bd, vd, xd = (t.to(dev) for t in (a, b, v, x))
    _lib.call("bam_selftest_umma", ad.data_ptr(), bd.data_ptr(), vd.data_ptr(), xd.data_ptr(),
              out.data_ptr())
    torch.cuda.synchronize()
    out = out.cpu()
    af, bf, vf, xf = (t.float() for t in (a, b, v, x))
    for i, ref in enumerate((af @ bf.t(), af @ vf, xf.t() @ vf)):
        err = (out[i] - ref).abs().max().item()
        assert err < 1e-2, f"selftest mode {i}: max err {err}"


def test_text_image_small():
    desc, _ = mask_ref.build_bitfield([("text", 128), ("image", 256), ("text", 384)])
    run_case(desc, 4, 2)


def test_causal_small_gqa():
    desc, _ = mask_ref.build_bitfield([("text", 1024)])
    run_case(desc, 8, 2)


def test_multimodal_partial_tiles():
    # non-aligned segments: many PARTIAL tiles, segments split across blocks
    desc, _ = mask_ref.build_bitfield([("text", 100), ("vision", 300), ("text", 77),
                                       ("audio", 211), ("text", 120), ("vision", 88),
                                       ("text", 128)])
    run_case(desc, 2, 2)


def test_prefix_lm_small_gqa():
    # config 5's prefix-LM pattern at 1K: bidirectional prefix, causal text
    desc, _ = mask_ref.build_bitfield([("prefix", 256), ("text", 768)])
    run_case(desc, 8, 2)


def test_emu_interleave_small_gqa():
    # config 4's pattern at 1K: distinct image names (bidirectional within one
    # image only), images not block-aligned, GQA 4 query heads per KV head
    desc, _ = mask_ref.build_bitfield([("text", 128), ("img0", 256), ("text", 64),
                                       ("img1", 192), ("text", 128), ("img2", 128),
                                       ("text", 128)])
    run_case(desc, 8, 2, seed=99)


def test_raw_descriptors():
    rng = np.random.default_rng(5)
    T = 768
    desc = []
    while len(desc) < T:
        run = int(rng.integers(1, 90))
        if rng.random() < 0.5:
            d = 1 | int(sum(2 << j for j in range(3) if rng.random() < 0.5))
        else:
            d = 2 << int(rng.integers(0, 3))
        desc += [d] * min(run, T - len(desc))
    run_case(desc, 2, 1)


def test_config1_full():
    # BASELINE.json config 1: 1 image + text, 4K, 8 heads
    desc, _ = mask_ref.build_bitfield([("text", 128), ("image", 1024), ("text", 2944)])
    run_case(desc, 8, 8)


def test_autograd_function():
    from paper_2503_11367_b200 import attention as A
    from paper_2503_11367_b200 import mask as M

    mask = M.build_bitfield([("text", 256), ("image", 256), ("text", 256)])
    q, k, v, do = inputs(768, 4, 4, seed=3)
    dev = torch.device("cuda")
    qd, kd, vd = (t.to(dev).requires_grad_(True) for t in (q, k, v))
    o = A.bitfield_attention(qd, kd, vd, mask)
    o.backward(do.to(dev))
    desc = np.asarray(mask.descriptors, dtype=np.int64)
    o_ref, q_g, k_g, v_g = attention_ref.attention_dense_autograd(q, k, v, do, desc, np.arange(768))
    assert_close("O", o.detach(), o_ref)
    assert_close("dQ", qd.grad, q_g)
    assert_close("dK", kd.grad, k_g)
    assert_close("dV", vd.grad, v_g)


@pytest.mark.parametrize("cfg_id", [2, 4])
def test_repeat_bitwise_deterministic(cfg_id):
    """Race detector: O, LSE, dK, dV have no atomics, so repeated runs on the
    same inputs must agree bit for bit (dQ uses fp32 reductions and may not)."""
    from paper_2503_11367_b200 import attention as A, mask as M
    from paper_2503_11367_b200.workloads import CONFIGS

    cfg = CONFIGS[cfg_id]
    mask = M.build_bitfield(cfg["segments"])
    plan = A.plan_for_mask(mask)
    T, dev = len(mask), torch.device("cuda")
    g = torch.Generator(device=dev).manual_seed(99)
    q = torch.randn(T, cfg["Hq"], 128, device=dev, generator=g, dtype=torch.bfloat16)
    k = torch.randn(T, cfg["Hkv"], 128, device=dev, generator=g, dtype=torch.bfloat16)
    v = torch.randn(T, cfg["Hkv"], 128, device=dev, generator=g, dtype=torch.bfloat16)
    do = torch.randn(T, cfg["Hq"], 128, device=dev, generator=g, dtype=torch.bfloat16)
    ref = None
    for _ in range(3):
        o, lse = A.attn_forward(q, k, v, plan)
        _, dk, dv = A.attn_backward(q, k, v, o, lse, do, plan, dkv_fp32=True)
        cur = [t.clone() for t in (o, lse, dk, dv)]
        if ref is None:
            ref = cur
        else:
            for name, a, b in zip(("O", "LSE", "dK", "dV"), cur, ref):
                assert torch.equal(a, b), f"{name} differs between identical runs (race?)"


@pytest.mark.parametrize("subblock", [1, 3, 8])
def test_split_kv_schedule_matches_whole_rows(subblock):
    """Intra-GPU subblocks (split-KV + aggregation kernel) against the fp32
    oracle (the north-star tolerance), and against the whole-row forward
    (fp32 partial merge: within bf16 rounding)."""
    from paper_2503_11367_b200 import attention as A, mask as M

    for Hq, Hkv in ((4, 2), (2, 2)):     # GQA pair kernel and the MHA kernel
        mask = M.build_bitfield([("text", 300), ("img0", 256), ("text", 500), ("img1", 200),
                                 ("text", 280)])
        plan = A.plan_for_mask(mask)
        T, dev = len(mask), torch.device("cuda")
        q, k, v, _ = inputs(T, Hq, Hkv, seed=7)
        qd, kd, vd = (t.to(dev) for t in (q, k, v))
        o, lse = A.attn_forward(qd, kd, vd, plan)
        sched = A.build_split_schedule(plan, subblock)
        assert sched.n_slots > 0 or subblock >= 8
        o2, lse2 = A.attn_forward(qd, kd, vd, plan, schedule=sched)
        desc = np.asarray(mask.descriptors, np.int64)
        o_ref, lse_ref = attention_ref.attention_fwd(q, k, v, desc, np.arange(T))
        assert_close(f"O split s={subblock} Hq={Hq}", o2, o_ref)
        assert max_abs(lse2.cpu(), lse_ref) <= 2e-3
        assert (o2.float() - o.float()).abs().max().item() < 1e-2
        assert (lse2 - lse).abs().max().item() < 1e-3
        # the schedule is the reference split_block / LPT piece order
        sizes = (sched.items[:, 2] - sched.items[:, 1]).cpu().tolist()
        assert sizes == sorted(sizes, reverse=True)
        assert max(sizes) <= subblock


def test_fwd_cta_pair_kernel_matches_one_cta():
    """The cta_group::2 forward (shared query-block pairs, union tile lists,
    K/V split across the two SMs) against the one-CTA head-pair kernel."""
    import os
    from paper_2503_11367_b200 import attention as A, mask as M

    segs = [("text", 384), ("img0", 512), ("text", 256), ("img1", 1024), ("text", 640)]
    mask = M.build_bitfield(segs)
    plan = A.plan_for_mask(mask)
    assert int(plan.counts[0]) > 0                # some pairs run on CTA pairs
    T, Hq, Hkv = len(mask), 8, 2
    dev = torch.device("cuda")
    g = torch.Generator(device=dev).manual_seed(21)
    q = torch.randn(T, Hq, 128, device=dev, generator=g, dtype=torch.bfloat16)
    k = torch.randn(T, Hkv, 128, device=dev, generator=g, dtype=torch.bfloat16)
    v = torch.randn(T, Hkv, 128, device=dev, generator=g, dtype=torch.bfloat16)
    old = os.environ.get("BAM_FWD_2CTA")
    try:
        os.environ["BAM_FWD_2CTA"] = "0"
        o1, l1 = A.attn_forward(q, k, v, plan)
        os.environ["BAM_FWD_2CTA"] = "1"
        o2, l2 = A.attn_forward(q, k, v, plan)
    finally:
        if old is None:
            os.environ.pop("BAM_FWD_2CTA", None)
        else:
            os.environ["BAM_FWD_2CTA"] = old
    torch.cuda.synchronize()
    assert (o1.float() - o2.float()).abs().max().item() < 1e-2
    assert (l1 - l2).abs().max().item() < 1e-3


def test_fwd_query_block_pairs_match_one_head_kernel():
    """MHA forward on query-block pairs (split-row CTA sharing K/V tiles over
    a union tile list) against the one-head kernel."""
    import os
    from paper_2503_11367_b200 import attention as A, mask as M

    segs = [("text", 384), ("img0", 512), ("text", 256), ("img1", 1024), ("text", 640)]
    mask = M.build_bitfield(segs)
    plan = A.plan_for_mask(mask)
    assert int(plan.counts[0]) > 0
    T, H = len(mask), 3
    dev = torch.device("cuda")
    g = torch.Generator(device=dev).manual_seed(22)
    q, k, v = (torch.randn(T, H, 128, device=dev, generator=g, dtype=torch.bfloat16)
               for _ in range(3))
    old = os.environ.get("BAM_FWD_QPAIRS")
    try:
        os.environ["BAM_FWD_QPAIRS"] = "0"
        o1, l1 = A.attn_forward(q, k, v, plan)
        os.environ["BAM_FWD_QPAIRS"] = "1"
        o2, l2 = A.attn_forward(q, k, v, plan)
    finally:
        if old is None:
            os.environ.pop("BAM_FWD_QPAIRS", None)
        else:
            os.environ["BAM_FWD_QPAIRS"] = old
    torch.cuda.synchronize()
    assert (o1.float() - o2.float()).abs().max().item() < 1e-2
    assert (l1 - l2).abs().max().item() < 1e-3


@pytest.mark.parametrize("Hq,Hkv", [(8, 2), (4, 4)])
def test_head_major_kv_matches_token_major(Hq, Hkv):
    """Head-major K/V [Hkv, T, 128] (the copy-engine CP gather's layout; only
    the TMA strides change) give bit-identical O, LSE, dK, dV to token-major
    K/V, for the GQA head-pair and the MHA query-pair / one-head kernels; the
    head-major dK/dV partial layout is the same numbers transposed."""
    from paper_2503_11367_b200 import attention as A, mask as M

    mask = M.build_bitfield([("text", 128), ("image", 1024), ("text", 2944)])
    plan = A.plan_for_mask(mask)
    T, dev = len(mask), torch.device("cuda")
    g = torch.Generator(device=dev).manual_seed(5)
    q = torch.randn(T, Hq, 128, device=dev, generator=g, dtype=torch.bfloat16)
    k = torch.randn(T, Hkv, 128, device=dev, generator=g, dtype=torch.bfloat16)
    v = torch.randn(T, Hkv, 128, device=dev, generator=g, dtype=torch.bfloat16)
    do = torch.randn(T, Hq, 128, device=dev, generator=g, dtype=torch.bfloat16)
    kh, vh = k.transpose(0, 1).contiguous(), v.transpose(0, 1).contiguous()
    o, lse = A.attn_forward(q, k, v, plan)
    oh, lseh = A.attn_forward(q, kh, vh, plan, kv_head_major=True)
    assert torch.equal(o, oh) and torch.equal(lse, lseh)
    ws = A.BackwardWorkspace(q, o, lse, do, plan, None)
    dk, dv = ws.main(k, v)
    ws.finalize()
    wsh = A.BackwardWorkspace(q, o, lse, do, plan, None)
    dkh, dvh = wsh.main(kh, vh, kv_head_major=True)
    wsh.finalize()
    assert torch.equal(dk, dkh) and torch.equal(dv, dvh)
    with pytest.raises(ValueError, match="head-major"):
        A.attn_forward(q, k, v, plan, kv_head_major=True)


def test_fwd_class_order_matches_head_pair_major():
    """The forward's class-major CTA order (BamAttnFwdParams.order_classes):
    the planner's geometric classes over the heavy-first order are the
    floor(log2(n_max / n)) ranges, and the kernel walked in that order writes
    bit-identical O / LSE to the head-pair-major order (it only reorders CTAs)."""
    import os
    from paper_2503_11367_b200 import attention as A, mask as M
    from paper_2503_11367_b200.workloads import emu_interleave

    mask = M.build_bitfield(emu_interleave(16 * 1024, seed=3))
    plan = A.plan_for_mask(mask)
    cnt = plan.row_cnt.cpu().numpy()[plan.fwd_order.cpu().numpy()]
    assert np.all(np.diff(cnt) <= 0)
    k_cls = np.array([min(int(cnt[0] // c).bit_length() - 1, 15) if c > 0 else 15 for c in cnt])
    want = [int(np.searchsorted(k_cls, c, side="left")) for c in range(16)] + [len(cnt)]
    got = plan.fwd_classes.cpu().tolist()
    assert got == want, (got, want)
    assert len(set(k_cls.tolist())) >= 3          # several classes present
    # shared query-block pairs (MHA): heavy-first by union length, then classes
    n_sh = int(plan.counts[0])
    assert n_sh > 1
    F = plan.fwd_pair_ids.shape[0]
    pid = plan.fwd_pair_ids.cpu().numpy()
    slot_off = plan.fwd_slot_off.cpu().numpy()
    w = np.array([slot_off[2 * pr + 1] - slot_off[2 * pr] for pr in pid[:n_sh]])
    assert np.all(np.diff(w) <= 0) and w[-1] > 0
    wk = [min(int(w[0] // c).bit_length() - 1, 15) for c in w] + [15] * (F - n_sh)
    want = [int(np.searchsorted(np.array(wk), c, side="left")) for c in range(16)] + [F]
    assert plan.fwd_pair_classes.cpu().tolist() == want
    dev = torch.device("cuda")
    for Hq, Hkv in ((8, 2), (2, 2)):     # GQA head pairs; MHA query-block pairs + rest
        T = len(mask)
        g = torch.Generator(device=dev).manual_seed(5)
        q = torch.randn(T, Hq, 128, device=dev, generator=g, dtype=torch.bfloat16)
        k = torch.randn(T, Hkv, 128, device=dev, generator=g, dtype=torch.bfloat16)
        v = torch.randn(T, Hkv, 128, device=dev, generator=g, dtype=torch.bfloat16)
        old = os.environ.get("BAM_FWD_CLASS_ORDER")
        try:
            os.environ["BAM_FWD_CLASS_ORDER"] = "0"
            o0, l0 = A.attn_forward(q, k, v, plan)
            os.environ["BAM_FWD_CLASS_ORDER"] = "1"
            o1, l1 = A.attn_forward(q, k, v, plan)
        finally:
            if old is None:
                os.environ.pop("BAM_FWD_CLASS_ORDER", None)
            else:
                os.environ["BAM_FWD_CLASS_ORDER"] = old
        torch.cuda.synchronize()
        assert torch.equal(o0, o1) and torch.equal(l0, l1), (Hq, Hkv)


def test_bwd_cta_pairs_match_single_ctas():
    """Backward CTA pairs (clusters of 2 multicasting Q/dO over union step lists,
    class 0 where a key block does not see the query block) against one CTA per
    key block (BAM_BWD_PAIRS=0): dK / dV bit-identical (a class-0 step adds exact
    zeros, the step order per key block is the same), dQ within fp32 reduction
    order."""
    import os
    from paper_2503_11367_b200 import attention as A, mask as M
    from paper_2503_11367_b200.workloads import emu_interleave

    mask = M.build_bitfield(emu_interleave(8 * 1024, seed=5))
    plan = A.plan_for_mask(mask)
    assert int(plan.pair_shared.sum()) > 0
    T, Hq, Hkv = len(mask), 4, 2
    dev = torch.device("cuda")
    g = torch.Generator(device=dev).manual_seed(8)
    q, do = (torch.randn(T, Hq, 128, device=dev, generator=g, dtype=torch.bfloat16)
             for _ in range(2))
    k, v = (torch.randn(T, Hkv, 128, device=dev, generator=g, dtype=torch.bfloat16)
            for _ in range(2))
    o, lse = A.attn_forward(q, k, v, plan)
    out = {}
    old = os.environ.get("BAM_BWD_PAIRS")
    try:
        for mode in ("1", "0"):
            os.environ["BAM_BWD_PAIRS"] = mode
            out[mode] = A.attn_backward(q, k, v, o, lse, do, plan, dkv_fp32=True)
    finally:
        if old is None:
            os.environ.pop("BAM_BWD_PAIRS", None)
        else:
            os.environ["BAM_BWD_PAIRS"] = old
    torch.cuda.synchronize()
    (dq1, dk1, dv1), (dq0, dk0, dv0) = out["1"], out["0"]
    assert torch.equal(dk1, dk0) and torch.equal(dv1, dv0)
    assert rel_l2(dq1, dq0) < 1e-3

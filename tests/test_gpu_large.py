"""Full-size (BASELINE.json configs 2-4, 32K-128K) GPU parity through checks
the fp32 oracle can afford:

* tile classes and W: bit-exact against the C restatement of
  block_workloads (oracle/c/bam_oracle.c);
* O, LSE and dQ on sampled query blocks (all heads): the oracle computes
  exactly those rows against all keys;
* dK, dV on sampled key blocks: the oracle sums the contributions of every
  query row whose tile with that key block is non-skip, using the kernel's
  (sample-validated) LSE and O for the softmax normaliser and D = rowsum(dO*O).

Tolerance as everywhere: max-abs 2e-2, relative-L2 1e-2 (bf16 vs fp32).
"""

import math

import numpy as np
import pytest
import torch

from oracle import attention_ref, mask_ref

pytestmark = pytest.mark.gpu

MAX_ABS, REL_L2 = 2e-2, 1e-2


def check(name, got, ref):
    got, ref = got.float().cpu(), ref.float().cpu()
    ma = (got - ref).abs().max().item()
    rl = ((got - ref).norm() / ref.norm().clamp_min(1e-12)).item()
    assert ma <= MAX_ABS and rl <= REL_L2, f"{name}: max-abs {ma:.3e} rel-L2 {rl:.3e}"


@pytest.mark.parametrize("cfg_id", [2, 3, 4])
def test_full_size_config(cfg_id):
    from paper_2503_11367_b200.workloads import CONFIGS

    cfg = CONFIGS[cfg_id]
    _full_size_parity(cfg["segments"], cfg["Hq"], cfg["Hkv"])


@pytest.mark.parametrize("name", ["causal", "prefix_lm", "multimodal"])
def test_full_size_sweep_128k(name):
    """BASELINE.json config 5: the 128K mask sweep at GQA 32q/8kv (multi_image
    is config 4 above).  The causal mask exercises 1024-entry tile lists."""
    from paper_2503_11367_b200.workloads import SWEEP_128K

    _full_size_parity(SWEEP_128K[name], 32, 8)


def _full_size_parity(segments, Hq, Hkv):
    from paper_2503_11367_b200 import attention as A, mask as M

    grp = Hq // Hkv
    mask = M.build_bitfield(segments)
    desc_d = mask.device_descriptors()
    T = desc_d.shape[0]
    nb = T // 128
    desc = desc_d.cpu().numpy()
    plan = A.build_plan(desc_d)

    ref_cls, ref_w = mask_ref.block_workloads_c(desc, 128)
    assert np.array_equal(plan.classes.cpu().numpy(), ref_cls)
    assert np.array_equal(plan.W.cpu().numpy(), ref_w)

    dev = torch.device("cuda")
    g = torch.Generator(device=dev).manual_seed(1234)
    q = torch.randn(T, Hq, 128, device=dev, generator=g, dtype=torch.bfloat16)
    k = torch.randn(T, Hkv, 128, device=dev, generator=g, dtype=torch.bfloat16)
    v = torch.randn(T, Hkv, 128, device=dev, generator=g, dtype=torch.bfloat16)
    do = torch.randn(T, Hq, 128, device=dev, generator=g, dtype=torch.bfloat16)
    o, lse = A.attn_forward(q, k, v, plan)
    dq, dk, dv = A.attn_backward(q, k, v, o, lse, do, plan, dkv_fp32=True)
    torch.cuda.synchronize()
    kc, vc = k.cpu(), v.cpu()

    # sampled query blocks: first, middle, last, and the heaviest row
    qblocks = sorted({0, nb // 2, nb - 1, int(np.argmax(ref_w))})
    rows = np.concatenate([np.arange(b * 128, (b + 1) * 128) for b in qblocks])
    rows_t = torch.from_numpy(rows)
    q_s, do_s = q.cpu()[rows_t], do.cpu()[rows_t]
    o_ref, lse_ref = attention_ref.attention_fwd(q_s, kc, vc, desc, rows)
    check("O", o.cpu()[rows_t], o_ref)
    assert (lse.cpu()[:, rows_t] - lse_ref).abs().max().item() <= 2e-3
    dq_ref, _, _ = attention_ref.attention_bwd(q_s, kc, vc, o_ref, lse_ref, do_s, desc, rows)
    check("dQ", dq.cpu()[rows_t], dq_ref)

    # sampled key blocks: contributions of every query row whose tile is non-skip
    scale = 1.0 / math.sqrt(128)
    kblocks = sorted({0, nb // 3, nb - 1})
    lse_c, o_c, q_c, do_c = lse.cpu(), o.cpu().float(), q.cpu().float(), do.cpu().float()
    for kb in kblocks:
        qb = np.nonzero(ref_cls[:, kb])[0]
        qrows = torch.from_numpy(np.concatenate([np.arange(b * 128, (b + 1) * 128) for b in qb]))
        keys = torch.arange(kb * 128, (kb + 1) * 128)
        allow = torch.from_numpy(mask_ref.dense_rows(desc, qrows.numpy(), keys.numpy()))
        dk_ref = torch.zeros(128, Hkv, 128)
        dv_ref = torch.zeros(128, Hkv, 128)
        for h in range(Hq):
            hk = h // grp
            Qh, dOh = q_c[qrows, h], do_c[qrows, h]
            Kh, Vh = kc[keys, hk].float(), vc[keys, hk].float()
            s = (Qh @ Kh.t()) * scale
            p = torch.exp(s - lse_c[h, qrows][:, None]).masked_fill(~allow, 0.0)
            dp = dOh @ Vh.t()
            D = (dOh * o_c[qrows, h]).sum(-1, keepdim=True)
            ds = p * (dp - D)
            dv_ref[:, hk] += p.t() @ dOh
            dk_ref[:, hk] += (ds.t() @ Qh) * scale
        check(f"dK[kb={kb}]", dk.cpu()[keys], dk_ref)
        check(f"dV[kb={kb}]", dv.cpu()[keys], dv_ref)


def test_full_dkdv_one_kv_group_config4():
    """SURVEY.md 8(d)'s full-size recipe for dK/dV: the complete dK and dV of one
    KV-head group (the last one: 4 query heads) at config 4 (128K), against an
    independent fp32 oracle pass -- its own forward (O, LSE) and backward per
    query block, blockwise-sparse over that row's non-skip key tiles
    (PAPER.md:616-619), the contributions summed at their key positions."""
    from paper_2503_11367_b200 import attention as A, mask as M
    from paper_2503_11367_b200.workloads import CONFIGS

    cfg = CONFIGS[4]
    Hq, Hkv = cfg["Hq"], cfg["Hkv"]
    grp, hk = Hq // Hkv, Hkv - 1
    mask = M.build_bitfield(cfg["segments"])
    desc_d = mask.device_descriptors()
    T = desc_d.shape[0]
    nb = T // 128
    desc = desc_d.cpu().numpy()
    plan = A.build_plan(desc_d)
    cls = plan.classes.cpu().numpy()
    dev = torch.device("cuda")
    g = torch.Generator(device=dev).manual_seed(4321)
    q = torch.randn(T, Hq, 128, device=dev, generator=g, dtype=torch.bfloat16)
    k = torch.randn(T, Hkv, 128, device=dev, generator=g, dtype=torch.bfloat16)
    v = torch.randn(T, Hkv, 128, device=dev, generator=g, dtype=torch.bfloat16)
    do = torch.randn(T, Hq, 128, device=dev, generator=g, dtype=torch.bfloat16)
    o, lse = A.attn_forward(q, k, v, plan)
    _, dk, dv = A.attn_backward(q, k, v, o, lse, do, plan, dkv_fp32=True)
    torch.cuda.synchronize()
    heads = slice(hk * grp, (hk + 1) * grp)
    qg, dog = q[:, heads].cpu(), do[:, heads].cpu()
    kg, vg = k[:, hk:hk + 1].cpu(), v[:, hk:hk + 1].cpu()
    dk_ref = torch.zeros(T, 128)
    dv_ref = torch.zeros(T, 128)
    for j in range(nb):
        kbs = np.nonzero(cls[j])[0]
        if kbs.size == 0:
            continue
        keys = np.concatenate([np.arange(b * 128, (b + 1) * 128) for b in kbs])
        rows = np.arange(j * 128, (j + 1) * 128)
        kt, rt = torch.from_numpy(keys), torch.from_numpy(rows)
        o_r, lse_r = attention_ref.attention_fwd(qg[rt], kg[kt], vg[kt], desc, rows, chunk=128,
                                                 k_pos=keys)
        _, dk_r, dv_r = attention_ref.attention_bwd(qg[rt], kg[kt], vg[kt], o_r, lse_r, dog[rt],
                                                    desc, rows, chunk=128, k_pos=keys)
        dk_ref[kt] += dk_r[:, 0]
        dv_ref[kt] += dv_r[:, 0]
    check(f"dK[kv head {hk}, all {T} keys]", dk.cpu()[:, hk], dk_ref)
    check(f"dV[kv head {hk}, all {T} keys]", dv.cpu()[:, hk], dv_ref)


def test_full_parity_config2():
    """full oracle parity at config 2 (32K image prefix + causal
    text, 32/32 heads): O, LSE and dQ of every row and dK / dV of every key,
    against an independent fp32 oracle pass per query block, blockwise-sparse
    over the row's non-skip key tiles."""
    from paper_2503_11367_b200 import attention as A, mask as M
    from paper_2503_11367_b200.workloads import CONFIGS

    cfg = CONFIGS[2]
    Hq, Hkv = cfg["Hq"], cfg["Hkv"]
    mask = M.build_bitfield(cfg["segments"])
    desc_d = mask.device_descriptors()
    T = desc_d.shape[0]
    nb = T // 128
    desc = desc_d.cpu().numpy()
    plan = A.build_plan(desc_d)
    cls = plan.classes.cpu().numpy()
    dev = torch.device("cuda")
    g = torch.Generator(device=dev).manual_seed(2468)
    q = torch.randn(T, Hq, 128, device=dev, generator=g, dtype=torch.bfloat16)
    k = torch.randn(T, Hkv, 128, device=dev, generator=g, dtype=torch.bfloat16)
    v = torch.randn(T, Hkv, 128, device=dev, generator=g, dtype=torch.bfloat16)
    do = torch.randn(T, Hq, 128, device=dev, generator=g, dtype=torch.bfloat16)
    o, lse = A.attn_forward(q, k, v, plan)
    dq, dk, dv = A.attn_backward(q, k, v, o, lse, do, plan, dkv_fp32=True)
    torch.cuda.synchronize()
    qc, kc, vc, doc = q.cpu(), k.cpu(), v.cpu(), do.cpu()
    o_ref, lse_ref, dq_ref = torch.empty(T, Hq, 128), torch.empty(Hq, T), torch.empty(T, Hq, 128)
    dk_ref, dv_ref = torch.zeros(T, Hkv, 128), torch.zeros(T, Hkv, 128)
    for j in range(nb):
        kbs = np.nonzero(cls[j])[0]
        keys = np.concatenate([np.arange(b * 128, (b + 1) * 128) for b in kbs])
        rows = np.arange(j * 128, (j + 1) * 128)
        kt, rt = torch.from_numpy(keys), torch.from_numpy(rows)
        o_r, lse_r = attention_ref.attention_fwd(qc[rt], kc[kt], vc[kt], desc, rows, chunk=128,
                                                 k_pos=keys)
        dq_r, dk_r, dv_r = attention_ref.attention_bwd(qc[rt], kc[kt], vc[kt], o_r, lse_r,
                                                       doc[rt], desc, rows, chunk=128, k_pos=keys)
        o_ref[rt], lse_ref[:, rt], dq_ref[rt] = o_r, lse_r, dq_r
        dk_ref[kt] += dk_r
        dv_ref[kt] += dv_r
    check("O (all rows)", o.cpu(), o_ref)
    assert (lse.cpu() - lse_ref).abs().max().item() <= 2e-3
    check("dQ (all rows)", dq.cpu(), dq_ref)
    check("dK (all keys)", dk.cpu(), dk_ref)
    check("dV (all keys)", dv.cpu(), dv_ref)

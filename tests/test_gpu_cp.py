"""GPU parity of the context-parallel plan on one device: CP ranks are
emulated one after another (the ranks' kernels never wait on each other, the
only exchange is NCCL), with the all-gather replaced by placing every global
block at its gathered row and the reduce-scatter by summing the partials.
Exercises the non-identity q_gid / k_row mappings of the kernels for every
distribution policy.  The real NCCL path runs under torchrun in
tools/cp_check.py and bench.py --gpus N."""

import numpy as np
import pytest
import torch

from oracle import attention_ref, mask_ref

pytestmark = pytest.mark.gpu

BLOCK = 128


def rel_l2(a, b):
    a, b = a.float().cpu(), b.float().cpu()
    return ((a - b).norm() / b.norm()).item()


@pytest.mark.parametrize("policy,world,Hq,Hkv", [("lpt", 4, 4, 2), ("zigzag", 2, 4, 2),
                                                 ("contiguous", 3, 4, 2), ("lpt", 3, 3, 3)])
def test_cp_emulated_ranks(policy, world, Hq, Hkv):
    from paper_2503_11367_b200 import attention as A
    from paper_2503_11367_b200 import cp

    segs = [("text", 256), ("img0", 512), ("text", 384), ("img1", 256), ("text", 640)]
    desc_l, _ = mask_ref.build_bitfield(segs)
    desc = np.asarray(desc_l, np.int64)
    T = desc.shape[0]
    g = torch.Generator().manual_seed(1234)
    q = torch.randn(T, Hq, 128, generator=g).to(torch.bfloat16)
    k = torch.randn(T, Hkv, 128, generator=g).to(torch.bfloat16)
    v = torch.randn(T, Hkv, 128, generator=g).to(torch.bfloat16)
    do = torch.randn(T, Hq, 128, generator=g).to(torch.bfloat16)
    dev = torch.device("cuda")
    d_desc = torch.from_numpy(desc).to(dev)
    qd, kd, vd, dod = (t.to(dev) for t in (q, k, v, do))
    o_ref, lse_ref = attention_ref.attention_fwd(q, k, v, desc, np.arange(T))
    dq_ref, dk_ref, dv_ref = attention_ref.attention_bwd(q, k, v, o_ref, lse_ref, do, desc,
                                                         np.arange(T))
    dk_sum = torch.zeros(T, Hkv, 128)
    dv_sum = torch.zeros(T, Hkv, 128)
    loads = []
    for rank in range(world):
        plan = cp.make_cp_plan(d_desc, world, rank, policy)
        lay = plan.layout
        loads.append(plan.assignment.loads.cpu().tolist())
        krow = lay.k_row.to(torch.int64)
        idx = (krow[:, None] * BLOCK + torch.arange(BLOCK, device=dev)[None, :]).reshape(-1)
        rows = world * lay.max_blocks * BLOCK
        k_all = torch.zeros(rows, Hkv, 128, dtype=torch.bfloat16, device=dev)
        v_all = torch.zeros_like(k_all)
        k_all[idx] = kd
        v_all[idx] = vd
        q_loc, do_loc = cp.shard_rows(qd, lay).contiguous(), cp.shard_rows(dod, lay).contiguous()
        o, lse = A.attn_forward(q_loc, k_all, v_all, plan.attn)
        dq, dk_all, dv_all = A.attn_backward(q_loc, k_all, v_all, o, lse, do_loc, plan.attn,
                                             dkv_fp32=True)
        torch.cuda.synchronize()
        pos = (lay.local_blocks.cpu().to(torch.int64)[:, None] * BLOCK +
               torch.arange(BLOCK)[None, :]).reshape(-1)
        assert rel_l2(o, o_ref[pos]) < 1e-2
        assert (o.float().cpu() - o_ref[pos]).abs().max() < 2e-2
        assert rel_l2(dq, dq_ref[pos]) < 1e-2
        dk_sum += dk_all[idx].cpu()
        dv_sum += dv_all[idx].cpu()
    assert rel_l2(dk_sum, dk_ref) < 1e-2 and (dk_sum - dk_ref).abs().max() < 2e-2
    assert rel_l2(dv_sum, dv_ref) < 1e-2 and (dv_sum - dv_ref).abs().max() < 2e-2
    # the device assignment is the reference policy, bit-exact
    from oracle import balance_ref
    _, W = mask_ref.block_workloads_np(desc, BLOCK)
    ref = {"lpt": balance_ref.lpt, "zigzag": balance_ref.zigzag,
           "contiguous": balance_ref.contiguous}[policy](list(W), world)
    assert tuple(loads[0]) == ref[1]


def test_head_groups_match_full():
    """The CP pipeline runs attention per KV-head group (h_begin / nh): each
    group must reproduce the full launch's heads exactly (O, LSE, dK, dV bit
    for bit; dQ up to fp32 reduction order)."""
    from paper_2503_11367_b200 import attention as A
    from paper_2503_11367_b200 import mask as M

    mask = M.build_bitfield([("text", 384), ("img0", 512), ("text", 640), ("img1", 256)])
    plan = A.plan_for_mask(mask)
    T, Hq, Hkv = len(mask), 8, 4
    dev = torch.device("cuda")
    g = torch.Generator(device=dev).manual_seed(5)
    q = torch.randn(T, Hq, 128, device=dev, generator=g, dtype=torch.bfloat16)
    k = torch.randn(T, Hkv, 128, device=dev, generator=g, dtype=torch.bfloat16)
    v = torch.randn(T, Hkv, 128, device=dev, generator=g, dtype=torch.bfloat16)
    do = torch.randn(T, Hq, 128, device=dev, generator=g, dtype=torch.bfloat16)
    o, lse = A.attn_forward(q, k, v, plan)
    dq, dk, dv = A.attn_backward(q, k, v, o, lse, do, plan, dkv_fp32=True)
    og, lg = torch.empty_like(o), torch.empty_like(lse)
    ws = None
    grp = Hq // Hkv
    parts = []
    for kv0, nkv in ((0, 2), (2, 2)):
        kg, vg = k[:, kv0:kv0 + nkv].contiguous(), v[:, kv0:kv0 + nkv].contiguous()
        A.attn_forward(q, kg, vg, plan, h_begin=kv0 * grp, nh=nkv * grp, out=(og, lg))
    assert torch.equal(og, o) and torch.equal(lg, lse)
    ws = A.BackwardWorkspace(q, o, lse, do, plan, None)
    for kv0, nkv in ((0, 2), (2, 2)):
        kg, vg = k[:, kv0:kv0 + nkv].contiguous(), v[:, kv0:kv0 + nkv].contiguous()
        parts.append(ws.main(kg, vg, h_begin=kv0 * grp, nh=nkv * grp))
    dqg = ws.finalize()
    assert torch.equal(torch.cat([p[0] for p in parts], 1), dk)
    assert torch.equal(torch.cat([p[1] for p in parts], 1), dv)
    assert (dqg.float() - dq.float()).abs().max().item() < 1e-2


def test_permute_blocks_gather_scatter_bit_exact():
    """Token permutation kernel (bam_permute_blocks): gather of several
    tensors in one launch and the inverse scatter, against plain indexing."""
    from paper_2503_11367_b200 import cp

    dev = torch.device("cuda")
    g = torch.Generator(device=dev).manual_seed(7)
    nb = 37
    T = nb * BLOCK
    owner = torch.randint(0, 3, (nb,), generator=g, device=dev, dtype=torch.int32)
    lay = cp.cp_layout(owner, 3, 1)
    q = torch.randn(T, 4, 128, device=dev, generator=g).to(torch.bfloat16)
    k = torch.randn(T, 2, 128, device=dev, generator=g).to(torch.bfloat16)
    w = torch.randn(T, 3, 8, device=dev, generator=g)           # fp32, 96-B rows
    rows = (lay.local_blocks.to(torch.int64)[:, None] * BLOCK +
            torch.arange(BLOCK, device=dev)[None, :]).reshape(-1)
    ql, kl, wl = cp.shard_rows(q, k, w, layout=lay)
    assert torch.equal(ql, q[rows]) and torch.equal(kl, k[rows]) and torch.equal(wl, w[rows])
    assert torch.equal(cp.shard_rows(q, lay), q[rows])
    out = torch.zeros_like(q)
    cp.unshard_rows(ql, lay, out)
    ref = torch.zeros_like(q)
    ref[rows] = q[rows]
    assert torch.equal(out, ref)
    # every rank's shard scattered back reassembles the sequence
    full = torch.empty_like(k)
    for r in range(3):
        lr = cp.cp_layout(owner, 3, r)
        cp.unshard_rows(cp.shard_rows(k, lr), lr, full)
    assert torch.equal(full, k)
    # misaligned rows are rejected with the library's message
    from paper_2503_11367_b200 import _lib
    bad = torch.zeros(T, 3, device=dev, dtype=torch.bfloat16)   # 6-B rows
    with pytest.raises(_lib.BamError, match="16-byte"):
        cp.shard_rows(bad, lay)


@pytest.mark.parametrize("head_major", [False, True])
def test_reduce_partials_bf16_bit_exact(head_major):
    """dK/dV reduce-scatter tail (bam_reduce_partials_bf16): the sum of the world
    partials in order, rounded to bf16, for both workspace layouts, bit-exact
    against sequential fp32 adds + torch's bf16 rounding; padded rows dropped."""
    from paper_2503_11367_b200 import _lib

    dev = torch.device("cuda")
    g = torch.Generator(device=dev).manual_seed(11)
    world, nkv, rows, n_local, d = 3, 5, 3 * BLOCK, 2 * BLOCK + 64, 128
    shape = (world, 2, nkv, rows, d) if head_major else (world, 2, rows, nkv, d)
    ws = torch.randn(shape, device=dev, generator=g) * 100
    acc = ws[0].clone()
    for p in range(1, world):
        acc = acc + ws[p]
    if head_major:
        acc = acc.transpose(1, 2)          # [2, rows, nkv, d]
    ref = acc[:, :n_local].to(torch.bfloat16)
    dk = torch.empty((n_local, nkv, d), dtype=torch.bfloat16, device=dev)
    dv = torch.empty_like(dk)
    per = rows * nkv * d
    head, row = (rows * d, d) if head_major else (d, nkv * d)
    _lib.call("bam_reduce_partials_bf16", ws.data_ptr(), world, 2 * per, per, head, row, nkv,
              n_local, dk.data_ptr(), dv.data_ptr())
    torch.cuda.synchronize()
    assert torch.equal(dk, ref[0]) and torch.equal(dv, ref[1])


@pytest.mark.parametrize("transport", ["nccl", "ce"])
def test_cp_single_rank_transports_match_local(transport):
    """cp_bitfield_attention on a one-rank NCCL process group, through both
    exchange transports (NCCL collectives; copy-engine pulls/pushes over
    symmetric memory): equal to the single-GPU autograd path."""
    import torch.distributed as dist

    from paper_2503_11367_b200 import attention as A
    from paper_2503_11367_b200 import cp
    from paper_2503_11367_b200 import mask as M

    if not dist.is_initialized():
        import socket
        with socket.socket() as sck:
            sck.bind(("127.0.0.1", 0))
            port = sck.getsockname()[1]
        dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0,
                                world_size=1, device_id=torch.device("cuda", 0))
    mask = M.build_bitfield([("text", 256), ("img0", 384), ("text", 512), ("img1", 128)])
    T, Hq, Hkv = len(mask), 8, 4
    dev = torch.device("cuda")
    g = torch.Generator(device=dev).manual_seed(3)
    q, k, v, do = (torch.randn(T, h, 128, device=dev, generator=g).to(torch.bfloat16)
                   for h in (Hq, Hkv, Hkv, Hq))
    plan = cp.make_cp_plan(mask, 1, 0, "lpt")
    outs = []
    for fn in ("local", transport):
        qd, kd, vd = (t.clone().requires_grad_(True) for t in (q, k, v))
        if fn == "local":
            o = A.bitfield_attention(qd, kd, vd, plan.attn)
        else:
            o = cp.cp_bitfield_attention(qd, kd, vd, plan, groups=2, transport=transport)
        o.backward(do)
        outs.append((o.detach(), qd.grad, kd.grad, vd.grad))
    for name, a, b in zip(("O", "dQ", "dK", "dV"), *outs):
        assert (a.float() - b.float()).abs().max().item() < 1e-2, name
    assert torch.equal(outs[0][0], outs[1][0])


def test_forward_waits_on_kv_arrival_flags():
    """The overlapped CP forward: the head-pair kernel starts while half of
    the key blocks (a 'peer' rank's rows) are still being copied on another
    stream, and waits per tile on the arrival flag that bam_stream_write_i32
    sets after the copy.  Must equal the forward on complete K/V."""
    from paper_2503_11367_b200 import _lib
    from paper_2503_11367_b200 import attention as A
    from paper_2503_11367_b200 import mask as M

    mask = M.build_bitfield([("text", 512), ("img0", 512), ("text", 512), ("img1", 512)])
    nb, T, Hq, Hkv = len(mask) // BLOCK, len(mask), 8, 2
    dev = torch.device("cuda")
    g = torch.Generator(device=dev).manual_seed(9)
    q = torch.randn(T, Hq, 128, device=dev, generator=g, dtype=torch.bfloat16)
    k = torch.randn(T, Hkv, 128, device=dev, generator=g, dtype=torch.bfloat16)
    v = torch.randn(T, Hkv, 128, device=dev, generator=g, dtype=torch.bfloat16)
    plan = A.plan_for_mask(mask)                 # k_row = identity: "rank r" owns rows r*nb/2..
    o_ref, lse_ref = A.attn_forward(q, k, v, plan)
    half = nb // 2 * BLOCK
    k2, v2 = torch.zeros_like(k), torch.zeros_like(v)
    k2[:half], v2[:half] = k[:half], v[:half]    # rank 0 (this rank): present at launch
    flags = torch.zeros(2, dtype=torch.int32, device=dev)
    side = torch.cuda.Stream()
    torch.cuda.synchronize()
    with torch.cuda.stream(side):
        torch.cuda._sleep(50_000_000)            # the peer's rows land well after the launch
        k2[half:].copy_(k[half:])
        v2[half:].copy_(v[half:])
        _lib.call("bam_stream_write_i32", flags[1:2].data_ptr(), 7)
    o, lse = A.attn_forward(q, k2, v2, plan, kv_ready=(flags, 7, 0, nb // 2))
    torch.cuda.synchronize()
    assert torch.equal(o, o_ref) and torch.equal(lse, lse_ref)


def test_cp_emulated_world8_config4_overlapped_forward():
    """The north-star shape at CP=8 with the copy-engine layout, ranks emulated
    one after another on one GPU: config 4 (128K EMU multi-image, GQA 32q/8kv),
    head-major gathered K/V [Hkv, 8*rows, d] whose peers' rows land on a side
    stream AFTER the forward starts, signalled through the world*Hkv = 64
    arrival flags (bam_stream_write_i32) that the kernel waits on per tile.
    Per rank: O/dQ of every local row against the single-GPU path (itself
    oracle-checked at this size in tests/test_gpu_large.py), the heaviest local
    query block against the fp32 oracle, and the dK/dV partials of all eight
    ranks summed against the single-GPU fp32 dK/dV."""
    from paper_2503_11367_b200 import _lib
    from paper_2503_11367_b200 import attention as A
    from paper_2503_11367_b200 import cp
    from paper_2503_11367_b200 import mask as M
    from paper_2503_11367_b200.workloads import CONFIGS

    world, cfg = 8, CONFIGS[4]
    Hq, Hkv = cfg["Hq"], cfg["Hkv"]
    mask = M.build_bitfield(cfg["segments"])
    d_desc = mask.device_descriptors()
    T = d_desc.shape[0]
    desc = d_desc.cpu().numpy()
    dev = torch.device("cuda")
    g = torch.Generator().manual_seed(1234)
    q, k, v, do = (torch.randn(T, h, 128, generator=g).to(torch.bfloat16)
                   for h in (Hq, Hkv, Hkv, Hq))
    qd, kd, vd, dod = (t.to(dev) for t in (q, k, v, do))
    full = A.plan_for_mask(mask)
    o_1, lse_1 = A.attn_forward(qd, kd, vd, full)
    dq_1, dk_1, dv_1 = A.attn_backward(qd, kd, vd, o_1, lse_1, dod, full, dkv_fp32=True)
    dk_sum = torch.zeros(T, Hkv, 128, device=dev)
    dv_sum = torch.zeros_like(dk_sum)
    side = torch.cuda.Stream()
    for rank in range(world):
        plan = cp.make_cp_plan(d_desc, world, rank, "lpt")
        lay = plan.layout
        rows = lay.max_blocks * BLOCK
        idx = (lay.k_row.to(torch.int64)[:, None] * BLOCK +
               torch.arange(BLOCK, device=dev)[None, :]).reshape(-1)
        k_all = torch.zeros(Hkv, world * rows, 128, dtype=torch.bfloat16, device=dev)
        v_all = torch.zeros_like(k_all)
        mine = torch.zeros(world * rows, dtype=torch.bool, device=dev)
        mine[rank * rows:(rank + 1) * rows] = True
        k_src = torch.zeros_like(k_all)
        v_src = torch.zeros_like(v_all)
        k_src[:, idx] = kd.transpose(0, 1)
        v_src[:, idx] = vd.transpose(0, 1)
        k_all[:, mine] = k_src[:, mine]          # this rank's rows: present at launch
        v_all[:, mine] = v_src[:, mine]
        # the peers' rows arrive by DMA (pinned host -> device, a copy engine, like the
        # NVLink pulls): the spinning forward CTAs occupy every SM, so a copy that
        # needed an SM (a same-device D2D copy kernel) could never run
        k_src_h, v_src_h = k_src.cpu().pin_memory(), v_src.cpu().pin_memory()
        flags = torch.zeros(world * Hkv, dtype=torch.int32, device=dev)
        epoch = 3 + rank
        q_loc, do_loc = cp.shard_rows(qd, dod, layout=lay)
        torch.cuda.synchronize()
        with torch.cuda.stream(side):
            torch.cuda._sleep(20_000_000)        # the peers' rows land after the launch
            for peer in range(world):
                if peer == rank:
                    continue
                sl = slice(peer * rows, (peer + 1) * rows)
                for h in range(Hkv):
                    k_all[h, sl].copy_(k_src_h[h, sl], non_blocking=True)
                    v_all[h, sl].copy_(v_src_h[h, sl], non_blocking=True)
                    _lib.call("bam_stream_write_i32", flags[peer * Hkv + h:].data_ptr(), epoch)
        o, lse = A.attn_forward(q_loc, k_all, v_all, plan.attn,
                                kv_ready=(flags, epoch, rank, lay.max_blocks), kv_head_major=True)
        torch.cuda.synchronize()
        assert int(flags.min().item()) in (0, epoch)
        ws = A.BackwardWorkspace(q_loc, o, lse, do_loc, plan.attn, None)
        dk_all, dv_all = ws.main(k_all, v_all, kv_head_major=True)
        dq = ws.finalize()
        dk_sum += dk_all[idx]
        dv_sum += dv_all[idx]
        pos = (lay.local_blocks.to(torch.int64)[:, None] * BLOCK +
               torch.arange(BLOCK, device=dev)[None, :]).reshape(-1)
        assert (o.float() - o_1[pos].float()).abs().max().item() < 2e-2, rank
        assert rel_l2(o, o_1[pos]) < 1e-2
        d = (dq.float() - dq_1[pos].float()).abs() - dq_1[pos].float().abs() * 2.0 ** -7
        assert d.max().item() < 2e-2 and rel_l2(dq, dq_1[pos]) < 1e-2, rank
        # the heaviest local query block against the oracle
        W = plan.attn.W[lay.local_blocks.long()]
        i = int(torch.argmax(W).item())
        b = int(lay.local_blocks[i].item())
        rws = np.arange(b * BLOCK, (b + 1) * BLOCK)
        rt = torch.from_numpy(rws)
        o_ref, lse_ref = attention_ref.attention_fwd(q[rt], k, v, desc, rws, chunk=128)
        dq_ref, _, _ = attention_ref.attention_bwd(q[rt], k, v, o_ref, lse_ref, do[rt], desc, rws,
                                                   chunk=128)
        sl = slice(i * BLOCK, (i + 1) * BLOCK)
        assert (o[sl].float().cpu() - o_ref).abs().max().item() < 2e-2
        assert (lse[:, sl].cpu() - lse_ref).abs().max().item() < 2e-3
        assert (dq[sl].float().cpu() - dq_ref).abs().max().item() < 2e-2
        assert rel_l2(dq[sl], dq_ref) < 1e-2
    assert rel_l2(dk_sum, dk_1) < 1e-2 and (dk_sum - dk_1).abs().max().item() < 2e-2
    assert rel_l2(dv_sum, dv_1) < 1e-2 and (dv_sum - dv_1).abs().max().item() < 2e-2


def test_kv_head_major_bit_exact():
    """bam_kv_head_major (the copy-engine gather's local step) against torch
    transposes: both destinations, row offsets, one and two outputs."""
    from paper_2503_11367_b200 import _lib

    dev = torch.device("cuda")
    g = torch.Generator(device=dev).manual_seed(4)
    for n, nkv in ((384, 8), (128, 3), (0, 2)):
        k = torch.randn(n, nkv, 128, device=dev, generator=g).to(torch.bfloat16)
        v = torch.randn(n, nkv, 128, device=dev, generator=g).to(torch.bfloat16)
        r0, o0, r1, o1 = n + 256, 128, 4 * n + 128, 2 * n
        k0 = torch.zeros(nkv, r0, 128, dtype=torch.bfloat16, device=dev)
        v0, k1, v1 = torch.zeros_like(k0), torch.zeros(nkv, r1, 128, dtype=torch.bfloat16,
                                                      device=dev), None
        v1 = torch.zeros_like(k1)
        _lib.call("bam_kv_head_major", k.data_ptr(), v.data_ptr(), n, nkv, k0.data_ptr(),
                  v0.data_ptr(), r0, o0, k1.data_ptr(), v1.data_ptr(), r1, o1)
        torch.cuda.synchronize()
        for dst, src, off in ((k0, k, o0), (v0, v, o0), (k1, k, o1), (v1, v, o1)):
            assert torch.equal(dst[:, off:off + n], src.transpose(0, 1))
            assert dst[:, :off].abs().sum().item() == 0 and dst[:, off + n:].abs().sum().item() == 0
    with pytest.raises(Exception, match="bam_kv_head_major"):
        _lib.call("bam_kv_head_major", k0.data_ptr(), v0.data_ptr(), 10, 2, k0.data_ptr(),
                  v0.data_ptr(), 5, 0, None, None, 0, 0)


def test_cp_emulated_mha_overlapped_forward():
    """MHA under the overlapped copy-engine forward: the query-block-pair kernel's
    union lists are local-first (bam_plan_build), so its CTAs start on this rank's
    key tiles and wait per tile on the per-(rank, head) arrival flags while the
    peers' rows land by DMA after the launch; O and dQ per rank against the
    single-GPU path, the dK/dV partials summed over the ranks against its dK/dV."""
    from paper_2503_11367_b200 import _lib
    from paper_2503_11367_b200 import attention as A
    from paper_2503_11367_b200 import cp
    from paper_2503_11367_b200 import mask as M

    world, Hq, Hkv = 4, 4, 4
    mask = M.build_bitfield([("image", 2048), ("text", 3072), ("img1", 1024), ("text", 2048)])
    d_desc = mask.device_descriptors()
    T = d_desc.shape[0]
    dev = torch.device("cuda")
    g = torch.Generator(device=dev).manual_seed(11)
    qd, kd, vd, dod = (torch.randn(T, h, 128, device=dev, generator=g, dtype=torch.bfloat16)
                       for h in (Hq, Hkv, Hkv, Hq))
    full = A.plan_for_mask(mask)
    o_1, lse_1 = A.attn_forward(qd, kd, vd, full)
    dq_1, dk_1, dv_1 = A.attn_backward(qd, kd, vd, o_1, lse_1, dod, full, dkv_fp32=True)
    dk_sum = torch.zeros(T, Hkv, 128, device=dev)
    dv_sum = torch.zeros_like(dk_sum)
    side = torch.cuda.Stream()
    n_pairs_seen = 0
    for rank in range(world):
        plan = cp.make_cp_plan(d_desc, world, rank, "lpt")
        lay = plan.layout
        n_pairs_seen += int(plan.attn.counts[0])
        rows = lay.max_blocks * BLOCK
        idx = (lay.k_row.to(torch.int64)[:, None] * BLOCK +
               torch.arange(BLOCK, device=dev)[None, :]).reshape(-1)
        k_src = torch.zeros(Hkv, world * rows, 128, dtype=torch.bfloat16, device=dev)
        v_src = torch.zeros_like(k_src)
        k_src[:, idx] = kd.transpose(0, 1)
        v_src[:, idx] = vd.transpose(0, 1)
        k_all, v_all = torch.zeros_like(k_src), torch.zeros_like(v_src)
        mine = slice(rank * rows, (rank + 1) * rows)
        k_all[:, mine] = k_src[:, mine]
        v_all[:, mine] = v_src[:, mine]
        k_src_h, v_src_h = k_src.cpu().pin_memory(), v_src.cpu().pin_memory()
        flags = torch.zeros(world * Hkv, dtype=torch.int32, device=dev)
        epoch = 5 + rank
        q_loc, do_loc = cp.shard_rows(qd, dod, layout=lay)
        torch.cuda.synchronize()
        with torch.cuda.stream(side):
            torch.cuda._sleep(5_000_000)         # the peers' rows land after the launch
            for peer in range(world):
                if peer == rank:
                    continue
                sl = slice(peer * rows, (peer + 1) * rows)
                for h in range(Hkv):
                    k_all[h, sl].copy_(k_src_h[h, sl], non_blocking=True)
                    v_all[h, sl].copy_(v_src_h[h, sl], non_blocking=True)
                    if h % 2 == 1:                # one flag per pair of KV heads
                        _lib.call("bam_stream_write_i32", flags[peer * Hkv + h - 1:].data_ptr(),
                                  epoch)
        o, lse = A.attn_forward(q_loc, k_all, v_all, plan.attn,
                                kv_ready=(flags, epoch, rank, lay.max_blocks, 2),
                                kv_head_major=True)
        torch.cuda.synchronize()
        ws = A.BackwardWorkspace(q_loc, o, lse, do_loc, plan.attn, None)
        dk_all, dv_all = ws.main(k_all, v_all, kv_head_major=True)
        dq = ws.finalize()
        dk_sum += dk_all[idx]
        dv_sum += dv_all[idx]
        pos = (lay.local_blocks.to(torch.int64)[:, None] * BLOCK +
               torch.arange(BLOCK, device=dev)[None, :]).reshape(-1)
        assert (o.float() - o_1[pos].float()).abs().max().item() < 2e-2, rank
        assert rel_l2(o, o_1[pos]) < 1e-2 and rel_l2(dq, dq_1[pos]) < 1e-2, rank
    assert n_pairs_seen > 0                       # the query-block-pair kernel ran
    assert rel_l2(dk_sum, dk_1) < 1e-2 and (dk_sum - dk_1).abs().max().item() < 2e-2
    assert rel_l2(dv_sum, dv_1) < 1e-2 and (dv_sum - dv_1).abs().max().item() < 2e-2


@pytest.mark.parametrize("policy,world", [("lpt", 1), ("lpt", 4), ("zigzag", 3), ("lpt", 8)])
def test_native_planner_matches_host_statement(policy, world):
    """bam_plan_build (one launch sequence, no host sync) against a host
    restatement with torch/Python of every list it builds: the gathered
    layout (cp.cp_layout), CSR rows (ascending; under CP grouped by owner in
    rotation order, this rank's key blocks first), CSC columns, heavy-first orders (stable sort by -count),
    the CTA-pair step lists (bam_build_pair_lists) and the forward pair /
    whole-row item compaction with its device counts."""
    from paper_2503_11367_b200 import _lib
    from paper_2503_11367_b200 import cp
    from paper_2503_11367_b200 import mask as M
    from paper_2503_11367_b200.workloads import emu_interleave

    mask = M.build_bitfield(emu_interleave(64 * 1024, seed=3))
    desc = mask.device_descriptors()
    dev = desc.device
    cls = None
    for rank in range(world):
        plan = cp.make_cp_plan(desc, world, rank, policy)
        at, lay = plan.attn, plan.layout
        if cls is None:
            cls = at.classes.cpu().numpy()
        nb = at.nb
        ref = cp.cp_layout(plan.assignment.owner, world, rank)
        assert torch.equal(lay.k_row.cpu(), ref.k_row.cpu())
        assert torch.equal(lay.local_blocks.cpu(), ref.local_blocks.cpu())
        assert lay.counts == ref.counts and lay.max_blocks == ref.max_blocks
        owner = plan.assignment.owner.cpu().numpy()
        q_gid = at.q_gid.cpu().numpy()
        row_off = at.row_off.cpu().numpy()
        rows = at.row_tiles.cpu().numpy()
        for j, b in enumerate(q_gid):
            kbs = np.nonzero(cls[b])[0]
            exp = [(kb << 2) | cls[b, kb] for kb in kbs]
            if world > 1:   # owners in rotation order rank, rank+1, ..., each ascending
                exp = [e for g in range(world) for e in exp
                       if owner[e >> 2] == (rank + g) % world]
            assert rows[row_off[j]:row_off[j + 1]].tolist() == exp
        col_off = at.col_off.cpu().numpy()
        cols = at.col_tiles.cpu().numpy()
        sub = cls[q_gid]                                  # [nq, nb]
        for kb in range(0, nb, 7):
            js = np.nonzero(sub[:, kb])[0]
            assert cols[col_off[kb]:col_off[kb + 1]].tolist() == [(j << 2) | sub[j, kb]
                                                                  for j in js]
        row_cnt = torch.from_numpy(np.diff(row_off)).to(torch.int64)
        col_cnt = torch.from_numpy(np.diff(col_off)).to(torch.int64)
        assert torch.equal(at.fwd_order.cpu().long(), torch.sort(-row_cnt, stable=True).indices)
        assert torch.equal(at.bwd_order.cpu().long(), torch.sort(-col_cnt, stable=True).indices)
        # step lists: the standalone bam_build_pair_lists over the same columns
        npairs = (nb + 1) // 2
        slot_kb = torch.empty(2 * npairs, dtype=torch.int32, device=dev)
        slot_cnt, slot_off = torch.empty_like(slot_kb), torch.empty(2 * npairs + 1,
                                                                    dtype=torch.int32, device=dev)
        shared = torch.empty(npairs, dtype=torch.int32, device=dev)
        _lib.call("bam_build_pair_lists", at.col_off.data_ptr(), at.col_tiles.data_ptr(),
                  at.bwd_order.data_ptr(), nb, slot_kb.data_ptr(), slot_cnt.data_ptr(),
                  slot_off.data_ptr(), None, shared.data_ptr())
        n_slot = int(slot_off[-1])
        tiles = torch.empty(max(n_slot, 1), dtype=torch.int32, device=dev)
        _lib.call("bam_build_pair_lists", at.col_off.data_ptr(), at.col_tiles.data_ptr(),
                  at.bwd_order.data_ptr(), nb, slot_kb.data_ptr(), slot_cnt.data_ptr(),
                  slot_off.data_ptr(), tiles.data_ptr(), shared.data_ptr())
        assert torch.equal(at.slot_kb, slot_kb) and torch.equal(at.slot_off, slot_off)
        assert torch.equal(at.pair_shared, shared)
        assert torch.equal(at.slot_tiles[:n_slot], tiles[:n_slot])
        # forward pairs -> shared pair ids + whole-row items of the other blocks
        fsh = None
        nq = len(q_gid)
        fp = (nq + 1) // 2
        fslot = at.fwd_slot_q.cpu().view(fp, 2)
        # recompute the shared flags from the union rule (8 u <= 9 max) on the rows
        asc = [sorted(rows[row_off[j]:row_off[j + 1]].tolist()) for j in range(nq)]
        fsh = []
        for pr in range(fp):
            a, b = fslot[pr].tolist()
            la = {e >> 2 for e in asc[a]} if a >= 0 else set()
            lb = {e >> 2 for e in asc[b]} if b >= 0 else set()
            mx = max(len(la), len(lb))
            fsh.append(b >= 0 and mx > 0 and 8 * len(la | lb) <= 9 * mx)
        # the forward union lists against bam_build_pair_lists' merge of the ascending rows
        rows_asc = torch.tensor([e for r in asc for e in r], dtype=torch.int32, device=dev)
        fq = torch.empty(2 * fp, dtype=torch.int32, device=dev)
        fcnt, foff = torch.empty_like(fq), torch.empty(2 * fp + 1, dtype=torch.int32, device=dev)
        fsh_d = torch.empty(fp, dtype=torch.int32, device=dev)
        _lib.call("bam_build_pair_lists", at.row_off.data_ptr(), rows_asc.data_ptr(),
                  at.fwd_order.data_ptr(), nq, fq.data_ptr(), fcnt.data_ptr(), foff.data_ptr(),
                  None, fsh_d.data_ptr())
        ftiles = torch.empty(max(int(foff[-1]), 1), dtype=torch.int32, device=dev)
        _lib.call("bam_build_pair_lists", at.row_off.data_ptr(), rows_asc.data_ptr(),
                  at.fwd_order.data_ptr(), nq, fq.data_ptr(), fcnt.data_ptr(), foff.data_ptr(),
                  ftiles.data_ptr(), fsh_d.data_ptr())
        assert torch.equal(at.fwd_slot_q, fq) and torch.equal(at.fwd_slot_off, foff)
        exp_t = ftiles[:int(foff[-1])].cpu().numpy().copy()
        if world > 1:   # each union list: owners in rotation order rank, rank+1, ...
            fo = foff.cpu().numpy()
            for sl in range(2 * fp):
                seg = exp_t[fo[sl]:fo[sl + 1]].tolist()
                exp_t[fo[sl]:fo[sl + 1]] = [e for g in range(world) for e in seg
                                            if owner[e >> 2] == (rank + g) % world]
        assert at.fwd_slot_tiles[:int(foff[-1])].cpu().tolist() == exp_t.tolist()
        assert fsh_d.cpu().tolist() == [int(x) for x in fsh]
        n_pairs, n_rest = at.counts.cpu().tolist()
        # shared pairs heavy-first by union length, ties by pair index (fwd_pair_w), and
        # their geometric work classes (the query-block-pair kernel's CTA order)
        fcnt_h = fcnt.cpu().tolist()
        want = sorted((pr for pr in range(fp) if fsh[pr]), key=lambda pr: (-fcnt_h[2 * pr], pr))
        assert at.fwd_pair_ids[:n_pairs].cpu().tolist() == want
        w_sorted = [fcnt_h[2 * pr] for pr in want] + [0] * (fp - n_pairs)
        kc = [min(int(w_sorted[0] // c).bit_length() - 1, 15) if c > 0 else 15
              for c in w_sorted] if n_pairs else [15] * fp
        assert at.fwd_pair_classes.cpu().tolist() == [
            next((i for i, x in enumerate(kc) if x >= c), fp) for c in range(16)] + [fp]
        rest = [j for pr in range(fp) if not fsh[pr] for j in fslot[pr].tolist() if j >= 0]
        assert n_rest == len(rest)
        items = at.fwd_rest_items[:n_rest].cpu().tolist()
        assert items == [[j, 0, int(row_cnt[j]), -1] for j in rest]


def test_copy_2d_and_kv_ready_validation():
    """bam_copy_2d (the strided copy-engine copies of the CP K/V pulls) against
    torch indexing; the C entry points reject kv_ready parameters the kernels
    cannot honour (a 64-bit per-rank mask, a positive rank stride)."""
    from paper_2503_11367_b200 import _lib
    from paper_2503_11367_b200 import attention as A
    from paper_2503_11367_b200 import cp
    from paper_2503_11367_b200 import mask as M

    dev = torch.device("cuda")
    g = torch.Generator(device=dev).manual_seed(2)
    src = torch.randn(3, 5, 128, 128, device=dev, generator=g).to(torch.bfloat16)  # [2,nkv,rows,d]-like
    dst = torch.zeros(5, 4 * 128, 128, dtype=torch.bfloat16, device=dev)
    row_b = 128 * 128 * 2
    _lib.call("bam_copy_2d", dst[1, 2 * 128:].data_ptr(), 4 * row_b, src[1, 1].data_ptr(), row_b,
              row_b, 3)
    torch.cuda.synchronize()
    ref = torch.zeros_like(dst)
    ref[1:4, 2 * 128:3 * 128] = src[1, 1:4]
    assert torch.equal(dst, ref)
    with pytest.raises(_lib.BamError):
        _lib.call("bam_copy_2d", dst.data_ptr(), 16, src.data_ptr(), 32, 32, 1)   # pitch < width

    mask = M.build_bitfield([("text", 512), ("img0", 512)])
    plan = A.plan_for_mask(mask)
    T = len(mask)
    q = torch.randn(T, 4, 128, device=dev, generator=g).to(torch.bfloat16)
    k = torch.randn(T, 2, 128, device=dev, generator=g).to(torch.bfloat16)
    flags = torch.zeros(8, dtype=torch.int32, device=dev)
    with pytest.raises(ValueError, match="kv_ready"):
        A.attn_forward(q, k, k, plan, kv_ready=(flags, 1, 0, 0))
    with pytest.raises(ValueError, match="kv_ready"):
        A.attn_forward(q, k, k, plan, kv_ready=(flags, 1, 70, 1))
    with pytest.raises(_lib.BamError, match="kv_ready"):   # flag groups must divide Hkv
        A.attn_forward(q, k, k, plan, kv_ready=(flags, 1, 0, 512, 3))
    # a rank that owns no query block cannot run (more ranks than blocks)
    with pytest.raises(ValueError, match="owns no query block"):
        cp.make_cp_plan(mask, 16, 15, "zigzag")

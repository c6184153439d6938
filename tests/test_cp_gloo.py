"""Multi-process (world_size 2, gloo, CPU) test of the context-parallel data
path: the product's layout (cp.cp_layout), K/V all-gather (cp.gather_kv) and
dK/dV reduce-scatter (cp.scatter_dkv), with the fp32 oracle standing in for
the attention kernels (which need a B200).  Per rank: the gathered K/V must
reproduce every global block at k_row[block], the local outputs must equal
the full-sequence oracle rows, and the reduce-scattered dK/dV must equal the
full-sequence gradients of the rank's own key blocks."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

BLOCK = 128


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, policy, result_dir):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from oracle import attention_ref, balance_ref, mask_ref
    from paper_2503_11367_b200 import cp

    torch.set_num_threads(1)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        segs = [("text", 256), ("img0", 384), ("text", 128), ("img1", 256), ("text", 256)]
        desc, _ = mask_ref.build_bitfield(segs)
        desc = np.asarray(desc, np.int64)
        T = desc.shape[0]
        nb = T // BLOCK
        _, W = mask_ref.block_workloads_np(desc, BLOCK)
        dist_fn = {"lpt": balance_ref.lpt, "zigzag": balance_ref.zigzag,
                   "contiguous": balance_ref.contiguous}[policy]
        gpu_blocks, _ = dist_fn(list(W), world)
        owner = torch.empty(nb, dtype=torch.int32)
        for g, blocks in enumerate(gpu_blocks):
            for b in blocks:
                owner[b] = g
        layout = cp.cp_layout(owner, world, rank)
        assert sorted(layout.local_blocks.tolist()) == sorted(gpu_blocks[rank])

        g = torch.Generator().manual_seed(1234)
        Hq, Hkv = 4, 2
        q = torch.randn(T, Hq, 128, generator=g)
        k = torch.randn(T, Hkv, 128, generator=g)
        v = torch.randn(T, Hkv, 128, generator=g)
        do = torch.randn(T, Hq, 128, generator=g)
        # the product's shard_rows is a CUDA kernel (tests/test_gpu_cp.py); here
        # the same block-row gather by indexing, to feed the gloo collectives
        rows = (layout.local_blocks.to(torch.int64)[:, None] * BLOCK +
                torch.arange(BLOCK)[None, :]).reshape(-1)
        q_loc, k_loc, v_loc, do_loc = (t.index_select(0, rows) for t in (q, k, v, do))

        k_all, v_all = cp.gather_kv(k_loc, v_loc, layout)
        assert k_all.shape[0] == world * layout.max_blocks * BLOCK
        krow = layout.k_row.to(torch.int64)
        gather_idx = (krow[:, None] * BLOCK + torch.arange(BLOCK)[None, :]).reshape(-1)
        assert torch.equal(k_all[gather_idx], k), "gathered K misplaced"
        assert torch.equal(v_all[gather_idx], v), "gathered V misplaced"

        pos = (layout.local_blocks.to(torch.int64)[:, None] * BLOCK +
               torch.arange(BLOCK)[None, :]).reshape(-1).numpy()
        k_g, v_g = k_all[gather_idx], v_all[gather_idx]
        o_loc, lse_loc = attention_ref.attention_fwd(q_loc, k_g, v_g, desc, pos)
        o_full, lse_full = attention_ref.attention_fwd(q, k, v, desc, np.arange(T))
        assert torch.allclose(o_loc, o_full[pos], atol=1e-5)
        dq_loc, dk_part, dv_part = attention_ref.attention_bwd(q_loc, k_g, v_g, o_loc, lse_loc,
                                                               do_loc, desc, pos)
        # place the global-order partials at their gathered rows, reduce-scatter
        dk_all = torch.zeros_like(k_all)
        dv_all = torch.zeros_like(v_all)
        dk_all[gather_idx] = dk_part
        dv_all[gather_idx] = dv_part
        dk_loc, dv_loc = cp.scatter_dkv(dk_all, dv_all, layout)
        dq_full, dk_full, dv_full = attention_ref.attention_bwd(q, k, v, o_full, lse_full, do, desc,
                                                                np.arange(T))
        assert torch.allclose(dq_loc, dq_full[pos], atol=1e-4)
        assert torch.allclose(dk_loc, dk_full[pos], atol=1e-4), (dk_loc - dk_full[pos]).abs().max()
        assert torch.allclose(dv_loc, dv_full[pos], atol=1e-4)
        open(os.path.join(result_dir, f"ok{rank}"), "w").close()
    finally:
        dist.destroy_process_group()


def _run(policy, tmp_path, world=2):
    mp.spawn(_worker, args=(world, _free_port(), policy, str(tmp_path)), nprocs=world, join=True)
    for r in range(world):
        assert os.path.exists(os.path.join(tmp_path, f"ok{r}"))


def test_cp_exchange_lpt(tmp_path):
    _run("lpt", tmp_path)


def test_cp_exchange_zigzag(tmp_path):
    _run("zigzag", tmp_path)


def test_cp_exchange_lpt_world4(tmp_path):
    # uneven per-rank block counts and padded shards across four ranks
    _run("lpt", tmp_path, world=4)


def test_cp_exchange_lpt_world8(tmp_path):
    # the north-star CP degree: eight ranks, 10 blocks -> some ranks own one block
    _run("lpt", tmp_path, world=8)


def test_cp_exchange_zigzag_world8(tmp_path):
    # zigzag with 2G = 16 chunks over 10 blocks: empty chunks, ranks without blocks
    _run("zigzag", tmp_path, world=8)


def test_cp_layout_unequal_counts():
    from paper_2503_11367_b200 import cp

    owner = torch.tensor([0, 1, 1, 1, 0, 2, 1], dtype=torch.int32)
    lay = [cp.cp_layout(owner, 3, r) for r in range(3)]
    assert lay[0].counts == [2, 4, 1] and lay[0].max_blocks == 4
    assert lay[1].local_blocks.tolist() == [1, 2, 3, 6]
    assert lay[2].local_blocks.tolist() == [5]
    # block b sits at owner*max + position among the owner's ascending blocks
    assert lay[0].k_row.tolist() == [0, 4, 5, 6, 1, 8, 7]


def _transport_worker(rank, world, port, fail_ranks, result_dir):
    """resolve_transport('auto') on a gloo group: the exchange 'fails' on the ranks
    in fail_ranks; every rank must reach the same choice (a per-rank
    fallback would leave ranks in mismatched collectives)."""
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from types import SimpleNamespace

    from paper_2503_11367_b200 import cp

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        def exchange(hkv, d, device, group=None):
            if rank in fail_ranks:
                raise RuntimeError("no peer mapping on this rank")
            return object()
        plan = SimpleNamespace(layout=SimpleNamespace(world=world), exchange=exchange)
        cp._TRANSPORT_CHOICE.clear()
        choice = cp.resolve_transport("auto", plan, 8, 128, torch.device("cpu"))
        with open(os.path.join(result_dir, f"choice{rank}"), "w") as fh:
            fh.write(choice)
        # forced transports and world 1 bypass the agreement
        assert cp.resolve_transport("nccl", plan, 8, 128, torch.device("cpu")) == "nccl"
        one = SimpleNamespace(layout=SimpleNamespace(world=1), exchange=exchange)
        assert cp.resolve_transport("auto", one, 8, 128, torch.device("cpu")) == "local"
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("fail_ranks,expected", [((), "ce"), ((1,), "nccl"), ((0, 2), "nccl")])
def test_transport_choice_is_collective(tmp_path, fail_ranks, expected):
    world = 3
    mp.spawn(_transport_worker, args=(world, _free_port(), fail_ranks, str(tmp_path)),
             nprocs=world, join=True)
    choices = {open(os.path.join(tmp_path, f"choice{r}")).read() for r in range(world)}
    assert choices == {expected}


def test_exchange_capacity():
    from paper_2503_11367_b200 import cp

    # headroom of 1/8, rounded up to 1024 tokens, capped at the (rounded) sequence
    assert cp.exchange_capacity(32896, 1024, 4) == 37888
    assert cp.exchange_capacity(1024, 8, 1) == 1024
    for rows, nb, world in ((128, 1024, 8), (16512, 1024, 8), (131072, 1024, 1)):
        cap = cp.exchange_capacity(rows, nb, world)
        assert cap >= rows and cap % 128 == 0

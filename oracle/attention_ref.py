"""fp32 CPU oracle for bitfield-masked attention (TEST INFRASTRUCTURE ONLY).

The reference has no attention code,
so this restates the semantics the north star fixes:

* mask: ``materialize`` (mask.py:106-112) -- text query sees keys k <= q that
  share a descriptor bit; a pure-modality query sees keys with an identical
  descriptor, non-causally;
* math: scaled dot-product attention with a row-wise softmax over the allowed
  keys, computed blockwise as in PAPER.md:616-619 (skip fully-masked
  128x128 tiles; only partial tiles need the element mask);
* GQA: query head h reads KV head h // (Hq // Hkv) (the usual convention;
  the reference is silent).

Tensors use the token-major layout of the product API: q [Tq, Hq, d],
k/v [Tk, Hkv, d]; ``q_pos`` are the global token positions of the query rows
(CP ranks own non-contiguous blocks); keys are the whole sequence 0..Tk-1.
Everything is computed in fp32 on the CPU with all host threads.
"""

from __future__ import annotations

import math

import numpy as np
import torch

from .mask_ref import dense_rows


def _rows_mask(desc_np: np.ndarray, rows: np.ndarray, cols=None) -> torch.Tensor:
    return torch.from_numpy(dense_rows(desc_np, rows, cols))


def attention_fwd(q, k, v, desc, q_pos, scale=None, chunk=512, k_pos=None):
    """Returns (O fp32 [Tq, Hq, d], LSE fp32 [Hq, Tq]).

    ``k_pos``: global positions of the rows of k/v (default: 0..Tk-1, the
    whole sequence).  Passing only the keys of a query block's non-skip
    tiles computes the same rows blockwise-sparse: skipped
    tiles contribute nothing."""
    q, k, v = q.float(), k.float(), v.float()
    Tq, Hq, d = q.shape
    Hkv = k.shape[1]
    grp = Hq // Hkv
    scale = 1.0 / math.sqrt(d) if scale is None else scale
    desc_np = np.asarray(desc.cpu().numpy() if torch.is_tensor(desc) else desc, dtype=np.int64)
    pos = np.asarray(q_pos.cpu().numpy() if torch.is_tensor(q_pos) else q_pos, dtype=np.int64)
    O = torch.empty(Tq, Hq, d)
    LSE = torch.empty(Hq, Tq)
    kk = k.permute(1, 0, 2)     # [Hkv, Tk, d]
    vv = v.permute(1, 0, 2)
    kp = None if k_pos is None else np.asarray(k_pos, dtype=np.int64)
    for r0 in range(0, Tq, chunk):
        r1 = min(r0 + chunk, Tq)
        allow = _rows_mask(desc_np, pos[r0:r1], kp)                # [R, Tk]
        qh = q[r0:r1].permute(1, 0, 2).reshape(Hkv, grp * (r1 - r0), d)
        s = torch.bmm(qh, kk.transpose(1, 2)).view(Hkv, grp, r1 - r0, -1) * scale
        s = s.masked_fill(~allow, float("-inf"))
        lse = torch.logsumexp(s, dim=-1)                            # [Hkv, grp, R]
        p = torch.exp(s - lse[..., None])
        o = torch.bmm(p.view(Hkv, grp * (r1 - r0), -1), vv).view(Hkv, grp, r1 - r0, d)
        O[r0:r1] = o.reshape(Hq, r1 - r0, d).permute(1, 0, 2)
        LSE[:, r0:r1] = lse.reshape(Hq, r1 - r0)
    return O, LSE


def attention_bwd(q, k, v, o, lse, do, desc, q_pos, scale=None, chunk=512, k_pos=None):
    """Gradients of sum(O * dO).  Returns (dQ [Tq, Hq, d], dK, dV [Tk, Hkv, d]),
    fp32; dK/dV are the contributions of these query rows only (the CP
    partials that a reduce-scatter sums).  ``k_pos`` as in attention_fwd."""
    q, k, v, o, do = q.float(), k.float(), v.float(), o.float(), do.float()
    Tq, Hq, d = q.shape
    Tk, Hkv, _ = k.shape
    grp = Hq // Hkv
    scale = 1.0 / math.sqrt(d) if scale is None else scale
    desc_np = np.asarray(desc.cpu().numpy() if torch.is_tensor(desc) else desc, dtype=np.int64)
    pos = np.asarray(q_pos.cpu().numpy() if torch.is_tensor(q_pos) else q_pos, dtype=np.int64)
    dQ = torch.empty(Tq, Hq, d)
    dK = torch.zeros(Hkv, Tk, d)
    dV = torch.zeros(Hkv, Tk, d)
    kk = k.permute(1, 0, 2)
    vv = v.permute(1, 0, 2)
    D_all = (do * o).sum(-1)                                        # [Tq, Hq]
    kp = None if k_pos is None else np.asarray(k_pos, dtype=np.int64)
    for r0 in range(0, Tq, chunk):
        r1 = min(r0 + chunk, Tq)
        R = r1 - r0
        allow = _rows_mask(desc_np, pos[r0:r1], kp)
        qh = q[r0:r1].permute(1, 0, 2).reshape(Hkv, grp * R, d)
        doh = do[r0:r1].permute(1, 0, 2).reshape(Hkv, grp * R, d)
        s = torch.bmm(qh, kk.transpose(1, 2)).view(Hkv, grp, R, Tk) * scale
        s = s.masked_fill(~allow, float("-inf"))
        l = lse[:, r0:r1].reshape(Hkv, grp, R, 1).float()
        p = torch.exp(s - l).view(Hkv, grp * R, Tk)
        dV += torch.bmm(p.transpose(1, 2), doh)
        dp = torch.bmm(doh, vv.transpose(1, 2))
        Dh = D_all[r0:r1].t().reshape(Hkv, grp * R, 1)
        ds = p * (dp - Dh)
        dQ[r0:r1] = (torch.bmm(ds, kk) * scale).view(Hq, R, d).permute(1, 0, 2)
        dK += torch.bmm(ds.transpose(1, 2), qh) * scale
    return dQ, dK.permute(1, 0, 2).contiguous(), dV.permute(1, 0, 2).contiguous()


def attention_dense_autograd(q, k, v, do, desc, q_pos, scale=None):
    """Independent dense formulation with torch autograd (small T only), used
    to cross-check ``attention_fwd`` / ``attention_bwd``."""
    q = q.float().clone().requires_grad_(True)
    k = k.float().clone().requires_grad_(True)
    v = v.float().clone().requires_grad_(True)
    Tq, Hq, d = q.shape
    grp = Hq // k.shape[1]
    scale = 1.0 / math.sqrt(d) if scale is None else scale
    desc_np = np.asarray(desc, dtype=np.int64)
    allow = _rows_mask(desc_np, np.asarray(q_pos, dtype=np.int64))
    kr = k.repeat_interleave(grp, dim=1)
    vr = v.repeat_interleave(grp, dim=1)
    s = torch.einsum("qhd,khd->hqk", q, kr) * scale
    s = s.masked_fill(~allow, float("-inf"))
    p = torch.softmax(s, dim=-1)
    o = torch.einsum("hqk,khd->qhd", p, vr)
    (o * do.float()).sum().backward()
    return o.detach(), q.grad, k.grad, v.grad

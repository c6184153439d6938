import math, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from oracle import mask_ref
from paper_2503_11367_b200 import attention as A, mask as M
scale_T = int(sys.argv[1]) if len(sys.argv) > 1 else 64
segs = [("text", 8*1024*scale_T//64), ("vision", 16*1024*scale_T//64), ("text", 16*1024*scale_T//64), ("audio", 16*1024*scale_T//64), ("text", 8*1024*scale_T//64)]
Hq = Hkv = int(sys.argv[2]) if len(sys.argv) > 2 else 4
mask = M.build_bitfield(segs); desc_d = mask.device_descriptors(); T = desc_d.shape[0]; nb = T // 128
desc = desc_d.cpu().numpy(); plan = A.build_plan(desc_d)
cls = plan.classes.cpu().numpy()
dev = torch.device("cuda"); g = torch.Generator(device=dev).manual_seed(1234)
q = torch.randn(T, Hq, 128, device=dev, generator=g, dtype=torch.bfloat16)
k = torch.randn(T, Hkv, 128, device=dev, generator=g, dtype=torch.bfloat16)
v = torch.randn(T, Hkv, 128, device=dev, generator=g, dtype=torch.bfloat16)
do = torch.randn(T, Hq, 128, device=dev, generator=g, dtype=torch.bfloat16)
o, lse = A.attn_forward(q, k, v, plan)
dq, dk, dv = A.attn_backward(q, k, v, o, lse, do, plan, dkv_fp32=True)
torch.cuda.synchronize()
scale = 1 / math.sqrt(128)
lse_c, o_c, q_c, do_c, kc, vc = lse.cpu(), o.cpu().float(), q.cpu().float(), do.cpu().float(), k.cpu(), v.cpu()
for kb in [0, 1, nb // 3, nb - 1]:
    qb = np.nonzero(cls[:, kb])[0]
    qrows = torch.from_numpy(np.concatenate([np.arange(b * 128, (b + 1) * 128) for b in qb]))
    keys = torch.arange(kb * 128, (kb + 1) * 128)
    allow = torch.from_numpy(mask_ref.dense_rows(desc, qrows.numpy(), keys.numpy()))
    for h in range(Hq):
        Qh, dOh = q_c[qrows, h], do_c[qrows, h]
        Kh, Vh = kc[keys, h].float(), vc[keys, h].float()
        s = (Qh @ Kh.t()) * scale
        p = torch.exp(s - lse_c[h, qrows][:, None]).masked_fill(~allow, 0.0)
        dp = dOh @ Vh.t()
        D = (dOh * o_c[qrows, h]).sum(-1, keepdim=True)
        ds = p * (dp - D)
        dvr = p.t() @ dOh; dkr = (ds.t() @ Qh) * scale
        # variants: bf16-rounded P / dS
        pb = p.to(torch.bfloat16).float(); dsb = ds.to(torch.bfloat16).float()
        dkb = (dsb.t() @ Qh) * scale
        e = lambda a, b: (((a - b).norm() / b.norm()).item(), (a - b).abs().max().item())
        print(f"T={T} kb={kb} nq={len(qb)} h={h} dV {e(dv.cpu()[keys, h], dvr)} dK {e(dk.cpu()[keys, h], dkr)} dK(bf16 dS ref) {e(dkb, dkr)} |dK| {dkr.norm().item():.3e}")

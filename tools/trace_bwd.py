#!/usr/bin/env python3
"""Per-step timeline of one backward CTA (needs a -DBAM_TRACE build, selected
with BAM_LIB_PATH).  Writes gpurun_out/trace_bwd.json: events x steps clock64."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2503_11367_b200 import _lib, attention as A, mask as M  # noqa: E402
from paper_2503_11367_b200.workloads import CONFIGS  # noqa: E402

cfg = CONFIGS[int(os.environ.get("CFG", "4"))]
mask = M.build_bitfield(cfg["segments"])
plan = A.plan_for_mask(mask)
T, dev = len(mask), torch.device("cuda")
g = torch.Generator(device=dev).manual_seed(1234)
q = torch.randn(T, cfg["Hq"], 128, device=dev, generator=g, dtype=torch.bfloat16)
k = torch.randn(T, cfg["Hkv"], 128, device=dev, generator=g, dtype=torch.bfloat16)
v = torch.randn(T, cfg["Hkv"], 128, device=dev, generator=g, dtype=torch.bfloat16)
do = torch.randn(T, cfg["Hq"], 128, device=dev, generator=g, dtype=torch.bfloat16)
buf = torch.zeros(20 * 4096, dtype=torch.int64, device=dev)
o, lse = A.attn_forward(q, k, v, plan)
A.attn_backward(q, k, v, o, lse, do, plan)
_lib.check(_lib.load().bam_set_trace_buffer(buf.data_ptr()))
A.attn_backward(q, k, v, o, lse, do, plan)
torch.cuda.synchronize()
tr = buf.view(20, 4096).cpu().tolist()
os.makedirs("gpurun_out", exist_ok=True)
with open("gpurun_out/trace_bwd.json", "w") as fh:
    json.dump(tr, fh)
print("ok")

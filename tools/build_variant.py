#!/usr/bin/env python3
"""Build an A/B variant of libbam.so: one source (or a comma-separated list)
recompiled with extra -D flags, linked with the default objects of the others.

  python tools/build_variant.py attn_fwd.cu libbam_x.so -DBAM_FWD_P_CHUNKS=4
  python tools/build_variant.py attn_fwd.cu,attn_bwd.cu libbam_clk.so -DBAM_CTA_CLOCK

The variant is selected at run time with BAM_LIB_PATH=<path>.
"""
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2503_11367_b200 import _build as b  # noqa: E402

srcs, out, *defs = sys.argv[1:]
srcs = srcs.split(",")
b.build_lib()
vobjs = []
for src in srcs:
    obj = os.path.join(b.OBJ, "variant_" + os.path.basename(out) + "_" + src + ".o")
    cmd = [b.NVCC, *b.ARCH, *b.FLAGS, *defs, "-Xptxas", "-v", "-c", os.path.join(b.CSRC, src),
           "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    sys.stderr.write(r.stderr)
    if r.returncode:
        sys.exit(r.returncode)
    vobjs.append(obj)
objs = [os.path.join(b.OBJ, os.path.basename(s) + ".o") for s in sorted(os.listdir(b.CSRC))
        if s.endswith(".cu") and s not in srcs] + vobjs
subprocess.run([b.NVCC, *b.ARCH, "-shared", "-o", os.path.join(b.PKG, out), *objs, "-lcudart"],
               check=True)
print(os.path.join(b.PKG, out))

#!/usr/bin/env python3
"""Build an A/B baseline of libbam.so: the given csrc/ sources taken from a git
revision (default HEAD), linked with the working tree's objects of the others.

  python tools/ab_variant.py libbam_base.so attn_fwd.cu [attn_bwd.cu ...] [--rev HEAD] [-DX=1]

Select it at run time with BAM_LIB_PATH=paper_2503_11367_b200/<out>.
"""
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2503_11367_b200 import _build as b  # noqa: E402

args = sys.argv[1:]
rev = "HEAD"
if "--rev" in args:
    i = args.index("--rev")
    rev = args[i + 1]
    del args[i:i + 2]
defs = [a for a in args if a.startswith("-D")]
out, *srcs = [a for a in args if not a.startswith("-D")]
b.build_lib()
objs = []
for src in srcs:
    text = subprocess.run(["git", "show", f"{rev}:paper_2503_11367_b200/csrc/{src}"],
                          capture_output=True, text=True, check=True, cwd=b.ROOT).stdout
    tmp = os.path.join("/tmp", f"ab_{rev}_{src}".replace("/", "_"))
    with open(tmp, "w") as fh:
        fh.write(text)
    obj = os.path.join(b.OBJ, f"ab_{os.path.basename(out)}_{src}.o")
    cmd = [b.NVCC, *b.ARCH, *b.FLAGS, "-I", b.CSRC, *defs, "-c", tmp, "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode:
        sys.stderr.write(r.stderr)
        sys.exit(r.returncode)
    objs.append(obj)
rest = [os.path.join(b.OBJ, s + ".o") for s in sorted(os.listdir(b.CSRC))
        if s.endswith(".cu") and s not in srcs]
subprocess.run([b.NVCC, *b.ARCH, "-shared", "-o", os.path.join(b.PKG, out), *rest, *objs,
                "-lcudart"], check=True)
print(os.path.join(b.PKG, out))

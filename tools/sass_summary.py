#!/usr/bin/env python3
"""Per-kernel SASS summary of libbam.so (cuobjdump -sass): counts of the
Blackwell instructions that prove the tcgen05 / TMEM / TMA paths --
UTCHMMA / UTCQMMA (tcgen05.mma), UTCBAR (tcgen05.commit), LDTM / STTM
(tcgen05.ld / st), UTMALDG (TMA tensor loads), UBLKCP / UBLKRED (bulk copies /
bulk reduce-adds), MUFU, FFMA2 / FADD2 / FMUL2 (packed fp32) -- and the
register count.  Writes a markdown table (default stdout).

    python tools/sass_summary.py [--lib paper_2503_11367_b200/libbam.so] [-o profiles/r02/sass.md]
"""
import argparse
import re
import subprocess
import sys

OPS = ["UTCHMMA", "UTCQMMA", "UTCBAR", "LDTM", "STTM", "UTMALDG", "UTMASTG", "UTMAREDG",
       "UBLKCP", "UBLKRED", "UBLKPF", "MUFU", "FFMA2", "FADD2", "FMUL2", "REDG", "SYNCS"]


def demangle(names):
    r = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True, text=True)
    out = r.stdout.splitlines()
    return out if len(out) == len(names) else names


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--lib", default="paper_2503_11367_b200/libbam.so")
    ap.add_argument("-o", "--output", default=None)
    args = ap.parse_args()
    sass = subprocess.run(["cuobjdump", "-sass", args.lib], capture_output=True, text=True,
                          check=True).stdout
    res = subprocess.run(["cuobjdump", "-res-usage", args.lib], capture_output=True,
                         text=True).stdout
    regs = {}
    for m in re.finditer(r"Function (\S+):\s*\n\s*REG:(\d+)", res):
        regs[m.group(1)] = int(m.group(2))
    kernels, cur = {}, None
    for line in sass.splitlines():
        m = re.match(r"\s*Function : (\S+)", line)
        if m:
            cur = m.group(1)
            kernels[cur] = {op: 0 for op in OPS}
            continue
        m = re.match(r"\s*/\*[0-9a-f]+\*/\s+(?:@!?U?P\w+\s+)?([A-Z0-9_]+)", line)
        if m and cur is not None:
            op = m.group(1)
            if op in kernels[cur]:
                kernels[cur][op] += 1
    names = list(kernels)
    pretty = demangle(names)
    cols = [op for op in OPS if any(k[op] for k in kernels.values())]
    lines = [f"# SASS instruction summary of `{args.lib}` (cuobjdump -sass, sm_100a)", "",
             "| kernel | regs | " + " | ".join(cols) + " |",
             "|---|---|" + "---|" * len(cols)]
    for raw, name in sorted(zip(names, pretty), key=lambda x: -sum(kernels[x[0]].values())):
        short = re.sub(r"\(.*", "", name)
        lines.append(f"| `{short}` | {regs.get(raw, '')} | " +
                     " | ".join(str(kernels[raw][op]) for op in cols) + " |")
    text = "\n".join(lines) + "\n"
    if args.output:
        with open(args.output, "w") as fh:
            fh.write(text)
    else:
        sys.stdout.write(text)


if __name__ == "__main__":
    main()

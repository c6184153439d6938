#!/usr/bin/env python3
"""Summarise ncu artefacts into markdown for profiles/.

    python tools/ncu_summary.py --launches gpurun_out/launches.csv \
        --report gpurun_out/prof_r01.ncu-rep > profiles/r01/ncu_summary.md
"""
import argparse
import collections
import csv
import io
import subprocess

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("sm__cycles_elapsed.avg.per_second", "SM clock"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "tensor pipe active % (elapsed)"),
    ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "XU (MUFU) pipe %"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA pipe %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("lts__t_sector_hit_rate.pct", "L2 hit rate %"),
    ("lts__t_sectors_srcunit_tex_op_red.sum", "L2 red sectors (dQ reductions)"),
    ("l1tex__m_xbar2l1tex_read_bytes.sum", "L2->SM bytes"),
    ("l1tex__m_l1tex2xbar_write_bytes.sum", "SM->L2 bytes"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "shared-memory LSU wavefronts"),
    ("l1tex__data_pipe_tc_wavefronts_mem_shared.sum", "shared-memory tensor-core wavefronts"),
    ("l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
     "shared-memory tensor-core wavefronts % of peak"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
     "shared-memory LSU wavefronts % of peak"),
    ("sm__icc_request_hit_rate.pct", "I-cache hit %"),
    ("launch__registers_per_thread", "registers / thread"),
    ("launch__shared_mem_per_block_dynamic", "dynamic smem / CTA"),
]


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h, data = rows[hi], rows[hi + 1:]
    ik, iv, iu = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    tot, cnt = collections.defaultdict(float), collections.Counter()
    scale = {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0,
             "second": 1e3, "s": 1e3}
    for r in data:
        name = r[ik].split("(")[0]
        tot[name] += float(r[iv].replace(",", "")) * scale.get(r[iu], 1.0)
        cnt[name] += 1
    s = sum(tot.values())
    out = ["| kernel | launches | total ms | share |", "|---|---|---|---|"]
    for k, v in sorted(tot.items(), key=lambda x: -x[1])[:12]:
        out.append(f"| `{k}` | {cnt[k]} | {v:.2f} | {100 * v / s:.1f}% |")
    return "\n".join(out)


def report(path):
    txt = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    h, u = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        d = {a: (b, c) for a, b, c in zip(h, u, r)}
        name = d.get("Kernel Name", ("", ""))[1].split("(")[0]
        out.append(f"\n### `{name}`\n\n| metric | value |\n|---|---|")
        for key, label in KEYS:
            if key in d:
                unit, val = d[key]
                out.append(f"| {label} (`{key}`) | {val} {unit} |")
    return "\n".join(out)


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--launches")
    ap.add_argument("--report")
    a = ap.parse_args()
    if a.launches:
        print("## Launch list (ncu --metrics gpu__time_duration.sum, bench.py --steps 2)\n")
        print("Cold-cache, serialised per launch: compare shares, not absolute times.\n")
        print(launches(a.launches))
    if a.report:
        print("\n## Full-set capture (ncu --set full), tools/run_attn.py --config 4\n")
        print(report(a.report))

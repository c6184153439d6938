#!/usr/bin/env python3
"""Per-step event offsets of one backward CTA from tools/trace_bwd.py's
gpurun_out/trace_bwd.json (clock64 stamps of thread 0 of each warp role),
relative to the compute warps seeing dP(s) ready; medians over the middle half
of the steps.

    python tools/trace_bwd_report.py [gpurun_out/trace_bwd.json]
"""
import json
import statistics as st
import sys

NAMES = {10: "tma: stage s free", 11: "mma: S(s) issue (stage full)",
         1: "mma: dP(s) issue (dQ^T(s-1) drained)", 12: "mma: dP(s) issued",
         2: "mma: P(s) chunk 1 ready seen", 14: "mma: dS(s) ready seen",
         3: "mma: dK(s) issued", 4: "cmp: S(s) seen", 5: "cmp: P(s) released",
         6: "cmp: dP(s) seen", 16: "cmp: dP(s) loaded", 17: "cmp: dS(s) stored",
         18: "cmp: proxy fence done", 7: "cmp: dS(s) arrive", 8: "dq: dQ^T(s) seen",
         13: "dq: staging buffer free", 15: "dq: staged", 9: "dq: bulk reduce issued"}
ORDER = [11, 4, 1, 12, 5, 6, 16, 17, 18, 2, 7, 14, 8, 3, 13, 15, 9, 10]

tr = json.load(open(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/trace_bwd.json"))
n = max(i for i in range(len(tr[4])) if tr[4][i] > 0) + 1
lo, hi = n // 4, 3 * n // 4
period = st.median(tr[4][s + 1] - tr[4][s] for s in range(lo, hi))
print(f"steps {n}, median period {period:.0f} clk (S(s) seen -> S(s+1) seen)")
print(f"{'event':42s} {'step s':>8s} {'step s+1':>9s}   (clk relative to cmp: dP(s) seen)")
for ev in ORDER:
    d0 = st.median(tr[ev][s] - tr[6][s] for s in range(lo, hi))
    d1 = st.median(tr[ev][s + 1] - tr[6][s] for s in range(lo, hi - 1))
    print(f"{ev:3d} {NAMES[ev]:38s} {d0:8.0f} {d1:9.0f}")

#!/usr/bin/env python3
"""Discrete-event model of the backward kernel's per-step pipeline (one CTA):
the MMA warp issues MMA groups in program order into an in-order tensor pipe
with a shallow queue; the compute warps turn S into P and dP into dS; the dQ
warps drain dQ^T.  Used to compare MMA issue orders before touching the
kernel; calibrated against the -DBAM_TRACE timeline (tools/trace_bwd.py,
2147 clk per step at config 4).

    python tools/bwd_schedule_sim.py
"""
import itertools

# tensor clk per group (M=128): bias+S^T TS (32+256), bias+dP^T, dV TS, dQ^T SS N=64
# (port-bound 48/k-step), dK SS N=128
DUR = {"S": 288, "dP": 288, "dV": 256, "dQ": 384, "dK": 256}
NMMA = {"S": 9, "dP": 9, "dV": 4, "dQ": 8, "dK": 4}


def simulate(order, steps=60, q_depth=4, notify=150, p_time=750, ds_time=520, drain=120,
             dq_order_dep=True):
    """order: the MMA warp's per-step program, a list of tokens
    ("S", k) issue S of step s+k; ("dP", k); ("dV", 0); ("dQ", 0); ("dK", 0);
    with implicit waits: dV(s) waits p_ready(s), dQ(s)/dK(s) wait ds_ready(s),
    dP(s) waits dq_empty(s-1) (dQ^T shares dP's TMEM columns), S(s) waits dV(s-1)
    issued (S overwrites P^T; tensor execution is in order)."""
    pipe_free = 0.0
    queue = []            # end times of MMAs in flight (for the issue-queue model)
    t_mma = 0.0           # MMA warp clock
    done = {}             # (kind, step) -> completion time
    issued = {}
    cmp_t = 0.0           # compute warps clock
    p_ready, ds_ready, dq_empty = {}, {}, {}

    def issue(kind, s):
        nonlocal pipe_free, t_mma
        # each MMA of the group starts when the pipe is free; the warp's issue of MMA i
        # blocks until fewer than q_depth MMAs are queued ahead of it
        n, dur = NMMA[kind], DUR[kind] / NMMA[kind]
        for _ in range(n):
            while len(queue) >= q_depth and queue[0] <= t_mma:
                queue.pop(0)
            if len(queue) >= q_depth:
                t_mma = queue.pop(0)
            start = max(pipe_free, t_mma)
            pipe_free = start + dur
            queue.append(pipe_free)
            t_mma += 2
        done[(kind, s)] = pipe_free
        issued[(kind, s)] = t_mma

    # software pipeline: the compute / dQ warps are advanced lazily as their inputs appear
    def advance_compute(upto):
        nonlocal cmp_t
        s = len(p_ready)
        while s <= upto:
            if ("S", s) not in done or ("dP", s) not in done:
                return
            t = max(cmp_t, done[("S", s)] + notify)
            p_ready[s] = t + p_time
            t = max(p_ready[s], done[("dP", s)] + notify)
            ds_ready[s] = t + ds_time
            cmp_t = ds_ready[s]
            s += 1

    def advance_dq(s):
        if ("dQ", s) in done and s not in dq_empty:
            dq_empty[s] = done[("dQ", s)] + notify + drain

    # prologue: S(0), dP(0)
    issue("S", 0)
    issue("dP", 0)
    advance_compute(0)
    for s in range(steps):
        for kind, k in order:
            st = s + k
            if kind == "dV":
                advance_compute(st)
                t_mma = max(t_mma, p_ready[st] + notify)
            elif kind in ("dQ", "dK"):
                advance_compute(st)
                if ("dQ", st) not in done or kind == "dQ":
                    t_mma = max(t_mma, ds_ready[st] + notify)
            elif kind == "dP":
                if st >= steps:
                    continue
                advance_dq(st - 1)
                t_mma = max(t_mma, dq_empty[st - 1] + notify)
            elif kind == "S":
                if st >= steps:
                    continue
            issue(kind, st)
            if kind == "dQ":
                advance_dq(st)
        advance_compute(s + 1)
    s_a, s_b = steps // 3, 2 * steps // 3
    return (done[("dK", s_b)] - done[("dK", s_a)]) / (s_b - s_a)


CURRENT = [("dV", 0), ("S", 1), ("dQ", 0), ("dK", 0), ("dP", 1)]

if __name__ == "__main__":
    print("tensor clk per step:", sum(DUR.values()))
    print("current order", CURRENT, "->", round(simulate(CURRENT)), "clk/step")
    cands = []
    toks = [("dV", 0), ("S", 1), ("dQ", 0), ("dK", 0), ("dP", 1)]
    for perm in itertools.permutations(toks):
        # legality: dP(s+1) after dQ(s) (TMEM columns); S(s+1) after dV(s) (P^T columns)
        if perm.index(("dP", 1)) < perm.index(("dQ", 0)):
            continue
        if perm.index(("S", 1)) < perm.index(("dV", 0)):
            continue
        try:
            cands.append((simulate(list(perm)), perm))
        except KeyError:
            continue
    for t, perm in sorted(cands)[:8]:
        print(round(t), perm)

#!/usr/bin/env python3
"""List-scheduling model of one CP rank's forward under the copy-engine gather
(config 4): whole-row CTAs (row, head pair) on 148 SMs, each doing its local
key tiles first and then waiting for its KV head's rows from the peers, which
land head by head ((h+1)/8 of the gather).  Compares the head-pair-major CTA
order with the geometric class order at N=4 / N=8 (N=8 cannot be measured on
the <=4-GPU boxes here; the N=4 prediction is checked against the measured
flag-wait share, profiles/r02/cta_tail/real_cp_n2_n4.jsonl).  Tile time is
calibrated on the measured N=4 forward (8.9 ms).

    python tools/fwd_order_sim.py [per-head-pull GB/s, default 300] [rotation-pull GB/s, 520]

The second part models the shipped arrival order: every row's remote tiles grouped
by owner in rotation order rank+1, rank+2, ... and the peers pulled one after
another in that order, peer p landing at rot(p)/(G-1) of the gather.
"""
import heapq
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2503_11367_b200.workloads import CONFIGS
def blocks_of(segs):
    b=[]
    for nm,c in segs: b += [nm]*(c//128)
    return np.array(b)
names=blocks_of(CONFIGS[4]['segments']); nb=len(names)
from collections import Counter
# row j's key blocks
def keys(j):
    if names[j]=='text': return list(range(j+1))
    return [i for i in range(nb) if names[i]==names[j]]
W=[len(keys(j)) for j in range(nb)]
def lpt(W,G):
    order=sorted(range(len(W)), key=lambda i:(-W[i],i)); loads=[0]*G; own=[0]*len(W)
    for i in order:
        g=min(range(G), key=lambda g:(loads[g],g)); loads[g]+=W[i]; own[i]=g
    return own
def sim(G, order_kind, rank=0, t_tile=0.0019, gather_ms=None, H=16, nsm=148, a=0.004):
    own=lpt(W,G)
    rows=[j for j in range(nb) if own[j]==rank]
    rows.sort(key=lambda j:(-W[j],j))
    # per row: local tile count, remote tiles per peer
    info={}
    for j in rows:
        ks=keys(j); loc=sum(1 for k in ks if own[k]==rank)
        rem=[k for k in ks if own[k]!=rank]; rem.sort()
        # remote tiles in ascending key order; peers interleaved by key id
        info[j]=(loc, [own[k] for k in rem])
    if gather_ms is None:
        gather_ms = (G-1)/G*448*1.048576/GBPS  # MiB->MB /GBps -> ms
    land=lambda h: (h+1)/8*gather_ms  # head h of every peer lands at (h+1)/8 of the gather
    if order_kind=='hp':
        seq=[(j,hp) for hp in range(H) for j in rows]
    else:
        mx=W[rows[0]]
        cls=lambda j: min(int(mx//W[j]).bit_length()-1,15)
        seq=[]
        for c in range(16):
            cr=[j for j in rows if cls(j)==c]
            seq += [(j,hp) for hp in range(H) for j in cr]
    h=[0.0]*nsm; heapq.heapify(h); end=0; waits=0
    for j,hp in seq:
        t=heapq.heappop(h); kvh=hp//2
        loc,rem=info[j]
        t2=t+a+loc*t_tile
        if rem:
            lt=land(kvh)
            if t2<lt: waits+=lt-t2; t2=lt
            t2+=len(rem)*t_tile
        end=max(end,t2); heapq.heappush(h,t2)
    busy=sum(a+W[j]*t_tile for j,hp in seq)
    return end, busy/nsm, waits
def simB(G, order_kind, gbps, rank=0, t_tile=0.0019, H=16, nsm=148, a=0.004):
    own=lpt(W,G)
    rows=[j for j in range(nb) if own[j]==rank]
    rows.sort(key=lambda j:(-W[j],j))
    T=(G-1)/G*448*1.048576/gbps
    rot=lambda p: (p-rank)%G   # 1..G-1
    land=lambda p: rot(p)/(G-1)*T
    info={}
    for j in rows:
        ks=keys(j); loc=sum(1 for k in ks if own[k]==rank)
        cnt=[0]*G
        for k in ks:
            if own[k]!=rank: cnt[own[k]]+=1
        info[j]=(loc,cnt)
    if order_kind=='hp':
        seq=[(j,hp) for hp in range(H) for j in rows]
    else:
        mx=W[rows[0]]
        cls=lambda j: min(int(mx//W[j]).bit_length()-1,15)
        seq=[]
        for c in range(16):
            cr=[j for j in rows if cls(j)==c]
            seq += [(j,hp) for hp in range(H) for j in cr]
    h=[0.0]*nsm; heapq.heapify(h); end=0; waits=0
    peers=sorted([p for p in range(G) if p!=rank], key=rot)
    for j,hp in seq:
        t=heapq.heappop(h)
        loc,cnt=info[j]
        t2=t+a+loc*t_tile
        for p in peers:
            if cnt[p]:
                lt=land(p)
                if t2<lt: waits+=lt-t2; t2=lt
                t2+=cnt[p]*t_tile
        end=max(end,t2); heapq.heappush(h,t2)
    return end, waits

GBPS = float(sys.argv[1]) if len(sys.argv) > 1 else 300.0   # per-(peer, head) pulls
for G in (4,8):
    for kind in ('hp','class'):
        e,lb,wt=sim(G,kind)
        e0,_,_=sim(G,kind,gather_ms=0.0)
        print(f"G={G} {kind:5s} span {e:.3f} ms (no-exchange {e0:.3f}) LB {lb:.3f} waits {wt:.1f} SM-ms -> wait share {wt/(148*e)*100:.2f}%")

# the shipped scheme: remote tiles grouped by owner in rotation order, pulls peer by
# peer in the same order (cp.SymmExchange.gather_overlapped; 520-557 GB/s measured at N=4)
ROT = float(sys.argv[2]) if len(sys.argv) > 2 else 520.0
for G in (4, 8):
    for kind in ("hp", "class"):
        e, wt = simB(G, kind, ROT)
        print(f"rotation pulls {ROT:.0f} GB/s G={G} {kind:5s} span {e:.3f} ms wait share "
              f"{wt / (148 * e) * 100:.2f}%")

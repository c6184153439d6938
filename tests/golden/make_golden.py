#!/usr/bin/env python3
"""Generate golden vectors by running the REFERENCE implementation.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py            # small cases + configs 1-2

The reference package (``mmplan``, /root/reference/pkg/src) is imported
read-only; its outputs are written as JSON fixtures next to this script.
Nothing at test time reads /root/reference.
"""

from __future__ import annotations

import json
import os
import random
import subprocess
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SRC = "/root/reference/pkg/src"
sys.path.insert(0, REF_SRC)

from mmplan import balance as ref_balance  # noqa: E402
from mmplan import mask as ref_mask  # noqa: E402


def rle(row):
    out = []
    for c in row:
        if out and out[-1][1] == c:
            out[-1][0] += 1
        else:
            out.append([1, c])
    return out


def random_segments(rng, max_total, names, max_run=96):
    # same generator shape as the reference hypothesis test (test_mask.py:155-170)
    segs, total = [], 0
    while total < 1 or (rng.random() < 0.7 and total < max_total):
        m = rng.choice(["text"] + names)
        c = min(rng.randint(1, max_run), max_total - total)
        if c == 0:
            break
        segs.append((m, c))
        total += c
    return segs


def mask_case(desc=None, segments=None, modalities=(), block_size=128, tag=""):
    if segments is not None:
        m = ref_mask.build_bitfield(segments)
    else:
        m = ref_mask.BitfieldMask(descriptors=tuple(desc), modalities=tuple(modalities))
    w = ref_mask.block_workloads(m, block_size)
    case = {"tag": tag, "block_size": block_size, "descriptors": list(m.descriptors),
            "modalities": list(m.modalities), "workloads": list(w.workloads),
            "classes_rle": [rle(r) for r in w.classes]}
    if segments is not None:
        case["segments"] = [[a, b] for a, b in segments]
    return case


def make_mask_cases():
    cases = []
    packed = [("text", 1), ("A", 2), ("B", 2), ("text", 3)]
    workseg = [("text", 1), ("A", 2), ("text", 2), ("B", 2), ("text", 1)]
    cases.append(mask_case(segments=packed, block_size=1, tag="packed_b1"))
    cases.append(mask_case(segments=workseg, block_size=1, tag="workload_vector_b1"))
    cases.append(mask_case(segments=[(m, c * 128) for m, c in workseg], block_size=128,
                           tag="workload_vector_b128"))
    cases.append(mask_case(segments=[("text", 8)], block_size=1, tag="causal_b1"))
    cases.append(mask_case(segments=[("A", 4), ("B", 4)], block_size=4, tag="cross_modality"))
    cases.append(mask_case(segments=[("text", 4)], block_size=2, tag="causal_diag"))
    rng = random.Random(0xB200)
    for i in range(80):
        bs = rng.choice([1, 7, 16, 32, 128])
        segs = random_segments(rng, 512 if bs > 1 else 160, ["A", "B", "C", "D"])
        cases.append(mask_case(segments=segs, block_size=bs, tag=f"random_segments_{i}"))
    # raw-descriptor masks: text tokens carry random subsets of modality bits,
    # modality tokens one bit (valid but not build_bitfield-shaped)
    for i in range(40):
        bs = rng.choice([1, 7, 16, 32, 128])
        T = rng.randint(1, 400 if bs > 1 else 120)
        nmod = rng.randint(1, 5)
        desc, cur = [], None
        while len(desc) < T:
            run = rng.randint(1, 64)
            if rng.random() < 0.5:
                d = 1 | sum((2 << j) for j in range(nmod) if rng.random() < 0.5)
            else:
                d = 2 << rng.randrange(nmod)
            if rng.random() < 0.2:      # token-level jitter inside a run
                run = 1
            desc += [d] * min(run, T - len(desc))
        cases.append(mask_case(desc=desc, modalities=[f"m{j}" for j in range(nmod)],
                               block_size=bs, tag=f"raw_{i}"))
    return cases


def make_validation_cases():
    out = []
    probes = [
        ([1 << 63], []), ([0], []), ([0b110], ["A", "B"]), ([1, 1, -1], []),
        ([1, 1 << 64], []), ([1, (1 << 61) | 1], []), ([1, 2, 0b1010, 0], ["A", "B", "C"]),
        ([3, 5, 2], ["A", "B"]),
    ]
    for desc, mods in probes:
        try:
            ref_mask.BitfieldMask(descriptors=tuple(desc), modalities=tuple(mods)).validate()
            msg = None
        except ref_mask.MaskError as e:
            msg = str(e)
        out.append({"descriptors": [str(d) for d in desc], "modalities": mods, "error": msg})
    for segs in ([(f"m{i}", 1) for i in range(61)], [("text", 0)], []):
        try:
            ref_mask.build_bitfield(segs)
            msg = None
        except ref_mask.MaskError as e:
            msg = str(e)
        out.append({"segments": [[a, b] for a, b in segs], "error": msg})
    return out


def assignment_doc(a):
    return {"gpu_blocks": [list(x) for x in a.gpu_blocks], "loads": list(a.loads),
            "imbalance": a.imbalance}


def make_balance_cases():
    rng = random.Random(0xBA1A)
    cases = []
    vecs = [([1, 2, 2, 4, 5, 2, 2, 8], 4), ([3] * 8, 4), ([2, 2, 2, 2], 2), ([3, 3, 2], 2),
            ([1, 2, 3, 4], 2), (list(range(1, 9)), 4), ([3, 3, 2, 2, 2], 2), ([0, 0, 0], 3)]
    for _ in range(150):
        G = rng.randint(1, 8)
        n = rng.randint(1, 300)
        vecs.append(([rng.randint(0, 64) for _ in range(n)], G))
    for _ in range(30):   # many ties
        G = rng.randint(1, 16)
        n = rng.randint(1, 1100) if rng.random() < 0.3 else rng.randint(1, 200)
        vecs.append(([rng.choice([1, 2, 3, 8]) for _ in range(n)], G))
    for w, G in vecs:
        c = {"workloads": w, "gpus": G,
             "lpt": assignment_doc(ref_balance.lpt_distribute(w, G)),
             "zigzag": assignment_doc(ref_balance.zigzag_distribute(w, G))}
        C = rng.randint(1, 8)
        s = rng.randint(1, 8)
        sch = ref_balance.intra_schedule(w, C, s)
        c["intra"] = {"compute_units": C, "subblock_size": s,
                      "compute_makespan": sch.compute_makespan,
                      "aggregation_cost": sch.aggregation_cost}
        if len(w) <= 64:
            c["intra"]["unit_tasks"] = [[[sb.block, sb.index, sb.size] for sb in u]
                                        for u in sch.unit_tasks]
        c["report"] = ref_balance.balance_report(w, G, C, s)
        if len(w) <= 10 and G <= 4:
            c["ilp"] = assignment_doc(ref_balance.ilp_optimal(w, G))
        cases.append(c)
    return cases


def config_workloads(segments, tag):
    m = ref_mask.build_bitfield(segments)
    t0 = time.time()
    w = ref_mask.block_workloads(m, 128)
    dt = time.time() - t0
    print(f"{tag}: reference block_workloads T={len(m)} took {dt:.1f}s", flush=True)
    return {"tag": tag, "segments": [[a, b] for a, b in segments], "block_size": 128,
            "workloads": list(w.workloads), "classes_rle": [rle(r) for r in w.classes],
            "reference_seconds": dt}


def write(name, obj):
    with open(os.path.join(HERE, name), "w") as fh:
        json.dump(obj, fh, separators=(",", ":"))
        fh.write("\n")


def main():
    write("mask_cases.json", make_mask_cases())
    write("validation_cases.json", make_validation_cases())
    write("balance_cases.json", make_balance_cases())
    # cp-distribute report on the reference fixture (cli.py:86-117), byte-exact
    fixture = "/root/reference/pkg/fixtures/mask-two-encoders.json"
    with open(fixture) as fh:
        write("mask_two_encoders_fixture.json", json.load(fh))
    out = os.path.join(HERE, "report_two_encoders.json")
    subprocess.run([sys.executable, "-c",
                    f"import sys; sys.path.insert(0, {REF_SRC!r}); from mmplan.cli import main; "
                    f"sys.exit(main(['cp-distribute', '--mask', {fixture!r}, '-o', {out!r}]))"],
                   check=True)
    # the reference's own pinned invocation (ref tests/test_cli.py:46-53), checked here
    # against the reference's committed golden (ref tests/golden/report_two_encoders.json)
    out_ilp = os.path.join(HERE, "report_two_encoders_ilp.json")
    subprocess.run([sys.executable, "-c",
                    f"import sys; sys.path.insert(0, {REF_SRC!r}); from mmplan.cli import main; "
                    f"sys.exit(main(['cp-distribute', '--mask', {fixture!r}, '-g', '4', '-c', '2', "
                    f"'-s', '2', '--ilp', '-o', {out_ilp!r}]))"],
                   check=True)
    with open(out_ilp, "rb") as a, open("/root/reference/pkg/tests/golden/report_two_encoders.json",
                                        "rb") as b:
        assert a.read() == b.read(), "reference CLI no longer reproduces its own golden"
    if "--skip-configs" not in sys.argv:
        write("config1_workloads.json",
              config_workloads([("text", 128), ("image", 1024), ("text", 2944)], "config1"))
        write("config2_workloads.json",
              config_workloads([("image", 8192), ("text", 24576)], "config2"))


if __name__ == "__main__":
    main()

"""``cp-distribute`` command -- drop-in for the hot-path subcommand of the
reference CLI (``mmplan cp-distribute``, cli.py:86-117, 172-186).

Block workloads and the four-policy report come from the GPU kernels; the
JSON document is byte-identical to the reference's (sorted keys, indent 2,
trailing newline, cli.py:35-41).  Exit codes follow cli.py:26-30: 0 ok,
2 unreadable input, 3 validation error, 5 exact-search budget exceeded.

Only the context-parallel subcommand is provided: ``plan`` / ``simulate`` /
``gantt`` / ``gen`` belong to the pipeline planner, outside this hot path.
"""

from __future__ import annotations

import argparse
import json
import sys

from . import balance
from . import mask as mask_mod

EXIT_OK = 0
EXIT_PARSE = 2
EXIT_INVALID = 3
EXIT_NO_PLAN = 4
EXIT_BUDGET = 5

REPORT_SCHEMA_VERSION = 1


def _write_json(doc: dict, path: str | None) -> None:
    text = json.dumps(doc, indent=2, sort_keys=True) + "\n"
    if path is None or path == "-":
        sys.stdout.write(text)
    else:
        with open(path, "w", encoding="utf-8") as fh:
            fh.write(text)


def cmd_cp_distribute(args: argparse.Namespace) -> int:
    mask = mask_mod.load_mask(args.mask)
    work = mask_mod.block_workloads(mask, args.block_size)
    workloads = list(work.workloads)
    report = balance.balance_report(
        workloads, num_gpus=args.gpus, compute_units=args.compute_units,
        subblock_size=args.subblock_size, alpha=args.alpha, beta=args.beta)
    doc = {
        "schema_version": REPORT_SCHEMA_VERSION,
        "block_size": work.block_size,
        "workloads": workloads,
        "gpus": args.gpus,
        "compute_units": args.compute_units,
        "subblock_size": args.subblock_size,
        "alpha": args.alpha,
        "beta": args.beta,
        "policies": report,
    }
    if args.ilp:
        optimal = balance.ilp_optimal(workloads, args.gpus)
        doc["ilp_optimal"] = {
            "loads": list(optimal.loads),
            "makespan": optimal.makespan,
            "imbalance": optimal.imbalance,
        }
    if args.measure:
        # measured makespans on this B200 (8(f)3); absent from the default,
        # byte-identical report
        from . import measure
        doc["measured"] = {
            "heads": args.heads, "kv_heads": args.kv_heads, "head_dim": 128,
            "unit": "ms of fwd+bwd kernels per rank (ranks emulated on one GPU)",
            "policies": measure.measure_policies(mask, args.gpus, args.subblock_size,
                                                 heads=args.heads, kv_heads=args.kv_heads),
        }
    _write_json(doc, args.output)
    return EXIT_OK


def build_parser() -> argparse.ArgumentParser:
    parser = argparse.ArgumentParser(
        prog="bam", description="B200 bitfield-masked context-parallel attention tools")
    sub = parser.add_subparsers(dest="command", required=True)
    p = sub.add_parser("cp-distribute",
                       help="compare context-parallel distribution policies on a mask")
    p.add_argument("--mask", required=True, help="mask document (segments or descriptors)")
    p.add_argument("--gpus", "-g", type=int, default=4)
    p.add_argument("--block-size", type=int, default=mask_mod.DEFAULT_BLOCK_SIZE)
    p.add_argument("--compute-units", "-c", type=int, default=4)
    p.add_argument("--subblock-size", "-s", type=int, default=2)
    p.add_argument("--alpha", type=float, default=balance.DEFAULT_ALPHA,
                   help="aggregation cost per extra subblock")
    p.add_argument("--beta", type=float, default=balance.DEFAULT_BETA,
                   help="aggregation cost per split query block")
    p.add_argument("--ilp", action="store_true",
                   help="also solve the exact assignment (small instances only)")
    p.add_argument("--output", "-o", default=None, help="report path (default stdout)")
    p.add_argument("--measure", action="store_true",
                   help="also run every rank's attention fwd+bwd per policy on this GPU and "
                        "report measured makespans (adds a 'measured' key)")
    p.add_argument("--heads", type=int, default=32, help="query heads for --measure")
    p.add_argument("--kv-heads", type=int, default=8, help="KV heads for --measure")
    p.set_defaults(func=cmd_cp_distribute)
    return parser


def main(argv: list[str] | None = None) -> int:
    parser = build_parser()
    args = parser.parse_args(argv)
    try:
        return args.func(args)
    except (FileNotFoundError, IsADirectoryError, json.JSONDecodeError) as exc:
        print(f"error: cannot read input: {exc}", file=sys.stderr)
        return EXIT_PARSE
    except balance.BudgetError as exc:
        print(f"error: {exc}", file=sys.stderr)
        return EXIT_BUDGET
    except ValueError as exc:
        print(f"error: {exc}", file=sys.stderr)
        return EXIT_INVALID


if __name__ == "__main__":
    sys.exit(main())

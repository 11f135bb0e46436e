"""`lindbench bench` on the GPU: the reference's kernel-benchmark command
(proj/tools/main.cpp:54-72, proj/src/commands.cpp:96-121) over lbg_run_bench,
with its CSV / JSON report formats (bench.cpp:202-248) plus the GPU columns.

    python -m paper_2603_18052_b200.lindbench bench [--dims 3,9,27] [--variants aos,soa]
        [--reps 50000] [--warmup 10] [--seed 42] [--batch 1] [--format csv|json]
        [--output PATH] [--machine NAME]

Exit codes as commands.hpp:14-17: 0 ok, 2 input error, 3 some cell failed.
"""
from __future__ import annotations

import argparse
import sys

import paper_2603_18052_b200 as lbg

EXIT_OK, EXIT_INPUT, EXIT_PARTIAL = 0, 2, 3


def _machine_name() -> str:
    try:
        import torch
        if torch.cuda.is_available():
            p = torch.cuda.get_device_properties(0)
            return f"{p.name} ({p.multi_processor_count} SMs, sm_{p.major}{p.minor})"
    except Exception:  # noqa: BLE001
        pass
    return "b200"


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="lindbench")
    sub = ap.add_subparsers(dest="cmd", required=True)
    b = sub.add_parser("bench", help="Time the propagation kernel variants")
    b.add_argument("--dims", default="3,9,27")
    b.add_argument("--variants", default="aos,soa")
    b.add_argument("--reps", type=int, default=50000)
    b.add_argument("--warmup", type=int, default=10)
    b.add_argument("--seed", type=int, default=lbg.SEED)
    b.add_argument("--batch", type=int, default=1, help="copies of the chain run at once (GPU extension)")
    b.add_argument("--format", choices=["csv", "json"], default="csv")
    b.add_argument("--output", default=None)
    b.add_argument("--machine", default=None, help="machine name in the report header")
    args = ap.parse_args(argv)
    try:
        dims = [int(x) for x in args.dims.split(",") if x]
        variants = [x for x in args.variants.split(",") if x]
        for v in variants:
            if v not in lbg.VARIANT:
                raise ValueError(f"bench: unknown variant: {v}")
        if args.reps < 1:
            raise ValueError("--reps must be positive")
    except ValueError as e:
        print(f"error: {e}", file=sys.stderr)
        return EXIT_INPUT
    cfgs, res = lbg.run_matrix(dims, variants, args.reps, args.warmup, args.seed, args.batch)
    machine = args.machine or _machine_name()
    text = (lbg.write_bench_json if args.format == "json" else lbg.write_bench_csv)(cfgs, res, machine)
    if args.output:
        with open(args.output, "w") as f:
            f.write(text)
    else:
        sys.stdout.write(text)
    for c, r in zip(cfgs, res):
        if r.failed:
            name = {0: "aos", 1: "soa", 2: "simd"}.get(c.variant, "?")
            print(f"error: bench cell failed: dim={c.dim} variant={name}: {r.error.decode()}", file=sys.stderr)
            return EXIT_PARTIAL
    return EXIT_OK


if __name__ == "__main__":
    sys.exit(main())

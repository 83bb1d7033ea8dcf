"""``count`` front door (reference cli.py:117-138 cmd_count).

    python -m paper_1503_00576_b200 count FILE [--format auto|text|binary]
        [--mode strict|symmetrize|normalize] [--workers W] [--pools P]

Prints the reference's three lines -- summary, phases, and the stable key=value record
(graph= vertices= edges= triangles= wedges= transitivity= preprocess_ms= count_ms=
total_ms= workers= pools=) -- with the counting, validation and wedge sum on the GPU.
Exit codes as the reference: 0 success, 1 data error, 2 usage error.  ``workers`` has no
effect on the GPU path; it is accepted and echoed so existing record parsers still work.
The reference's bench / generate / convert subcommands are out of scope.
"""
from __future__ import annotations

import argparse
import os
import sys

from . import io as gio
from .count import count_with_timings, default_workers, warm_kernel
from .graph import GraphValidationError
from .metrics import CountOverflowError, transitivity, wedge_count

WORKERS_ENV = "TRICOUNT_WORKERS"

DATA_ERRORS = (GraphValidationError, gio.ParseError, gio.BadMagicError, gio.TruncatedFileError,
               OSError, ValueError, RuntimeError, CountOverflowError)


def _env_workers() -> int:
    value = os.environ.get(WORKERS_ENV)
    if value:
        try:
            return int(value)
        except ValueError:
            pass
    return default_workers()


def build_parser() -> argparse.ArgumentParser:
    parser = argparse.ArgumentParser(
        prog="tricount-b200",
        description="Exact triangle counting on B200: degree-ordered orientation and "
        "per-edge adjacency intersections in sm_100a kernels.")
    sub = parser.add_subparsers(dest="command", required=True)
    p = sub.add_parser("count", help="count triangles in a graph file")
    p.add_argument("input", help="edge list file (text or TRI1 binary)")
    p.add_argument("--format", choices=("auto", "text", "binary"), default="auto",
                   help="input format (default: sniff the magic bytes)")
    p.add_argument("--mode", choices=gio.READ_MODES, default="symmetrize",
                   help="edge list interpretation (default symmetrize)")
    p.add_argument("--workers", type=int, default=None,
                   help=f"accepted for compatibility (default ${WORKERS_ENV} or CPU count)")
    p.add_argument("--pools", type=int, default=1,
                   help="independent contiguous edge partitions (default 1)")
    return parser


def cmd_count(args) -> int:
    g = gio.load_graph(args.input, args.format, args.mode)
    workers = args.workers if args.workers is not None else _env_workers()
    warm_kernel()
    triangles, timings = count_with_timings(g, workers, pools=args.pools)
    wedges = wedge_count(g)
    ratio = transitivity(triangles, wedges)
    print(f"{args.input}: {g.num_vertices} vertices, {g.num_undirected_edges} undirected edges; "
          f"{triangles} triangles, transitivity {ratio:.6f}")
    print(f"phases: preprocess {timings.preprocess_ms:.3f} ms, count {timings.count_ms:.3f} ms "
          f"({workers} workers, {args.pools} pools; file parsing excluded)")
    print(f"graph={args.input} vertices={g.num_vertices} edges={g.num_undirected_edges} "
          f"triangles={triangles} wedges={wedges} transitivity={ratio:.6f} "
          f"preprocess_ms={timings.preprocess_ms:.3f} count_ms={timings.count_ms:.3f} "
          f"total_ms={timings.total_ms:.3f} workers={workers} pools={args.pools}")
    return 0


def main(argv=None) -> int:
    parser = build_parser()
    try:
        args = parser.parse_args(argv)
    except SystemExit as e:
        return int(e.code) if isinstance(e.code, int) else 2
    try:
        return cmd_count(args)
    except DATA_ERRORS as e:
        print(f"error: {e}", file=sys.stderr)
        return 1


if __name__ == "__main__":
    sys.exit(main())

"""Command line: ``python -m paper_2508_18224_b200 bench``.

Mirrors the reference's ``blockattn bench`` (cli.py:149-242): the same CSV
columns (``BENCH_COLUMNS``), one row per (engine, phase), the value-independent
meter counters next to the measured time.  The backend column is ``cuda``;
times are CUDA-event medians / minima over ``--repeat`` runs of the device
operators (kv_major phases, the query-major forward, the kv_major backward).
Errors (bad config, malformed selection) exit with status 2 as in the
reference (cli.py:281-288).
"""

from __future__ import annotations

import argparse
import csv
import statistics
import sys

from .config import ConfigError, load_config_file, make_config
from .selection import SelectionError

BENCH_COLUMNS = (
    "engine", "phase", "backend", "repeat", "median_s", "min_s",
    "bytes_loaded", "bytes_stored", "flops", "task_count", "inner_iterations",
)


def _time(fn, repeat):
    import torch

    times, result = [], None
    for _ in range(repeat):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        result = fn()
        e1.record()
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1) / 1e3)
    return result, statistics.median(times), min(times)


def cmd_bench(args) -> int:
    import torch

    from . import TrafficMeter, build_inverse_index, kv_major, query_major, select_topk_blocks

    cfg = load_config_file(args.config) if args.config else make_config(
        N=2048, d_K=64, d_V=64, h=4, h_K=1, B_K=64, T=8, W=128)
    dtype = {"bf16": torch.bfloat16, "f32": torch.float32, "f64": torch.float64}[args.dtype]
    g = torch.Generator(device="cuda").manual_seed(args.seed)
    mk = lambda *s: torch.randn(*s, device="cuda", generator=g).to(dtype)  # noqa: E731
    L = lambda x: x.permute(0, 2, 1)  # noqa: E731  storage (N, heads, d) -> logical (N, d, heads)
    Q, K, V = L(mk(cfg.N, cfg.h, cfg.d_K)), L(mk(cfg.N, cfg.h_K, cfg.d_K)), L(mk(cfg.N, cfg.h_K, cfg.d_V))
    dOut = L(mk(cfg.N, cfg.h, cfg.d_V))
    scores = torch.rand(cfg.h_K, cfg.N, cfg.b, device="cuda", generator=g)
    sel = select_topk_blocks(scores, cfg)
    inv = build_inverse_index(sel, cfg)
    rows = []

    def record(engine, phase, counters, med, best):
        rows.append({"engine": engine, "phase": phase, "backend": "cuda", "repeat": args.repeat,
                     "median_s": format(med, ".6e"), "min_s": format(best, ".6e"),
                     "bytes_loaded": counters.bytes_loaded, "bytes_stored": counters.bytes_stored,
                     "flops": counters.flops, "task_count": counters.task_count,
                     "inner_iterations": counters.inner_iterations})

    def run_stats():
        m = TrafficMeter()
        return kv_major.compute_softmax_stats(Q, K, sel, cfg, meter=m), m

    (stats, m), med, best = _time(run_stats, args.repeat)
    record("kv_major", "stats", m.phase("stats"), med, best)

    def run_block():
        m = TrafficMeter()
        return kv_major.block_pass_forward(Q, K, V, inv, stats, cfg, meter=m), m

    (buf, m), med, best = _time(run_block, args.repeat)
    record("kv_major", "block_pass", m.phase("block_pass"), med, best)

    def run_reduce():
        m = TrafficMeter()
        return kv_major.reduce_forward(buf, inv, stats, cfg, meter=m), m

    (_, m), med, best = _time(run_reduce, args.repeat)
    record("kv_major", "reduce", m.phase("reduce"), med, best)
    (res, med, best) = _time(lambda: kv_major.selected_forward(Q, K, V, sel, cfg), args.repeat)
    record("kv_major", "forward_fused", res[1].phase("block_pass"), med, best)
    (res, med, best) = _time(lambda: query_major.selected_forward(Q, K, V, sel, cfg), args.repeat)
    record("query_major", "forward", res[1].phase("query_major"), med, best)
    (res, med, best) = _time(lambda: kv_major.selected_backward(Q, K, V, sel, dOut, cfg), args.repeat)
    for name, counters in res[3].as_rows():
        record("kv_major", f"backward_{name}", counters, med, best)
    (res, med, best) = _time(lambda: query_major.selected_backward(Q, K, V, sel, dOut, cfg), args.repeat)
    record("query_major", "backward", res[3].phase("query_major"), med, best)
    out = open(args.csv, "w", newline="") if args.csv else sys.stdout
    try:
        w = csv.DictWriter(out, fieldnames=BENCH_COLUMNS)
        w.writeheader()
        w.writerows(rows)
    finally:
        if args.csv:
            out.close()
    return 0


def build_parser() -> argparse.ArgumentParser:
    parser = argparse.ArgumentParser(prog="paper_2508_18224_b200",
                                     description="B200 FSA / NSA operators")
    sub = parser.add_subparsers(dest="command", required=True)
    p = sub.add_parser("bench", help="CUDA-event micro-benchmarks of the device operators")
    p.add_argument("--config", help="key = value config file (reference format)")
    p.add_argument("--seed", type=int, default=0)
    p.add_argument("--repeat", type=int, default=3)
    p.add_argument("--dtype", choices=("bf16", "f32", "f64"), default="bf16")
    p.add_argument("--csv", help="output CSV path (defaults to stdout)")
    p.set_defaults(fn=cmd_bench)
    return parser


def main(argv=None) -> int:
    args = build_parser().parse_args(argv)
    try:
        return args.fn(args)
    except (ConfigError, SelectionError, FileNotFoundError) as exc:
        print(f"error: {exc}", file=sys.stderr)
        return 2


if __name__ == "__main__":
    sys.exit(main())

"""Latency / throughput of the NSA step at every BASELINE.json GPU shape (1 GPU).

    python tools/sweep.py [--steps K] [--warmup W]

Per config: forward and forward+backward ms (CUDA events on the launching
stream, max of nothing -- one GPU), tokens/s, and effective TFLOP/s on the
algorithmic FLOPs of SURVEY 8(d) (selected 4/10 d B_K R, sliding 4/10 d h
sum_t min(t+1, W), compressed 4 d h sum_t floor((t+1)/B_K)); R is read from the
inverse index.  Synthetic N(0,1) bf16 inputs, U[0,1) gates.
"""

import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2508_18224_b200 as fsa  # noqa: E402
from paper_2508_18224_b200 import nsa  # noqa: E402

CONFIGS = [
    ("llama3-8b-attn-32k", dict(N=32768, h=32, h_K=8), True),
    ("llama3-8b-attn-64k (north_star target)", dict(N=65536, h=32, h_K=8), True),
    ("qwen2.5-7b-attn-64k (fwd)", dict(N=65536, h=28, h_K=4), False),
    ("gqa1-stress-64k", dict(N=65536, h=16, h_K=16), True),
    ("qwen3-14b-attn-128k", dict(N=131072, h=40, h_K=8), True),
]


def flops(cfg, R):
    d, N, W = cfg.d_K, cfg.N, cfg.W
    slide = sum(min(t + 1, W) for t in range(N))
    formed = sum((t + 1) // cfg.B_K for t in range(N))
    fwd = 4.0 * d * cfg.B_K * R + 4.0 * d * cfg.h * slide + 4.0 * d * cfg.h * formed
    bwd = 10.0 * d * cfg.B_K * R + 10.0 * d * cfg.h * slide
    return fwd, bwd


def time_it(fn, steps, warmup):
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / steps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=2)
    ap.add_argument("--nsa", action="store_true",
                    help="also time the selected branch alone: FSA (kv-major, tcgen05) vs the NSA "
                         "query-major baseline (query_major.selected_forward)")
    ap.add_argument("--full", action="store_true",
                    help="also time the step with the compressed-branch + gate backward (full=True)")
    a = ap.parse_args()
    rows = []
    for name, spec, bwd in CONFIGS:
        cfg = fsa.make_config(N=spec["N"], d_K=128, d_V=128, h=spec["h"], h_K=spec["h_K"], B_K=64,
                              T=16, W=512)
        g = torch.Generator(device="cuda").manual_seed(0)
        bf = torch.bfloat16
        q = torch.randn(cfg.N, cfg.h, 128, device="cuda", dtype=bf, generator=g)
        k = torch.randn(cfg.N, cfg.h_K, 128, device="cuda", dtype=bf, generator=g)
        v = torch.randn(cfg.N, cfg.h_K, 128, device="cuda", dtype=bf, generator=g)
        do = torch.randn(cfg.N, cfg.h, 128, device="cuda", dtype=bf, generator=g)
        tau = torch.rand(cfg.N, 3, device="cuda", generator=g)
        _, ctx = nsa.nsa_forward(q, k, v, tau, cfg)
        R = int(ctx.inv.offsets[:, -1].to(torch.int64).sum()) * cfg.g
        f_fwd, f_bwd = flops(cfg, R)
        ms_f = time_it(lambda: nsa.nsa_forward(q, k, v, tau, cfg), a.steps, a.warmup)
        row = {"config": name, "N": cfg.N, "h": cfg.h, "h_K": cfg.h_K, "g": cfg.g, "R": R,
               "fwd_ms": round(ms_f, 3), "fwd_tflops": round(f_fwd / ms_f / 1e9, 1),
               "fwd_tokens_s": round(cfg.N / ms_f * 1e3, 1)}
        if bwd:
            def step():
                _, c_ = nsa.nsa_forward(q, k, v, tau, cfg)
                nsa.nsa_backward(c_, do)
            ms = time_it(step, a.steps, a.warmup)
            row.update({"fwd_bwd_ms": round(ms, 3), "fwd_bwd_tflops": round((f_fwd + f_bwd) / ms / 1e9, 1),
                        "fwd_bwd_tokens_s": round(cfg.N / ms * 1e3, 1)})
        if a.nsa:
            from paper_2508_18224_b200 import kv_major, query_major
            L = lambda x: x.permute(0, 2, 1)  # noqa: E731  logical (N, d, h) views
            sel = ctx.sel
            row["sel_fwd_fsa_ms"] = round(time_it(
                lambda: kv_major.selected_forward(L(q), L(k), L(v), sel, cfg), a.steps, a.warmup), 3)
            row["sel_fwd_nsa_ms"] = round(time_it(
                lambda: query_major.selected_forward(L(q), L(k), L(v), sel, cfg), a.steps, a.warmup), 3)
            row["fsa_speedup"] = round(row["sel_fwd_nsa_ms"] / row["sel_fwd_fsa_ms"], 2)
            if bwd:
                row["sel_bwd_fsa_ms"] = round(time_it(
                    lambda: kv_major.selected_backward(L(q), L(k), L(v), sel, L(do), cfg), 2, 1), 3)
                row["sel_bwd_nsa_ms"] = round(time_it(
                    lambda: query_major.selected_backward(L(q), L(k), L(v), sel, L(do), cfg), 2, 1), 3)
                row["fsa_bwd_speedup"] = round(row["sel_bwd_nsa_ms"] / row["sel_bwd_fsa_ms"], 2)
        if a.full and bwd:
            def full_step():
                _, c_ = nsa.nsa_forward(q, k, v, tau, cfg)
                nsa.nsa_backward(c_, do, full=True)
            row["fwd_bwd_full_ms"] = round(time_it(full_step, 2, 1), 3)
        rows.append(row)
        print(json.dumps(row), flush=True)
        del q, k, v, do, tau, ctx
        torch.cuda.empty_cache()
    print("\n| config | N | g | fwd ms | fwd TFLOP/s | fwd+bwd ms | fwd+bwd TFLOP/s | fwd+bwd tokens/s |")
    print("|---|---|---|---|---|---|---|---|")
    for r in rows:
        print(f"| {r['config']} | {r['N']} | {r['g']} | {r['fwd_ms']} | {r['fwd_tflops']} | "
              f"{r.get('fwd_bwd_ms', '-')} | {r.get('fwd_bwd_tflops', '-')} | {r.get('fwd_bwd_tokens_s', '-')} |")
    if a.nsa:
        print("\n| config | g | selected fwd FSA ms | NSA query-major ms | FSA speed-up | "
              "selected bwd FSA ms | NSA query-major bwd ms | FSA bwd speed-up |")
        print("|---|---|---|---|---|---|---|---|")
        for r in rows:
            print(f"| {r['config']} | {r['g']} | {r['sel_fwd_fsa_ms']} | {r['sel_fwd_nsa_ms']} | {r['fsa_speedup']}x | "
                  f"{r.get('sel_bwd_fsa_ms', '-')} | {r.get('sel_bwd_nsa_ms', '-')} | {r.get('fsa_bwd_speedup', '-')}x |")


if __name__ == "__main__":
    main()

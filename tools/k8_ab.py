"""A/B timing of one C-ABI entry point under env-selected kernel variants.

    python tools/k8_ab.py --entry fsa_sel_bwd --env FSA_K8_VARIANT --variants 0,1,2,3 [--N 131072 --h 40 --h_K 8]

Runs one NSA forward + backward, then times the selected-branch backward
(K8: fsa_sel_bwd) or forward (K5: fsa_sel_fwd) alone, CUDA events, median of
--iters, alternating variants so clock drift hits all of them alike.
"""
import argparse
import ctypes
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2508_18224_b200 as fsa  # noqa: E402
from paper_2508_18224_b200 import _lib, nsa  # noqa: E402
from paper_2508_18224_b200.kv_major import _backward_core  # noqa: E402


# entries called by nsa_backward (others are timed inside nsa_forward)
BACKWARD = ("fsa_slide_bwd", "fsa_dq_reduce_add", "fsa_gate_backward_fold", "fsa_bwd_delta",
            "fsa_stage_f16_ops")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--N", type=int, default=131072)
    ap.add_argument("--h", type=int, default=40)
    ap.add_argument("--h_K", type=int, default=8)
    ap.add_argument("--entry", default="fsa_sel_bwd")
    ap.add_argument("--env", default="FSA_K8_VARIANT")
    ap.add_argument("--variants", default="0,1")
    ap.add_argument("--iters", type=int, default=7)
    a = ap.parse_args()
    cfg = fsa.make_config(N=a.N, d_K=128, d_V=128, h=a.h, h_K=a.h_K, B_K=64, T=16, W=512)
    g = torch.Generator(device="cuda").manual_seed(0)
    mk = lambda *s: torch.randn(*s, device="cuda", dtype=torch.bfloat16, generator=g)  # noqa: E731
    q, k, v, do = mk(a.N, a.h, 128), mk(a.N, a.h_K, 128), mk(a.N, a.h_K, 128), mk(a.N, a.h, 128)
    tau = torch.rand(a.N, 3, device="cuda", generator=g)
    out, ctx = nsa.nsa_forward(q, k, v, tau, cfg)
    nsa.nsa_backward(ctx, do)
    torch.cuda.synchronize()
    orig = _lib.call
    times = {}

    def timed(name, *args):
        if name != a.entry:
            return orig(name, *args)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        r = orig(name, *args)
        e1.record()
        timed.ev.append((e0, e1))
        return r
    timed.ev = []
    _lib.call = timed
    variants = a.variants.split(",")
    res = {vv: [] for vv in variants}
    for it in range(a.iters + 1):
        for vv in variants:
            os.environ[a.env] = vv
            timed.ev = []
            if a.entry == "fsa_sel_bwd":
                _backward_core(cfg, torch.bfloat16, q, k, v, do, ctx.sel, ctx.inv, ctx.out_sel, ctx.lse_sel)
            elif a.entry in BACKWARD:
                nsa.nsa_backward(ctx, do)
            else:
                nsa.nsa_forward(q, k, v, tau, cfg)
            torch.cuda.synchronize()
            if it > 0:
                res[vv].append(sum(e0.elapsed_time(e1) for e0, e1 in timed.ev))
    _lib.call = orig
    rows = int(ctx.inv.offsets[:, -1].sum()) * cfg.g
    fl = {"fsa_sel_bwd": 10, "fsa_sel_fwd": 4}.get(a.entry, 0) * 128 * 64 * rows
    for vv in variants:
        m = statistics.median(res[vv])
        tf = f"{fl / m / 1e9:.0f} TFLOP/s  " if fl else ""
        print(f"N={a.N} h={a.h} {a.entry} {a.env}={vv}: {m:.3f} ms  {tf}(min {min(res[vv]):.3f})")


if __name__ == "__main__":
    main()

"""Run one kernel stage on a small bf16 problem (hang isolation / quick timing).

    python tools/stage_check.py <stage> [N]
stages: slide_fwd cmp_fwd sel_fwd sel_bwd slide_bwd nsa nsa_full
"""

import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2508_18224_b200 as fsa  # noqa: E402
from paper_2508_18224_b200 import kv_major  # noqa: E402


def main():
    stage = sys.argv[1]
    N = int(sys.argv[2]) if len(sys.argv) > 2 and stage != "shape" else 2048
    g = torch.Generator(device="cuda").manual_seed(0)
    mk = lambda *s: torch.randn(*s, device="cuda", dtype=torch.bfloat16, generator=g)  # noqa: E731
    if stage in ("llama", "shape"):  # 2 NSA fwd+bwd steps (profile the second)
        # shape: python tools/stage_check.py shape N h h_K
        NN, hh, hk = (32768, 32, 8) if stage == "llama" else (int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4]))
        cfg = fsa.make_config(N=NN, d_K=128, d_V=128, h=hh, h_K=hk, B_K=64, T=16, W=512)
        q, k, v, do = mk(cfg.N, hh, 128), mk(cfg.N, hk, 128), mk(cfg.N, hk, 128), mk(cfg.N, hh, 128)
        tau = torch.rand(cfg.N, 3, device="cuda", generator=g)
        for _ in range(2):
            out, ctx = fsa.nsa_forward(q, k, v, tau, cfg)
            fsa.nsa_backward(ctx, do)
        torch.cuda.synchronize()
        print(stage, "ok", flush=True)
        return
    cfg = fsa.make_config(N=N, d_K=128, d_V=128, h=8, h_K=2, B_K=64, T=8, W=256)
    q, k, v, do = mk(N, 8, 128), mk(N, 2, 128), mk(N, 2, 128), mk(N, 8, 128)
    L = lambda x: x.permute(0, 2, 1)  # noqa: E731
    t0 = time.time()
    if stage == "slide_fwd":
        r = fsa.sliding_attention_forward(L(q), L(k), L(v), cfg)
    elif stage == "cmp_fwd":
        c = fsa.compress_kv(L(k), L(v), cfg)
        r = fsa.compressed_attention_forward(L(q), c, cfg)
    elif stage == "sel_fwd":
        sel = fsa.select_topk_blocks(torch.rand(2, N, cfg.b, device="cuda", generator=g), cfg)
        r = kv_major.selected_forward(L(q), L(k), L(v), sel, cfg)
    elif stage == "sel_bwd":
        sel = fsa.select_topk_blocks(torch.rand(2, N, cfg.b, device="cuda", generator=g), cfg)
        r = kv_major.selected_backward(L(q), L(k), L(v), sel, L(do), cfg)
    elif stage == "slide_bwd":
        r = fsa.sliding_attention_backward(L(q), L(k), L(v), L(do), cfg)
    elif stage == "nsa":
        out, ctx = fsa.nsa_forward(q, k, v, torch.rand(N, 3, device="cuda", generator=g), cfg)
        r = fsa.nsa_backward(ctx, do)
    elif stage == "nsa_full":  # + the compressed-branch backward (K8 compressed mode)
        out, ctx = fsa.nsa_forward(q, k, v, torch.rand(N, 3, device="cuda", generator=g), cfg)
        r = fsa.nsa_backward(ctx, do, full=True)
    torch.cuda.synchronize()
    print(f"{stage} N={N} ok {time.time() - t0:.3f}s", flush=True)


if __name__ == "__main__":
    main()

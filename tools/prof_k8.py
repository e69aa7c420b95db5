"""One NSA step, then one extra selected-branch backward (K8) launch for ncu:
    ncu -k regex:tc_sel_bwd --launch-skip 2 --launch-count 1 python tools/prof_k8.py"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2508_18224_b200 as fsa  # noqa: E402
from paper_2508_18224_b200 import nsa  # noqa: E402
from paper_2508_18224_b200.kv_major import _backward_core  # noqa: E402

g = torch.Generator(device="cuda").manual_seed(0)
cfg = fsa.make_config(N=32768, d_K=128, d_V=128, h=32, h_K=8, B_K=64, T=16, W=512)
mk = lambda *s: torch.randn(*s, device="cuda", dtype=torch.bfloat16, generator=g)  # noqa: E731
q, k, v, do = mk(cfg.N, 32, 128), mk(cfg.N, 8, 128), mk(cfg.N, 8, 128), mk(cfg.N, 32, 128)
tau = torch.rand(cfg.N, 3, device="cuda", generator=g)
out, ctx = nsa.nsa_forward(q, k, v, tau, cfg)
nsa.nsa_backward(ctx, do)
_backward_core(cfg, torch.bfloat16, q, k, v, do, ctx.sel, ctx.inv, ctx.out_sel, ctx.lse_sel)
torch.cuda.synchronize()

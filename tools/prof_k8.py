"""One NSA step, then one extra selected-branch forward (K5) and backward (K8)
launch for ncu:
    ncu -k regex:tc_sel_bwd --launch-skip 1 --launch-count 1 python tools/prof_k8.py [N h h_K]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2508_18224_b200 as fsa  # noqa: E402
from paper_2508_18224_b200 import nsa  # noqa: E402
from paper_2508_18224_b200.kv_major import _backward_core  # noqa: E402

N, h, hk = (int(x) for x in sys.argv[1:4]) if len(sys.argv) > 3 else (32768, 32, 8)
g = torch.Generator(device="cuda").manual_seed(0)
cfg = fsa.make_config(N=N, d_K=128, d_V=128, h=h, h_K=hk, B_K=64, T=16, W=512)
mk = lambda *s: torch.randn(*s, device="cuda", dtype=torch.bfloat16, generator=g)  # noqa: E731
q, k, v, do = mk(cfg.N, h, 128), mk(cfg.N, hk, 128), mk(cfg.N, hk, 128), mk(cfg.N, h, 128)
tau = torch.rand(cfg.N, 3, device="cuda", generator=g)
out, ctx = nsa.nsa_forward(q, k, v, tau, cfg)
nsa.nsa_backward(ctx, do)
nsa.nsa_forward(q, k, v, tau, cfg)
_backward_core(cfg, torch.bfloat16, q, k, v, do, ctx.sel, ctx.inv, ctx.out_sel, ctx.lse_sel)
torch.cuda.synchronize()

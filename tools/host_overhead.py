"""Host cost of issuing one NSA fwd+bwd step (no sync) vs its device time."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2508_18224_b200 as fsa  # noqa: E402
from paper_2508_18224_b200 import nsa  # noqa: E402

cfg = fsa.make_config(N=32768, d_K=128, d_V=128, h=32, h_K=8, B_K=64, T=16, W=512)
g = torch.Generator(device="cuda").manual_seed(0)
mk = lambda *s: torch.randn(*s, device="cuda", dtype=torch.bfloat16, generator=g)  # noqa: E731
q, k, v, do = mk(cfg.N, 32, 128), mk(cfg.N, 8, 128), mk(cfg.N, 8, 128), mk(cfg.N, 32, 128)
tau = torch.rand(cfg.N, 3, device="cuda", generator=g)


def step():
    _, ctx = nsa.nsa_forward(q, k, v, tau, cfg)
    return nsa.nsa_backward(ctx, do)


for _ in range(3):
    step()
torch.cuda.synchronize()
# host issue cost: a step issued while the GPU is still busy with a long queue
t0 = time.perf_counter()
for _ in range(10):
    step()
t1 = time.perf_counter()
torch.cuda.synchronize()
t2 = time.perf_counter()
print(f"host issue {1e3 * (t1 - t0) / 10:.2f} ms/step, wall {1e3 * (t2 - t0) / 10:.2f} ms/step")

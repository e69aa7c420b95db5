"""Re-run the compressed-branch backward (full NSA backward) many times and
check the results are bit-identical run to run (race hunting).
    python tools/stress_cmp.py [runs] [N h h_K B_K]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2508_18224_b200 as fsa  # noqa: E402

runs = int(sys.argv[1]) if len(sys.argv) > 1 else 50
N, h, hk, bk = (int(x) for x in sys.argv[2:6]) if len(sys.argv) > 5 else (2048, 7, 1, 32)
cfg = fsa.make_config(N=N, d_K=128, d_V=128, h=h, h_K=hk, B_K=bk, T=6, W=128)
g = torch.Generator(device="cuda").manual_seed(0)
mk = lambda *s: torch.randn(*s, device="cuda", dtype=torch.bfloat16, generator=g)  # noqa: E731
q, k, v, do = mk(N, h, 128), mk(N, hk, 128), mk(N, hk, 128), mk(N, h, 128)
tau = torch.rand(N, 3, device="cuda", generator=g)
ref = None
bad = 0
for i in range(runs):
    _, ctx = fsa.nsa.nsa_forward(q, k, v, tau, cfg)
    got = fsa.nsa.nsa_backward(ctx, do, full=True)
    got = [x.clone() for x in got]
    if ref is None:
        ref = got
        continue
    diffs = [(name, float((a - b).abs().max())) for name, a, b in zip(("dQ", "dK", "dV", "dtau"), got, ref)
             if not torch.equal(a, b)]
    if diffs:
        bad += 1
        print("run", i, "differs:", diffs, flush=True)
print(f"{runs} runs, {bad} differing", flush=True)

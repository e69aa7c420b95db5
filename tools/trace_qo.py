"""Timeline of CTA 0 of the sliding-window dQ kernel (fsa_debug_qo_trace)."""
import ctypes
import os
import sys

os.environ["FSA_TRACE_LIB"] = "1"  # the trace build (build.py --trace)
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2508_18224_b200 as fsa  # noqa: E402
from paper_2508_18224_b200 import _lib, nsa  # noqa: E402

g = torch.Generator(device="cuda").manual_seed(0)
cfg = fsa.make_config(N=32768, d_K=128, d_V=128, h=32, h_K=8, B_K=64, T=16, W=512)
mk = lambda *s: torch.randn(*s, device="cuda", dtype=torch.bfloat16, generator=g)  # noqa: E731
q, k, v, do = mk(cfg.N, 32, 128), mk(cfg.N, 8, 128), mk(cfg.N, 8, 128), mk(cfg.N, 32, 128)
tau = torch.rand(cfg.N, 3, device="cuda", generator=g)
out, ctx = nsa.nsa_forward(q, k, v, tau, cfg)
nsa.nsa_backward(ctx, do)
torch.cuda.synchronize()
buf = torch.zeros(4 * 128 * 8 + 3072, dtype=torch.int64, device="cuda")
lib = _lib.lib()
lib.fsa_debug_qo_trace(ctypes.c_void_p(buf.data_ptr()))
L = lambda x: x.permute(0, 2, 1)  # noqa: E731
fsa.sliding_attention_forward(L(q), L(k), L(v), cfg)
torch.cuda.synchronize()
lib.fsa_debug_qo_trace(None)
tb = buf.cpu()
t = tb[: 4 * 128 * 8].view(4, 128, 8)
its = tb[4 * 128 * 8:]
t0 = int(t[0, 0, 0])
print("wg tile   S_iss  S_land  P_done  PV_iss  epi_wait  O_done  epi_done  iters")
for u in range(40):
    for w in range(2):
        r = [int(t[w, u, j]) - t0 if int(t[w, u, j]) else -1 for j in range(7)] + [int(t[w, u, 7])]
        print(f"{w:2d} {u:4d} " + " ".join(f"{x:8d}" for x in r) + f"   S batch {int(t[w + 2, u, 0]) - t0} -> {int(t[w + 2, u, 1]) - t0}  P by warp " + " ".join(str(int(t[w + 2, u, 2 + q]) - t0) for q in range(4)))

print("MMA loop iteration start times (first 60):")
print([int(x) - t0 for x in its[:60]])
print("per iteration: [start, after PV streams, after S streams] (iterations 10..30)")
for i in range(10, 30):
    print(i, int(its[i]) - t0, int(its[1024 + i]) - int(its[i]), int(its[2048 + i]) - int(its[1024 + i]))

import torch, sys, os
sys.path.insert(0, '/root/repo')
import paper_2508_18224_b200 as fsa
from paper_2508_18224_b200 import _lib
import ctypes
cfg = fsa.make_config(N=32768, d_K=128, d_V=128, h=32, h_K=8, B_K=64, T=16, W=512)
g = torch.Generator(device="cuda").manual_seed(0)
q = torch.randn(cfg.N, 32, 128, device="cuda", generator=g).to(torch.bfloat16)
kc = torch.randn(cfg.b, 8, 128, device="cuda", generator=g)
sc = torch.empty(8, cfg.N, cfg.b, device="cuda")
s = _lib.shape_of(cfg)
def run():
    _lib.call("fsa_importance_scores", ctypes.byref(s), _lib.dt_code(torch.bfloat16), _lib.ptr(q), _lib.ptr(kc), _lib.ptr(sc), _lib.stream())
for _ in range(3): run()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10): run()
e1.record(); torch.cuda.synchronize()
print("fsa_importance_scores (SIMT fp32) ms:", e0.elapsed_time(e1) / 10)

"""Per-item timeline of CTA 0 of the K5 selected forward kernel (trace build:
fsa_debug_sel_fwd_trace).  python tools/trace_k5.py [N h h_K]"""
import ctypes
import os
import sys

os.environ["FSA_TRACE_LIB"] = "1"  # the trace build (build.py --trace)
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2508_18224_b200 as fsa  # noqa: E402
from paper_2508_18224_b200 import _lib, nsa  # noqa: E402


def main():
    N, h, hk = (int(x) for x in sys.argv[1:4]) if len(sys.argv) > 3 else (32768, 32, 8)
    g = torch.Generator(device="cuda").manual_seed(0)
    cfg = fsa.make_config(N=N, d_K=128, d_V=128, h=h, h_K=hk, B_K=64, T=16, W=512)
    mk = lambda *s: torch.randn(*s, device="cuda", dtype=torch.bfloat16, generator=g)  # noqa: E731
    q, k, v = mk(N, h, 128), mk(N, hk, 128), mk(N, hk, 128)
    tau = torch.rand(N, 3, device="cuda", generator=g)
    nsa.nsa_forward(q, k, v, tau, cfg)
    torch.cuda.synchronize()
    buf = torch.zeros(256 * 8, dtype=torch.int64, device="cuda")
    lib = _lib.lib()
    lib.fsa_debug_sel_fwd_trace(ctypes.c_void_p(buf.data_ptr()))
    nsa.nsa_forward(q, k, v, tau, cfg)
    torch.cuda.synchronize()
    lib.fsa_debug_sel_fwd_trace(None)
    t = buf.view(256, 8).cpu()
    t0 = int(t[0, 0])
    names = ["gather", "S_iss", "S_land", "P_done", "PV_iss", "O_land", "stored", "-"]
    print("item " + " ".join(f"{n:>9}" for n in names) + "   (cycles from item 0 gather)")
    for i in range(0, 120):
        row = [int(t[i, j]) - t0 if int(t[i, j]) else -1 for j in range(8)]
        print(f"{i:4d} " + " ".join(f"{x:9d}" for x in row))


if __name__ == "__main__":
    main()

"""Per-item timeline of CTA 0 of the K8 backward kernel (debug builds of the
trace hook, fsa_debug_bwd_trace).  python tools/trace_k8.py [sel|slide]"""
import ctypes
import os
import sys

os.environ["FSA_TRACE_LIB"] = "1"  # the trace build (build.py --trace)
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2508_18224_b200 as fsa  # noqa: E402
from paper_2508_18224_b200 import _lib, nsa  # noqa: E402


def main():
    mode = sys.argv[1] if len(sys.argv) > 1 else "sel"
    g = torch.Generator(device="cuda").manual_seed(0)
    cfg = fsa.make_config(N=32768, d_K=128, d_V=128, h=32, h_K=8, B_K=64, T=16, W=512)
    mk = lambda *s: torch.randn(*s, device="cuda", dtype=torch.bfloat16, generator=g)  # noqa: E731
    q, k, v, do = mk(cfg.N, 32, 128), mk(cfg.N, 8, 128), mk(cfg.N, 8, 128), mk(cfg.N, 32, 128)
    tau = torch.rand(cfg.N, 3, device="cuda", generator=g)
    out, ctx = nsa.nsa_forward(q, k, v, tau, cfg)
    nsa.nsa_backward(ctx, do)
    torch.cuda.synchronize()
    buf = torch.zeros(256 * 16, dtype=torch.int64, device="cuda")
    if os.environ.get("K8_PROBE"):
        buf[255 * 16 + 15] = 1  # raw S/dP completion probe (slot 13)
    lib = _lib.lib()
    lib.fsa_debug_bwd_trace(ctypes.c_void_p(buf.data_ptr()))
    if mode == "sel":
        from paper_2508_18224_b200.kv_major import _backward_core
        _backward_core(cfg, torch.bfloat16, q, k, v, do, ctx.sel, ctx.inv, ctx.out_sel, ctx.lse_sel)
    else:
        nsa.nsa_backward(ctx, do)  # selected then sliding launch: the sliding one overwrites
    torch.cuda.synchronize()
    lib.fsa_debug_bwd_trace(None)
    t = buf.view(256, 16).cpu()
    if mode == "sel":
        pass
    t0 = int(t[0, 0])
    names = ["gather", "sdp_iss", "sdp_land", "pds_done", "prod_iss", "prod_land", "dq_tmem", "dq_store", "prod_rdy", "pds_w0", "pds_w1", "pds_w2", "sdp_start", "sdp_raw", "ld_land", "ld_ready"]
    print("item " + " ".join(f"{n:>9}" for n in names) + "   (cycles from item 0 gather)")
    prev = None
    for i in range(0, 120):
        row = [int(t[i, j]) - t0 if int(t[i, j]) else -1 for j in range(16)]
        print(f"{i:4d} " + " ".join(f"{x:9d}" for x in row))


if __name__ == "__main__":
    main()

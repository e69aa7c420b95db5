"""Time the selected-attention kernels on a BASELINE shape (development probe).

    python tools/probe_sel.py [--N 32768 --h 32 --h_K 8]
"""

import argparse
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2508_18224_b200 as fsa  # noqa: E402
from paper_2508_18224_b200 import _lib, kv_major  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--N", type=int, default=32768)
    ap.add_argument("--h", type=int, default=32)
    ap.add_argument("--h_K", type=int, default=8)
    ap.add_argument("--T", type=int, default=16)
    ap.add_argument("--iters", type=int, default=10)
    a = ap.parse_args()
    cfg = fsa.make_config(N=a.N, d_K=128, d_V=128, h=a.h, h_K=a.h_K, B_K=64, T=a.T)
    g = torch.Generator(device="cuda").manual_seed(0)
    q = torch.randn(cfg.N, cfg.h, 128, device="cuda", dtype=torch.bfloat16, generator=g)
    k = torch.randn(cfg.N, cfg.h_K, 128, device="cuda", dtype=torch.bfloat16, generator=g)
    v = torch.randn(cfg.N, cfg.h_K, 128, device="cuda", dtype=torch.bfloat16, generator=g)
    scores = torch.rand(cfg.h_K, cfg.N, cfg.b, device="cuda", generator=g)
    sel = fsa.select_topk_blocks(scores, cfg)
    inv = fsa.build_inverse_index(sel, cfg)
    nnz = int(inv.offsets[:, -1].sum())
    R = nnz * cfg.g
    flops = 4.0 * 128 * 64 * R
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    for it in range(a.iters + 2):
        ev[0].record()
        out, lse = kv_major._fused_forward(cfg, torch.bfloat16, q, k, v, sel, inv)
        ev[1].record()
    torch.cuda.synchronize()
    # separate timing of K5 and K6
    (ob_code, ob_dt), _ = _lib.buffer_dtypes(cfg, torch.bfloat16)
    rows = _lib.partial_rows(cfg, torch.bfloat16)
    obuf = torch.empty((rows, 128), dtype=ob_dt, device="cuda")
    ml = torch.empty((rows, 2), dtype=torch.float32, device="cuda")
    s = _lib.shape_of(cfg)
    v16, vscale = _lib.v_to_f16(cfg, v)
    t5, t6 = [], []
    for it in range(a.iters + 2):
        ev[0].record()
        _lib.call("fsa_sel_fwd", ctypes.byref(s), _lib.DT_BF16, _lib.FWD_LOCAL, _lib.ptr(q), _lib.ptr(k),
                  _lib.ptr(v16), _lib.ptr(inv.offsets), _lib.ptr(inv.qlist), _lib.ptr(inv.work), None,
                  _lib.ptr(obuf), ob_code, _lib.ptr(ml), _lib.stream())
        ev[1].record()
        o2 = torch.empty((cfg.N, cfg.h, 128), dtype=torch.float32, device="cuda")
        l2 = torch.empty((cfg.h, cfg.N), dtype=torch.float32, device="cuda")
        ev[2].record()
        _lib.call("fsa_merge_fwd", ctypes.byref(s), _lib.DT_BF16, _lib.MERGE_LOCAL, _lib.ptr(sel.idx),
                  _lib.ptr(inv.work), _lib.ptr(obuf), ob_code, _lib.ptr(ml), None, None, _lib.ptr(o2), _lib.ptr(l2), None,
                  None, 0, _lib.ptr(vscale), _lib.stream())
        ev[3].record()
        torch.cuda.synchronize()
        if it >= 2:
            t5.append(ev[0].elapsed_time(ev[1]))
            t6.append(ev[2].elapsed_time(ev[3]))
    k5 = float(np.median(t5))
    k6 = float(np.median(t6))
    print(f"N={cfg.N} h={cfg.h} h_K={cfg.h_K} nnz/kvh={nnz / cfg.h_K:.0f} R={R}")
    print(f"K5 sel_fwd  {k5:.3f} ms  {flops / k5 / 1e9:.1f} TFLOP/s  (obuf {ob_dt})")
    merge_bytes = R * (2 * 128 + 8) + cfg.h * cfg.N * (128 * 4 + 4) + cfg.h_K * cfg.N * cfg.T * 4
    print(f"K6 merge    {k6:.3f} ms  {merge_bytes / k6 / 1e6:.1f} GB/s")


if __name__ == "__main__":
    main()

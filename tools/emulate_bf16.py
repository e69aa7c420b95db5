"""Numpy emulation of the tensor-core selected-attention numerics (K5 + merge,
K8 + dQ reduce) to find which bf16 rounding drives elementwise parity
violations against the float64 oracle.

    python tools/emulate_bf16.py [--N 4096] [--variants ...]

Each variant toggles one rounding: P in the forward PV product, the O_i/l_i
partials, delta's source, P / dS in the backward, the dq partials.
"""

from __future__ import annotations

import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import fsa_oracle as O  # noqa: E402


def bf(x):
    return torch.from_numpy(np.ascontiguousarray(x)).to(torch.bfloat16).double().numpy()


def f16(x):
    return np.asarray(x, dtype=np.float16).astype(np.float64)


def f16_rows(x):
    """fp16 with a power-of-two scale per row (last axis): max |row| -> [2^14, 2^15)."""
    mx = np.abs(x).max(-1, keepdims=True)
    e = np.where(mx > 0, 14 - np.floor(np.log2(np.where(mx > 0, mx, 1))), 0)
    s = np.exp2(e)
    return f16(x * s) / s


def rnd(x, mode):
    return {"bf16": bf, "f16": f16, "f16r": f16_rows, "f32": f32, "exact": (lambda y: y)}[mode](x)


def f32(x):
    return np.asarray(x, dtype=np.float32).astype(np.float64)


def emulate(Q, K, V, dO, idx, c, v):
    """Q (N,d,h) etc. in the oracle layout; returns out (N,d,h), dQ (N,d,h)."""
    N, d, h = Q.shape
    g, T, BK = c.g, c.T, c.B_K
    out = np.zeros((N, d, h))
    dQ = np.zeros((N, d, h))
    lse_all = np.zeros((h, N))
    for j in range(h):
        kh = j // g
        for t0 in range(0, N, 256):
            ts = np.arange(t0, min(N, t0 + 256))
            sel = idx[kh, ts]                      # (n, T)
            live = sel >= 0
            blk = np.where(live, sel, 0)
            keys = blk[:, :, None] * BK + np.arange(BK)[None, None, :]  # (n,T,64)
            Kk = K[keys, :, kh]                    # (n,T,64,d)
            Vk = V[keys, :, kh]
            q = Q[ts, :, j]                        # (n,d)
            do = dO[ts, :, j]
            S = np.einsum("nd,ntkd->ntk", q, Kk) * c.scale
            vis = (keys <= ts[:, None, None]) & live[:, :, None]
            S = np.where(vis, S, -np.inf)
            # ---- forward: per-block local stats, bf16 P, bf16 partial O_i / l_i
            mi = S.max(-1)                         # (n,T)
            mi_s = np.where(np.isfinite(mi), mi, 0.0)
            e = np.where(vis, np.exp(f32(S - mi_s[..., None])), 0.0)
            li = e.sum(-1)
            Pf = rnd(e, v["fwd_p"])
            Oi = np.einsum("ntk,ntkd->ntd", Pf, Vk)
            part = Oi / np.where(li > 0, li, 1)[..., None]
            part = rnd(part, v["obuf"])
            m = np.where(live, mi_s, -np.inf).max(-1)
            wgt = np.where(live, np.exp(mi_s - m[:, None]) * li, 0.0)
            l = wgt.sum(-1)
            o = (wgt[..., None] * part).sum(1) / l[:, None]
            lse = m + np.log(l)
            if v["out_bf16"]:
                o = bf(o)
            out[ts, :, j] = o
            lse_all[j, ts] = lse
            # ---- backward
            if v["delta_exact"]:
                Pe = np.where(vis, np.exp(S - lse[:, None, None]), 0.0)
                ex = (np.einsum("ntk,ntkd->nd", Pe, Vk) * do).sum(-1)
                delta = ex
            else:
                delta = (o * do).sum(-1)
            P = np.where(vis, np.exp(f32(S - f32(lse)[:, None, None])), 0.0)
            dP = np.einsum("nd,ntkd->ntk", do, Vk)
            dS = P * (dP - delta[:, None, None])
            if v["ds_q"] == "f16r":  # per-row scaled fp16 dS against fp16 K (exact)
                dSq = f16_rows(dS)
            else:
                dSq = rnd(dS, v["ds_q"])
            dqp = np.einsum("ntk,ntkd->ntd", dSq, Kk) * c.scale
            dqp = rnd(dqp, v["dq_part"])
            dQ[ts, :, j] = np.where(live[..., None], dqp, 0).sum(1)
    return out, dQ


def viol(got, ref, rtol=2e-2):
    rms = np.sqrt(np.mean(ref * ref))
    err = np.abs(got - ref)
    bound = rtol * rms + rtol * np.abs(ref)
    return int((err > bound).sum()), float((err / bound).max())


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--N", type=int, default=4096)
    ap.add_argument("--h", type=int, default=8)
    ap.add_argument("--hk", type=int, default=2)
    ap.add_argument("--T", type=int, default=16)
    ap.add_argument("--seed", type=int, default=5)
    a = ap.parse_args()
    kw = dict(N=a.N, d_K=128, d_V=128, h=a.h, h_K=a.hk, B_K=64, T=a.T, W=512)
    c = O.cfg_of(**kw)
    Q, K, V = (bf(x) for x in O.make_qkv(c, a.seed))
    dO = bf(O.make_dout(c, a.seed))
    idx = O.select_topk(O.make_scores(c, a.seed), c)
    want_out, _ = O.selected_forward(Q, K, V, idx, c)
    want_dQ = O.selected_backward(Q, K, V, idx, dO, c)[0]
    base = dict(fwd_p="bf16", obuf="bf16", out_bf16=False, delta_exact=False, ds_q="bf16",
                dq_part="bf16")
    variants = {
        "gpu (as built)": {},
        "A: f16 P, f16r obuf, f16r dq": dict(fwd_p="f16", obuf="f16r", dq_part="f16r"),
        "A + narrow out": dict(fwd_p="f16", obuf="f16r", dq_part="f16r", out_bf16=True),
        "B: A + f16r dS(q)": dict(fwd_p="f16", obuf="f16r", dq_part="f16r", ds_q="f16r"),
        "C: A with f32 dq": dict(fwd_p="f16", obuf="f16r", dq_part="f32"),
        "D: bf16 fwd, f16r dq": dict(dq_part="f16r"),
        "E: f16 P, bf16 obuf, f16r dq": dict(fwd_p="f16", dq_part="f16r"),
    }
    for name, ch in variants.items():
        v = dict(base, **ch)
        o, dq = emulate(Q, K, V, dO, idx, c, v)
        vo, wo = viol(o, want_out)
        vq, wq = viol(dq, want_dQ)
        print(f"{name:28s} out: {vo:6d} bad (worst {wo:.2f})   dQ: {vq:6d} bad (worst {wq:.2f})", flush=True)


if __name__ == "__main__":
    main()

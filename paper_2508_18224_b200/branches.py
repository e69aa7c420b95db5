"""Compressed and sliding-window branches plus the gated combine, on the device.

API of the reference's ``branches.py`` (branches.py:18-104).  Additionally
``sliding_attention_backward`` exposes the band-masked gradient the
reference only reaches through ``dense_backward(band_mask)`` (oracle.py:102-131).
"""

from __future__ import annotations

import ctypes
import dataclasses

import torch

from . import _lib
from .config import as_headed, compute_dtype, logical, to_device
from .types import AttentionOutput


@dataclasses.dataclass
class CompressedKV:
    """Mean-pooled KV (logical (b, d, h_K)) and first-block prefix means
    (logical (min(B_K-1, N), d, h_K)), in the accumulator dtype."""

    K_cmp: torch.Tensor
    V_cmp: torch.Tensor
    K_prefix: torch.Tensor
    V_prefix: torch.Tensor


def compress_kv(K, V, cfg) -> CompressedKV:
    """branches.py:34-44 (K1)."""
    k0, v0 = to_device(K), to_device(V)
    dt = compute_dtype(k0, v0)
    k = as_headed(k0, cfg.N, cfg.d_K, cfg.h_K, "K", dt)
    v = as_headed(v0, cfg.N, cfg.d_V, cfg.h_K, "V", dt)
    acc = _lib.acc_dtype(dt)
    dev = k.device
    n_pref = min(cfg.B_K - 1, cfg.N)
    Kc = torch.empty((cfg.b, cfg.h_K, cfg.d_K), dtype=acc, device=dev)
    Vc = torch.empty((cfg.b, cfg.h_K, cfg.d_V), dtype=acc, device=dev)
    Kp = torch.empty((n_pref, cfg.h_K, cfg.d_K), dtype=acc, device=dev)
    Vp = torch.empty((n_pref, cfg.h_K, cfg.d_V), dtype=acc, device=dev)
    s = _lib.shape_of(cfg)
    _lib.call("fsa_compress_kv", ctypes.byref(s), _lib.dt_code(dt), _lib.ptr(k), _lib.ptr(v),
              _lib.ptr(Kc), _lib.ptr(Vc), _lib.ptr(Kp), _lib.ptr(Vp), _lib.stream())
    return CompressedKV(logical(Kc), logical(Vc), logical(Kp), logical(Vp))


def _tc_qo(cfg, dt) -> bool:
    """The query-outer tensor-core forward's configuration (tc_qo_supported)."""
    return (dt == torch.bfloat16 and cfg.d_K == 128 and cfg.d_V == 128 and cfg.h % cfg.h_K == 0
            and cfg.g <= 128 and cfg.N < (1 << 30))


def _cmp_workspace(cfg, dev):
    s = _lib.shape_of(cfg)
    n = _lib.lib().fsa_cmp_workspace_bytes(ctypes.byref(s))
    return torch.empty(max(1, n), dtype=torch.uint8, device=dev)


def _cmp_storage(cmp: CompressedKV, acc):
    return tuple(to_device(x, acc).permute(0, 2, 1).contiguous()
                 for x in (cmp.K_cmp, cmp.V_cmp, cmp.K_prefix, cmp.V_prefix))


def compressed_attention_forward(Q, cmp: CompressedKV, cfg, *, scores_out: bool = False):
    """branches.py:47-78 (K2).  With ``scores_out`` also returns the
    importance scores (selection.py:105-120) from the same pass."""
    q0 = to_device(Q)
    if tuple(cmp.K_cmp.shape) != (cfg.b, cfg.d_K, cfg.h_K):
        raise ValueError(f"shape mismatch for K_cmp: got {tuple(cmp.K_cmp.shape)}")
    dt = compute_dtype(q0, to_device(cmp.K_cmp))
    q = as_headed(q0, cfg.N, cfg.d_K, cfg.h, "Q", dt)
    acc = _lib.acc_dtype(dt)
    Kc, Vc, Kp, Vp = _cmp_storage(cmp, acc)
    dev = q.device
    out = torch.empty((cfg.N, cfg.h, cfg.d_V), dtype=acc, device=dev)
    lse = torch.empty((cfg.h, cfg.N), dtype=acc, device=dev)
    s = _lib.shape_of(cfg)
    ws = _cmp_workspace(cfg, dev)
    ops = _lib.F16Ops(cfg, dev).stage(q=q) if _tc_qo(cfg, dt) else None
    _lib.call("fsa_cmp_attn_fwd", ctypes.byref(s), _lib.dt_code(dt), _lib.ptr(q), _lib.ptr(Kc),
              _lib.ptr(Vc), _lib.ptr(Kp), _lib.ptr(Vp), _lib.ptr(out), _lib.ptr(lse), None,
              _lib.ptr(ws), None if ops is None else _lib.ptr(ops.q),
              None if ops is None else _lib.ptr(ops.scales), _lib.stream())
    scores = None
    if scores_out:  # every block, causal or not (selection.py:105-120)
        scores = torch.empty((cfg.h_K, cfg.N, cfg.b), dtype=acc, device=dev)
        _lib.call("fsa_importance_scores", ctypes.byref(s), _lib.dt_code(dt), _lib.ptr(q),
                  _lib.ptr(Kc), _lib.ptr(scores), _lib.stream())
    res = AttentionOutput(out=logical(out), lse=lse)
    return (res, scores) if scores_out else res


def sliding_attention_forward(Q, K, V, cfg) -> AttentionOutput:
    """branches.py:81-83: causal attention over the last W positions (K10)."""
    ts = [to_device(x) for x in (Q, K, V)]
    dt = compute_dtype(*ts)
    q = as_headed(ts[0], cfg.N, cfg.d_K, cfg.h, "Q", dt)
    k = as_headed(ts[1], cfg.N, cfg.d_K, cfg.h_K, "K", dt)
    v = as_headed(ts[2], cfg.N, cfg.d_V, cfg.h_K, "V", dt)
    out, lse = _slide_fwd_storage(cfg, dt, q, k, v)
    return AttentionOutput(out=logical(out), lse=lse)


def _slide_fwd_storage(cfg, dt, q, k, v, v16=None):
    """K10 on storage tensors.  The bf16 tensor-core path reads V as its
    scaled fp16 copy ``v16 = (V16, vscale)`` (made here when not given)."""
    dev, acc = q.device, _lib.acc_dtype(dt)
    out = torch.empty((cfg.N, cfg.h, cfg.d_V), dtype=acc, device=dev)
    lse = torch.empty((cfg.h, cfg.N), dtype=acc, device=dev)
    s = _lib.shape_of(cfg)
    vscale = None
    if _tc_qo(cfg, dt):
        v, vscale = v16 if v16 is not None else _lib.v_to_f16(cfg, v)
    _lib.call("fsa_slide_fwd", ctypes.byref(s), _lib.dt_code(dt), _lib.ptr(q), _lib.ptr(k),
              _lib.ptr(v), _lib.ptr(vscale), _lib.ptr(out), _lib.ptr(lse), _lib.stream())
    return out, lse


def _slide_bwd_storage(cfg, dt, q, k, v, do, out, lse, accumulate_into=None, delta=None, ops=None):
    """K11.  With ``accumulate_into=(dQ, dK, dV)`` the sliding gradients are
    added onto those tensors in-kernel (tensor-core path) and they are returned.
    ``delta`` (h, N) may be passed precomputed (fsa_gate_backward); ``ops``:
    staged fp16 operands (_lib.F16Ops holding K16 and dO16 of this do)."""
    dev, acc = q.device, _lib.acc_dtype(dt)
    s = _lib.shape_of(cfg)
    st = _lib.stream()
    if delta is None:
        delta = torch.empty((cfg.h, cfg.N), dtype=acc, device=dev)
        _lib.call("fsa_bwd_delta", ctypes.byref(s), _lib.dt_code(dt), _lib.ptr(out), _lib.ptr(do),
                  _lib.ptr(delta), st)
    nws = _lib.lib().fsa_slide_bwd_workspace_bytes(ctypes.byref(s), _lib.dt_code(dt))
    ws = torch.empty(nws, dtype=torch.uint8, device=dev) if nws else None
    if accumulate_into is not None and ws is not None:
        dQ, dK, dV = accumulate_into
        accumulate = 1
    else:
        dQ = torch.empty((cfg.N, cfg.h, cfg.d_K), dtype=acc, device=dev)
        dK = torch.empty((cfg.N, cfg.h_K, cfg.d_K), dtype=acc, device=dev)
        dV = torch.empty((cfg.N, cfg.h_K, cfg.d_V), dtype=acc, device=dev)
        accumulate = 0
    if ws is not None and ops is None:  # tensor-core path: fp16 operands
        ops = _lib.F16Ops.of(cfg, q, k, v, do)
    elif ws is None:
        ops = None
    qq, kk, vv, dd = (q, k, v, do) if ops is None else (ops.q, ops.k, ops.v, ops.dout)
    _lib.call("fsa_slide_bwd", ctypes.byref(s), _lib.dt_code(dt), _lib.ptr(qq), _lib.ptr(kk),
              _lib.ptr(vv), _lib.ptr(dd), _lib.ptr(lse), _lib.ptr(delta), _lib.ptr(dQ), _lib.ptr(dK),
              _lib.ptr(dV), _lib.ptr(ws), accumulate, None if ops is None else _lib.ptr(ops.scales),
              st)
    if accumulate_into is not None and not accumulate:
        aQ, aK, aV = accumulate_into
        aQ += dQ
        aK += dK
        aV += dV
        return aQ, aK, aV
    return dQ, dK, dV


def sliding_attention_backward(Q, K, V, dOut, cfg):
    """Gradients of sum(sliding_attention_forward(...).out * dOut) (K11),
    the band-mask case of oracle.py:102-131.  Returns (dQ, dK, dV) logical."""
    ts = [to_device(x) for x in (Q, K, V, dOut)]
    dt = compute_dtype(*ts)
    q = as_headed(ts[0], cfg.N, cfg.d_K, cfg.h, "Q", dt)
    k = as_headed(ts[1], cfg.N, cfg.d_K, cfg.h_K, "K", dt)
    v = as_headed(ts[2], cfg.N, cfg.d_V, cfg.h_K, "V", dt)
    do = as_headed(ts[3], cfg.N, cfg.d_V, cfg.h, "dOut", dt)
    out, lse = _slide_fwd_storage(cfg, dt, q, k, v)
    dQ, dK, dV = _slide_bwd_storage(cfg, dt, q, k, v, do, out, lse)
    return logical(dQ), logical(dK), logical(dV)


def validate_gates(tau, cfg) -> torch.Tensor:
    """branches.py:86-92."""
    t = to_device(tau)
    if not t.is_floating_point():
        t = t.to(torch.float64)
    if tuple(t.shape) != (cfg.N, 3):
        raise ValueError(f"shape mismatch for gates: expected {(cfg.N, 3)}, got {tuple(t.shape)}")
    if bool(((t < 0) | (t > 1)).any()):
        raise ValueError("gate values must lie in [0, 1]")
    return t


def gated_combine(outs, tau, cfg) -> AttentionOutput:
    """branches.py:95-104 (K12): out = sum_c tau[:, c] * out_c; lse is NaN."""
    t = validate_gates(tau, cfg)
    if len(outs) != 3:
        raise ValueError("expected exactly three branch outputs")
    shapes = {tuple(o.out.shape) for o in outs}
    if len(shapes) != 1:
        raise ValueError(f"shape mismatch across branches: {sorted(shapes)}")
    xs = [to_device(o.out) for o in outs]
    acc = _lib.acc_dtype(compute_dtype(*xs))
    st = [as_headed(x, cfg.N, cfg.d_V, cfg.h, "out", acc) for x in xs]
    tt = t.to(acc).contiguous()
    out = torch.empty_like(st[0])
    s = _lib.shape_of(cfg)
    _lib.call("fsa_gated_combine", ctypes.byref(s), _lib.dt_code(acc), _lib.ptr(st[0]),
              _lib.ptr(st[1]), _lib.ptr(st[2]), _lib.ptr(tt), _lib.ptr(out), 1, _lib.stream())
    lse = torch.full((cfg.h, cfg.N), float("nan"), dtype=acc, device=out.device)
    return AttentionOutput(out=logical(out), lse=lse)

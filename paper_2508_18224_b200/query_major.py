"""NSA query-major selected attention -- the paper's baseline schedule.

Same API as the reference's ``query_major.py``: one task per (kv head,
token) batching the group's g query heads, walking the token's selected KV
blocks in ascending order with an online softmax (query_major.py:45-69,
_core.pyx:134-181).  On B200 the task's g rows are far below the M = 64/128
rows a tcgen05 MMA needs, so this schedule runs on CUDA cores
(``fsa_qm_fwd``); it exists as the FSA-vs-NSA comparison point (SURVEY 8(f)
rank 1, ``tools/sweep.py --nsa``).  The traffic meter is the reference's
closed form (query_major.py:32-42), including the min_tile padding.

The backward (query_major.py:72-115) recomputes the forward and scatters
dK / dV with atomics (``fsa_qm_bwd``) -- the reduction FSA's KV-block-major
backward replaces with single-writer tasks.
"""

from __future__ import annotations

import ctypes

import torch

from . import _lib
from .config import logical
from .kv_major import _intake
from .meter import TrafficMeter
from .selection import SelectionTensor, validate_selection
from .types import AttentionOutput


def _meter_forward(sel: SelectionTensor, cfg, meter: TrafficMeter) -> None:
    """query_major.py:32-42."""
    ph = meter.phase("query_major")
    bpe = cfg.bytes_per_elem
    pad = max(cfg.g, cfg.min_tile)
    steps = int(sel.row_lengths().sum())
    ph.task_count += cfg.h_K * cfg.N
    ph.inner_iterations += steps
    ph.bytes_loaded += (cfg.h_K * cfg.N * pad * cfg.d_K + steps * cfg.B_K * (cfg.d_K + cfg.d_V)) * bpe
    ph.bytes_stored += cfg.h_K * cfg.N * cfg.g * cfg.d_V * bpe
    ph.flops += steps * 2 * pad * cfg.B_K * (cfg.d_K + cfg.d_V)


def tc_supported(cfg, dt) -> bool:
    """bf16, d = 128, B_K = 64, g <= 16, T <= 16: the tcgen05 query-major forward."""
    return (dt == torch.bfloat16 and cfg.d_K == 128 and cfg.d_V == 128 and cfg.B_K == 64
            and cfg.g <= 16 and max(cfg.g, cfg.min_tile) <= 16 and cfg.T <= 16)


def selected_forward(Q, K, V, sel: SelectionTensor, cfg) -> tuple[AttentionOutput, TrafficMeter]:
    """query_major.py:45-69 on the device: (AttentionOutput, TrafficMeter).
    bf16 d = 128 runs the tcgen05 kernel (``fsa_qm_fwd_tc``: the g heads padded
    to max(g, min_tile) on the MMA's N side, a K/V tile load per (token, block
    pair)); other shapes the CUDA-core kernel (``fsa_qm_fwd``)."""
    dt, q, k, v, _ = _intake(cfg, Q, K, V)
    validate_selection(sel, cfg)
    acc = _lib.acc_dtype(dt)
    out = torch.empty((cfg.N, cfg.h, cfg.d_V), dtype=acc, device=q.device)
    lse = torch.empty((cfg.h, cfg.N), dtype=acc, device=q.device)
    s = _lib.shape_of(cfg)
    if tc_supported(cfg, dt):
        v16, vscale = _lib.v_to_f16(cfg, v)
        _lib.call("fsa_qm_fwd_tc", ctypes.byref(s), _lib.ptr(q), _lib.ptr(k), _lib.ptr(v16),
                  _lib.ptr(vscale), _lib.ptr(sel.idx), _lib.ptr(out), _lib.ptr(lse),
                  int(cfg.min_tile), _lib.stream())
    else:
        _lib.call("fsa_qm_fwd", ctypes.byref(s), _lib.dt_code(dt), _lib.ptr(q), _lib.ptr(k),
                  _lib.ptr(v), _lib.ptr(sel.idx), _lib.ptr(out), _lib.ptr(lse), _lib.stream())
    meter = TrafficMeter()
    _meter_forward(sel, cfg, meter)
    return AttentionOutput(out=logical(out), lse=lse), meter


def _meter_backward(sel: SelectionTensor, cfg, meter: TrafficMeter) -> None:
    """query_major.py:101-114."""
    ph = meter.phase("query_major")
    bpe = cfg.bytes_per_elem
    pad = max(cfg.g, cfg.min_tile)
    steps = int(sel.row_lengths().sum())
    ph.task_count += cfg.h_K * cfg.N
    ph.inner_iterations += steps
    ph.bytes_loaded += (cfg.h_K * cfg.N * (pad * cfg.d_K + cfg.g * cfg.d_V)
                        + 2 * steps * cfg.B_K * (cfg.d_K + cfg.d_V)) * bpe
    ph.bytes_stored += (cfg.h_K * cfg.N * cfg.g * cfg.d_K + steps * cfg.B_K * (cfg.d_K + cfg.d_V)) * bpe
    ph.flops += steps * 2 * pad * cfg.B_K * (4 * cfg.d_K + 3 * cfg.d_V)


def selected_backward(Q, K, V, sel: SelectionTensor, dOut, cfg):
    """query_major.py:72-115 on the device: (dQ, dK, dV, TrafficMeter).

    Recomputes the forward (``fsa_qm_fwd``) as the reference does
    (_core.pyx:193), then ``fsa_bwd_delta`` and ``fsa_qm_bwd``: per (kv head,
    token) task, dQ rows written once, dK / dV rows scattered with atomics
    (the query-major schedule has no single writer per KV row; summation
    order is therefore not fixed -- within tolerance, not bit-reproducible)."""
    dt, q, k, v, do = _intake(cfg, Q, K, V, dOut)
    validate_selection(sel, cfg)
    acc = _lib.acc_dtype(dt)
    dev = q.device
    out = torch.empty((cfg.N, cfg.h, cfg.d_V), dtype=acc, device=dev)
    lse = torch.empty((cfg.h, cfg.N), dtype=acc, device=dev)
    delta = torch.empty((cfg.h, cfg.N), dtype=acc, device=dev)
    dQ = torch.empty((cfg.N, cfg.h, cfg.d_K), dtype=acc, device=dev)
    dK = torch.empty((cfg.N, cfg.h_K, cfg.d_K), dtype=acc, device=dev)
    dV = torch.empty((cfg.N, cfg.h_K, cfg.d_V), dtype=acc, device=dev)
    s = _lib.shape_of(cfg)
    st = _lib.stream()
    _lib.call("fsa_qm_fwd", ctypes.byref(s), _lib.dt_code(dt), _lib.ptr(q), _lib.ptr(k),
              _lib.ptr(v), _lib.ptr(sel.idx), _lib.ptr(out), _lib.ptr(lse), st)
    _lib.call("fsa_bwd_delta", ctypes.byref(s), _lib.dt_code(dt), _lib.ptr(out), _lib.ptr(do),
              _lib.ptr(delta), st)
    _lib.call("fsa_qm_bwd", ctypes.byref(s), _lib.dt_code(dt), _lib.ptr(q), _lib.ptr(k), _lib.ptr(v),
              _lib.ptr(do), _lib.ptr(sel.idx), _lib.ptr(lse), _lib.ptr(delta), _lib.ptr(dQ),
              _lib.ptr(dK), _lib.ptr(dV), st)
    meter = TrafficMeter()
    _meter_backward(sel, cfg, meter)
    return logical(dQ), logical(dK), logical(dV), meter

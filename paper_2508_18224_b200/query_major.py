"""NSA query-major selected attention -- the paper's baseline schedule.

Same API as the reference's ``query_major.py``: one task per (kv head,
token) batching the group's g query heads, walking the token's selected KV
blocks in ascending order with an online softmax (query_major.py:45-69,
_core.pyx:134-181).  On B200 the task's g rows are far below the M = 64/128
rows a tcgen05 MMA needs, so this schedule runs on CUDA cores
(``fsa_qm_fwd``); it exists as the FSA-vs-NSA comparison point (SURVEY 8(f)
rank 1, ``tools/sweep.py --nsa``).  The traffic meter is the reference's
closed form (query_major.py:32-42), including the min_tile padding.

The query-major backward (query_major.py:72-115) is not built in this round:
``kv_major.selected_backward`` computes the same gradients.
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


def selected_forward(Q, K, V, sel: SelectionTensor, cfg) -> tuple[AttentionOutput, TrafficMeter]:
    """query_major.py:45-69 on the device: (AttentionOutput, TrafficMeter)."""
    dt, q, k, v, _ = _intake(cfg, Q, K, V)
    validate_selection(sel, cfg)
    acc = _lib.acc_dtype(dt)
    out = torch.empty((cfg.N, cfg.h, cfg.d_V), dtype=acc, device=q.device)
    lse = torch.empty((cfg.h, cfg.N), dtype=acc, device=q.device)
    s = _lib.shape_of(cfg)
    _lib.call("fsa_qm_fwd", ctypes.byref(s), _lib.dt_code(dt), _lib.ptr(q), _lib.ptr(k),
              _lib.ptr(v), _lib.ptr(sel.idx), _lib.ptr(out), _lib.ptr(lse), _lib.stream())
    meter = TrafficMeter()
    _meter_forward(sel, cfg, meter)
    return AttentionOutput(out=logical(out), lse=lse), meter


def selected_backward(Q, K, V, sel: SelectionTensor, dOut, cfg):
    """query_major.py:72-115 -- not built this round (same gradients as
    kv_major.selected_backward)."""
    raise NotImplementedError("query-major backward is not built; use kv_major.selected_backward")

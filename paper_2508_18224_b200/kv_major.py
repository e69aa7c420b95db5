"""FSA KV-block-major selected attention on the device.

Same operator API as the reference's ``kv_major.py`` (names, keyword flags,
return types, error messages).  The arithmetic runs in the CUDA kernels:

* ``selected_forward`` -- fused fast path: one pass over the
  (kv head, block) tasks emits per-block local (m_i, l_i) and O_i / l_i into
  a slot-indexed partial buffer, then the merge kernel combines the <= T
  partials of each (head, token) in ascending block order.  No separate
  statistics pre-pass; exact by softmax shift invariance.
* ``compute_softmax_stats`` / ``block_pass_forward`` / ``reduce_forward`` --
  the reference's three-phase API (kv_major.py:105-242), served by the same
  kernels in STATS / GLOBAL / REDUCE modes.
* ``selected_backward`` -- recompute forward, delta, per-task backward with
  single-writer dK/dV per (kv head, block), ascending-block dQ reduction.
"""

from __future__ import annotations

import ctypes
import dataclasses

import numpy as np
import torch

from . import _lib
from .config import as_headed, compute_dtype, logical, to_device
from .meter import TrafficMeter, backward_meter, forward_meter, meter_block_pass, meter_reduce, meter_stats
from .selection import InverseIndex, SelectionTensor, build_inverse_index
from .types import AttentionOutput


@dataclasses.dataclass
class SoftmaxStats:
    """Per (query head, token) max and exp-sum of the selected logits, (h, N)."""

    m: torch.Tensor
    l: torch.Tensor


class OutputBuffer:
    """Slot-indexed partial rows of ``block_pass_forward``.

    Device storage ``data`` is (h, N, T, d_V): the partial of query head j,
    token t against its slot-th selected block.  ``rows[j][i]`` gives the
    reference's per-task view (n_valid rows in slot order, kv_major.py:50-76),
    materialised on demand; ``write`` keeps the single-writer guard.
    """

    def __init__(self, data: torch.Tensor, inv: InverseIndex, cfg):
        self.data = data
        self._inv = inv
        self._cfg = cfg
        nv = inv.n_valid
        self.written = np.repeat(nv > 0, cfg.g, axis=0)  # (h, b)
        self._rows = None

    def _region(self, j, i):
        cfg = self._cfg
        kh = j // cfg.g
        off = self._inv.offsets[kh]
        a, b_ = int(off[i]), int(off[i + 1])
        ent = self._inv.qlist[kh, a:b_].to(torch.int64)
        t, s = ent // cfg.T, ent % cfg.T
        return self.data[j, t, s]

    @property
    def rows(self):
        if self._rows is None:
            cfg = self._cfg
            self._rows = [[self._region(j, i) if self.written[j, i] else None for i in range(cfg.b)]
                          for j in range(cfg.h)]
        return self._rows

    def write(self, j: int, i: int, region, reserved: int) -> None:
        if region.shape[0] > reserved:
            raise ValueError(f"buffer overflow: task ({j}, {i}) wrote {region.shape[0]} rows "
                             f"into a region reserved for {reserved}")
        if self.rows[j][i] is not None:
            raise ValueError(f"buffer region ({j}, {i}) written twice")
        self.rows[j][i] = region

    @property
    def peak_elements(self) -> int:
        nv = self._inv.n_valid
        return int(nv.sum(axis=1).max() * self._cfg.d_V)


# ---------------------------------------------------------------------------
# shared intake
# ---------------------------------------------------------------------------

def _intake(cfg, Q, K, V=None, dOut=None):
    ts = [to_device(x) for x in (Q, K, V, dOut) if x is not None]
    dt = compute_dtype(*ts)
    q = as_headed(Q, cfg.N, cfg.d_K, cfg.h, "Q", dt)
    k = as_headed(K, cfg.N, cfg.d_K, cfg.h_K, "K", dt)
    v = as_headed(V, cfg.N, cfg.d_V, cfg.h_K, "V", dt) if V is not None else None
    do = as_headed(dOut, cfg.N, cfg.d_V, cfg.h, "dOut", dt) if dOut is not None else None
    return dt, q, k, v, do


def _sel_partials(cfg, dt, q, k, v, inv, v16=None):
    """K5 in LOCAL mode: slot-indexed partials O_i / l_i and (m_i, l_i).
    On the tensor-core path (fp16 obuf) V is read as its scaled fp16 copy
    (``v16 = (V16, vscale)`` from fsa_v_to_f16, made here when not given).
    Returns (obuf, ml, obuf code, vscale or None)."""
    dev = q.device
    acc = _lib.acc_dtype(dt)
    (ob_code, ob_dtype), _ = _lib.buffer_dtypes(cfg, dt)
    vscale = None
    if ob_code == _lib.DT_F16:
        v, vscale = v16 if v16 is not None else _lib.v_to_f16(cfg, v)
    rows = _lib.partial_rows(cfg, dt)  # item-major on the tensor-core path
    obuf = torch.empty((rows, cfg.d_V), dtype=ob_dtype, device=dev)
    ml = torch.empty((rows, 2), dtype=acc, device=dev)
    s = _lib.shape_of(cfg)
    _lib.call("fsa_sel_fwd", ctypes.byref(s), _lib.dt_code(dt), _lib.FWD_LOCAL, _lib.ptr(q),
              _lib.ptr(k), _lib.ptr(v), _lib.ptr(inv.offsets), _lib.ptr(inv.qlist), _lib.ptr(inv.work),
              None, _lib.ptr(obuf), ob_code, _lib.ptr(ml), _lib.stream())
    return obuf, ml, ob_code, vscale


def _tc_partials(cfg, dt) -> bool:
    """bf16 d = 128 B_K = 64: the tensor-core path (fp16 partials)."""
    (ob_code, _), _ = _lib.buffer_dtypes(cfg, dt)
    return ob_code == _lib.DT_F16


def _fused_forward(cfg, dt, q, k, v, sel, inv):
    """K5 (LOCAL) + K6 (LOCAL merge): returns out storage (N, h, d_V) and lse
    (h, N), both in the accumulator dtype (f32 for bf16 inputs)."""
    dev = q.device
    acc = _lib.acc_dtype(dt)
    obuf, ml, ob_code, vscale = _sel_partials(cfg, dt, q, k, v, inv)
    s = _lib.shape_of(cfg)
    st = _lib.stream()
    out = torch.empty((cfg.N, cfg.h, cfg.d_V), dtype=acc, device=dev)
    lse = torch.empty((cfg.h, cfg.N), dtype=acc, device=dev)
    _lib.call("fsa_merge_fwd", ctypes.byref(s), _lib.dt_code(dt), _lib.MERGE_LOCAL,
              _lib.ptr(sel.idx), _lib.ptr(inv.work), _lib.ptr(obuf), ob_code, _lib.ptr(ml), None,
              None, _lib.ptr(out),
              _lib.ptr(lse), None, None, 0, _lib.ptr(vscale), st)
    return out, lse


# ---------------------------------------------------------------------------
# reference phase API
# ---------------------------------------------------------------------------

def compute_softmax_stats(Q, K, sel: SelectionTensor, cfg, *, shared_max: bool = False,
                          meter: TrafficMeter | None = None) -> SoftmaxStats:
    """kv_major.py:105-149: exact (m, l), merged in ascending block order."""
    dt, q, k, _, _ = _intake(cfg, Q, K)
    inv = build_inverse_index(sel, cfg)
    dev, acc = q.device, _lib.acc_dtype(dt)
    ml = torch.empty((cfg.h, cfg.N, cfg.T, 2), dtype=acc, device=dev)
    s = _lib.shape_of(cfg)
    st = _lib.stream()
    acc_code = _lib.dt_code(acc)
    if _tc_partials(cfg, dt):  # K5 STATS mode on tcgen05
        _lib.call("fsa_sel_fwd_phase", ctypes.byref(s), _lib.FWD_STATS, _lib.ptr(q), _lib.ptr(k), None,
                  None, _lib.ptr(inv.offsets), _lib.ptr(inv.qlist), _lib.ptr(inv.work), None, None,
                  _lib.ptr(ml), st)
    else:
        _lib.call("fsa_sel_fwd", ctypes.byref(s), _lib.dt_code(dt), _lib.FWD_STATS, _lib.ptr(q),
                  _lib.ptr(k), _lib.ptr(k), _lib.ptr(inv.offsets), _lib.ptr(inv.qlist),
                  _lib.ptr(inv.work), None, None, acc_code, _lib.ptr(ml), st)
    m = torch.empty((cfg.h, cfg.N), dtype=acc, device=dev)
    l = torch.empty_like(m)
    _lib.call("fsa_merge_fwd", ctypes.byref(s), _lib.dt_code(dt), _lib.MERGE_STATS,
              _lib.ptr(sel.idx), _lib.ptr(inv.work), None, acc_code, _lib.ptr(ml), None, None, None, None, _lib.ptr(m),
              _lib.ptr(l), int(bool(shared_max)), None, st)
    if meter is not None:
        meter_stats(meter, inv.n_valid, cfg)
    return SoftmaxStats(m=m, l=l)


def block_pass_forward(Q, K, V, inv: InverseIndex, stats: SoftmaxStats, cfg, *,
                       meter: TrafficMeter | None = None, task_order=None) -> OutputBuffer:
    """kv_major.py:152-204: unnormalised exp(z - m) @ V_i per (head, block).

    Tasks are independent CTAs writing disjoint slots, so any execution order
    gives bit-identical buffers; ``task_order`` is validated as in the
    reference (kv_major.py:173-177)."""
    if task_order is not None:
        order = np.asarray(task_order).reshape(-1)
        if order.size != cfg.h * cfg.b or not np.array_equal(np.sort(order), np.arange(cfg.h * cfg.b)):
            raise ValueError("task_order must be a permutation of all tasks")
    dt, q, k, v, _ = _intake(cfg, Q, K, V)
    dev, acc = q.device, _lib.acc_dtype(dt)
    mg = to_device(stats.m, acc).contiguous()
    obuf = torch.zeros((cfg.h, cfg.N, cfg.T, cfg.d_V), dtype=acc, device=dev)
    s = _lib.shape_of(cfg)
    if _tc_partials(cfg, dt):  # K5 GLOBAL mode on tcgen05 (P . V in fp16 on the scaled V copy)
        v16, vscale = _lib.v_to_f16(cfg, v)
        _lib.call("fsa_sel_fwd_phase", ctypes.byref(s), _lib.FWD_GLOBAL, _lib.ptr(q), _lib.ptr(k),
                  _lib.ptr(v16), _lib.ptr(vscale), _lib.ptr(inv.offsets), _lib.ptr(inv.qlist),
                  _lib.ptr(inv.work), _lib.ptr(mg), _lib.ptr(obuf), None, _lib.stream())
    else:
        _lib.call("fsa_sel_fwd", ctypes.byref(s), _lib.dt_code(dt), _lib.FWD_GLOBAL, _lib.ptr(q),
                  _lib.ptr(k), _lib.ptr(v), _lib.ptr(inv.offsets), _lib.ptr(inv.qlist),
                  _lib.ptr(inv.work), _lib.ptr(mg), _lib.ptr(obuf), _lib.dt_code(acc), None,
                  _lib.stream())
    if meter is not None:
        meter_block_pass(meter, inv.n_valid, cfg)
    return OutputBuffer(obuf, inv, cfg)


def reduce_forward(buf: OutputBuffer, inv: InverseIndex, stats: SoftmaxStats, cfg, *,
                   meter: TrafficMeter | None = None) -> AttentionOutput:
    """kv_major.py:207-242: ascending-block sum of partials, one division by l."""
    nv = inv.n_valid
    if buf._rows is not None:  # the per-task view was touched: honour its edits
        for j in range(cfg.h):
            for i in range(cfg.b):
                if buf._rows[j][i] is None and nv[j // cfg.g, i] != 0:
                    raise ValueError(f"missing buffer region for task ({j}, {i})")
    data = buf.data
    dev, acc = data.device, data.dtype
    dt = acc
    mg = to_device(stats.m, acc).contiguous()
    lg = to_device(stats.l, acc).contiguous()
    sel_idx = _selection_of(inv, cfg)
    out = torch.empty((cfg.N, cfg.h, cfg.d_V), dtype=dt, device=dev)
    lse = torch.empty((cfg.h, cfg.N), dtype=acc, device=dev)
    s = _lib.shape_of(cfg)
    _lib.call("fsa_merge_fwd", ctypes.byref(s), _lib.dt_code(dt), _lib.MERGE_REDUCE,
              _lib.ptr(sel_idx), None, _lib.ptr(data), _lib.dt_code(acc), None, _lib.ptr(mg),
              _lib.ptr(lg), _lib.ptr(out), _lib.ptr(lse), None, None, 0, None, _lib.stream())
    if meter is not None:
        meter_reduce(meter, nv, cfg)
    return AttentionOutput(out=logical(out), lse=lse)


def _selection_of(inv: InverseIndex, cfg) -> torch.Tensor:
    from .selection import selection_from_inverse
    cached = getattr(inv, "_sel_idx", None)
    if cached is None:
        cached = selection_from_inverse(inv, cfg).idx
        inv._sel_idx = cached
    return cached


def selected_forward(Q, K, V, sel: SelectionTensor, cfg, *, shared_max: bool = False,
                     task_order=None) -> tuple[AttentionOutput, TrafficMeter]:
    """kv_major.py:245-261 (fused path; ``shared_max`` only moves the internal
    shift, which the fused local-statistics form makes irrelevant)."""
    if task_order is not None:
        order = np.asarray(task_order).reshape(-1)
        if order.size != cfg.h * cfg.b or not np.array_equal(np.sort(order), np.arange(cfg.h * cfg.b)):
            raise ValueError("task_order must be a permutation of all tasks")
    dt, q, k, v, _ = _intake(cfg, Q, K, V)
    inv = build_inverse_index(sel, cfg)
    out, lse = _fused_forward(cfg, dt, q, k, v, sel, inv)
    return AttentionOutput(out=logical(out), lse=lse), forward_meter(inv.n_valid, cfg)


def _backward_core(cfg, dt, q, k, v, do, sel, inv, out, lse, delta=None):
    """K7 + K8 + K9 on storage-layout tensors; returns dQ, dK, dV storage (acc dtype).
    ``delta`` (h, N) may be passed precomputed (fsa_gate_backward)."""
    dev, acc = q.device, _lib.acc_dtype(dt)
    s = _lib.shape_of(cfg)
    st = _lib.stream()
    if delta is None:
        delta = torch.empty((cfg.h, cfg.N), dtype=acc, device=dev)
        _lib.call("fsa_bwd_delta", ctypes.byref(s), _lib.dt_code(dt), _lib.ptr(out), _lib.ptr(do),
                  _lib.ptr(delta), st)
    _, (dq_code, dq_dtype) = _lib.buffer_dtypes(cfg, dt)
    dq_buf = _lib.dq_buffer(cfg, dq_code, dq_dtype, dev)
    dK = torch.empty((cfg.N, cfg.h_K, cfg.d_K), dtype=acc, device=dev)
    dV = torch.empty((cfg.N, cfg.h_K, cfg.d_V), dtype=acc, device=dev)
    ops = _lib.F16Ops.of(cfg, q, k, v, do) if dq_code == _lib.DT_F16R else None  # tensor-core path
    qq, kk, vv, dd = (q, k, v, do) if ops is None else (ops.q, ops.k, ops.v, ops.dout)
    _lib.call("fsa_sel_bwd", ctypes.byref(s), _lib.dt_code(dt), _lib.ptr(qq), _lib.ptr(kk),
              _lib.ptr(vv), _lib.ptr(dd), _lib.ptr(lse), _lib.ptr(delta), _lib.ptr(inv.offsets),
              _lib.ptr(inv.qlist), _lib.ptr(inv.work), _lib.ptr(dq_buf), dq_code, _lib.ptr(dK),
              _lib.ptr(dV), None if ops is None else _lib.ptr(ops.scales), st)
    dQ = torch.empty((cfg.N, cfg.h, cfg.d_K), dtype=acc, device=dev)
    _lib.call("fsa_dq_reduce", ctypes.byref(s), _lib.dt_code(dt), _lib.ptr(sel.idx),
              _lib.ptr(dq_buf), dq_code, _lib.ptr(dQ), st)
    return dQ, dK, dV


def selected_backward(Q, K, V, sel: SelectionTensor, dOut, cfg, *, shared_max: bool = False):
    """kv_major.py:264-355: gradients of sum(out * dOut) w.r.t. Q, K, V, in the
    input layouts, plus the traffic meter.  Recomputes the forward as the
    reference does."""
    dt, q, k, v, do = _intake(cfg, Q, K, V, dOut)
    inv = build_inverse_index(sel, cfg)
    out, lse = _fused_forward(cfg, dt, q, k, v, sel, inv)
    dQ, dK, dV = _backward_core(cfg, dt, q, k, v, do, sel, inv, out, lse)
    return logical(dQ), logical(dK), logical(dV), backward_meter(inv.n_valid, cfg)

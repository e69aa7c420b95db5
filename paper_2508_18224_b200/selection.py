"""Block selection, validation and the inverse index on the device.

Mirrors the reference's ``selection.py`` API (names, argument order,
``SelectionError`` messages).  ``select_topk_blocks`` runs the K3 kernel and
``build_inverse_index`` the K4 counting sort (csrc/select.cu, csrc/inverse.cu);
the resulting ``InverseIndex`` lives on the GPU as CSR and materialises the
reference's list-of-arrays view only when a caller asks for it.
"""

from __future__ import annotations

import ctypes
import dataclasses
import struct

import numpy as np
import torch

from . import _lib
from .config import as_headed, to_device

SENTINEL = -1


class SelectionError(ValueError):
    """Malformed selection tensor (selection.py:26)."""


class SelectionTensor:
    """``idx`` (h_K, N, T) int32 on the device: ascending block ids, -1 padded."""

    def __init__(self, idx):
        t = to_device(idx)
        if t.dim() != 3:
            raise SelectionError("malformed selection: idx must be 3-d (h_K, N, T)")
        self.idx = t.to(torch.int32).contiguous()
        self._inverse_cache = None
        self._trusted = False   # produced by select_topk_blocks -> valid by construction

    def row_lengths(self) -> torch.Tensor:
        return (self.idx != SENTINEL).sum(dim=2)

    def nnz(self) -> int:
        return int((self.idx != SENTINEL).sum())

    def __repr__(self):
        return f"SelectionTensor(shape={tuple(self.idx.shape)})"


def _raise_flags(bits: int) -> None:
    for bit, msg in _lib.SEL_FLAGS:
        if bits & bit:
            raise SelectionError(msg)


def _shape_check(sel: SelectionTensor, cfg) -> None:
    shp = tuple(sel.idx.shape)
    if shp != (cfg.h_K, cfg.N, cfg.T):
        raise SelectionError(f"malformed selection: shape {shp} != {(cfg.h_K, cfg.N, cfg.T)}")


def validate_selection(sel: SelectionTensor, cfg) -> None:
    """selection.py:49-75 on the device; raises the reference's first message."""
    _shape_check(sel, cfg)
    flags = torch.zeros(1, dtype=torch.int32, device=sel.idx.device)
    s = _lib.shape_of(cfg)
    _lib.call("fsa_validate_selection", ctypes.byref(s), _lib.ptr(sel.idx), _lib.ptr(flags),
              _lib.stream())
    _raise_flags(int(flags.item()))


def select_topk_blocks(scores, cfg) -> SelectionTensor:
    """selection.py:78-102: own block + top-(T-1) causal blocks, ties to the
    lower index, -inf/NaN never selected.  Scores f32 or f64 are compared
    exactly as given (no rounding)."""
    sc = to_device(scores)
    if sc.dtype not in (torch.float32, torch.float64):
        sc = sc.to(torch.float32)
    if tuple(sc.shape) != (cfg.h_K, cfg.N, cfg.b):
        raise ValueError(
            f"shape mismatch for scores: expected {(cfg.h_K, cfg.N, cfg.b)}, got {tuple(sc.shape)}")
    sc = sc.contiguous()
    idx = torch.empty((cfg.h_K, cfg.N, cfg.T), dtype=torch.int32, device=sc.device)
    s = _lib.shape_of(cfg)
    _lib.call("fsa_select_topk", ctypes.byref(s), _lib.dt_code(sc.dtype), _lib.ptr(sc),
              _lib.ptr(idx), _lib.stream())
    sel = SelectionTensor(idx)
    sel._trusted = True
    return sel


def importance_scores_from_compressed(Q, K_cmp, cfg) -> torch.Tensor:
    """selection.py:105-120 -> (h_K, N, b) in the accumulator dtype."""
    q = to_device(Q)
    kc = to_device(K_cmp)
    if tuple(q.shape) != (cfg.N, cfg.d_K, cfg.h):
        raise ValueError(f"shape mismatch for Q: got {tuple(q.shape)}")
    if tuple(kc.shape) != (cfg.b, cfg.d_K, cfg.h_K):
        raise ValueError(f"shape mismatch for K_cmp: got {tuple(kc.shape)}")
    dtype = torch.float64 if torch.float64 in (q.dtype, kc.dtype) else q.dtype
    if dtype not in (torch.float32, torch.float64, torch.bfloat16):
        dtype = torch.float32
    qs = as_headed(q, cfg.N, cfg.d_K, cfg.h, "Q", dtype)
    acc = _lib.acc_dtype(dtype)
    kcs = kc.to(acc).permute(0, 2, 1).contiguous()
    out = torch.empty((cfg.h_K, cfg.N, cfg.b), dtype=acc, device=qs.device)
    s = _lib.shape_of(cfg)
    _lib.call("fsa_importance_scores", ctypes.byref(s), _lib.dt_code(dtype), _lib.ptr(qs),
              _lib.ptr(kcs), _lib.ptr(out), _lib.stream())
    return out


class InverseIndex:
    """Per (kv head, block): ascending attending tokens (selection.py:123-143).

    Device form: ``offsets`` (h_K, b+1) int32 CSR and ``qlist`` (h_K, N*T)
    int32 entries ``t*T + slot``.  ``queries``/``n_valid`` are host views
    built on first use.
    """

    def __init__(self, offsets: torch.Tensor, qlist: torch.Tensor, cfg, work=None):
        self.offsets = offsets
        self.qlist = qlist
        self.work = work  # tensor-core work plan (include/fsa_b200.h)
        self._cfg = cfg
        self._n_valid = None
        self._queries = None

    @property
    def n_valid(self) -> np.ndarray:
        if self._n_valid is None:
            off = self.offsets.to(torch.int64).cpu().numpy()
            self._n_valid = np.diff(off, axis=1)
        return self._n_valid

    @property
    def queries(self):
        if self._queries is None:
            cfg = self._cfg
            off = self.offsets.cpu().numpy().astype(np.int64)
            ql = self.qlist.cpu().numpy()
            self._queries = [
                [(ql[kh, off[kh, i]:off[kh, i + 1]] // cfg.T).astype(np.int32) for i in range(cfg.b)]
                for kh in range(cfg.h_K)]
        return self._queries

    def slots(self, kh: int, i: int) -> dict:
        return {int(t): s for s, t in enumerate(self.queries[kh][i])}

    def slot_of(self, kh: int, i: int, t: int) -> int:
        q = self.queries[kh][i]
        pos = int(np.searchsorted(q, t))
        if pos >= len(q) or q[pos] != t:
            raise KeyError(f"token {t} does not attend block {i} of KV head {kh}")
        return pos


def build_inverse_index(sel: SelectionTensor, cfg, *, validate: bool | None = None) -> InverseIndex:
    """selection.py:146-169: stable counting sort on the device, memoised on
    ``sel``.  Validation flags are computed by the same kernel; they are read
    back (one sync) unless the selection came from select_topk_blocks."""
    cached = getattr(sel, "_inverse_cache", None)
    if cached is not None:
        return cached
    _shape_check(sel, cfg)
    dev = sel.idx.device
    s = _lib.shape_of(cfg)
    ws_bytes = _lib.lib().fsa_inverse_workspace_bytes(ctypes.byref(s))
    ws = torch.empty(max(1, ws_bytes), dtype=torch.uint8, device=dev)
    offsets = torch.empty((cfg.h_K, cfg.b + 1), dtype=torch.int32, device=dev)
    qlist = torch.empty((cfg.h_K, cfg.N * cfg.T), dtype=torch.int32, device=dev)
    # work plan: item prefix [h_K*b + 1], a scheduler counter slot (tc_sched.cuh)
    # and the list position of every selection entry (include/fsa_b200.h)
    nw = _lib.lib().fsa_work_plan_bytes(ctypes.byref(s)) // 4
    work = torch.empty((nw,), dtype=torch.int32, device=dev)
    flags = torch.zeros(1, dtype=torch.int32, device=dev)
    _lib.call("fsa_build_inverse", ctypes.byref(s), _lib.ptr(sel.idx), _lib.ptr(ws),
              _lib.ptr(offsets), _lib.ptr(qlist), _lib.ptr(work), _lib.ptr(flags), _lib.stream())
    if validate is None:
        validate = not getattr(sel, "_trusted", False)
    if validate:
        _raise_flags(int(flags.item()))
    inv = InverseIndex(offsets, qlist, cfg, work)
    sel._inverse_cache = inv
    return inv


def selection_from_inverse(inv: InverseIndex, cfg) -> SelectionTensor:
    """Rebuild the canonical selection from the CSR (selection.py:172-181)."""
    dev = inv.offsets.device
    idx = torch.full((cfg.h_K * cfg.N * cfg.T,), SENTINEL, dtype=torch.int32, device=dev)
    for kh in range(cfg.h_K):
        off = inv.offsets[kh].to(torch.int64)
        counts = off[1:] - off[:-1]
        nnz = int(off[-1])
        blocks = torch.repeat_interleave(torch.arange(cfg.b, device=dev, dtype=torch.int32), counts)
        ent = inv.qlist[kh, :nnz].to(torch.int64)
        idx[kh * cfg.N * cfg.T + ent] = blocks
    return SelectionTensor(idx.view(cfg.h_K, cfg.N, cfg.T))


def self_block_selection(cfg) -> SelectionTensor:
    dev = _lib.require_device()
    idx = torch.full((cfg.h_K, cfg.N, cfg.T), SENTINEL, dtype=torch.int32, device=dev)
    idx[:, :, 0] = (torch.arange(cfg.N, device=dev) // cfg.B_K).to(torch.int32)
    return SelectionTensor(idx)


def full_selection(cfg) -> SelectionTensor:
    if cfg.T != cfg.b:
        raise ValueError(f"full selection needs T == b (T={cfg.T}, b={cfg.b})")
    dev = _lib.require_device()
    own = torch.arange(cfg.N, device=dev)[:, None] // cfg.B_K
    cols = torch.arange(cfg.b, device=dev)[None, :]
    idx = torch.where(cols <= own, cols, torch.full_like(cols, SENTINEL)).to(torch.int32)
    return SelectionTensor(idx.expand(cfg.h_K, cfg.N, cfg.T).contiguous())


def save_selection(sel: SelectionTensor, path) -> None:
    """Fixture format: little-endian int32 header (h_K, N, T), row-major body (selection.py:201-206)."""
    arr = sel.idx.cpu().numpy().astype("<i4")
    with open(path, "wb") as fh:
        fh.write(struct.pack("<3i", *arr.shape))
        fh.write(np.ascontiguousarray(arr).tobytes())


def load_selection(path) -> SelectionTensor:
    raw = open(path, "rb").read()
    if len(raw) < 12:
        raise SelectionError("malformed selection: truncated fixture header")
    h_K, N, T = struct.unpack("<3i", raw[:12])
    body = np.frombuffer(raw[12:], dtype="<i4")
    if min(h_K, N, T) < 1 or body.size != h_K * N * T:
        raise SelectionError("malformed selection: fixture size mismatch")
    return SelectionTensor(body.reshape(h_K, N, T).astype(np.int32))

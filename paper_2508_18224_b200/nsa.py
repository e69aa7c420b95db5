"""One NSA attention forward + backward, end to end on the device.

This is the training-path composition of the reference operators (the
pipeline of test_branches.py:167-192 / scenario.py:47-56, plus the
backward the reference provides for the selected and sliding branches):

  forward : compress_kv (K1) -> compressed attention + importance scores (K2)
            -> top-k (K3) -> inverse index (K4) -> FSA selected forward
            (K5 + K6) -> sliding window (K10) -> gated combine (K12)
  backward: gate scaling -> selected backward (K7 + K8 + K9) and sliding
            backward (K11); dQ/dK/dV summed over the two branches.

The compressed branch and the gates have no backward in the reference
(SURVEY 2.3 K13); they are not differentiated here either.

Everything operates on storage-layout tensors: Q (N, h, d), K/V (N, h_K, d),
tau (N, 3) in the accumulator dtype.  No host synchronisation happens inside
``forward``/``backward`` (the selection is valid by construction, so its
validity flags are not read back), so a step can be captured in a CUDA graph.
"""

from __future__ import annotations

import ctypes
import dataclasses

import torch

from . import _lib
from .kv_major import _backward_core, _sel_partials
from .branches import _cmp_workspace, _slide_bwd_storage, _slide_fwd_storage, _tc_qo
from .config import make_config
from .selection import SelectionTensor, build_inverse_index


@dataclasses.dataclass
class NSAContext:
    cfg: object
    dtype: torch.dtype
    q: torch.Tensor
    k: torch.Tensor
    v: torch.Tensor
    tau: torch.Tensor
    sel: SelectionTensor
    inv: object
    out_sel: torch.Tensor
    lse_sel: torch.Tensor
    out_slide: torch.Tensor
    lse_slide: torch.Tensor
    out_cmp: torch.Tensor
    scores: torch.Tensor
    # compressed branch (for nsa_backward(..., full=True))
    k_cmp: torch.Tensor = None
    v_cmp: torch.Tensor = None
    lse_cmp: torch.Tensor = None
    # tensor-core path: the fp16 operands staged by the forward (Q16, V16 and
    # their scales, _lib.F16Ops); the backward adds K16 and dO16
    ops: object = None


def _check(x, name, shape, dtype, dev):
    """Storage-layout intake of the step (the device path reads raw pointers):
    the reference's shape message (config.py:149-154), one dtype, one device,
    contiguous storage.  No host synchronisation."""
    if not isinstance(x, torch.Tensor):
        raise TypeError(f"{name} must be a torch tensor on the device")
    if tuple(x.shape) != tuple(shape):
        raise ValueError(f"shape mismatch for {name}: expected {tuple(shape)}, got {tuple(x.shape)}")
    if x.dtype != dtype:
        raise ValueError(f"{name} has dtype {x.dtype}; the step runs in {dtype} (all of Q, K, V, dOut)")
    if x.device != dev:
        raise ValueError(f"{name} is on {x.device}, Q on {dev}")
    if not x.is_contiguous():
        raise ValueError(f"{name} must be contiguous storage ({', '.join(map(str, shape))}); "
                         "use the operator API for logical (N, d, h) views")


def _gates(tau, cfg, acc, dev):
    """tau (N, 3) in the accumulator dtype, contiguous (a bf16 tau is cast)."""
    if not isinstance(tau, torch.Tensor) or tuple(tau.shape) != (cfg.N, 3):
        shp = tuple(tau.shape) if hasattr(tau, "shape") else type(tau).__name__
        raise ValueError(f"shape mismatch for gates: expected {(cfg.N, 3)}, got {shp}")
    if tau.device != dev:
        raise ValueError(f"gates are on {tau.device}, Q on {dev}")
    return tau.to(acc).contiguous()


# The tensor-core kernels index (token, head) rows with 32-bit offsets: a
# problem (or a kv-head chunk of it) runs on them while N * h stays below this.
TC_MAX_TOKEN_HEADS = 1 << 23


@dataclasses.dataclass
class ChunkedNSAContext:
    """Forward state of a kv-head-chunked step: one NSAContext per chunk of
    kv heads [lo, hi) (query heads [g lo, g hi))."""
    cfg: object
    dtype: torch.dtype
    chunks: list  # [(kv_lo, kv_hi, NSAContext)]


def kv_chunk_bytes(cfg, kv_heads: int) -> int:
    """Device bytes of the transient buffers one chunk of ``kv_heads`` kv heads
    allocates on top of the step's inputs and outputs (bf16 tensor-core path):
    the importance scores (fp32 [h_K][N][b]), the FSA slot partials of the
    forward (fp16 O rows + fp32 (m, l), items padded to 128 rows) or of the
    backward (fp16 dq rows + exponents), whichever is larger, and the chunk's
    fp16 operand copies and head slices."""
    g, rows = cfg.g, cfg.g * cfg.N * cfg.T * kv_heads
    scores = kv_heads * cfg.N * cfg.b * 4
    partials = max(int(rows * 1.05) * (2 * cfg.d_V + 8), rows * (2 * cfg.d_K + 4))
    per_token = kv_heads * g * (cfg.d_K * 2 * 4 + cfg.d_V * 4 * 4)  # q/dout slices + fp16 copies, fp32 branch outs
    return scores + partials + cfg.N * per_token


def plan_kv_chunk(cfg, budget_bytes: int | None = None) -> int:
    """kv heads per chunk: the largest divisor of h_K whose chunk keeps
    N * h under TC_MAX_TOKEN_HEADS (the tensor-core path) and, when a budget
    is given, whose transient buffers fit it.  h_K means no chunking."""
    best = 1
    for c in range(1, cfg.h_K + 1):
        if cfg.h_K % c:
            continue
        if cfg.N * cfg.g * c >= TC_MAX_TOKEN_HEADS and c > 1:
            break
        if budget_bytes is not None and kv_chunk_bytes(cfg, c) > budget_bytes and c > 1:
            break
        best = c
    return best


def _chunk_cfg(cfg, kv_heads):
    return make_config(N=cfg.N, d_K=cfg.d_K, d_V=cfg.d_V, h=cfg.g * kv_heads, h_K=kv_heads,
                       B_K=cfg.B_K, T=cfg.T, B_Q=cfg.B_Q, W=cfg.W,
                       bytes_per_elem=cfg.bytes_per_elem, min_tile=cfg.min_tile)


def _nsa_forward_chunked(q, k, v, tau, cfg, kv_chunk, keep_scores=False):
    """Buffer-reusing schedule (PAPER.md:267 -- "process a subset of query
    heads at each time, reusing the buffers"): the step runs one chunk of
    kv heads (and their g query heads each) at a time, so the scores, the
    slot partials and the dq partials are sized for the chunk and released
    before the next one.  Every operator is independent per kv head
    (selection.py:116-119, kv_major.py:127-140), so the result equals the
    unchunked step bit for bit."""
    dt = q.dtype
    dev = q.device
    _check(q, "Q", (cfg.N, cfg.h, cfg.d_K), dt, dev)
    _check(k, "K", (cfg.N, cfg.h_K, cfg.d_K), dt, dev)
    _check(v, "V", (cfg.N, cfg.h_K, cfg.d_V), dt, dev)
    if kv_chunk < 1 or cfg.h_K % kv_chunk:
        raise ValueError(f"kv_chunk={kv_chunk} does not divide h_K={cfg.h_K}")
    sub = _chunk_cfg(cfg, kv_chunk)
    out = torch.empty((cfg.N, cfg.h, cfg.d_V), dtype=dt, device=dev)
    chunks = []
    for lo in range(0, cfg.h_K, kv_chunk):
        hi = lo + kv_chunk
        qs = q.narrow(1, lo * cfg.g, kv_chunk * cfg.g).contiguous()
        ks, vs = k.narrow(1, lo, kv_chunk).contiguous(), v.narrow(1, lo, kv_chunk).contiguous()
        o, c = nsa_forward(qs, ks, vs, tau, sub, kv_chunk=kv_chunk, keep_scores=keep_scores)
        out.narrow(1, lo * cfg.g, kv_chunk * cfg.g).copy_(o)
        chunks.append((lo, hi, c))
    return out, ChunkedNSAContext(cfg, dt, chunks)


def _nsa_backward_chunked(ctx: ChunkedNSAContext, dout, full):
    cfg, dt = ctx.cfg, ctx.dtype
    dev = dout.device
    _check(dout, "dOut", (cfg.N, cfg.h, cfg.d_V), dt, dev)
    acc = _lib.acc_dtype(dt)
    dQ = torch.empty((cfg.N, cfg.h, cfg.d_K), dtype=acc, device=dev)
    dK = torch.empty((cfg.N, cfg.h_K, cfg.d_K), dtype=acc, device=dev)
    dV = torch.empty((cfg.N, cfg.h_K, cfg.d_V), dtype=acc, device=dev)
    dtau = torch.zeros((cfg.N, 3), dtype=acc, device=dev) if full else None
    for lo, hi, c in ctx.chunks:
        g0, g1 = lo * cfg.g, hi * cfg.g
        grads = nsa_backward(c, dout.narrow(1, g0, g1 - g0).contiguous(), full=full)
        dQ.narrow(1, g0, g1 - g0).copy_(grads[0])
        dK.narrow(1, lo, hi - lo).copy_(grads[1])
        dV.narrow(1, lo, hi - lo).copy_(grads[2])
        if full:
            dtau += grads[3]  # the gate gradient sums over every head of a token
    return (dQ, dK, dV, dtau) if full else (dQ, dK, dV)


def nsa_forward(q, k, v, tau, cfg, *, heads=None, kv_chunk=None, keep_scores=False):
    """Returns (combined out (N, h, d_V), ctx).

    Storage-layout inputs: q (N, h, d_K), k (N, h_K, d_K), v (N, h_K, d_V), one
    dtype, contiguous, on the device; tau (N, 3) (cast to the accumulator dtype).

    ``heads=(lo, hi)``: compute only query heads lo..hi-1 of every kv group
    (the query-head split of parallel.shard_plan).  The compressed branch and
    the block selection still see the whole group -- the importance scores
    sum over all g heads of a group (selection.py:105-120) -- then the
    selected and sliding branches and the combine run on the sub-group only.
    Out and ctx describe the sub-problem (h = h_K * (hi - lo)).

    ``kv_chunk=c``: the buffer-reusing schedule -- c kv heads at a time (c
    divides h_K), the ctx a ChunkedNSAContext; "auto" sizes c from the free
    device memory (plan_kv_chunk).  Problems with N * h >= TC_MAX_TOKEN_HEADS
    are chunked automatically so that every chunk runs on the tensor-core
    kernels.  ``keep_scores=True`` keeps the importance scores (h_K N b
    floats) in ctx.scores; by default they are released once the selection
    is made."""
    if kv_chunk == "auto":
        free, _ = torch.cuda.mem_get_info(q.device)
        kv_chunk = plan_kv_chunk(cfg, int(free * 0.8))
    elif kv_chunk is None and heads is None and cfg.N * cfg.h >= TC_MAX_TOKEN_HEADS \
            and q.dtype == torch.bfloat16:
        kv_chunk = plan_kv_chunk(cfg)
    if kv_chunk is not None and kv_chunk < cfg.h_K:
        if heads is not None:
            raise ValueError("heads= and kv_chunk= do not combine")
        return _nsa_forward_chunked(q, k, v, tau, cfg, int(kv_chunk), keep_scores)
    dt = q.dtype
    acc = _lib.acc_dtype(dt)
    dev = q.device
    _check(q, "Q", (cfg.N, cfg.h, cfg.d_K), dt, dev)
    _check(k, "K", (cfg.N, cfg.h_K, cfg.d_K), dt, dev)
    _check(v, "V", (cfg.N, cfg.h_K, cfg.d_V), dt, dev)
    tau = _gates(tau, cfg, acc, dev)
    s = _lib.shape_of(cfg)
    st = _lib.stream()
    (ob_code, _), _ = _lib.buffer_dtypes(cfg, dt)
    # tensor-core path: the P.V products read V as its power-of-two scaled fp16
    # copy and the compressed attention's S runs on the fp16 copy of Q (the
    # operands its backward recomputes S from)
    ops = _lib.F16Ops(cfg, dev).stage(q=q, v=v) if _tc_qo(cfg, dt) else None
    v16 = None if ops is None else (ops.v, ops.block(2))
    n_pref = min(cfg.B_K - 1, cfg.N)
    Kc = torch.empty((cfg.b, cfg.h_K, cfg.d_K), dtype=acc, device=dev)
    Vc = torch.empty((cfg.b, cfg.h_K, cfg.d_V), dtype=acc, device=dev)
    Kp = torch.empty((max(n_pref, 1), cfg.h_K, cfg.d_K), dtype=acc, device=dev)
    Vp = torch.empty((max(n_pref, 1), cfg.h_K, cfg.d_V), dtype=acc, device=dev)
    _lib.call("fsa_compress_kv", ctypes.byref(s), _lib.dt_code(dt), _lib.ptr(k), _lib.ptr(v),
              _lib.ptr(Kc), _lib.ptr(Vc), _lib.ptr(Kp), _lib.ptr(Vp), st)
    out_cmp = torch.empty((cfg.N, cfg.h, cfg.d_V), dtype=acc, device=dev)
    lse_cmp = torch.empty((cfg.h, cfg.N), dtype=acc, device=dev)
    scores = torch.empty((cfg.h_K, cfg.N, cfg.b), dtype=acc, device=dev)
    ws = _cmp_workspace(cfg, dev)
    _lib.call("fsa_cmp_attn_fwd", ctypes.byref(s), _lib.dt_code(dt), _lib.ptr(q), _lib.ptr(Kc),
              _lib.ptr(Vc), _lib.ptr(Kp), _lib.ptr(Vp), _lib.ptr(out_cmp), _lib.ptr(lse_cmp),
              _lib.ptr(scores), _lib.ptr(ws), None if ops is None else _lib.ptr(ops.q),
              None if ops is None else _lib.ptr(ops.scales), st)
    idx = torch.empty((cfg.h_K, cfg.N, cfg.T), dtype=torch.int32, device=dev)
    _lib.call("fsa_select_topk", ctypes.byref(s), _lib.dt_code(acc), _lib.ptr(scores),
              _lib.ptr(idx), st)
    if not keep_scores:  # h_K N b floats: release them before the partial buffers are allocated
        scores = None
    sel = SelectionTensor(idx)
    sel._trusted = True
    if heads is not None:
        lo, hi = heads
        if not 0 <= lo < hi <= cfg.g:
            raise ValueError(f"heads {heads} outside the group of {cfg.g} query heads")
        sub = make_config(N=cfg.N, d_K=cfg.d_K, d_V=cfg.d_V, h=cfg.h_K * (hi - lo), h_K=cfg.h_K,
                          B_K=cfg.B_K, T=cfg.T, B_Q=cfg.B_Q, W=cfg.W,
                          bytes_per_elem=cfg.bytes_per_elem, min_tile=cfg.min_tile)

        def take(x, axis):  # heads axis of a storage tensor -> the sub-group's heads
            shp = list(x.shape)
            y = x.reshape(shp[:axis] + [cfg.h_K, cfg.g] + shp[axis + 1:])
            y = y.narrow(axis + 1, lo, hi - lo)
            return y.reshape(shp[:axis] + [sub.h] + shp[axis + 1:]).contiguous()

        q, out_cmp, lse_cmp = take(q, 1), take(out_cmp, 1), take(lse_cmp, 0)
        cfg = sub
        s = _lib.shape_of(cfg)
        if ops is not None:  # the sub-group's Q16 (its own scale); V16 carries over
            sops = _lib.F16Ops(cfg, dev).stage(q=q)
            sops.v = ops.v
            sops.block(2).copy_(ops.block(2))
            ops = sops
    inv = build_inverse_index(sel, cfg, validate=False)
    # K5 writes the slot partials; the sliding branch runs before the merge so
    # that K6 can apply the gated combine (K12) in the same pass
    obuf, ml, ob_code, vscale = _sel_partials(cfg, dt, q, k, v, inv, v16=v16)
    out_slide, lse_slide = _slide_fwd_storage(cfg, dt, q, k, v, v16=v16)
    out_sel = torch.empty((cfg.N, cfg.h, cfg.d_V), dtype=acc, device=dev)
    lse_sel = torch.empty((cfg.h, cfg.N), dtype=acc, device=dev)
    out = torch.empty((cfg.N, cfg.h, cfg.d_V), dtype=dt, device=dev)
    _lib.call("fsa_merge_combine_fwd", ctypes.byref(s), _lib.dt_code(dt), _lib.ptr(sel.idx),
              _lib.ptr(inv.work), _lib.ptr(obuf), ob_code, _lib.ptr(ml), _lib.ptr(vscale), _lib.ptr(out_cmp),
              _lib.ptr(out_slide), _lib.ptr(tau), _lib.ptr(out_sel), _lib.ptr(lse_sel), _lib.ptr(out),
              st)
    del obuf, ml
    ctx = NSAContext(cfg, dt, q, k, v, tau, sel, inv, out_sel, lse_sel, out_slide, lse_slide,
                     out_cmp, scores, Kc, Vc, lse_cmp, ops)
    return out, ctx


def nsa_backward(ctx: NSAContext, dout, *, full: bool = False):
    """Returns (dQ, dK, dV) storage tensors in the accumulator dtype: the
    gradients through the selected and sliding branches, the ones the
    reference differentiates.  With ``full=True`` also through the compressed
    branch (attention over the pooled rows, the pooling and the prefix means;
    no reference backward -- SURVEY 8(f) rank 3) and returns
    (dQ, dK, dV, dtau) with the gate gradient dtau (N, 3).
    dout: (N, h, d_V) storage in the step's dtype, contiguous, on the device.

    The gate (branches.py:103, d_c = tau_c dOut) folds into each branch's
    statistics: tau exp(z - lse) = exp(z - (lse - ln tau)) and delta_c =
    sum out_c * dOut, so every branch backward reads the raw dOut -- no gated
    (and, in bf16, rounded) cotangent copies."""
    if isinstance(ctx, ChunkedNSAContext):
        return _nsa_backward_chunked(ctx, dout, full)
    cfg, dt = ctx.cfg, ctx.dtype
    _check(dout, "dOut", (cfg.N, cfg.h, cfg.d_V), dt, ctx.q.device)
    s = _lib.shape_of(cfg)
    st = _lib.stream()
    acc = _lib.acc_dtype(dt)
    dev = dout.device
    delta_sel = torch.empty((cfg.h, cfg.N), dtype=acc, device=dev)
    delta_slide = torch.empty_like(delta_sel)
    lse_sel, lse_slide = torch.empty_like(delta_sel), torch.empty_like(delta_sel)
    if full:
        delta_cmp, lse_cmp = torch.empty_like(delta_sel), torch.empty_like(delta_sel)
        dtau = torch.empty((cfg.N, 3), dtype=acc, device=dev)
        _lib.call("fsa_gate_backward_full_fold", ctypes.byref(s), _lib.dt_code(dt),
                  _lib.ptr(dout), _lib.ptr(ctx.tau), _lib.ptr(ctx.out_cmp), _lib.ptr(ctx.out_sel),
                  _lib.ptr(ctx.out_slide), _lib.ptr(ctx.lse_cmp), _lib.ptr(ctx.lse_sel),
                  _lib.ptr(ctx.lse_slide), _lib.ptr(delta_cmp), _lib.ptr(delta_sel),
                  _lib.ptr(delta_slide), _lib.ptr(lse_cmp), _lib.ptr(lse_sel), _lib.ptr(lse_slide),
                  _lib.ptr(dtau), st)
    else:
        _lib.call("fsa_gate_backward_fold", ctypes.byref(s), _lib.dt_code(dt), _lib.ptr(dout),
                  _lib.ptr(ctx.tau), _lib.ptr(ctx.out_sel), _lib.ptr(ctx.out_slide),
                  _lib.ptr(ctx.lse_sel), _lib.ptr(ctx.lse_slide), _lib.ptr(delta_sel),
                  _lib.ptr(delta_slide), _lib.ptr(lse_sel), _lib.ptr(lse_slide), st)
    # tensor-core operands: the forward staged Q16 / V16, the backward adds K16 / dO16
    ops = ctx.ops.stage(k=ctx.k, dout=dout) if ctx.ops is not None else None
    dQ, dK, dV = _sel_slide_backward(ctx, dout, delta_sel, delta_slide, lse_sel, lse_slide, ops)
    if not full:
        return dQ, dK, dV
    nws = _lib.lib().fsa_cmp_bwd_fold_workspace_bytes(ctypes.byref(s), _lib.dt_code(dt))
    ws = torch.empty(max(nws, 1), dtype=torch.uint8, device=dev)
    _lib.call("fsa_cmp_bwd_fold", ctypes.byref(s), _lib.dt_code(dt), _lib.ptr(ctx.q),
              _lib.ptr(ctx.k_cmp), _lib.ptr(ctx.v_cmp), _lib.ptr(dout), _lib.ptr(ctx.tau),
              _lib.ptr(lse_cmp), _lib.ptr(delta_cmp), _lib.ptr(dQ), _lib.ptr(dK), _lib.ptr(dV),
              None if ops is None else _lib.ptr(ops.q), None if ops is None else _lib.ptr(ops.dout),
              None if ops is None else _lib.ptr(ops.scales), _lib.ptr(ws), st)
    return dQ, dK, dV, dtau


def _sel_slide_backward(ctx: NSAContext, dout, delta_sel, delta_slide, lse_sel, lse_slide, ops):
    """Selected + sliding backward from the raw dOut with the gate folded into
    each branch's statistics (lse - ln tau, delta = sum out * dOut).  ``ops``:
    the fp16 operands (_lib.F16Ops) of the tensor-core path."""
    cfg, dt = ctx.cfg, ctx.dtype
    s = _lib.shape_of(cfg)
    st = _lib.stream()
    acc = _lib.acc_dtype(dt)
    _, (dq_code, dq_dtype) = _lib.buffer_dtypes(cfg, dt)
    if dq_code != _lib.DT_F16R:  # generic (f32 / f64 / small shapes) path
        dQ, dK, dV = _backward_core(cfg, dt, ctx.q, ctx.k, ctx.v, dout, ctx.sel, ctx.inv,
                                    ctx.out_sel, lse_sel, delta=delta_sel)
        return _slide_bwd_storage(cfg, dt, ctx.q, ctx.k, ctx.v, dout, ctx.out_slide, lse_slide,
                                  accumulate_into=(dQ, dK, dV), delta=delta_slide, ops=ops)
    # tensor-core path: K8 (selected) writes dK/dV and the fp16 dq partials;
    # the sliding backward adds its dK/dV in-kernel and writes its fp32 dQ
    # rows, which the dQ reduce (K9) adds while summing the partials -- every
    # gradient element is written once, with no read-modify-write pass over dQ
    dev = dout.device
    inv = ctx.inv
    dq_buf = _lib.dq_buffer(cfg, dq_code, dq_dtype, dev)
    dK = torch.empty((cfg.N, cfg.h_K, cfg.d_K), dtype=acc, device=dev)
    dV = torch.empty((cfg.N, cfg.h_K, cfg.d_V), dtype=acc, device=dev)
    _lib.call("fsa_sel_bwd", ctypes.byref(s), _lib.dt_code(dt), _lib.ptr(ops.q), _lib.ptr(ops.k),
              _lib.ptr(ops.v), _lib.ptr(ops.dout), _lib.ptr(lse_sel), _lib.ptr(delta_sel),
              _lib.ptr(inv.offsets), _lib.ptr(inv.qlist), _lib.ptr(inv.work), _lib.ptr(dq_buf),
              dq_code, _lib.ptr(dK), _lib.ptr(dV), _lib.ptr(ops.scales), st)
    dQ_slide = torch.empty((cfg.N, cfg.h, cfg.d_K), dtype=acc, device=dev)
    nws = _lib.lib().fsa_slide_bwd_workspace_bytes(ctypes.byref(s), _lib.dt_code(dt))
    ws = torch.empty(max(nws, 1), dtype=torch.uint8, device=dev)
    _lib.call("fsa_slide_bwd", ctypes.byref(s), _lib.dt_code(dt), _lib.ptr(ops.q), _lib.ptr(ops.k),
              _lib.ptr(ops.v), _lib.ptr(ops.dout), _lib.ptr(lse_slide), _lib.ptr(delta_slide),
              _lib.ptr(dQ_slide), _lib.ptr(dK), _lib.ptr(dV), _lib.ptr(ws), 2, _lib.ptr(ops.scales),
              st)
    dQ = torch.empty((cfg.N, cfg.h, cfg.d_K), dtype=acc, device=dev)
    _lib.call("fsa_dq_reduce_add", ctypes.byref(s), _lib.dt_code(dt), _lib.ptr(ctx.sel.idx),
              _lib.ptr(dq_buf), dq_code, _lib.ptr(dQ_slide), _lib.ptr(dQ), st)
    return dQ, dK, dV


def nsa_forward_backward(q, k, v, tau, dout, cfg, *, full: bool = False, kv_chunk=None):
    """One full step: forward then backward; returns (out, dQ, dK, dV[, dtau]).
    With ``kv_chunk`` each chunk's backward follows its forward directly, so
    only one chunk's forward state is alive at a time (the forward's branch
    outputs and statistics of the other chunks are never held together)."""
    if kv_chunk == "auto":
        free, _ = torch.cuda.mem_get_info(q.device)
        kv_chunk = plan_kv_chunk(cfg, int(free * 0.8))
    elif kv_chunk is None and cfg.N * cfg.h >= TC_MAX_TOKEN_HEADS and q.dtype == torch.bfloat16:
        kv_chunk = plan_kv_chunk(cfg)
    if kv_chunk is None or kv_chunk >= cfg.h_K:
        out, ctx = nsa_forward(q, k, v, tau, cfg)
        return (out,) + tuple(nsa_backward(ctx, dout, full=full))
    if kv_chunk < 1 or cfg.h_K % kv_chunk:
        raise ValueError(f"kv_chunk={kv_chunk} does not divide h_K={cfg.h_K}")
    dt, dev = q.dtype, q.device
    _check(dout, "dOut", (cfg.N, cfg.h, cfg.d_V), dt, dev)
    acc = _lib.acc_dtype(dt)
    out = torch.empty((cfg.N, cfg.h, cfg.d_V), dtype=dt, device=dev)
    dQ = torch.empty((cfg.N, cfg.h, cfg.d_K), dtype=acc, device=dev)
    dK = torch.empty((cfg.N, cfg.h_K, cfg.d_K), dtype=acc, device=dev)
    dV = torch.empty((cfg.N, cfg.h_K, cfg.d_V), dtype=acc, device=dev)
    dtau = torch.zeros((cfg.N, 3), dtype=acc, device=dev) if full else None
    for lo in range(0, cfg.h_K, kv_chunk):
        g0, n = lo * cfg.g, kv_chunk * cfg.g
        sub = _chunk_cfg(cfg, kv_chunk)
        o, c = nsa_forward(q.narrow(1, g0, n).contiguous(), k.narrow(1, lo, kv_chunk).contiguous(),
                           v.narrow(1, lo, kv_chunk).contiguous(), tau, sub, kv_chunk=kv_chunk,
                           keep_scores=False)
        out.narrow(1, g0, n).copy_(o)
        grads = nsa_backward(c, dout.narrow(1, g0, n).contiguous(), full=full)
        del c
        dQ.narrow(1, g0, n).copy_(grads[0])
        dK.narrow(1, lo, kv_chunk).copy_(grads[1])
        dV.narrow(1, lo, kv_chunk).copy_(grads[2])
        if full:
            dtau += grads[3]
    return (out, dQ, dK, dV, dtau) if full else (out, dQ, dK, dV)

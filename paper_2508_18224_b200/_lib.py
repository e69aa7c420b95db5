"""ctypes binding of libfsa_b200.so (include/fsa_b200.h).

The shared library is built in-tree by ``python -m paper_2508_18224_b200.build``
(or ``__graft_entry__.build()``).  There is no fallback: if the library is
missing or no CUDA device is present, every operator raises.
"""

from __future__ import annotations

import ctypes
import os

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
# FSA_TRACE_LIB=1 loads the trace build (build.py --trace: the product kernels
# plus the include/fsa_b200_trace.h timeline hooks; development tools only)
TRACE = os.environ.get("FSA_TRACE_LIB") == "1"
LIB_PATH = os.path.join(_HERE, "libfsa_b200_trace.so" if TRACE else "libfsa_b200.so")

FSA_OK, FSA_ERR_INVALID, FSA_ERR_CUDA, FSA_ERR_UNSUPPORTED = 0, 1, 2, 3
DT_F32, DT_F64, DT_BF16, DT_I32, DT_F16, DT_F16R = 0, 1, 2, 3, 4, 5
FWD_LOCAL, FWD_STATS, FWD_GLOBAL = 0, 1, 2
MERGE_LOCAL, MERGE_STATS, MERGE_REDUCE = 0, 1, 2

SEL_FLAGS = (  # bit, message -- in the reference's check order (selection.py:59-75)
    (1, "malformed selection: empty row"),
    (2, "malformed selection: entry after sentinel"),
    (4, "malformed selection: block index out of range"),
    (8, "malformed selection: non-causal entry"),
    (16, "malformed selection: duplicate entry"),
    (32, "malformed selection: not strictly increasing"),
)


class FsaShape(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int64) for n in ("N", "d_K", "d_V", "h", "h_K", "B_K", "T", "W")] + [
        ("scale", ctypes.c_double)]


_vp, _i, _i64, _sz = ctypes.c_void_p, ctypes.c_int, ctypes.c_int64, ctypes.c_size_t
_sp = ctypes.POINTER(FsaShape)
_ip = ctypes.POINTER(ctypes.c_int)

# symbol -> argtypes (restype int unless noted); must match include/fsa_b200.h
SIGNATURES = {
    "fsa_last_error": ([], ctypes.c_char_p),
    "fsa_abi_version": ([], _i),
    "fsa_device_check": ([], _i),
    "fsa_buffer_dtypes": ([_sp, _i, _ip, _ip], _i),
    "fsa_v_to_f16": ([_sp, _i, _vp, _vp, _vp, _vp], _i),
    "fsa_stage_f16_ops": ([_sp, _i] + [_vp] * 9 + [_vp], _i),
    "fsa_compress_kv": ([_sp, _i, _vp, _vp, _vp, _vp, _vp, _vp, _vp], _i),
    "fsa_importance_scores": ([_sp, _i, _vp, _vp, _vp, _vp], _i),
    "fsa_select_topk": ([_sp, _i, _vp, _vp, _vp], _i),
    "fsa_validate_selection": ([_sp, _vp, _vp, _vp], _i),
    "fsa_inverse_workspace_bytes": ([_sp], _sz),
    "fsa_work_plan_bytes": ([_sp], _sz),
    "fsa_partial_rows": ([_sp, _i], _i64),
    "fsa_build_inverse": ([_sp, _vp, _vp, _vp, _vp, _vp, _vp, _vp], _i),
    "fsa_sel_fwd": ([_sp, _i, _i, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _i, _vp, _vp], _i),
    "fsa_sel_fwd_phase": ([_sp, _i, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp], _i),
    "fsa_merge_fwd": ([_sp, _i, _i, _vp, _vp, _vp, _i, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _i, _vp, _vp], _i),
    "fsa_merge_combine_fwd": ([_sp, _i, _vp, _vp, _vp, _i, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp], _i),
    "fsa_bwd_delta": ([_sp, _i, _vp, _vp, _vp, _vp], _i),
    "fsa_sel_bwd": ([_sp, _i, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _i, _vp, _vp, _vp, _vp], _i),
    "fsa_dq_reduce": ([_sp, _i, _vp, _vp, _i, _vp, _vp], _i),
    "fsa_dq_reduce_add": ([_sp, _i, _vp, _vp, _i, _vp, _vp, _vp], _i),
    "fsa_cmp_workspace_bytes": ([_sp], _sz),
    "fsa_cmp_attn_fwd": ([_sp, _i, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp], _i),
    "fsa_slide_fwd": ([_sp, _i, _vp, _vp, _vp, _vp, _vp, _vp, _vp], _i),
    "fsa_slide_bwd_workspace_bytes": ([_sp, _i], _sz),
    "fsa_slide_bwd": ([_sp, _i, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _i, _vp, _vp], _i),
    "fsa_gated_combine": ([_sp, _i, _vp, _vp, _vp, _vp, _vp, _i, _vp], _i),
    "fsa_gate_scale": ([_sp, _i, _vp, _vp, _i, _vp, _vp], _i),
    "fsa_gate_backward": ([_sp, _i, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp], _i),
    "fsa_gate_backward_fold": ([_sp, _i] + [_vp] * 10 + [_vp], _i),
    "fsa_gate_backward_full_fold": ([_sp, _i] + [_vp] * 15 + [_vp], _i),
    "fsa_cmp_bwd_fold_workspace_bytes": ([_sp, _i], _sz),
    "fsa_cmp_bwd_fold": ([_sp, _i] + [_vp] * 14 + [_vp], _i),
    "fsa_cmp_bwd_workspace_bytes": ([_sp, _i], _sz),
    "fsa_cmp_bwd": ([_sp, _i, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp], _i),
    "fsa_gate_backward_full": ([_sp, _i] + [_vp] * 13, _i),
    "fsa_qm_fwd_tc": ([_sp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _i, _vp], _i),
    "fsa_qm_fwd": ([_sp, _i, _vp, _vp, _vp, _vp, _vp, _vp, _vp], _i),
    "fsa_qm_bwd": ([_sp, _i, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp], _i),
    "fsa_check_finite": ([_i, _vp, _i64, _vp, _vp], _i),
}


# include/fsa_b200_trace.h: only in libfsa_b200_trace.so
TRACE_SIGNATURES = {
    "fsa_debug_bwd_trace": ([_vp], None),
    "fsa_debug_dq_trace": ([_vp], None),
    "fsa_debug_qo_trace": ([_vp], None),
    "fsa_debug_sel_fwd_trace": ([_vp], None),
    "fsa_debug_gather4_test": ([_vp, ctypes.c_int64, _vp, _vp, _i, _i, _vp, _vp, ctypes.c_int64, _vp], _i),
}


class FsaError(RuntimeError):
    """A CUDA-side failure reported through the C-ABI."""


_lib = None


def lib():
    """Load the library once; raise loudly when it is missing."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is not built; run `python -m paper_2508_18224_b200.build` "
                "(the FSA operators have no CPU fallback)")
        l = ctypes.CDLL(LIB_PATH)
        for name, (args, res) in {**SIGNATURES, **(TRACE_SIGNATURES if TRACE else {})}.items():
            fn = getattr(l, name)
            fn.argtypes = args
            fn.restype = res
        _lib = l
    return _lib


def last_error() -> str:
    return lib().fsa_last_error().decode(errors="replace")


def call(name, *args):
    rc = getattr(lib(), name)(*args)
    if rc != FSA_OK:
        msg = last_error()
        if rc == FSA_ERR_INVALID:
            raise ValueError(f"{name}: {msg}")
        raise FsaError(f"{name}: {msg}")
    return rc


_checked_devices = set()


def require_device():
    """The operators only run on a CUDA (sm_100a) device."""
    if not torch.cuda.is_available():
        raise RuntimeError("the FSA B200 operators need a CUDA device (no CPU fallback)")
    dev = torch.cuda.current_device()
    if dev not in _checked_devices:
        call("fsa_device_check")
        _checked_devices.add(dev)
    return torch.device("cuda", dev)


def shape_of(cfg) -> FsaShape:
    return FsaShape(cfg.N, cfg.d_K, cfg.d_V, cfg.h, cfg.h_K, cfg.B_K, cfg.T, cfg.W, cfg.scale)


def ptr(t):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def stream():
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def dt_code(dtype) -> int:
    if dtype == torch.float32:
        return DT_F32
    if dtype == torch.float64:
        return DT_F64
    if dtype == torch.bfloat16:
        return DT_BF16
    raise ValueError(f"unsupported dtype {dtype} (float32, float64 or bfloat16)")


def acc_dtype(dtype):
    return torch.float64 if dtype == torch.float64 else torch.float32


_TORCH_OF = {DT_F32: torch.float32, DT_F64: torch.float64, DT_BF16: torch.bfloat16,
             DT_F16: torch.float16, DT_F16R: torch.uint8}


def buffer_dtypes(cfg, dtype):
    """((obuf code, torch dtype), (dq_buf code, torch dtype)) for a problem; the
    tensor-core path uses fp16 obuf and FSA_DT_F16R dq_buf (bytes)."""
    s = shape_of(cfg)
    ob, dq = ctypes.c_int(), ctypes.c_int()
    call("fsa_buffer_dtypes", ctypes.byref(s), dt_code(dtype), ctypes.byref(ob), ctypes.byref(dq))
    if (dtype == torch.bfloat16 and ob.value != DT_F16 and cfg.d_K == 128 and cfg.d_V == 128
            and cfg.B_K == 64 and cfg.N * cfg.h >= (1 << 23)):
        _warn_large_once(cfg)
    return (ob.value, _TORCH_OF[ob.value]), (dq.value, _TORCH_OF[dq.value])


_WARNED_LARGE = False


def _warn_large_once(cfg):
    """The tensor-core kernels index (token, head) rows with 32-bit offsets
    (N h < 2^23); a larger single call runs the CUDA-core kernels -- say so once."""
    global _WARNED_LARGE
    if not _WARNED_LARGE:
        import warnings
        warnings.warn(f"N*h = {cfg.N * cfg.h} >= 2^23: this call runs the CUDA-core kernels, not "
                      "the tensor-core ones; nsa_forward / nsa_forward_backward chunk by kv head "
                      "automatically (kv_chunk), or shard the kv heads", RuntimeWarning, stacklevel=3)
        _WARNED_LARGE = True


def partial_rows(cfg, dtype) -> int:
    """Rows of the obuf / ml partial buffers (item-major tiles on the
    tensor-core path, slot-indexed h N T otherwise; include/fsa_b200.h)."""
    s = shape_of(cfg)
    return int(lib().fsa_partial_rows(ctypes.byref(s), dt_code(dtype)))


def dq_buffer(cfg, code, dtype, dev):
    """The dq partial buffer: slot-indexed rows [h N T][d_K] of dtype, or for
    FSA_DT_F16R the fp16 rows followed by 4 int8 exponents per row
    (include/fsa_b200.h)."""
    rows = cfg.h * cfg.N * cfg.T
    if code == DT_F16R:
        return torch.empty(rows * (2 * cfg.d_K + 4), dtype=torch.uint8, device=dev)
    return torch.empty((rows, cfg.d_K), dtype=dtype, device=dev)


def v_to_f16(cfg, v):
    """fsa_v_to_f16: the power-of-two scaled fp16 copy of V (N, h_K, d_V) and
    its per-kv-head scales -- the value operand of the tensor-core P.V products."""
    v16 = torch.empty(v.shape, dtype=torch.float16, device=v.device)
    vscale = torch.empty(2 * cfg.h_K, dtype=torch.float32, device=v.device)
    s = shape_of(cfg)
    call("fsa_v_to_f16", ctypes.byref(s), dt_code(v.dtype), ptr(v), ptr(v16), ptr(vscale), stream())
    return v16, vscale


class F16Ops:
    """fsa_stage_f16_ops: the fp16 operands of the bf16 tensor-core path
    (Q16, K16, V16, dO16, power-of-two scaled per kv head / kv group) and their
    scale blocks ``scales`` ([4][2 h_K] floats: s_Q, s_K, s_V, s_dO).  The
    forward stages Q (compressed-attention S) and V (every P.V product); the
    backward adds K and dOut."""

    def __init__(self, cfg, dev):
        self.cfg = cfg
        self.scales = torch.empty(8 * cfg.h_K, dtype=torch.float32, device=dev)
        self.q = self.k = self.v = self.dout = None

    def block(self, i):
        """scale block i (0 Q, 1 K, 2 V, 3 dOut): [2 h_K] floats, scales first."""
        hk = self.cfg.h_K
        return self.scales[2 * hk * i:2 * hk * (i + 1)]

    def stage(self, q=None, k=None, v=None, dout=None):
        src = (q, k, v, dout)
        dst = [None if x is None else torch.empty(x.shape, dtype=torch.float16, device=x.device)
               for x in src]
        s = shape_of(self.cfg)
        dt = next(x.dtype for x in src if x is not None)
        call("fsa_stage_f16_ops", ctypes.byref(s), dt_code(dt), *(ptr(x) for x in src),
             *(ptr(x) for x in dst), ptr(self.scales), stream())
        for name, x in zip(("q", "k", "v", "dout"), dst):
            if x is not None:
                setattr(self, name, x)
        return self

    @classmethod
    def of(cls, cfg, q, k, v, dout):
        return cls(cfg, q.device).stage(q, k, v, dout)

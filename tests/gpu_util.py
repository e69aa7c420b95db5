"""Helpers shared by the GPU parity tests."""

from __future__ import annotations

import json
import os

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


def _report(rec):
    """FSA_PARITY_REPORT=<file>: append one JSON line per comparison (violation
    counts, max normalised error) -- the evidence behind profiles/*parity*."""
    path = os.environ.get("FSA_PARITY_REPORT")
    if path:
        with open(path, "a") as fh:
            fh.write(json.dumps(rec) + "\n")


def assert_close(got, ref, dtype, what="", grad=False):
    """Tolerance per north_star and SURVEY 8(d), elementwise for every dtype:

        |got - ref| <= rtol * |ref| + rtol * RMS(ref)

    rtol = 1e-4 (f32), 2e-2 (bf16); f64 at the reference's own 1e-9 scale.
    ``ref`` is the float64 oracle run on the dtype-rounded inputs.  The
    normwise error ||err|| / ||ref|| is reported alongside as a diagnostic
    only.  ``grad`` is kept for call-site documentation."""
    got = np.asarray(got, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    assert got.shape == ref.shape, (what, got.shape, ref.shape)
    if dtype == "f64":
        tol = 1e-9 * max(1.0, float(np.abs(ref).max()) if ref.size else 1.0)
        err = float(np.abs(got - ref).max()) if ref.size else 0.0
        assert err <= tol, f"{what}: max abs err {err:.3e} > {tol:.1e}"
        return
    rtol = 1e-4 if dtype == "f32" else 2e-2
    atol = rtol * max(rms(ref), 1e-30)
    err = np.abs(got - ref)
    bound = atol + rtol * np.abs(ref)
    bad = ~(err <= bound)  # NaN counts as a violation
    nbad = int(bad.sum())
    worst = float((err / bound).max()) if ref.size else 0.0
    normwise = float(np.linalg.norm(err) / max(np.linalg.norm(ref), 1e-300)) if ref.size else 0.0
    _report(dict(what=what, dtype=dtype, n=int(ref.size), violations=nbad,
                 worst_err_over_bound=worst, normwise=normwise))
    assert nbad == 0, (f"{what}: {nbad}/{bad.size} elements outside |err| <= {rtol}*|ref| + "
                       f"{rtol}*RMS(ref) (atol {atol:.2e}); worst err/bound {worst:.2f}, "
                       f"normwise {normwise:.2e}")

"""Load golden fixtures (tests/golden/*.npz) and regenerate their inputs.

Fixtures come from the real reference (tests/golden/make_golden.py); inputs are
regenerated from the stored seed through the same PCG64 streams
(``oracle.fsa_oracle.make_qkv`` restates rng.py:14-39) and the same rounding.
"""

from __future__ import annotations

import json
import os

import numpy as np

from oracle import fsa_oracle as O

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def round_inputs(x, dtype):
    if dtype in (None, "None", "f64"):
        return np.asarray(x, dtype=np.float64)
    if dtype == "f32":
        return np.asarray(x, dtype=np.float32).astype(np.float64)
    if dtype == "bf16":
        import torch
        return torch.from_numpy(np.asarray(x, dtype=np.float64)).to(torch.bfloat16).double().numpy()
    raise ValueError(dtype)


def load(name):
    return np.load(os.path.join(GOLDEN, name + ".npz"))


def case(name):
    """Return (cfg_kwargs, oracle Cfg, inputs dict, fixture)."""
    z = load(name)
    kw = json.loads(str(z["cfg"]))
    c = O.cfg_of(**kw)
    seed = int(z["seed"])
    rt = str(z["round_to"])
    Q, K, V = O.make_qkv(c, seed)
    dOut = O.make_dout(c, seed)
    Q, K, V, dOut = (round_inputs(x, rt) for x in (Q, K, V, dOut))
    tau = O.make_gates(c, seed)
    return kw, c, dict(Q=Q, K=K, V=V, dOut=dOut, tau=tau, round_to=rt), z


def stride_of(z):
    return int(z["token_stride"]) if "token_stride" in z.files else 1


FULL_CASES = ["case_kv_small", "case_rect_dims", "case_pipeline", "case_g8_bk1", "case_unit",
              "case_tiny_fp32", "case_d128_bf16"]

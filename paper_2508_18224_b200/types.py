"""Result records shared by the operators (oracle.py:20-23 in the reference)."""

from __future__ import annotations

import dataclasses

import torch


@dataclasses.dataclass
class AttentionOutput:
    out: torch.Tensor  # logical (N, d_V, h)
    lse: torch.Tensor  # (h, N)

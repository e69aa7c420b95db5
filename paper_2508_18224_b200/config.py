"""Attention configuration, mirroring the reference's ``config.py``.

Same record (``AttentionConfig``), same derived fields (g, b, scale), same
defaults (B_Q = min(16, N), W = min(512, N)), same error type and messages
(config.py:26-143), so configs and config files are interchangeable with the
reference.  ``as_headed`` is the device-side analogue of config.py:146-155:
it validates the logical (token, feature, head) shape and returns the
(token, head, feature) storage the kernels read.
"""

from __future__ import annotations

import dataclasses
import math

import numpy as np
import torch

from . import _lib


class ConfigError(ValueError):
    """An AttentionConfig invariant is violated (config.py:26)."""


@dataclasses.dataclass(frozen=True)
class AttentionConfig:
    N: int
    d_K: int
    d_V: int
    h: int
    h_K: int
    B_K: int
    T: int
    B_Q: int | None = None
    W: int | None = None
    bytes_per_elem: int = 2
    min_tile: int = 8
    g: int = 0
    b: int = 0

    @property
    def d(self) -> int:
        if self.d_K != self.d_V:
            raise ConfigError(f"non-uniform head dims (d_K={self.d_K}, d_V={self.d_V})")
        return self.d_K

    @property
    def scale(self) -> float:
        return 1.0 / math.sqrt(self.d_K)


_REQUIRED = ("N", "d_K", "d_V", "h", "h_K", "B_K", "T")
_INT_KEYS = _REQUIRED + ("B_Q", "W", "bytes_per_elem", "min_tile")


def validate_config(cfg: AttentionConfig) -> AttentionConfig:
    """Resolve defaults and derived fields; report every violation at once."""
    low = [f"{k} must be >= 1" for k in _REQUIRED if getattr(cfg, k) < 1]
    if low:
        raise ConfigError("; ".join(low))
    B_Q = min(16, cfg.N) if cfg.B_Q is None else cfg.B_Q
    W = min(512, cfg.N) if cfg.W is None else cfg.W
    b = cfg.N // cfg.B_K
    rules = [
        (cfg.h % cfg.h_K != 0, "h not divisible by h_K"),
        (cfg.N % cfg.B_K != 0, "N not divisible by B_K"),
        (cfg.N % cfg.B_K == 0 and cfg.T > b, f"T exceeds b={b}"),
        (not 1 <= B_Q <= cfg.N, "B_Q out of range [1, N]"),
        (not 1 <= W <= cfg.N, "W out of range [1, N]"),
        (cfg.min_tile < 1, "min_tile must be >= 1"),
        (cfg.bytes_per_elem not in (2, 4, 8), "bytes_per_elem not in {2, 4, 8}"),
    ]
    bad = [msg for broken, msg in rules if broken]
    if bad:
        raise ConfigError("; ".join(bad))
    return dataclasses.replace(cfg, B_Q=B_Q, W=W, g=cfg.h // cfg.h_K, b=b)


def make_config(**kwargs) -> AttentionConfig:
    return validate_config(AttentionConfig(**kwargs))


def parse_config_text(text: str) -> AttentionConfig:
    """``key = value`` lines with ``#`` comments (config.py:112-133)."""
    vals: dict[str, int] = {}
    for n, raw in enumerate(text.splitlines(), start=1):
        body = raw.split("#", 1)[0].strip()
        if not body:
            continue
        key, eq, val = body.partition("=")
        if not eq:
            raise ConfigError(f"line {n}: expected 'key = value', got {raw!r}")
        key = key.strip()
        if key not in _INT_KEYS:
            raise ConfigError(f"line {n}: unknown config key {key!r}")
        try:
            vals[key] = int(val.strip())
        except ValueError:
            raise ConfigError(f"line {n}: non-integer value for {key!r}") from None
    missing = [k for k in _REQUIRED if k not in vals]
    if missing:
        raise ConfigError("missing required config keys: " + ", ".join(missing))
    return make_config(**vals)


def load_config_file(path) -> AttentionConfig:
    with open(path, "r", encoding="utf-8") as fh:
        return parse_config_text(fh.read())


# ---------------------------------------------------------------------------
# tensor intake
# ---------------------------------------------------------------------------

#: check finiteness of every operator input (config.py:152-154); the training
#: path (nsa.py) turns this off because it needs one device->host sync per call.
CHECK_FINITE = True


def to_device(x, dtype=None) -> torch.Tensor:
    """numpy / CPU inputs are uploaded (float64 numpy stays float64, the
    reference's precision); CUDA tensors pass through."""
    dev = _lib.require_device()
    if isinstance(x, np.ndarray) or not torch.is_tensor(x):
        x = torch.as_tensor(np.asarray(x))
    if x.device != dev:
        x = x.to(dev, non_blocking=True)
    if dtype is not None and x.dtype != dtype:
        x = x.to(dtype)
    return x


def check_finite(x: torch.Tensor, name: str) -> None:
    flag = torch.zeros(1, dtype=torch.int32, device=x.device)
    _lib.call("fsa_check_finite", _lib.dt_code(x.dtype), _lib.ptr(x), x.numel(), _lib.ptr(flag),
              _lib.stream())
    if int(flag.item()):
        raise ValueError(f"{name} contains non-finite entries")


def as_headed(x, tokens: int, dim: int, heads: int, name: str, dtype=None) -> torch.Tensor:
    """Validate a logical (token, feature, head) tensor and return contiguous
    (token, head, feature) storage on the device."""
    x = to_device(x, dtype)
    if tuple(x.shape) != (tokens, dim, heads):
        raise ValueError(f"shape mismatch for {name}: expected {(tokens, dim, heads)}, got {tuple(x.shape)}")
    if x.dtype not in (torch.float32, torch.float64, torch.bfloat16):
        x = x.to(torch.float32)
    st = x.permute(0, 2, 1).contiguous()
    if CHECK_FINITE:
        check_finite(st, name)
    return st


def compute_dtype(*xs) -> torch.dtype:
    """The arithmetic type of a call: float64 if any input is float64, else
    float32 if any is float32, else bfloat16."""
    dts = {x.dtype for x in xs if torch.is_tensor(x)} | {
        torch.float64 for x in xs if isinstance(x, np.ndarray)}
    if torch.float64 in dts:
        return torch.float64
    if torch.float32 in dts or not dts:
        return torch.float32
    return torch.bfloat16


def logical(storage: torch.Tensor) -> torch.Tensor:
    """(token, head, feature) storage -> logical (token, feature, head) view."""
    return storage.permute(0, 2, 1)

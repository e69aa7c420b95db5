"""Multi-GPU partitioning of the NSA operator path.

Every hot-path operator is independent per KV head: scores and top-k per kv
head (selection.py:89-99, :116-119), the inverse index per kv head
(selection.py:157-166), the FSA tasks per (query head j, block i) with j in
the group of kv head j // g (kv_major.py:127-140, :183-203, :302-324), and
the three branches per head (branches.py:34-104).  So rank p of P owns the
kv heads [p h_K / P, (p + 1) h_K / P), their g query heads, and the whole
sequence, and runs the unmodified single-GPU path on that slice: **no
collective on the data path**.  NCCL appears only off the clock, to gather
results for validation (``gather_heads``), and as the timing barrier.

A second axis -- independent sequences (batch) -- needs no code at all: each
rank runs its own sequence; ``bench.py`` uses it for its weak-scaling line.

Storage layouts (include/fsa_b200.h): Q/out/dQ (N, h, d), K/V/dK/dV
(N, h_K, d) -> the head axis is dim 1; lse/m/l (h, N), scores (h_K, N, b) and
idx (h_K, N, T) -> the head axis is dim 0.
"""

from __future__ import annotations

import dataclasses

import torch

from .config import AttentionConfig, ConfigError, make_config


@dataclasses.dataclass(frozen=True)
class KVShard:
    """The slice of a problem one rank owns."""

    rank: int
    world: int
    kv_lo: int  # kv heads [kv_lo, kv_hi)
    kv_hi: int
    q_lo: int   # query heads [q_lo, q_hi) = g * [kv_lo, kv_hi)
    q_hi: int
    cfg: AttentionConfig  # the per-rank problem (h = g * (kv_hi - kv_lo))


def shard_kv_heads(cfg: AttentionConfig, rank: int, world: int) -> KVShard:
    """Contiguous kv-head partition of ``cfg`` over ``world`` ranks."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} for world size {world}")
    if cfg.h_K % world:
        raise ConfigError(f"h_K={cfg.h_K} kv heads cannot be split evenly over {world} ranks")
    per = cfg.h_K // world
    lo, hi = rank * per, (rank + 1) * per
    sub = make_config(N=cfg.N, d_K=cfg.d_K, d_V=cfg.d_V, h=cfg.g * per, h_K=per, B_K=cfg.B_K,
                      T=cfg.T, B_Q=cfg.B_Q, W=cfg.W, bytes_per_elem=cfg.bytes_per_elem,
                      min_tile=cfg.min_tile)
    return KVShard(rank, world, lo, hi, cfg.g * lo, cfg.g * hi, sub)


def slice_heads(x: torch.Tensor, lo: int, hi: int, dim: int) -> torch.Tensor:
    """Rows [lo, hi) of the head axis ``dim`` as a contiguous tensor."""
    return x.narrow(dim, lo, hi - lo).contiguous()


def shard_inputs(shard: KVShard, q, k, v, dout=None):
    """Per-rank Q (N, h, d), K, V (N, h_K, d) [, dOut (N, h, d)] storage slices."""
    out = [slice_heads(q, shard.q_lo, shard.q_hi, 1), slice_heads(k, shard.kv_lo, shard.kv_hi, 1),
           slice_heads(v, shard.kv_lo, shard.kv_hi, 1)]
    if dout is not None:
        out.append(slice_heads(dout, shard.q_lo, shard.q_hi, 1))
    return tuple(out)


def gather_heads(local: torch.Tensor, dim: int, group=None) -> torch.Tensor:
    """Concatenate every rank's head slice along ``dim`` (rank order), over the
    process group's backend (NCCL on GPUs, gloo in the CPU tests).  Off the
    hot path: used to validate a sharded run against the oracle."""
    import torch.distributed as dist

    world = dist.get_world_size(group)
    if world == 1:
        return local
    moved = local.movedim(dim, 0).contiguous()
    parts = [torch.empty_like(moved) for _ in range(world)]
    dist.all_gather(parts, moved, group=group)
    return torch.cat(parts, 0).movedim(0, dim).contiguous()

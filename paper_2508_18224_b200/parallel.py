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

When the ranks outnumber the kv heads (Qwen2.5-7B: h_K = 4 at P = 8) the
second axis is the query heads *inside* a kv group (``QueryShard``): the
``world / h_K`` ranks of a kv head split its g query heads.  Each of them
recomputes the group's importance scores and block selection (they sum over
all g heads, selection.py:105-120; the compressed pass is the cheap one) and
runs the selected and sliding branches for its own heads only
(``nsa.nsa_forward(..., heads=(lo, hi))``).  The forward still needs no
collective; the backward's dK / dV of the kv head are partial sums over the
rank's query heads, so they are summed over the kv head's ranks -- one
all_reduce of N·(d_K + d_V)·4 bytes per kv head, the only exchange step.

A third axis -- independent sequences (batch) -- needs no code at all: each
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


@dataclasses.dataclass(frozen=True)
class QueryShard:
    """One rank's query heads [lo, hi) of kv head ``kv`` (ranks > kv heads)."""

    rank: int
    world: int
    kv: int          # the kv head this rank works on
    lo: int          # query heads [lo, hi) within the group (absolute: kv * g + lo ...)
    hi: int
    peers: tuple     # ranks sharing the kv head (the dK / dV all_reduce group)
    group_cfg: AttentionConfig  # the whole group (h = g, h_K = 1): scores, selection
    cfg: AttentionConfig        # this rank's sub-problem (h = hi - lo, h_K = 1)


def shard_query_heads(cfg: AttentionConfig, rank: int, world: int) -> QueryShard:
    """world = r * h_K ranks: r ranks per kv head, each with a contiguous run of
    the group's g query heads (sizes differ by at most one)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} for world size {world}")
    if world % cfg.h_K:
        raise ConfigError(f"{world} ranks are not a multiple of h_K={cfg.h_K} kv heads")
    r = world // cfg.h_K
    if r > cfg.g:
        raise ConfigError(f"{r} ranks per kv head exceed the group size g={cfg.g}")
    kv, sub = divmod(rank, r)
    lo, hi = sub * cfg.g // r, (sub + 1) * cfg.g // r
    common = dict(N=cfg.N, d_K=cfg.d_K, d_V=cfg.d_V, h_K=1, B_K=cfg.B_K, T=cfg.T, B_Q=cfg.B_Q,
                  W=cfg.W, bytes_per_elem=cfg.bytes_per_elem, min_tile=cfg.min_tile)
    return QueryShard(rank, world, kv, lo, hi, tuple(range(kv * r, (kv + 1) * r)),
                      make_config(h=cfg.g, **common), make_config(h=hi - lo, **common))


def shard_plan(cfg: AttentionConfig, rank: int, world: int):
    """KV-head shards when they divide, else query-head shards within groups."""
    if cfg.h_K % world == 0:
        return shard_kv_heads(cfg, rank, world)
    return shard_query_heads(cfg, rank, world)


def query_shard_inputs(shard: QueryShard, q, k, v, dout=None):
    """The kv head's whole query group (N, g, d), its K / V (N, 1, d) and this
    rank's dOut heads (N, hi - lo, d)."""
    g = shard.group_cfg.h
    out = [slice_heads(q, shard.kv * g, (shard.kv + 1) * g, 1),
           slice_heads(k, shard.kv, shard.kv + 1, 1), slice_heads(v, shard.kv, shard.kv + 1, 1)]
    if dout is not None:
        out.append(slice_heads(dout, shard.kv * g + shard.lo, shard.kv * g + shard.hi, 1))
    return tuple(out)


def query_shard_step(shard: QueryShard, q_group, k, v, tau, dout=None, group=None):
    """NSA forward (and backward if dout is given) of one query shard on the
    device: returns out (N, hi - lo, d) [, dQ (N, hi - lo, d), dK, dV (N, 1, d)].
    dK / dV are all_reduced over the kv head's ranks (``group``: a process
    group of ``shard.peers``; None when the shard is alone)."""
    from . import nsa

    out, ctx = nsa.nsa_forward(q_group, k, v, tau, shard.group_cfg, heads=(shard.lo, shard.hi))
    if dout is None:
        return out
    dQ, dK, dV = nsa.nsa_backward(ctx, dout)
    if group is not None:
        import torch.distributed as dist

        dist.all_reduce(dK, group=group)
        dist.all_reduce(dV, group=group)
    return out, dQ, dK, dV

"""Value-independent traffic counters (the reference's ``meter.py``).

The reference fills a ``TrafficMeter`` inside its Python task loops
(kv_major.py:89-102, :186-203, :229-241, :285-354).  Here the counters are the
same exact integers, computed in closed form from the inverse index's
per-(kv head, block) row counts ``n_valid`` -- they never depend on tensor
values, so nothing is read back from the kernels except ``n_valid``.
"""

from __future__ import annotations

import dataclasses

import numpy as np

PHASES = ("stats", "block_pass", "reduce", "query_major")


@dataclasses.dataclass
class PhaseCounters:
    bytes_loaded: int = 0
    bytes_stored: int = 0
    flops: int = 0
    task_count: int = 0
    inner_iterations: int = 0

    @property
    def bytes_total(self) -> int:
        return self.bytes_loaded + self.bytes_stored

    def merged(self, other: "PhaseCounters") -> "PhaseCounters":
        return PhaseCounters(*(getattr(self, f.name) + getattr(other, f.name)
                               for f in dataclasses.fields(self)))

    def add(self, **kw) -> None:
        for k, v in kw.items():
            setattr(self, k, getattr(self, k) + int(v))


@dataclasses.dataclass
class TrafficMeter:
    phases: dict = dataclasses.field(default_factory=dict)

    def phase(self, name: str) -> PhaseCounters:
        return self.phases.setdefault(name, PhaseCounters())

    def merged(self, other: "TrafficMeter") -> "TrafficMeter":
        out = TrafficMeter({k: dataclasses.replace(v) for k, v in self.phases.items()})
        for k, v in other.phases.items():
            out.phases[k] = out.phase(k).merged(v)
        return out

    @property
    def total_bytes(self) -> int:
        return sum(p.bytes_total for p in self.phases.values())

    @property
    def total_flops(self) -> int:
        return sum(p.flops for p in self.phases.values())

    def as_rows(self):
        for name in PHASES:
            if name in self.phases:
                yield name, self.phases[name]
        for name in sorted(set(self.phases) - set(PHASES)):
            yield name, self.phases[name]


def _tiles(nv, B_Q):
    return -(-nv // B_Q)


def meter_stats(meter: TrafficMeter, nv: np.ndarray, cfg) -> None:
    """compute_softmax_stats accounting: per kv head, tiles of B_Q rows."""
    it = _tiles(nv, cfg.B_Q)
    live = nv > 0
    meter.phase("stats").add(
        task_count=cfg.h_K * cfg.b, inner_iterations=it.sum(),
        bytes_loaded=(((cfg.B_K + nv) * cfg.d_K) * cfg.bytes_per_elem)[live].sum(),
        bytes_stored=(nv * cfg.bytes_per_elem)[live].sum(),
        flops=(2 * it * cfg.B_Q * cfg.B_K * cfg.d_K)[live].sum())


def meter_block_pass(meter: TrafficMeter, nv: np.ndarray, cfg) -> None:
    """block_pass_forward accounting, g query heads per kv head."""
    it = _tiles(nv, cfg.B_Q)
    live = nv > 0
    bpe, g = cfg.bytes_per_elem, cfg.g
    meter.phase("block_pass").add(
        task_count=cfg.h * cfg.b, inner_iterations=g * it.sum(),
        bytes_loaded=g * ((cfg.B_K * (cfg.d_K + cfg.d_V) + nv * (cfg.d_K + 1)) * bpe)[live].sum(),
        bytes_stored=g * (nv * cfg.d_V * bpe).sum(),
        flops=g * (2 * it * cfg.B_Q * cfg.B_K * (cfg.d_K + cfg.d_V))[live].sum())


def meter_reduce(meter: TrafficMeter, nv: np.ndarray, cfg) -> None:
    nnz = nv.sum(axis=1)
    bpe = cfg.bytes_per_elem
    meter.phase("reduce").add(
        task_count=cfg.h * cfg.N, inner_iterations=cfg.g * nnz.sum(),
        bytes_loaded=cfg.g * ((nnz * cfg.d_V + cfg.N) * bpe).sum(),
        bytes_stored=cfg.h * cfg.N * cfg.d_V * bpe)


def forward_meter(nv, cfg) -> TrafficMeter:
    nv = np.asarray(nv, dtype=np.int64)
    m = TrafficMeter()
    meter_stats(m, nv, cfg)
    meter_block_pass(m, nv, cfg)
    meter_reduce(m, nv, cfg)
    return m


def backward_meter(nv, cfg) -> TrafficMeter:
    """selected_backward: forward recompute + backward tasks + reductions."""
    nv = np.asarray(nv, dtype=np.int64)
    m = forward_meter(nv, cfg)
    it = _tiles(nv, cfg.B_Q)
    live = nv > 0
    bpe, g = cfg.bytes_per_elem, cfg.g
    dsum = cfg.d_K + cfg.d_V
    m.phase("block_pass").add(
        task_count=cfg.h * cfg.b, inner_iterations=g * it.sum(),
        bytes_loaded=g * ((cfg.B_K * dsum + nv * dsum + 3 * nv) * bpe)[live].sum(),
        bytes_stored=g * ((nv * cfg.d_K + cfg.B_K * dsum) * bpe)[live].sum(),
        flops=g * (2 * it * cfg.B_Q * cfg.B_K * (3 * cfg.d_K + 2 * cfg.d_V))[live].sum())
    nnz = nv.sum(axis=1)
    touched = int(live.sum())
    m.phase("reduce").add(
        task_count=cfg.h * cfg.N, inner_iterations=g * nnz.sum(),
        bytes_loaded=2 * cfg.h * cfg.N * cfg.d_V * bpe + g * (nnz * cfg.d_K * bpe).sum()
        + touched * g * cfg.B_K * dsum * bpe,
        bytes_stored=cfg.h * cfg.N * bpe + cfg.h * cfg.N * cfg.d_K * bpe + touched * cfg.B_K * dsum * bpe)
    return m

"""KV-head sharding (paper_2508_18224_b200/parallel.py) on CPU with gloo,
world size 2: each rank runs the NSA fwd+bwd pipeline (the oracle as the
stand-in compute -- there is no GPU here) on its shard, the head slices are
all-gathered, and rank 0 checks the result against the unsharded problem.
Sharding by kv head must be bit-exact."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import fsa_oracle as O
from paper_2508_18224_b200 import make_config
from paper_2508_18224_b200.config import ConfigError
from paper_2508_18224_b200.parallel import gather_heads, shard_inputs, shard_kv_heads

KW = dict(N=256, d_K=16, d_V=16, h=8, h_K=4, B_K=16, T=4, W=32)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _storage(x):  # logical (N, d, heads) -> storage (N, heads, d)
    return torch.from_numpy(np.ascontiguousarray(x.transpose(0, 2, 1)))


def _logical(t):
    return t.permute(0, 2, 1).numpy()


def _worker(rank, world, port, outdir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        cfg = make_config(**KW)
        c = O.cfg_of(**KW)
        Q, K, V = O.make_qkv(c, 7)
        dO = O.make_dout(c, 7)
        tau = O.make_gates(c, 7)
        sh = shard_kv_heads(cfg, rank, world)
        q, k, v, do = shard_inputs(sh, _storage(Q), _storage(K), _storage(V), _storage(dO))
        cs = O.cfg_of(N=sh.cfg.N, d_K=sh.cfg.d_K, d_V=sh.cfg.d_V, h=sh.cfg.h, h_K=sh.cfg.h_K,
                      B_K=sh.cfg.B_K, T=sh.cfg.T, W=sh.cfg.W)
        r = O.nsa_forward_backward_group(_logical(q), _logical(k), _logical(v), _logical(do), tau, cs)
        full = {
            "idx": gather_heads(torch.from_numpy(r["idx"]), 0),
            "out": gather_heads(_storage(r["out"]), 1),
            "dQ": gather_heads(_storage(r["dQ_sel"] + r["g_slide"][0]), 1),
            "dK": gather_heads(_storage(r["dK_sel"] + r["g_slide"][1]), 1),
            "dV": gather_heads(_storage(r["dV_sel"] + r["g_slide"][2]), 1),
        }
        if rank == 0:
            np.savez(os.path.join(outdir, "sharded.npz"), **{n: t.numpy() for n, t in full.items()})
    finally:
        dist.destroy_process_group()


def test_kv_head_shards_gather_bit_exact(tmp_path):
    world = 2
    mp.start_processes(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world,
                       join=True, start_method="spawn")
    got = np.load(tmp_path / "sharded.npz")
    c = O.cfg_of(**KW)
    Q, K, V = O.make_qkv(c, 7)
    dO = O.make_dout(c, 7)
    tau = O.make_gates(c, 7)
    r = O.nsa_forward_backward_group(Q, K, V, dO, tau, c)
    assert np.array_equal(got["idx"], r["idx"])
    assert np.array_equal(got["out"], _storage(r["out"]).numpy())
    for name, ref in (("dQ", r["dQ_sel"] + r["g_slide"][0]), ("dK", r["dK_sel"] + r["g_slide"][1]),
                      ("dV", r["dV_sel"] + r["g_slide"][2])):
        assert np.array_equal(got[name], _storage(ref).numpy()), name


def test_shard_plan():
    cfg = make_config(N=1024, d_K=128, d_V=128, h=32, h_K=8, B_K=64, T=16, W=512)
    shards = [shard_kv_heads(cfg, r, 4) for r in range(4)]
    assert [(s.kv_lo, s.kv_hi, s.q_lo, s.q_hi) for s in shards] == [
        (0, 2, 0, 8), (2, 4, 8, 16), (4, 6, 16, 24), (6, 8, 24, 32)]
    assert all(s.cfg.h == 8 and s.cfg.h_K == 2 and s.cfg.g == 4 for s in shards)
    with pytest.raises(ConfigError, match="cannot be split evenly"):
        shard_kv_heads(cfg, 0, 3)
    with pytest.raises(ValueError):
        shard_kv_heads(cfg, 4, 4)


# ---------------------------------------------------------------------------
# query-head split (ranks > kv heads, e.g. Qwen2.5-7B h_K = 4 at P = 8)
# ---------------------------------------------------------------------------

QKW = dict(N=256, d_K=16, d_V=16, h=6, h_K=1, B_K=16, T=4, W=32)


def _qworker(rank, world, port, outdir):
    from paper_2508_18224_b200.parallel import query_shard_inputs, shard_plan

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        cfg = make_config(**QKW)
        c = O.cfg_of(**QKW)
        Q, K, V = O.make_qkv(c, 5)
        dO = O.make_dout(c, 5)
        tau = O.make_gates(c, 5)
        sh = shard_plan(cfg, rank, world)
        qg, k, v, do = query_shard_inputs(sh, _storage(Q), _storage(K), _storage(V), _storage(dO))
        # the oracle as the stand-in for nsa.nsa_forward(..., heads=(lo, hi)):
        # group scores and selection, then the sub-group's branches
        gc = O.cfg_of(N=c.N, d_K=c.d_K, d_V=c.d_V, h=sh.group_cfg.h, h_K=1, B_K=c.B_K, T=c.T, W=c.W)
        sc = O.cfg_of(N=c.N, d_K=c.d_K, d_V=c.d_V, h=sh.cfg.h, h_K=1, B_K=c.B_K, T=c.T, W=c.W)
        Qg, Kl, Vl, dOs = _logical(qg), _logical(k), _logical(v), _logical(do)
        cmp = O.compress_kv(Kl, Vl, gc)
        idx = O.select_topk(O.importance_scores(Qg, cmp.K_cmp, gc), gc)
        Qs = np.ascontiguousarray(Qg[:, :, sh.lo:sh.hi])
        outs = [O.compressed_forward(Qs, cmp, sc)[0], O.selected_forward(Qs, Kl, Vl, idx, sc)[0],
                O.sliding_forward(Qs, Kl, Vl, sc)[0]]
        out, _ = O.gated_combine(outs, tau, sc)
        gs = O.selected_backward(Qs, Kl, Vl, idx, dOs * tau[:, 1][:, None, None], sc)
        gl = O.sliding_backward(Qs, Kl, Vl, dOs * tau[:, 2][:, None, None], sc)
        dK = _storage(gs[1] + gl[1])
        dV = _storage(gs[2] + gl[2])
        group = dist.new_group(list(sh.peers))
        dist.all_reduce(dK, group=group)  # the query-head split's one exchange step
        dist.all_reduce(dV, group=group)
        full = {"out": gather_heads(_storage(out), 1), "dQ": gather_heads(_storage(gs[0] + gl[0]), 1),
                "dK": dK, "dV": dV, "idx": torch.from_numpy(idx)}
        if rank == 0:
            np.savez(os.path.join(outdir, "qsharded.npz"), **{n: t.numpy() for n, t in full.items()})
    finally:
        dist.destroy_process_group()


def test_query_head_shards_match_unsharded(tmp_path):
    world = 2
    mp.start_processes(_qworker, args=(world, _free_port(), str(tmp_path)), nprocs=world,
                       join=True, start_method="spawn")
    got = np.load(tmp_path / "qsharded.npz")
    c = O.cfg_of(**QKW)
    Q, K, V = O.make_qkv(c, 5)
    dO = O.make_dout(c, 5)
    tau = O.make_gates(c, 5)
    r = O.nsa_forward_backward_group(Q, K, V, dO, tau, c)
    assert np.array_equal(got["idx"], r["idx"])  # every rank selects from the whole group
    assert np.array_equal(got["out"], _storage(r["out"]).numpy())  # per-head: bit-exact
    assert np.array_equal(got["dQ"], _storage(r["dQ_sel"] + r["g_slide"][0]).numpy())
    for name, ref in (("dK", r["dK_sel"] + r["g_slide"][1]), ("dV", r["dV_sel"] + r["g_slide"][2])):
        np.testing.assert_allclose(got[name], _storage(ref).numpy(), rtol=1e-12, atol=1e-12)


def test_shard_plan_axes():
    from paper_2508_18224_b200.parallel import KVShard, QueryShard, shard_plan

    qwen = make_config(N=4096, d_K=128, d_V=128, h=28, h_K=4, B_K=64, T=16, W=512)
    assert isinstance(shard_plan(qwen, 1, 4), KVShard)
    plan = [shard_plan(qwen, r, 8) for r in range(8)]
    assert all(isinstance(s, QueryShard) for s in plan)
    assert [(s.kv, s.lo, s.hi) for s in plan[:2]] == [(0, 0, 3), (0, 3, 7)]
    assert plan[5].peers == (4, 5) and plan[5].cfg.h == 4 and plan[5].group_cfg.h == 7
    with pytest.raises(ConfigError):
        shard_plan(qwen, 0, 6)

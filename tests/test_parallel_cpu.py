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

"""The sharded NSA step on the device, as separate processes.

Two ranks (spawned processes, one CUDA context each; on a one-GPU box both
use cuda:0) run the product path -- ``parallel.shard_kv_heads`` /
``shard_query_heads`` -> ``nsa.nsa_forward`` -> ``nsa.nsa_backward`` -- on
their slice; the slices are gathered over a gloo group (host copies: NCCL
refuses two ranks on one device) and rank 0 compares them with the unsharded
run of the same path.  Every operator is independent per kv head
(selection.py:116-119, :157-166; kv_major.py:127-140), so the kv-head split
must be bit-exact; the query-head split (ranks > kv heads) sums dK / dV over
its ranks with the one all_reduce of the path."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

KW = dict(N=4096, d_K=128, d_V=128, h=16, h_K=4, B_K=64, T=16, W=512)
QKW = dict(N=4096, d_K=128, d_V=128, h=6, h_K=1, B_K=64, T=16, W=512)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _inputs(kw, seed):
    g = torch.Generator().manual_seed(seed)
    mk = lambda *s: torch.randn(*s, generator=g).to(torch.bfloat16)  # noqa: E731
    q, k, v, do = mk(kw["N"], kw["h"], 128), mk(kw["N"], kw["h_K"], 128), mk(kw["N"], kw["h_K"], 128), \
        mk(kw["N"], kw["h"], 128)
    tau = torch.rand(kw["N"], 3, generator=g)
    return q, k, v, do, tau


def _gather_cpu(x, dim):
    from paper_2508_18224_b200.parallel import gather_heads
    return gather_heads(x.detach().cpu(), dim)


def _worker(rank, world, port, outdir, mode):
    import paper_2508_18224_b200 as fsa
    from paper_2508_18224_b200 import nsa, parallel

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(rank % torch.cuda.device_count())
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        kw = KW if mode == "kv" else QKW
        cfg = fsa.make_config(**kw)
        q, k, v, do, tau = (x.cuda() for x in _inputs(kw, 11))
        if mode == "kv":
            sh = parallel.shard_kv_heads(cfg, rank, world)
            qs, ks, vs, dos = parallel.shard_inputs(sh, q, k, v, do)
            out, ctx = nsa.nsa_forward(qs, ks, vs, tau, sh.cfg)
            dQ, dK, dV = nsa.nsa_backward(ctx, dos)
            res = {"out": _gather_cpu(out, 1), "dQ": _gather_cpu(dQ, 1), "dK": _gather_cpu(dK, 1),
                   "dV": _gather_cpu(dV, 1), "idx": _gather_cpu(ctx.sel.idx, 0)}
        else:
            sh = parallel.shard_plan(cfg, rank, world)
            qg, ks, vs, dos = parallel.query_shard_inputs(sh, q, k, v, do)
            out, ctx = nsa.nsa_forward(qg, ks, vs, tau, sh.group_cfg, heads=(sh.lo, sh.hi))
            dQ, dK, dV = nsa.nsa_backward(ctx, dos)
            dK, dV = dK.cpu(), dV.cpu()
            group = dist.new_group(list(sh.peers))
            dist.all_reduce(dK, group=group)  # the split's one exchange step
            dist.all_reduce(dV, group=group)
            res = {"out": _gather_cpu(out, 1), "dQ": _gather_cpu(dQ, 1), "dK": dK, "dV": dV,
                   "idx": ctx.sel.idx.cpu()}
        torch.cuda.synchronize()
        if rank == 0:
            torch.save({n: t.float() if t.is_floating_point() else t for n, t in res.items()},
                       os.path.join(outdir, f"{mode}.pt"))
    finally:
        dist.destroy_process_group()


def _unsharded(kw):
    import paper_2508_18224_b200 as fsa
    from paper_2508_18224_b200 import nsa

    cfg = fsa.make_config(**kw)
    q, k, v, do, tau = (x.cuda() for x in _inputs(kw, 11))
    out, ctx = nsa.nsa_forward(q, k, v, tau, cfg)
    dQ, dK, dV = nsa.nsa_backward(ctx, do)
    return {"out": out.float().cpu(), "dQ": dQ.cpu(), "dK": dK.cpu(), "dV": dV.cpu(),
            "idx": ctx.sel.idx.cpu()}


def test_kv_head_shards_two_processes_bit_exact(tmp_path):
    mp.start_processes(_worker, args=(2, _free_port(), str(tmp_path), "kv"), nprocs=2, join=True,
                       start_method="spawn")
    got = torch.load(tmp_path / "kv.pt")
    want = _unsharded(KW)
    for name in ("idx", "out", "dQ", "dK", "dV"):
        assert torch.equal(got[name], want[name]), name


def test_query_head_shards_two_processes(tmp_path):
    """h_K = 1 over two ranks: each rank selects from the whole group and runs
    its 3 of the 6 query heads; out / dQ are per head (bit-exact); dK / dV are
    the all_reduced partial sums: a different fp32 summation order, and the
    fp16 backward operands are staged with the rank's own power-of-two scales
    (max over its heads), so P / dS round differently at 2^-11 -- measured
    1.1e-5 of max|dK|."""
    mp.start_processes(_worker, args=(2, _free_port(), str(tmp_path), "q"), nprocs=2, join=True,
                       start_method="spawn")
    got = torch.load(tmp_path / "q.pt")
    want = _unsharded(QKW)
    for name in ("idx", "out", "dQ"):
        assert torch.equal(got[name], want[name]), name
    for name in ("dK", "dV"):
        ref = want[name]
        err = (got[name] - ref).abs().max().item()
        assert err <= 1e-4 * ref.abs().max().item() + 1e-6, (name, err)

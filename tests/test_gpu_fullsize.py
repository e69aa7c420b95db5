"""Full-size parity of the NSA step at every BASELINE.json GPU shape and at
north_star's target (Llama-3-8B attention, 64K tokens).

Whole-array parity: for one complete KV group of every configuration the
float64 oracle (oracle.selected_forward_backward, sliding_forward/backward,
compressed_forward, select_topk -- pinned to the reference by
test_oracle_golden.py) runs on the group's whole sequence, in worker
processes (one per query head for the selected branch, one each for the
sliding branch, the compressed branch and the top-k), and every element of
out / out_sel / out_slide / out_cmp / lse / dQ / dK / dV of that group and
its (N, T) selection are compared.  In addition, on the whole device result:

* selection: ascending, causal, own block present, row length min(own+1, T),
  and bit-exact against the oracle's top-k on the GPU's own scores;
* inverse index: CSR round trip back to the selection, nnz closed form;
* forward: out (gated combine), out/lse of every branch on sampled tokens;
* backward: dQ rows on sampled tokens, dK/dV rows of sampled KV blocks, and
  for every kv head the identity sum_s dV[s] = sum_t sum_{j in group}
  (tau1 + tau2)[t] dOut[t, j] (softmax rows sum to one).
Tolerances as tests/gpu_util.assert_close (bf16: elementwise 2e-2 |ref| + 2e-2 RMS(ref)).
"""

import numpy as np
import pytest
import torch

import paper_2508_18224_b200 as fsa
from gpu_util import assert_close
from oracle import fsa_oracle as O
from paper_2508_18224_b200 import nsa
from paper_2508_18224_b200.selection import selection_from_inverse

pytestmark = pytest.mark.gpu

# BASELINE.json configs[1..4]; B_K = 64, T = 16, W = 512
CONFIGS = {
    "llama3_8b_32k": dict(N=32768, h=32, h_K=8, bwd=True),
    "llama3_8b_64k": dict(N=65536, h=32, h_K=8, bwd=True),  # north_star's target
    "qwen25_7b_64k_fwd": dict(N=65536, h=28, h_K=4, bwd=False),
    "gqa1_64k": dict(N=65536, h=16, h_K=16, bwd=True),
    "qwen3_14b_128k": dict(N=131072, h=40, h_K=8, bwd=True),
}


def _np(t):
    return t.detach().float().cpu().numpy()


@pytest.mark.parametrize("name", list(CONFIGS))
def test_fullsize_nsa_step(name):
    spec = CONFIGS[name]
    kw = dict(N=spec["N"], d_K=128, d_V=128, h=spec["h"], h_K=spec["h_K"], B_K=64, T=16, W=512)
    cfg = fsa.make_config(**kw)
    c = O.cfg_of(**kw)
    gen = torch.Generator(device="cuda").manual_seed(7)
    bf = torch.bfloat16
    q = torch.randn(c.N, c.h, 128, device="cuda", dtype=bf, generator=gen)
    k = torch.randn(c.N, c.h_K, 128, device="cuda", dtype=bf, generator=gen)
    v = torch.randn(c.N, c.h_K, 128, device="cuda", dtype=bf, generator=gen)
    do = torch.randn(c.N, c.h, 128, device="cuda", dtype=bf, generator=gen)
    tau = torch.rand(c.N, 3, device="cuda", generator=gen)
    out, ctx = nsa.nsa_forward(q, k, v, tau, cfg, keep_scores=True)
    if spec["bwd"]:
        dQ, dK, dV = nsa.nsa_backward(ctx, do)
    torch.cuda.synchronize()
    # determinism: no floating-point atomics, fixed reduction orders -> a second
    # run (different dynamic task-to-CTA assignment) is bit-identical
    out2, ctx2 = nsa.nsa_forward(q, k, v, tau, cfg)
    assert torch.equal(out2, out) and torch.equal(ctx2.sel.idx, ctx.sel.idx)
    if spec["bwd"]:
        for a_, b_ in zip(nsa.nsa_backward(ctx2, do), (dQ, dK, dV)):
            assert torch.equal(a_, b_), "backward not bit-identical across runs"
    del out2, ctx2

    # ---- selection structure on the whole result
    idx = ctx.sel.idx
    own = torch.arange(c.N, device="cuda") // c.B_K
    live = idx >= 0
    want_len = torch.clamp(own + 1, max=c.T)
    assert torch.equal(live.sum(-1), want_len.expand(c.h_K, -1).to(live.sum(-1).dtype))
    assert bool((idx <= own[None, :, None]).all()), "non-causal block selected"
    assert bool((idx == own[None, :, None]).any(-1).all()), "own block missing"
    a, b_ = idx[..., 1:], idx[..., :-1]
    assert bool(((a > b_) | (a < 0)).all()), "selection rows not strictly ascending"
    # ---- inverse index: CSR round trip and closed-form nnz (test_selection.py:208-215)
    assert torch.equal(selection_from_inverse(ctx.inv, cfg).idx, idx)
    nnz = c.B_K * sum(min(jb + 1, c.T) for jb in range(c.b))
    assert (ctx.inv.offsets[:, -1].to(torch.int64) == nnz).all()

    # ---- sampled tokens: selection bit-exact on the GPU's scores, forward, dQ
    rng = np.random.default_rng(c.N + c.h)
    toks = np.unique(np.concatenate([[0, 1, 62, 63, 64, 65, 511, 512, c.N - 1],
                                     rng.integers(0, c.N, 23)]))
    tt = torch.from_numpy(toks).cuda()
    idx_rows = idx[:, tt].cpu().numpy()
    score_rows = ctx.scores[:, tt].double().cpu().numpy()
    np.testing.assert_array_equal(O.select_topk_rows(score_rows, toks, c), idx_rows)
    Kc, Vc = _np(k), _np(v)
    pooled = O.pooled_kv(Kc, Vc, c)
    tau_np = tau.double().cpu().numpy()
    r = O.nsa_rows(_np(q[tt]), toks, Kc, Vc, idx_rows, tau_np[toks], pooled, c,
                   dO_rows=_np(do[tt]) if spec["bwd"] else None)
    assert_close(_np(out[tt]), r["out"], "bf16", f"{name} out")
    assert_close(_np(ctx.out_sel[tt]), r["out_sel"], "bf16", f"{name} out_sel")
    assert_close(_np(ctx.out_slide[tt]), r["out_slide"], "bf16", f"{name} out_slide")
    assert_close(_np(ctx.out_cmp[tt]), r["out_cmp"], "bf16", f"{name} out_cmp")
    for br in ("sel", "slide"):
        got = getattr(ctx, "lse_" + br)[:, tt].double().cpu().numpy()
        assert np.abs(got - r["lse_" + br]).max() < 2e-2, f"{name} lse_{br}"
    if not spec["bwd"]:
        return
    assert_close(_np(dQ[tt]), r["dQ"], "bf16", f"{name} dQ", grad=True)

    # ---- sampled KV blocks: dK / dV rows (selected + sliding branches)
    idx_np = idx.cpu().numpy()
    q_of = lambda ts: _np(q[torch.from_numpy(np.asarray(ts)).cuda()])  # noqa: E731
    do_of = lambda ts: _np(do[torch.from_numpy(np.asarray(ts)).cuda()])  # noqa: E731
    for kh, i in ((c.h_K - 1, c.b // 2), (0, c.b - 1), (c.h_K // 2, c.b - 7)):
        rk, rv = O.block_grads(i, kh, q_of, Kc, Vc, do_of, tau_np, idx_np[kh], c)
        sl = slice(i * c.B_K, (i + 1) * c.B_K)
        assert_close(_np(dK[sl, kh]), rk, "bf16", f"{name} dK block {i} kv {kh}", grad=True)
        assert_close(_np(dV[sl, kh]), rv, "bf16", f"{name} dV block {i} kv {kh}", grad=True)

    # ---- every block at once: sum_s dV[s] = sum_t (tau1 + tau2) sum_{j in grp} dOut[t, j]
    w = (tau[:, 1] + tau[:, 2]).double()
    rhs = (do.double() * w[:, None, None]).sum(0).view(c.h_K, c.g, 128).sum(1)
    lhs = dV.double().sum(0)
    err = (lhs - rhs).norm() / rhs.norm()
    assert float(err) < 1e-2, f"{name}: dV column-sum identity off by {float(err):.2e}"


# ---------------------------------------------------------------------------
# whole-array parity of one complete KV group (every element, every branch)
# ---------------------------------------------------------------------------

_G = {}  # the group's float64 inputs, shared copy-on-write with the forked workers


def _oracle_part(task):
    """One piece of the float64 oracle for the group in _G, run in a worker;
    arrays come back as float32 (8e-8 relative, far below the bf16 bound)."""
    from threadpoolctl import threadpool_limits

    kind, j = task
    g, c1, cg, bwd = _G["g"], _G["c1"], _G["cg"], _G["bwd"]
    Q, K, V, dO, tau = _G["Q"], _G["K"], _G["V"], _G["dO"], _G["tau"]
    f32 = lambda x: np.asarray(x, dtype=np.float32)  # noqa: E731
    with threadpool_limits(1):
        if kind == "sel":  # query head j of the group (its dK/dV share: summed in head order)
            q = Q[:, :, j:j + 1]
            if bwd:
                d = dO[:, :, j:j + 1] * tau[:, 1][:, None, None]
                out, lse, dq, dk, dv = O.selected_forward_backward(q, K, V, _G["idx"], d, c1)
                return kind, j, dict(out=f32(out), lse=lse, dQ=f32(dq), dK=dk, dV=dv)
            out, lse = O.selected_forward(q, K, V, _G["idx"], c1)
            return kind, j, dict(out=f32(out), lse=lse)
        if kind == "slide":
            out, lse = O.sliding_forward(Q, K, V, cg)
            res = dict(out=f32(out), lse=lse)
            if bwd:
                dq, dk, dv = O.sliding_backward(Q, K, V, dO * tau[:, 2][:, None, None], cg)
                res.update(dQ=f32(dq), dK=dk, dV=dv)
            return kind, j, res
        if kind == "cmp":
            cmp = O.compress_kv(K, V, cg)
            out, lse = O.compressed_forward(Q, cmp, cg)
            scores = O.importance_scores(Q, cmp.K_cmp, cg)
            return kind, j, dict(out=f32(out), lse=lse, scores=scores)
        if kind == "topk":  # on the GPU's own scores (fp32 -> f64 exact)
            return kind, j, dict(idx=O.select_topk(_G["scores"], cg))
    raise ValueError(kind)


def _whole_group(name, spec, q, k, v, do, tau, out, ctx, grads, kh):
    import multiprocessing as mp

    N, g = spec["N"], spec["h"] // spec["h_K"]
    kw = dict(N=N, d_K=128, d_V=128, h=g, h_K=1, B_K=64, T=16, W=512)
    js = slice(kh * g, (kh + 1) * g)
    lg = lambda x: np.ascontiguousarray(_np(x).transpose(0, 2, 1)).astype(np.float64)  # noqa: E731
    _G.clear()
    _G.update(g=g, bwd=spec["bwd"], cg=O.cfg_of(**kw), c1=O.cfg_of(**dict(kw, h=1)),
              Q=lg(q[:, js]), K=lg(k[:, kh:kh + 1]), V=lg(v[:, kh:kh + 1]),
              dO=lg(do[:, js]) if spec["bwd"] else None, tau=tau.double().cpu().numpy(),
              idx=ctx.sel.idx[kh:kh + 1].cpu().numpy(),
              scores=ctx.scores[kh:kh + 1].double().cpu().numpy())
    tasks = [("topk", 0), ("slide", 0), ("cmp", 0)] + [("sel", j) for j in range(g)]
    import os
    with mp.get_context("fork").Pool(max(1, min(len(tasks), os.cpu_count() or 1))) as pool:
        parts = {}
        for kind, j, res in pool.imap_unordered(_oracle_part, tasks):
            parts[(kind, j)] = res
    # selection of the whole group: bit-exact on the GPU's own scores
    np.testing.assert_array_equal(parts[("topk", 0)]["idx"], _G["idx"])
    lay = lambda x: x.transpose(0, 2, 1)  # noqa: E731  oracle (N, d, h) -> storage (N, h, d)
    sel_out = np.concatenate([parts[("sel", j)]["out"] for j in range(g)], axis=2)
    sel_lse = np.concatenate([parts[("sel", j)]["lse"] for j in range(g)], axis=0)
    sl, cm = parts[("slide", 0)], parts[("cmp", 0)]
    t = _G["tau"]
    want = (t[:, 0][:, None, None] * cm["out"].astype(np.float64)
            + t[:, 1][:, None, None] * sel_out + t[:, 2][:, None, None] * sl["out"])
    tag = f"{name} kv{kh} (whole group)"
    assert_close(_np(out[:, js]), lay(want), "bf16", f"{tag} out")
    assert_close(_np(ctx.out_sel[:, js]), lay(sel_out), "bf16", f"{tag} out_sel")
    assert_close(_np(ctx.out_slide[:, js]), lay(sl["out"]), "bf16", f"{tag} out_slide")
    assert_close(_np(ctx.out_cmp[:, js]), lay(cm["out"]), "bf16", f"{tag} out_cmp")
    for br, ref in (("sel", sel_lse), ("slide", sl["lse"]), ("cmp", cm["lse"])):
        got = getattr(ctx, "lse_" + br)[js].double().cpu().numpy()
        err = float(np.abs(got - ref).max())
        assert err < 2e-2, f"{tag} lse_{br}: max abs err {err:.2e}"
    # importance scores of the causal blocks (the ones top-k reads)
    rows = np.arange(0, N, 4)  # every 4th token (the scores are N x b)
    causal = np.arange(N // 64)[None, :] <= (rows // 64)[:, None]
    assert_close(_G["scores"][0][rows][causal], cm["scores"][0][rows][causal], "bf16",
                 f"{tag} scores")
    if not spec["bwd"]:
        return
    dQ, dK, dV = grads
    sel_dq = np.concatenate([parts[("sel", j)]["dQ"] for j in range(g)], axis=2)
    want_dq = sel_dq.astype(np.float64) + sl["dQ"]
    want_dk = sl["dK"].copy()
    want_dv = sl["dV"].copy()
    sk = sum(parts[("sel", j)]["dK"] for j in range(g))  # ascending head order
    sv = sum(parts[("sel", j)]["dV"] for j in range(g))
    want_dk, want_dv = sk + want_dk, sv + want_dv
    assert_close(_np(dQ[:, js]), lay(want_dq), "bf16", f"{tag} dQ", grad=True)
    assert_close(_np(dK[:, kh:kh + 1]), lay(want_dk), "bf16", f"{tag} dK", grad=True)
    assert_close(_np(dV[:, kh:kh + 1]), lay(want_dv), "bf16", f"{tag} dV", grad=True)


@pytest.mark.parametrize("name", list(CONFIGS))
def test_fullsize_whole_group(name):
    """Every element of one whole KV group (the last) against the float64 oracle."""
    spec = CONFIGS[name]
    kw = dict(N=spec["N"], d_K=128, d_V=128, h=spec["h"], h_K=spec["h_K"], B_K=64, T=16, W=512)
    cfg = fsa.make_config(**kw)
    gen = torch.Generator(device="cuda").manual_seed(11)
    bf = torch.bfloat16
    N, h, hk = spec["N"], spec["h"], spec["h_K"]
    q = torch.randn(N, h, 128, device="cuda", dtype=bf, generator=gen)
    k = torch.randn(N, hk, 128, device="cuda", dtype=bf, generator=gen)
    v = torch.randn(N, hk, 128, device="cuda", dtype=bf, generator=gen)
    do = torch.randn(N, h, 128, device="cuda", dtype=bf, generator=gen)
    tau = torch.rand(N, 3, device="cuda", generator=gen)
    out, ctx = nsa.nsa_forward(q, k, v, tau, cfg, keep_scores=True)
    grads = nsa.nsa_backward(ctx, do) if spec["bwd"] else None
    torch.cuda.synchronize()
    _whole_group(name, spec, q, k, v, do, tau, out, ctx, grads, hk - 1)


# ---------------------------------------------------------------------------
# long context through the buffer-reusing kv-head-chunked schedule (512K tokens,
# Qwen3-14B shape: N h = 21M >= 2^23, so nsa_forward chunks by kv head itself)
# ---------------------------------------------------------------------------

def test_long_context_512k_chunked_sampled():
    N, h, h_K = 524288, 40, 8
    kw = dict(N=N, d_K=128, d_V=128, h=h, h_K=h_K, B_K=64, T=16, W=512)
    cfg = fsa.make_config(**kw)
    gen = torch.Generator(device="cuda").manual_seed(11)
    bf = torch.bfloat16
    q = torch.randn(N, h, 128, device="cuda", dtype=bf, generator=gen)
    k = torch.randn(N, h_K, 128, device="cuda", dtype=bf, generator=gen)
    v = torch.randn(N, h_K, 128, device="cuda", dtype=bf, generator=gen)
    do = torch.randn(N, h, 128, device="cuda", dtype=bf, generator=gen)
    tau = torch.rand(N, 3, device="cuda", generator=gen)
    out, ctx = nsa.nsa_forward(q, k, v, tau, cfg)  # auto-chunked (N h >= 2^23)
    assert isinstance(ctx, nsa.ChunkedNSAContext)
    lo, hi, c0 = ctx.chunks[0]
    assert (lo, hi) == (0, fsa.plan_kv_chunk(cfg))
    dQ, dK, dV = nsa.nsa_backward(ctx, do)
    torch.cuda.synchronize()
    g, sub, idx0 = cfg.g, c0.cfg, c0.sel.idx.clone()
    del ctx, c0
    torch.cuda.empty_cache()
    # the first chunk's sub-problem, re-run with its scores kept: same selection
    qs, ks, vs = q[:, lo * g:hi * g].contiguous(), k[:, lo:hi].contiguous(), v[:, lo:hi].contiguous()
    _, cs = nsa.nsa_forward(qs, ks, vs, tau, sub, keep_scores=True)
    assert torch.equal(cs.sel.idx, idx0)
    c = O.cfg_of(N=N, d_K=128, d_V=128, h=sub.h, h_K=sub.h_K, B_K=64, T=16, W=512)
    rng = np.random.default_rng(5)
    toks = np.unique(np.concatenate([[0, 63, 64, 300000, N - 1], rng.integers(0, N, 11)]))
    tt = torch.from_numpy(toks).cuda()
    idx_rows = idx0[:, tt].cpu().numpy()
    np.testing.assert_array_equal(
        O.select_topk_rows(cs.scores[:, tt].double().cpu().numpy(), toks, c), idx_rows)
    del cs
    Kc, Vc = _np(ks), _np(vs)
    r = O.nsa_rows(_np(qs[tt]), toks, Kc, Vc, idx_rows, tau.double().cpu().numpy()[toks],
                   O.pooled_kv(Kc, Vc, c), c, dO_rows=_np(do[tt, lo * g:hi * g]))
    assert_close(_np(out[tt, lo * g:hi * g]), r["out"], "bf16", "512K out")
    assert_close(_np(dQ[tt, lo * g:hi * g]), r["dQ"], "bf16", "512K dQ", grad=True)
    # every kv head: sum_s dV[s] = sum_t (tau1 + tau2) sum_{j in grp} dOut[t, j]
    w = (tau[:, 1] + tau[:, 2]).double()
    rhs = (do.double() * w[:, None, None]).sum(0).view(h_K, g, 128).sum(1)
    err = (dV.double().sum(0) - rhs).norm() / rhs.norm()
    assert float(err) < 1e-2, f"512K dV column-sum identity off by {float(err):.2e}"

"""Full-size parity of the NSA step at every BASELINE.json GPU shape.

The whole-array oracle cannot run at 32K-128K tokens, so parity here rests on
(1) size-independent structure checked on the whole device result and
(2) the oracle's sampled-row restatement (oracle.nsa_rows / block_grads,
pinned to the whole-array oracle by test_oracle_golden.py) on sampled tokens
and KV blocks:

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
    out, ctx = nsa.nsa_forward(q, k, v, tau, cfg)
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

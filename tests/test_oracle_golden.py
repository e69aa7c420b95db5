"""Pin the CPU oracle (oracle/fsa_oracle.py) to the real reference's outputs.

The fixtures were produced by importing the reference package itself
(tests/golden/make_golden.py).  Tolerances follow the reference's own tests
(1e-10 forward, 1e-9 backward, test_kv_major.py / test_acceptance.py).
"""

import json

import numpy as np
import pytest

from golden_io import FULL_CASES, case, load, stride_of
from oracle import fsa_oracle as O


def _tol(z):
    return 1e-10 if z["out"].dtype == np.float64 else 2e-5


@pytest.mark.parametrize("name", FULL_CASES)
def test_selection_and_inverse_bit_exact(name):
    kw, c, inp, z = case(name)
    if str(z["sel_mode"]) == "random_uniform":
        scores = O.make_scores(c, int(z["seed"]))
    else:
        cmp = O.compress_kv(inp["K"], inp["V"], c)
        scores = O.importance_scores(inp["Q"], cmp.K_cmp, c)
    idx = O.select_topk(scores, c)
    np.testing.assert_array_equal(idx, z["idx"])
    inv = O.build_inverse(idx, c)
    np.testing.assert_array_equal(inv.offsets, z["inv_offsets"])
    np.testing.assert_array_equal(np.concatenate(inv.tok), z["inv_tok"])
    np.testing.assert_array_equal(inv.n_valid, z["n_valid"])


@pytest.mark.parametrize("name", FULL_CASES)
def test_forward_backward_match_reference(name):
    kw, c, inp, z = case(name)
    st = stride_of(z)
    tol = _tol(z)
    idx = z["idx"]
    out, lse = O.selected_forward(inp["Q"], inp["K"], inp["V"], idx, c)
    scale = max(1.0, float(np.abs(z["out"]).max()))
    assert np.abs(out[::st] - z["out"]).max() <= tol * scale
    assert np.abs(lse - z["lse"]).max() <= tol * max(1.0, float(np.abs(z["lse"]).max()))
    stats = O.softmax_stats(inp["Q"], inp["K"], idx, c)
    assert np.abs(stats.m - z["m"]).max() <= tol * 10
    assert np.abs(stats.l - z["l"]).max() <= tol * 10 * max(1.0, float(z["l"].max()))
    stats = O.softmax_stats(inp["Q"], inp["K"], idx, c, shared_max=True)
    np.testing.assert_allclose(stats.m, z["m_sh"], atol=tol * 10)
    np.testing.assert_allclose(stats.l, z["l_sh"], rtol=tol * 10, atol=tol * 10)
    dQ, dK, dV = O.selected_backward(inp["Q"], inp["K"], inp["V"], idx, inp["dOut"], c)
    btol = 1e-9 if z["dQ"].dtype == np.float64 else 5e-5
    for got, key in ((dQ, "dQ"), (dK, "dK"), (dV, "dV")):
        ref = z[key]
        assert np.abs(got[::st] - ref).max() <= btol * max(1.0, float(np.abs(ref).max())), key


@pytest.mark.parametrize("name", FULL_CASES)
def test_branches_match_reference(name):
    kw, c, inp, z = case(name)
    st = stride_of(z)
    tol = _tol(z)
    cmp = O.compress_kv(inp["K"], inp["V"], c)
    for key, got in zip(("K_cmp", "V_cmp", "K_prefix", "V_prefix"), cmp):
        np.testing.assert_allclose(got, z[key], atol=tol, rtol=tol)
    sc = O.importance_scores(inp["Q"], cmp.K_cmp, c)
    np.testing.assert_allclose(sc[:, ::st], z["scores_cmp"], atol=tol * 10, rtol=tol)
    o, l = O.compressed_forward(inp["Q"], cmp, c)
    np.testing.assert_allclose(o[::st], z["cmp_out"], atol=tol * 10, rtol=tol)
    np.testing.assert_allclose(l, z["cmp_lse"], atol=tol * 10, rtol=tol)
    if "slide_out" in z.files:
        so, sl = O.sliding_forward(inp["Q"], inp["K"], inp["V"], c)
        np.testing.assert_allclose(so[::st], z["slide_out"], atol=tol * 10, rtol=tol)
        np.testing.assert_allclose(sl, z["slide_lse"], atol=tol * 10, rtol=tol)
        g = O.sliding_backward(inp["Q"], inp["K"], inp["V"], inp["dOut"], c)
        btol = 1e-9 if z["dQ"].dtype == np.float64 else 5e-5
        for got, key in zip(g, ("slide_dQ", "slide_dK", "slide_dV")):
            ref = z[key]
            assert np.abs(got[::st] - ref).max() <= btol * max(1.0, float(np.abs(ref).max())), key
        sel_out, _ = O.selected_forward(inp["Q"], inp["K"], inp["V"], z["idx"], c)
        comb, lse = O.gated_combine((o, sel_out, so), inp["tau"], c)
        np.testing.assert_allclose(comb[::st], z["comb_out"], atol=tol * 10, rtol=tol)
        assert np.isnan(lse).all()


@pytest.mark.parametrize("name", FULL_CASES)
def test_dense_truth_agrees(name):
    kw, c, inp, z = case(name)
    if "dense_out" not in z.files:
        pytest.skip("large case: dense truth not stored")
    allow = O.selection_mask(z["idx"], c)
    out, lse = O.dense_forward(inp["Q"], inp["K"], inp["V"], allow, c)
    np.testing.assert_allclose(out, z["dense_out"], atol=1e-10)
    np.testing.assert_allclose(lse, z["dense_lse"], atol=1e-10)


@pytest.mark.parametrize("name", FULL_CASES)
def test_meter_closed_forms(name):
    kw, c, inp, z = case(name)
    want_f = json.loads(str(z["meter_fwd"]))
    want_b = json.loads(str(z["meter_bwd"]))
    assert O.meter_forward(z["n_valid"], c) == want_f
    assert O.meter_backward(z["n_valid"], c) == want_b


def _kat_scores(z, tag, c):
    if tag + "__scores" in z.files:
        return z[tag + "__scores"]
    seed, f32 = (int(v) for v in z[tag + "__seed"])
    s = O.make_scores(c, seed)
    return s.astype(np.float32).astype(np.float64) if f32 else s


def test_selection_kats():
    z = load("selection_kats")
    tags = sorted({k.split("__")[0] for k in z.files})
    assert len(tags) >= 9
    for tag in tags:
        c = O.cfg_of(**json.loads(str(z[tag + "__cfg"])))
        idx = O.select_topk(_kat_scores(z, tag, c), c)
        np.testing.assert_array_equal(idx, z[tag + "__idx"], err_msg=tag)


def test_malformed_messages():
    z = load("malformed")
    c = O.cfg_of(**json.loads(str(z["cfg"])))
    msgs = json.loads(str(z["messages"]))
    for tag, msg in msgs.items():
        with pytest.raises(O.OracleSelectionError) as exc:
            O.validate_selection(z["idx_" + tag], c)
        assert str(exc.value) == msg, tag


def test_acceptance_sweep():
    z = load("acceptance_sweep")
    for n in range(int(z["count"])):
        p = f"s{n}__"
        c = O.cfg_of(**json.loads(str(z[p + "cfg"])))
        seed = int(z[p + "seed"])
        Q, K, V = O.make_qkv(c, seed)
        idx = O.select_topk(O.make_scores(c, seed), c)
        np.testing.assert_array_equal(idx, z[p + "idx"])
        out, lse = O.selected_forward(Q, K, V, idx, c)
        assert np.abs(out - z[p + "out"]).max() <= 1e-10
        g = O.selected_backward(Q, K, V, idx, O.make_dout(c, seed), c)
        for got, key in zip(g, ("dQ", "dK", "dV")):
            assert np.abs(got - z[p + key]).max() <= 1e-9


def test_sampled_row_restatement_matches_whole_array_oracle():
    """oracle.nsa_rows / block_grads (used by the full-size GPU parity tests)
    against the whole-array oracle pinned above, on a small problem."""
    kw = dict(N=512, d_K=16, d_V=16, h=8, h_K=2, B_K=16, T=4, W=64)
    c = O.cfg_of(**kw)
    Q, K, V = O.make_qkv(c, 11)
    dO = O.make_dout(c, 11)
    tau = O.make_gates(c, 11)
    cmp = O.compress_kv(K, V, c)
    idx = O.select_topk(O.importance_scores(Q, cmp.K_cmp, c), c)
    o_sel, l_sel = O.selected_forward(Q, K, V, idx, c)
    o_sl, l_sl = O.sliding_forward(Q, K, V, c)
    o_cmp, l_cmp = O.compressed_forward(Q, cmp, c)
    out, _ = O.gated_combine((o_cmp, o_sel, o_sl), tau, c)
    g_sel = O.selected_backward(Q, K, V, idx, dO * tau[:, 1][:, None, None], c)
    g_sl = O.sliding_backward(Q, K, V, dO * tau[:, 2][:, None, None], c)
    st = lambda x: np.ascontiguousarray(x.transpose(0, 2, 1))  # noqa: E731
    Qs, Ks, Vs, dOs = st(Q), st(K), st(V), st(dO)
    toks = np.array([0, 5, 14, 15, 16, 63, 64, 200, 511])
    scores = O.importance_scores(Q, cmp.K_cmp, c)
    np.testing.assert_array_equal(O.select_topk_rows(scores[:, toks], toks, c), idx[:, toks])
    pooled = O.pooled_kv(Ks, Vs, c)
    r = O.nsa_rows(Qs[toks], toks, Ks, Vs, idx[:, toks], tau[toks], pooled, c, dO_rows=dOs[toks])
    for name, ref in (("out", out), ("out_sel", o_sel), ("out_slide", o_sl), ("out_cmp", o_cmp)):
        np.testing.assert_allclose(r[name], st(ref)[toks], rtol=1e-10, atol=1e-12, err_msg=name)
    for name, ref in (("lse_sel", l_sel), ("lse_slide", l_sl), ("lse_cmp", l_cmp)):
        np.testing.assert_allclose(r[name], ref[:, toks], rtol=1e-10, atol=1e-12, err_msg=name)
    np.testing.assert_allclose(r["dQ"], st(g_sel[0] + g_sl[0])[toks], rtol=1e-9, atol=1e-12)
    for kh, i in ((0, 0), (1, 7), (1, 31)):
        dK, dV = O.block_grads(i, kh, lambda ts: Qs[ts], Ks, Vs, lambda ts: dOs[ts], tau, idx[kh], c)
        sl = slice(i * c.B_K, (i + 1) * c.B_K)
        np.testing.assert_allclose(dK, (g_sel[1] + g_sl[1])[sl, :, kh], rtol=1e-9, atol=1e-12)
        np.testing.assert_allclose(dV, (g_sel[2] + g_sl[2])[sl, :, kh], rtol=1e-9, atol=1e-12)


def test_compressed_backward_and_gate_grad_vs_autograd():
    """The compressed branch and the gate have no backward in the reference
    (parity unpinned); the oracle's analytic gradients are pinned to float64
    torch autograd of the same forward semantics (branches.py:34-104)."""
    import torch
    kw = dict(N=256, d_K=8, d_V=12, h=4, h_K=2, B_K=16, T=4, W=32)
    c = O.cfg_of(**kw)
    Q, K, V = O.make_qkv(c, 5)
    dO = O.make_dout(c, 5)
    tau = O.make_gates(c, 5)
    tQ, tK, tV = (torch.from_numpy(x).requires_grad_(True) for x in (Q, K, V))
    n_pref = min(c.B_K - 1, c.N)
    Kc = tK.reshape(c.b, c.B_K, c.d_K, c.h_K).mean(1)
    Vc = tV.reshape(c.b, c.B_K, c.d_V, c.h_K).mean(1)
    Vp = torch.cumsum(tV[:n_pref], 0) / torch.arange(1, n_pref + 1, dtype=torch.float64)[:, None, None]
    formed = (torch.arange(c.N) + 1) // c.B_K
    outs = []
    for j in range(c.h):
        kh = j // c.g
        z = (tQ[:, :, j] @ Kc[:, :, kh].T) * c.scale
        z = z.masked_fill(torch.arange(c.b)[None, :] >= formed[:, None], float("-inf"))
        ready = formed > 0
        p = torch.softmax(z[ready], dim=1)
        o = torch.zeros(c.N, c.d_V, dtype=torch.float64)
        o = o.index_put((torch.nonzero(ready)[:, 0],), p @ Vc[:, :, kh])
        o = o.index_put((torch.arange(n_pref),), Vp[:, :, kh])
        outs.append(o)
    out = torch.stack(outs, dim=2)
    (out * torch.from_numpy(dO)).sum().backward()
    dQ, dK, dV = O.compressed_backward(Q, K, V, dO, c)
    np.testing.assert_allclose(dQ, tQ.grad.numpy(), rtol=1e-10, atol=1e-12)
    np.testing.assert_allclose(dK, tK.grad.numpy(), rtol=1e-10, atol=1e-12)
    np.testing.assert_allclose(dV, tV.grad.numpy(), rtol=1e-10, atol=1e-12)
    # also equal to the forward restatement's output
    o_cmp, _ = O.compressed_forward(Q, O.compress_kv(K, V, c), c)
    np.testing.assert_allclose(out.detach().numpy(), o_cmp, rtol=1e-12, atol=1e-12)
    # gate gradient vs autograd
    o_sel, _ = O.selected_forward(Q, K, V, O.select_topk(O.make_scores(c, 5), c), c)
    o_sl, _ = O.sliding_forward(Q, K, V, c)
    tt = torch.from_numpy(tau).requires_grad_(True)
    comb = sum(tt[:, i][:, None, None] * torch.from_numpy(x) for i, x in enumerate((o_cmp, o_sel, o_sl)))
    (comb * torch.from_numpy(dO)).sum().backward()
    np.testing.assert_allclose(O.gate_grad((o_cmp, o_sel, o_sl), dO, c), tt.grad.numpy(),
                               rtol=1e-10, atol=1e-12)

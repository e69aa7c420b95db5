"""GPU parity: the CUDA path against the reference's golden fixtures and the
CPU oracle on identical inputs.

Selections are compared bit-exactly; floating-point results within the
north_star tolerances (f64: the reference's own 1e-10/1e-9, f32: rtol 1e-4,
bf16: rtol 2e-2, each with an RMS-scaled absolute floor -- gpu_util.assert_close).
All calls go through the package API -> ctypes -> libfsa_b200.so.
"""

import json

import numpy as np
import pytest
import torch

import paper_2508_18224_b200 as fsa
from paper_2508_18224_b200 import kv_major
from golden_io import FULL_CASES, case, load, round_inputs, stride_of
from gpu_util import DT, assert_close, dev, host
from oracle import fsa_oracle as O

pytestmark = pytest.mark.gpu


def _cfg(kw):
    return fsa.make_config(**kw)


# ---------------------------------------------------------------------------
# K3 top-k selection: bit-exact
# ---------------------------------------------------------------------------

def test_select_topk_golden_kats():
    z = load("selection_kats")
    tags = sorted({k.split("__")[0] for k in z.files})
    for tag in tags:
        kw = json.loads(str(z[tag + "__cfg"]))
        cfg = _cfg(kw)
        c = O.cfg_of(**kw)
        if tag + "__scores" in z.files:
            scores = z[tag + "__scores"]
        else:
            seed, f32 = (int(v) for v in z[tag + "__seed"])
            scores = O.make_scores(c, seed)
            if f32:
                scores = scores.astype(np.float32).astype(np.float64)
        sel = fsa.select_topk_blocks(torch.from_numpy(scores).cuda(), cfg)
        np.testing.assert_array_equal(host(sel.idx), z[tag + "__idx"], err_msg=tag)
        if np.array_equal(scores.astype(np.float32).astype(np.float64), scores):
            sel32 = fsa.select_topk_blocks(torch.from_numpy(scores).float().cuda(), cfg)
            np.testing.assert_array_equal(host(sel32.idx), z[tag + "__idx"], err_msg=tag + " f32")


@pytest.mark.parametrize("kw", [
    dict(N=4096, d_K=8, d_V=8, h=2, h_K=2, B_K=64, T=16),
    dict(N=2048, d_K=8, d_V=8, h=4, h_K=4, B_K=16, T=7),
    dict(N=512, d_K=8, d_V=8, h=1, h_K=1, B_K=4, T=32),
    dict(N=1024, d_K=8, d_V=8, h=1, h_K=1, B_K=8, T=33),
    dict(N=640, d_K=8, d_V=8, h=2, h_K=1, B_K=5, T=1),
])
@pytest.mark.parametrize("sdt", ["f32", "f64"])
def test_select_topk_random_vs_oracle(kw, sdt):
    c = O.cfg_of(**kw)
    rng = np.random.default_rng(kw["N"] + kw["T"])
    scores = rng.standard_normal((c.h_K, c.N, c.b))
    scores[rng.uniform(size=scores.shape) < 0.1] = 0.25  # ties
    scores[rng.uniform(size=scores.shape) < 0.01] = -np.inf
    scores[rng.uniform(size=scores.shape) < 0.01] = np.nan
    if sdt == "f32":
        scores = scores.astype(np.float32).astype(np.float64)
    want = O.select_topk(scores, c)
    t = torch.from_numpy(scores).cuda()
    if sdt == "f32":
        t = t.float()
    got = fsa.select_topk_blocks(t, _cfg(kw))
    np.testing.assert_array_equal(host(got.idx), want)


@pytest.mark.parametrize("kw", [
    dict(N=16384, d_K=8, d_V=8, h=2, h_K=2, B_K=16, T=16),   # b = 1024 (32 candidates / lane)
    dict(N=32768, d_K=8, d_V=8, h=1, h_K=1, B_K=16, T=16),   # b = 2048: streamed rows
    dict(N=8192, d_K=8, d_V=8, h=1, h_K=1, B_K=2, T=32),     # b = 4096
    dict(N=4112, d_K=8, d_V=8, h=1, h_K=1, B_K=4, T=8),      # b = 1028: streamed rows
    dict(N=4800, d_K=8, d_V=8, h=1, h_K=1, B_K=16, T=32),    # b = 300, T = 32
    dict(N=2048, d_K=8, d_V=8, h=1, h_K=1, B_K=64, T=1),     # b = 32, T = 1
])
def test_select_topk_ties_and_specials(kw):
    """Radix-select path (f32): heavy exact ties at the T-th key, +inf
    (ties the own block; wins on index), -0.0 vs +0.0, -inf / NaN."""
    c = O.cfg_of(**kw)
    rng = np.random.default_rng(kw["b"] if "b" in kw else kw["N"])
    scores = np.round(rng.standard_normal((c.h_K, c.N, c.b)) * 2) / 2  # few distinct values
    u = rng.uniform(size=scores.shape)
    scores[u < 0.02] = np.inf
    scores[(u >= 0.02) & (u < 0.05)] = -0.0
    scores[(u >= 0.05) & (u < 0.08)] = 0.0
    scores[(u >= 0.08) & (u < 0.10)] = -np.inf
    scores[(u >= 0.10) & (u < 0.11)] = np.nan
    scores = scores.astype(np.float32).astype(np.float64)
    want = O.select_topk(scores, c)
    got = fsa.select_topk_blocks(torch.from_numpy(scores).float().cuda(), _cfg(kw))
    np.testing.assert_array_equal(host(got.idx), want)


def test_malformed_selection_messages():
    z = load("malformed")
    cfg = _cfg(json.loads(str(z["cfg"])))
    for tag, msg in json.loads(str(z["messages"])).items():
        sel = fsa.SelectionTensor(z["idx_" + tag])
        with pytest.raises(fsa.SelectionError) as exc:
            fsa.validate_selection(sel, cfg)
        assert str(exc.value) == msg, tag
        with pytest.raises(fsa.SelectionError) as exc:
            fsa.build_inverse_index(fsa.SelectionTensor(z["idx_" + tag]), cfg)
        assert str(exc.value) == msg, tag


# ---------------------------------------------------------------------------
# K4 inverse index: bit-exact CSR
# ---------------------------------------------------------------------------

@pytest.mark.parametrize("name", FULL_CASES)
def test_inverse_index_golden(name):
    kw, c, inp, z = case(name)
    cfg = _cfg(kw)
    sel = fsa.SelectionTensor(z["idx"])
    inv = fsa.build_inverse_index(sel, cfg)
    assert fsa.build_inverse_index(sel, cfg) is inv
    np.testing.assert_array_equal(host(inv.offsets).astype(np.int64), z["inv_offsets"])
    np.testing.assert_array_equal(inv.n_valid, z["n_valid"])
    toks = np.concatenate([host(inv.qlist[kh, : int(z["inv_offsets"][kh, -1])]) // c.T
                           for kh in range(c.h_K)])
    np.testing.assert_array_equal(toks, z["inv_tok"])
    back = fsa.selection_from_inverse(inv, cfg)
    np.testing.assert_array_equal(host(back.idx), z["idx"])


def test_inverse_large_vs_oracle():
    kw = dict(N=32768, d_K=8, d_V=8, h=2, h_K=2, B_K=64, T=16)
    c = O.cfg_of(**kw)
    idx = O.select_topk(O.make_scores(c, 3), c)
    want = O.build_inverse(idx, c)
    inv = fsa.build_inverse_index(fsa.SelectionTensor(idx), _cfg(kw))
    np.testing.assert_array_equal(host(inv.offsets).astype(np.int64), want.offsets)
    for kh in range(c.h_K):
        ql = host(inv.qlist[kh, : want.offsets[kh, -1]])
        np.testing.assert_array_equal(ql // c.T, want.tok[kh])
        np.testing.assert_array_equal(ql % c.T, want.slot[kh])


# ---------------------------------------------------------------------------
# selected attention forward / backward
# ---------------------------------------------------------------------------

def _dtype_for(z, requested):
    return requested


@pytest.mark.parametrize("name", FULL_CASES)
def test_selected_forward_golden(name):
    kw, c, inp, z = case(name)
    cfg = _cfg(kw)
    st = stride_of(z)
    dt = "f64" if inp["round_to"] in ("None", "f64") else ("f32" if inp["round_to"] == "f32" else "bf16")
    for run_dt in sorted({"f64", dt}):
        tdt = DT[run_dt]
        Q, K, V = (dev(inp[k], tdt) for k in "QKV")
        sel = fsa.SelectionTensor(z["idx"])
        res, meter = kv_major.selected_forward(Q, K, V, sel, cfg)
        tol_dt = run_dt if run_dt != "f64" or z["out"].dtype == np.float64 else "f32"
        assert_close(host(res.out)[::st], z["out"], tol_dt, f"{name} out {run_dt}")
        assert_close(host(res.lse), z["lse"], tol_dt if tol_dt != "bf16" else "f32", f"{name} lse {run_dt}")
        want = json.loads(str(z["meter_fwd"]))
        got = {k: dict(bytes_loaded=p.bytes_loaded, bytes_stored=p.bytes_stored, flops=p.flops,
                       task_count=p.task_count, inner_iterations=p.inner_iterations)
               for k, p in meter.phases.items()}
        assert got == want


@pytest.mark.parametrize("name", ["case_kv_small", "case_rect_dims", "case_g8_bk1", "case_unit",
                                  "case_tiny_fp32"])
def test_phase_api_golden(name):
    kw, c, inp, z = case(name)
    cfg = _cfg(kw)
    st = stride_of(z)
    Q, K, V = (dev(inp[k]) for k in "QKV")
    tol = "f64" if z["out"].dtype == np.float64 else "f32"
    sel = fsa.SelectionTensor(z["idx"])
    stats = kv_major.compute_softmax_stats(Q, K, sel, cfg)
    assert_close(host(stats.m), z["m"], tol, "m")
    assert_close(host(stats.l), z["l"], tol, "l")
    sh = kv_major.compute_softmax_stats(Q, K, sel, cfg, shared_max=True)
    assert_close(host(sh.m), z["m_sh"], tol, "m_sh")
    assert_close(host(sh.l), z["l_sh"], tol, "l_sh")
    inv = fsa.build_inverse_index(sel, cfg)
    buf = kv_major.block_pass_forward(Q, K, V, inv, stats, cfg)
    res = kv_major.reduce_forward(buf, inv, stats, cfg)
    assert_close(host(res.out)[::st], z["out"], tol, "reduce out")
    res_sh = kv_major.reduce_forward(kv_major.block_pass_forward(Q, K, V, inv, sh, cfg), inv, sh, cfg)
    assert_close(host(res_sh.out)[::st], z["out_sh"], tol, "shared-max out")


@pytest.mark.parametrize("kw", [
    dict(N=4096, d_K=128, d_V=128, h=8, h_K=2, B_K=64, T=16),   # GQA 4 (Llama-shaped)
    dict(N=2048, d_K=128, d_V=128, h=5, h_K=1, B_K=64, T=16),   # GQA 5 (Qwen3-shaped)
])
def test_phase_api_tensor_core_bf16(kw):
    """compute_softmax_stats / block_pass_forward (kv_major.py:105-204) on the
    tcgen05 K5 kernel in STATS / GLOBAL mode for bf16 d = 128, then
    reduce_forward, against the oracle on the bf16-rounded inputs: m, l in the
    fp32 tolerance (S products are exact in fp32 accumulation), out in bf16's."""
    c = O.cfg_of(**kw)
    cfg = _cfg(kw)
    Q, K, V = (round_inputs(x, "bf16") for x in O.make_qkv(c, 9))
    idx = O.select_topk(O.make_scores(c, 9), c)
    tQ, tK, tV = (dev(x, torch.bfloat16) for x in (Q, K, V))
    sel = fsa.SelectionTensor(idx)
    inv = fsa.build_inverse_index(sel, cfg)
    for shared in (False, True):
        want = O.softmax_stats(Q, K, idx, c, shared_max=shared)
        stats = kv_major.compute_softmax_stats(tQ, tK, sel, cfg, shared_max=shared)
        assert_close(host(stats.m), want.m, "f32", f"tc m shared={shared}")
        assert_close(host(stats.l), want.l, "f32", f"tc l shared={shared}")
        buf = kv_major.block_pass_forward(tQ, tK, tV, inv, stats, cfg)
        res = kv_major.reduce_forward(buf, inv, stats, cfg)
        regions = O.block_pass(Q, K, V, idx, want, c)
        want_out, want_lse = O.reduce_regions(regions, want, c, inv=O.build_inverse(idx, c))
        assert_close(host(res.out), want_out, "bf16", f"tc phase out shared={shared}")
        assert_close(host(res.lse), want_lse, "f32", f"tc phase lse shared={shared}")
        # a GLOBAL row of one (head, block) task against the reference region
        j, i = cfg.h - 1, 3
        rows = O.build_inverse(idx, c).queries(j // c.g, i)
        assert_close(host(buf.rows[j][i]), regions[j][i], "bf16", "tc GLOBAL region")


@pytest.mark.parametrize("name", FULL_CASES)
def test_selected_backward_golden(name):
    kw, c, inp, z = case(name)
    cfg = _cfg(kw)
    st = stride_of(z)
    tdt = torch.float64
    Q, K, V, dO = (dev(inp[k], tdt) for k in ("Q", "K", "V", "dOut"))
    dQ, dK, dV, meter = kv_major.selected_backward(Q, K, V, fsa.SelectionTensor(z["idx"]), dO, cfg)
    tol = "f64" if z["dQ"].dtype == np.float64 else "f32"
    for got, key in ((dQ, "dQ"), (dK, "dK"), (dV, "dV")):
        assert_close(host(got)[::st], z[key], tol, f"{name} {key}", grad=True)
    want = json.loads(str(z["meter_bwd"]))
    got = {k: dict(bytes_loaded=p.bytes_loaded, bytes_stored=p.bytes_stored, flops=p.flops,
                   task_count=p.task_count, inner_iterations=p.inner_iterations)
           for k, p in meter.phases.items()}
    assert got == want


@pytest.mark.parametrize("run_dt", ["f32", "bf16"])
@pytest.mark.parametrize("kw", [
    dict(N=2048, d_K=64, d_V=64, h=4, h_K=1, B_K=64, T=8, W=128),       # BASELINE cfg 1 (tiny)
    dict(N=4096, d_K=128, d_V=128, h=8, h_K=2, B_K=64, T=16, W=512),    # Llama-shaped, short
    dict(N=2048, d_K=128, d_V=128, h=5, h_K=1, B_K=64, T=16, W=512),    # GQA 5 (Qwen3)
    dict(N=2048, d_K=128, d_V=128, h=2, h_K=2, B_K=64, T=16, W=512),    # GQA 1
    dict(N=16384, d_K=128, d_V=128, h=8, h_K=4, B_K=64, T=16, W=512),   # >> tasks than SMs
])
def test_selected_fwd_bwd_vs_oracle(kw, run_dt):
    """Oracle fed the dtype-rounded inputs, compared in that dtype's tolerance."""
    c = O.cfg_of(**kw)
    cfg = _cfg(kw)
    Q, K, V = (round_inputs(x, run_dt) for x in O.make_qkv(c, 5))
    dO = round_inputs(O.make_dout(c, 5), run_dt)
    idx = O.select_topk(O.make_scores(c, 5), c)
    want_out, want_lse = O.selected_forward(Q, K, V, idx, c)
    tdt = DT[run_dt]
    tQ, tK, tV, tdO = (dev(x, tdt) for x in (Q, K, V, dO))
    sel = fsa.SelectionTensor(idx)
    res, _ = kv_major.selected_forward(tQ, tK, tV, sel, cfg)
    assert_close(host(res.out), want_out, run_dt, "out")
    assert_close(host(res.lse), want_lse, "f32" if run_dt == "bf16" else run_dt, "lse")
    want = O.selected_backward(Q, K, V, idx, dO, c)
    got = kv_major.selected_backward(tQ, tK, tV, sel, tdO, cfg)
    for g_, w_, name in zip(got[:3], want, ("dQ", "dK", "dV")):
        assert_close(host(g_), w_, run_dt, name, grad=True)


@pytest.mark.parametrize("chunk", [256, 1024, 4096])
def test_token_chunked_plan_vs_oracle(chunk, monkeypatch):
    """Token-chunked work plan (common.cuh): tasks are (kv head, chunk, block)
    sub-lists.  Forced small chunks give the same forward bit for bit as a
    single chunk, and match the oracle (kv_major.py:245-261)."""
    kw = dict(N=8192, d_K=128, d_V=128, h=10, h_K=2, B_K=64, T=16, W=512)
    c = O.cfg_of(**kw)
    cfg = _cfg(kw)
    Q, K, V = (round_inputs(x, "bf16") for x in O.make_qkv(c, 7))
    idx = O.select_topk(O.make_scores(c, 7), c)
    tQ, tK, tV = (dev(x, torch.bfloat16) for x in (Q, K, V))
    monkeypatch.setenv("FSA_CHUNK_TOKENS", str(1 << 30))
    one, _ = kv_major.selected_forward(tQ, tK, tV, fsa.SelectionTensor(idx), cfg)
    monkeypatch.setenv("FSA_CHUNK_TOKENS", str(chunk))
    res, _ = kv_major.selected_forward(tQ, tK, tV, fsa.SelectionTensor(idx), cfg)
    assert torch.equal(res.out, one.out) and torch.equal(res.lse, one.lse)
    want_out, want_lse = O.selected_forward(Q, K, V, idx, c)
    assert_close(host(res.out), want_out, "bf16", "out")
    assert_close(host(res.lse), want_lse, "f32", "lse")


def test_acceptance_sweep_golden():
    z = load("acceptance_sweep")
    for n in range(int(z["count"])):
        p = f"s{n}__"
        kw = json.loads(str(z[p + "cfg"]))
        c = O.cfg_of(**kw)
        cfg = _cfg(kw)
        seed = int(z[p + "seed"])
        Q, K, V = (dev(x) for x in O.make_qkv(c, seed))
        sel = fsa.select_topk_blocks(torch.from_numpy(O.make_scores(c, seed)).cuda(), cfg)
        np.testing.assert_array_equal(host(sel.idx), z[p + "idx"])
        res, _ = kv_major.selected_forward(Q, K, V, sel, cfg)
        assert np.abs(host(res.out) - z[p + "out"]).max() <= 1e-10
        g = kv_major.selected_backward(Q, K, V, sel, dev(O.make_dout(c, seed)), cfg)
        for got, key in zip(g[:3], ("dQ", "dK", "dV")):
            assert np.abs(host(got) - z[p + key]).max() <= 1e-9


def test_bit_identical_repeats_and_task_order():
    kw = dict(N=1024, d_K=128, d_V=128, h=8, h_K=2, B_K=64, T=8)
    c = O.cfg_of(**kw)
    cfg = _cfg(kw)
    Q, K, V = (dev(x, torch.bfloat16) for x in O.make_qkv(c, 1))
    sel = fsa.SelectionTensor(O.select_topk(O.make_scores(c, 1), c))
    a, _ = kv_major.selected_forward(Q, K, V, sel, cfg)
    b, _ = kv_major.selected_forward(Q, K, V, sel, cfg,
                                     task_order=np.random.default_rng(0).permutation(cfg.h * cfg.b))
    assert torch.equal(a.out, b.out) and torch.equal(a.lse, b.lse)
    dO = dev(O.make_dout(c, 1), torch.bfloat16)
    g1 = kv_major.selected_backward(Q, K, V, sel, dO, cfg)
    g2 = kv_major.selected_backward(Q, K, V, sel, dO, cfg)
    for x, y in zip(g1[:3], g2[:3]):
        assert torch.equal(x, y)
    with pytest.raises(ValueError, match="task_order must be a permutation"):
        kv_major.selected_forward(Q, K, V, sel, cfg, task_order=[0, 0, 1])


# ---------------------------------------------------------------------------
# branches
# ---------------------------------------------------------------------------

@pytest.mark.parametrize("name", FULL_CASES)
def test_branches_golden(name):
    kw, c, inp, z = case(name)
    cfg = _cfg(kw)
    st = stride_of(z)
    tol = "f64" if z["out"].dtype == np.float64 else "f32"
    Q, K, V, dO = (dev(inp[k]) for k in ("Q", "K", "V", "dOut"))
    cmp = fsa.compress_kv(K, V, cfg)
    for key in ("K_cmp", "V_cmp", "K_prefix", "V_prefix"):
        assert_close(host(getattr(cmp, key)), z[key], tol, key)
    sc = fsa.importance_scores_from_compressed(Q, cmp.K_cmp, cfg)
    assert_close(host(sc)[:, ::st], z["scores_cmp"], tol, "scores")
    res, sc2 = fsa.compressed_attention_forward(Q, cmp, cfg, scores_out=True)
    assert_close(host(res.out)[::st], z["cmp_out"], tol, "cmp out")
    assert_close(host(res.lse), z["cmp_lse"], tol, "cmp lse")
    assert_close(host(sc2)[:, ::st], z["scores_cmp"], tol, "fused scores")
    if "slide_out" in z.files:
        sl = fsa.sliding_attention_forward(Q, K, V, cfg)
        assert_close(host(sl.out)[::st], z["slide_out"], tol, "slide out")
        assert_close(host(sl.lse), z["slide_lse"], tol, "slide lse")
        g = fsa.sliding_attention_backward(Q, K, V, dO, cfg)
        for got, key in zip(g, ("slide_dQ", "slide_dK", "slide_dV")):
            assert_close(host(got)[::st], z[key], tol, key)
        sel_res, _ = kv_major.selected_forward(Q, K, V, fsa.SelectionTensor(z["idx"]), cfg)
        comb = fsa.gated_combine((res, sel_res, sl), torch.from_numpy(inp["tau"]).cuda(), cfg)
        assert_close(host(comb.out)[::st], z["comb_out"], tol, "combined")
        assert torch.isnan(comb.lse).all()


def test_gate_errors():
    kw = dict(N=32, d_K=8, d_V=8, h=4, h_K=2, B_K=8, T=2)
    cfg = _cfg(kw)
    c = O.cfg_of(**kw)
    Q, K, V = (dev(x) for x in O.make_qkv(c, 12))
    r = fsa.sliding_attention_forward(Q, K, V, cfg)
    bad = np.zeros((cfg.N, 3))
    bad[0, 0] = 1.5
    with pytest.raises(ValueError, match="gate values"):
        fsa.gated_combine((r, r, r), bad, cfg)
    with pytest.raises(ValueError, match="expected exactly three"):
        fsa.gated_combine((r, r), np.zeros((cfg.N, 3)), cfg)


# ---------------------------------------------------------------------------
# full NSA step (the bench workload) vs the oracle composition
# ---------------------------------------------------------------------------

@pytest.mark.parametrize("run_dt", ["f32", "bf16"])
def test_nsa_step_vs_oracle(run_dt):
    kw = dict(N=2048, d_K=128, d_V=128, h=8, h_K=2, B_K=64, T=8, W=256)
    c = O.cfg_of(**kw)
    cfg = _cfg(kw)
    Q, K, V = (round_inputs(x, run_dt) for x in O.make_qkv(c, 9))
    dO = round_inputs(O.make_dout(c, 9), run_dt)
    tau = O.make_gates(c, 9)
    tdt = DT[run_dt]
    q, k, v, do = (dev(x, tdt).permute(0, 2, 1).contiguous() for x in (Q, K, V, dO))
    acc = torch.float32
    out, ctx = fsa.nsa_forward(q, k, v, torch.from_numpy(tau).to("cuda", acc), cfg, keep_scores=True)
    # selection parity on the GPU's own scores (SURVEY 8(c) score-path caveat)
    scores = host(ctx.scores).astype(np.float64)
    idx = O.select_topk(scores, c)
    np.testing.assert_array_equal(host(ctx.sel.idx), idx)
    cmp = O.compress_kv(K, V, c)
    # the fused pipeline fills the blocks top-k can read: i < own block
    causal = np.arange(c.b)[None, None, :] < (np.arange(c.N) // c.B_K)[None, :, None]
    causal = np.broadcast_to(causal, scores.shape)
    assert_close(scores[causal], O.importance_scores(Q, cmp.K_cmp, c)[causal],
                 "f32" if run_dt == "f32" else "bf16", "scores")
    o_cmp, _ = O.compressed_forward(Q, cmp, c)
    o_sel, _ = O.selected_forward(Q, K, V, idx, c)
    o_sl, _ = O.sliding_forward(Q, K, V, c)
    want, _ = O.gated_combine((o_cmp, o_sel, o_sl), tau, c)
    assert_close(host(out.permute(0, 2, 1)), want, run_dt, "combined")
    dQ, dK, dV = fsa.nsa_backward(ctx, do)
    gs = O.selected_backward(Q, K, V, idx, dO * tau[:, 1][:, None, None], c)
    gl = O.sliding_backward(Q, K, V, dO * tau[:, 2][:, None, None], c)
    for got, a, b, name in zip((dQ, dK, dV), gs, gl, ("dQ", "dK", "dV")):
        assert_close(host(got.permute(0, 2, 1)), a + b, run_dt, name, grad=True)
    # full NSA backward: + the compressed branch (no reference backward: the
    # float64 oracle, pinned to autograd) and the gate gradient
    fQ, fK, fV, dtau = fsa.nsa_backward(ctx, do, full=True)
    gc = O.compressed_backward(Q, K, V, dO * tau[:, 0][:, None, None], c)
    for got, a, b, cc, name in zip((fQ, fK, fV), gs, gl, gc, ("dQ", "dK", "dV")):
        assert_close(host(got.permute(0, 2, 1)), a + b + cc, run_dt, name + " (full)", grad=True)
    want_tau = O.gate_grad((o_cmp, o_sel, o_sl), dO, c)
    assert_close(host(dtau), want_tau, run_dt, "dtau", grad=True)


@pytest.mark.parametrize("kw,run_dt", [
    (dict(N=512, d_K=16, d_V=24, h=4, h_K=2, B_K=16, T=4, W=64), "f64"),
    (dict(N=1000, d_K=32, d_V=32, h=6, h_K=3, B_K=8, T=5, W=40), "f32"),
    # tensor-core path (bf16, d = 128): K8 compressed mode + query-outer dQ
    (dict(N=4096, d_K=128, d_V=128, h=8, h_K=2, B_K=32, T=8, W=256), "bf16"),
    (dict(N=2048, d_K=128, d_V=128, h=7, h_K=1, B_K=32, T=6, W=128), "bf16"),
    (dict(N=4800, d_K=128, d_V=128, h=4, h_K=4, B_K=16, T=8, W=64), "bf16"),
])
def test_compressed_backward_vs_oracle(kw, run_dt):
    """fsa_cmp_bwd (generic kernels) at the reference's own tolerances for f64."""
    c = O.cfg_of(**kw)
    cfg = _cfg(kw)
    Q, K, V = (round_inputs(x, run_dt) for x in O.make_qkv(c, 13))
    dO = round_inputs(O.make_dout(c, 13), run_dt)
    tau = O.make_gates(c, 13)
    tdt = DT[run_dt]
    q, k, v, do = (dev(x, tdt).permute(0, 2, 1).contiguous() for x in (Q, K, V, dO))
    acc = torch.float64 if run_dt == "f64" else torch.float32
    out, ctx = fsa.nsa_forward(q, k, v, torch.from_numpy(tau).to("cuda", acc), cfg)
    fQ, fK, fV, dtau = fsa.nsa_backward(ctx, do, full=True)
    idx = host(ctx.sel.idx)
    gs = O.selected_backward(Q, K, V, idx, dO * tau[:, 1][:, None, None], c)
    gl = O.sliding_backward(Q, K, V, dO * tau[:, 2][:, None, None], c)
    gc = O.compressed_backward(Q, K, V, dO * tau[:, 0][:, None, None], c)
    for got, a, b, cc, name in zip((fQ, fK, fV), gs, gl, gc, ("dQ", "dK", "dV")):
        assert_close(host(got.permute(0, 2, 1)), a + b + cc, run_dt, name, grad=True)
    cmp = O.compress_kv(K, V, c)
    outs = (O.compressed_forward(Q, cmp, c)[0], O.selected_forward(Q, K, V, idx, c)[0],
            O.sliding_forward(Q, K, V, c)[0])
    assert_close(host(dtau), O.gate_grad(outs, dO, c), run_dt, "dtau", grad=True)


# ---------------------------------------------------------------------------
# tensor-core sliding-window and compressed branches (bf16, d = 128)
# ---------------------------------------------------------------------------

@pytest.mark.parametrize("kw", [
    dict(N=2048, d_K=128, d_V=128, h=8, h_K=2, B_K=64, T=8, W=512),
    dict(N=1280, d_K=128, d_V=128, h=2, h_K=2, B_K=64, T=8, W=100),     # g=1, W not /64
    dict(N=1024, d_K=128, d_V=128, h=16, h_K=2, B_K=32, T=8, W=64),     # g=8, B_K=32
    dict(N=960, d_K=128, d_V=128, h=5, h_K=1, B_K=64, T=4, W=300),      # g=5: scores unfused
])
def test_tc_window_branches_vs_oracle(kw):
    c = O.cfg_of(**kw)
    cfg = _cfg(kw)
    Q, K, V = (round_inputs(x, "bf16") for x in O.make_qkv(c, 21))
    tQ, tK, tV = (dev(x, torch.bfloat16) for x in (Q, K, V))
    sl = fsa.sliding_attention_forward(tQ, tK, tV, cfg)
    want_o, want_l = O.sliding_forward(Q, K, V, c)
    assert_close(host(sl.out), want_o, "bf16", "slide out")
    assert_close(host(sl.lse), want_l, "f32", "slide lse")
    cmp = fsa.compress_kv(tK, tV, cfg)
    res, sc = fsa.compressed_attention_forward(tQ, cmp, cfg, scores_out=True)
    ocmp = O.compress_kv(K, V, c)
    # the tensor-core path reads bf16-rounded pooled rows: feed the oracle the same
    kc16 = round_inputs(host(cmp.K_cmp).astype(np.float64), "bf16")
    vc16 = round_inputs(host(cmp.V_cmp).astype(np.float64), "bf16")
    want_o, want_l = O.compressed_forward(Q, O.Compressed(kc16, vc16, ocmp.K_prefix, ocmp.V_prefix), c)
    assert_close(host(res.out), want_o, "bf16", "cmp out")
    assert_close(host(res.lse), want_l, "f32" if False else "bf16", "cmp lse")
    assert_close(host(sc), O.importance_scores(Q, host(cmp.K_cmp).astype(np.float64), c), "f32",
                 "scores")
    # fused scores of the pipeline: every block a token's top-k reads
    out, ctx = fsa.nsa_forward(tQ.permute(0, 2, 1).contiguous(), tK.permute(0, 2, 1).contiguous(),
                               tV.permute(0, 2, 1).contiguous(),
                               torch.full((cfg.N, 3), 1.0 / 3, device="cuda"), cfg, keep_scores=True)
    fused = host(ctx.scores)
    full = host(sc)
    causal = np.arange(c.b)[None, None, :] < (np.arange(c.N) // c.B_K)[None, :, None]
    causal = np.broadcast_to(causal, fused.shape)
    assert_close(fused[causal], O.importance_scores(Q, host(cmp.K_cmp).astype(np.float64), c)[causal],
                 "bf16", "fused scores")
    assert full.shape == fused.shape


@pytest.mark.parametrize("kw", [
    dict(N=2048, d_K=128, d_V=128, h=8, h_K=2, B_K=64, T=8, W=512),
    dict(N=1280, d_K=128, d_V=128, h=2, h_K=2, B_K=64, T=8, W=100),
    dict(N=8192, d_K=128, d_V=128, h=8, h_K=4, B_K=64, T=8, W=512),     # many tasks per CTA
])
def test_tc_sliding_backward_vs_oracle(kw):
    c = O.cfg_of(**kw)
    cfg = _cfg(kw)
    Q, K, V = (round_inputs(x, "bf16") for x in O.make_qkv(c, 22))
    dO = round_inputs(O.make_dout(c, 22), "bf16")
    tQ, tK, tV, tdO = (dev(x, torch.bfloat16) for x in (Q, K, V, dO))
    got = fsa.sliding_attention_backward(tQ, tK, tV, tdO, cfg)
    want = O.sliding_backward(Q, K, V, dO, c)
    for g_, w_, name in zip(got, want, ("dQ", "dK", "dV")):
        assert_close(host(g_), w_, "bf16", name, grad=True)


# ---------------------------------------------------------------------------
# NSA query-major baseline (query_major.py:45-69): same outputs as the FSA
# kv-major path / the oracle, reference meter closed form
# ---------------------------------------------------------------------------

@pytest.mark.parametrize("kw,run_dt", [
    (dict(N=512, d_K=32, d_V=48, h=8, h_K=2, B_K=16, T=4), "f64"),
    (dict(N=1024, d_K=64, d_V=64, h=4, h_K=4, B_K=32, T=6), "f32"),
    (dict(N=2048, d_K=128, d_V=128, h=16, h_K=2, B_K=64, T=8), "bf16"),
    (dict(N=1024, d_K=128, d_V=128, h=7, h_K=1, B_K=64, T=5), "bf16"),
    (dict(N=4096, d_K=128, d_V=128, h=8, h_K=2, B_K=64, T=16), "bf16"),    # tcgen05, g = 4
    (dict(N=2048, d_K=128, d_V=128, h=5, h_K=1, B_K=64, T=16), "bf16"),    # g = 5
    (dict(N=2048, d_K=128, d_V=128, h=2, h_K=2, B_K=64, T=16), "bf16"),    # g = 1
    (dict(N=1024, d_K=128, d_V=128, h=32, h_K=2, B_K=64, T=11), "bf16"),   # g = 16: N side 16
])
def test_query_major_forward_vs_oracle(kw, run_dt):
    c = O.cfg_of(**kw)
    cfg = _cfg(kw)
    Q, K, V = (round_inputs(x, run_dt) for x in O.make_qkv(c, 31))
    idx = O.select_topk(O.make_scores(c, 31), c)
    tq, tk, tv = (dev(x, DT[run_dt]) for x in (Q, K, V))
    res, meter = fsa.query_major.selected_forward(tq, tk, tv, fsa.SelectionTensor(idx), cfg)
    want_o, want_l = O.selected_forward(Q, K, V, idx, c)
    assert_close(host(res.out), want_o, run_dt, "qm out")
    assert_close(host(res.lse), want_l, "f64" if run_dt == "f64" else "f32", "qm lse")
    ph = meter.phases["query_major"]
    steps = int((idx != -1).sum())
    pad = max(c.g, c.min_tile)
    assert ph.task_count == c.h_K * c.N and ph.inner_iterations == steps
    assert ph.flops == steps * 2 * pad * c.B_K * (c.d_K + c.d_V)


@pytest.mark.parametrize("kw,run_dt", [
    (dict(N=512, d_K=32, d_V=48, h=8, h_K=2, B_K=16, T=4), "f64"),
    (dict(N=1056, d_K=64, d_V=64, h=4, h_K=4, B_K=32, T=6), "f32"),
    (dict(N=2048, d_K=128, d_V=128, h=16, h_K=2, B_K=64, T=8), "bf16"),
    (dict(N=1024, d_K=128, d_V=128, h=7, h_K=1, B_K=64, T=5), "bf16"),
])
def test_query_major_backward_vs_oracle(kw, run_dt):
    """query_major.py:72-115: same gradients as the oracle, reference meter."""
    c = O.cfg_of(**kw)
    cfg = _cfg(kw)
    Q, K, V = (round_inputs(x, run_dt) for x in O.make_qkv(c, 37))
    dO = round_inputs(O.make_dout(c, 37), run_dt)
    idx = O.select_topk(O.make_scores(c, 37), c)
    tq, tk, tv, tdo = (dev(x, DT[run_dt]) for x in (Q, K, V, dO))
    dQ, dK, dV, meter = fsa.query_major.selected_backward(tq, tk, tv, fsa.SelectionTensor(idx), tdo, cfg)
    want = O.selected_backward(Q, K, V, idx, dO, c)
    for g_, w_, name in zip((dQ, dK, dV), want, ("dQ", "dK", "dV")):
        assert_close(host(g_), w_, run_dt, "qm " + name, grad=True)
    ph = meter.phases["query_major"]
    steps = int((idx != -1).sum())
    pad = max(c.g, c.min_tile)
    assert ph.task_count == c.h_K * c.N and ph.inner_iterations == steps
    assert ph.flops == steps * 2 * pad * c.B_K * (4 * c.d_K + 3 * c.d_V)


def test_cli_bench_csv(tmp_path):
    """python -m paper_2508_18224_b200 bench: the reference's CSV columns, one row per phase."""
    import csv as _csv

    from paper_2508_18224_b200 import cli
    cfgf = tmp_path / "tiny.cfg"
    cfgf.write_text("N = 1024\nd_K = 64\nd_V = 64\nh = 4\nh_K = 1\nB_K = 64\nT = 8\n")
    out = tmp_path / "bench.csv"
    assert cli.main(["bench", "--config", str(cfgf), "--repeat", "2", "--dtype", "f32",
                     "--csv", str(out)]) == 0
    rows = list(_csv.DictReader(open(out)))
    assert tuple(rows[0].keys()) == cli.BENCH_COLUMNS
    phases = {(r["engine"], r["phase"]) for r in rows}
    assert {("kv_major", "stats"), ("kv_major", "block_pass"), ("kv_major", "reduce"),
            ("query_major", "forward")} <= phases
    assert all(float(r["median_s"]) > 0 for r in rows)


@pytest.mark.parametrize("full", [False, True])
def test_window_backward_partial_tile_repeatable(full):
    """g = 7: the TMA boxes fill 126 of a tile's 128 rows.  The two spare rows
    must be zero, or stale shared memory (NaN patterns) leaks into dK / dV
    through 0 * NaN (seen as rare NaN runs before the fix): 30 reruns must be
    finite and bit-identical."""
    N, h, hk = 2048, 7, 1
    cfg = fsa.make_config(N=N, d_K=128, d_V=128, h=h, h_K=hk, B_K=32, T=6, W=128)
    g = torch.Generator(device="cuda").manual_seed(3)
    mk = lambda *s: torch.randn(*s, device="cuda", dtype=torch.bfloat16, generator=g)  # noqa: E731
    q, k, v, do = mk(N, h, 128), mk(N, hk, 128), mk(N, hk, 128), mk(N, h, 128)
    tau = torch.rand(N, 3, device="cuda", generator=g)
    ref = None
    for _ in range(30):
        _, ctx = fsa.nsa.nsa_forward(q, k, v, tau, cfg)
        got = [x.clone() for x in fsa.nsa.nsa_backward(ctx, do, full=full)]
        assert all(bool(torch.isfinite(x).all()) for x in got)
        if ref is None:
            ref = got
        else:
            assert all(torch.equal(a, b) for a, b in zip(got, ref))


def test_query_head_split_matches_unsharded():
    """parallel.QueryShard on the device: the two ranks of a kv head (simulated
    in one process) reproduce the unsharded step; dK / dV are the sum of the
    ranks' partials (the all_reduce of the multi-GPU run)."""
    from paper_2508_18224_b200 import parallel

    cfg = fsa.make_config(N=4096, d_K=128, d_V=128, h=7, h_K=1, B_K=64, T=8, W=256)
    g = torch.Generator(device="cuda").manual_seed(11)
    mk = lambda *s: torch.randn(*s, device="cuda", dtype=torch.bfloat16, generator=g)  # noqa: E731
    q, k, v, do = mk(cfg.N, 7, 128), mk(cfg.N, 1, 128), mk(cfg.N, 1, 128), mk(cfg.N, 7, 128)
    tau = torch.rand(cfg.N, 3, device="cuda", generator=g)
    out, ctx = fsa.nsa.nsa_forward(q, k, v, tau, cfg)
    dQ, dK, dV = fsa.nsa.nsa_backward(ctx, do)
    parts = []
    for rank in range(2):
        sh = parallel.shard_plan(cfg, rank, 2)
        qg, kk, vv, dd = parallel.query_shard_inputs(sh, q, k, v, do)
        parts.append(parallel.query_shard_step(sh, qg, kk, vv, tau, dd))
    o2 = torch.cat([p[0] for p in parts], 1)
    dq2 = torch.cat([p[1] for p in parts], 1)
    dk2, dv2 = parts[0][2] + parts[1][2], parts[0][3] + parts[1][3]
    assert torch.allclose(o2.float(), out.float(), rtol=1e-2, atol=1e-2)
    for got, ref in ((dq2, dQ), (dk2, dK), (dv2, dV)):
        err = (got - ref).abs().max().item()
        assert err <= 1e-3 * ref.abs().max().item(), err


# NSA step on the tensor-core path over group sizes / windows / budgets the
# BASELINE shapes do not reach (partial items, windows not a multiple of 64,
# T = 1, g = 3, 6, 16, several kv heads): out, dQ, dK, dV, dtau vs the oracle.
@pytest.mark.parametrize("kw", [
    dict(N=1536, d_K=128, d_V=128, h=6, h_K=2, B_K=64, T=1, W=100),
    dict(N=1024, d_K=128, d_V=128, h=16, h_K=1, B_K=64, T=16, W=700),
    dict(N=3072, d_K=128, d_V=128, h=9, h_K=3, B_K=64, T=5, W=64),
    dict(N=1088, d_K=128, d_V=128, h=6, h_K=1, B_K=64, T=3, W=1),
    dict(N=1088, d_K=128, d_V=128, h=2, h_K=2, B_K=64, T=4, W=333),
    dict(N=512, d_K=128, d_V=128, h=128, h_K=1, B_K=64, T=4, W=128),
    # T > 32 (the dQ reduce of the tensor-core backward at T in (32, b])
    dict(N=4096, d_K=128, d_V=128, h=8, h_K=2, B_K=64, T=48, W=256),
    dict(N=4160, d_K=128, d_V=128, h=5, h_K=1, B_K=64, T=64, W=512),
])
def test_nsa_step_shapes_vs_oracle(kw):
    _nsa_step_vs_oracle(kw)


# seeded random shapes: group sizes 2..12, budgets 1..24, windows 1..900, N up to 3K,
# B_K 64 (tensor-core path) or 32 / 16 (SIMT path)
def _fuzz_shapes(n=6, seed=2026):
    rng = np.random.default_rng(seed)
    out = []
    for _ in range(n):
        B_K = int(rng.choice([64, 64, 64, 32, 16]))
        b = int(rng.integers(4, 3072 // B_K + 1))
        h_K = int(rng.integers(1, 4))
        g = int(rng.integers(2, 13))
        out.append(dict(N=b * B_K, d_K=128, d_V=128, h=g * h_K, h_K=h_K, B_K=B_K,
                        T=int(rng.integers(1, min(24, b) + 1)), W=int(rng.integers(1, 900))))
    return out


@pytest.mark.parametrize("kw", _fuzz_shapes())
def test_nsa_step_fuzz_vs_oracle(kw):
    _nsa_step_vs_oracle(kw)


def _nsa_step_vs_oracle(kw):
    c = O.cfg_of(**kw)
    cfg = _cfg(kw)
    Q, K, V = (round_inputs(x, "bf16") for x in O.make_qkv(c, 21))
    dO = round_inputs(O.make_dout(c, 21), "bf16")
    tau = O.make_gates(c, 21)
    q, k, v, do = (dev(x, torch.bfloat16).permute(0, 2, 1).contiguous() for x in (Q, K, V, dO))
    out, ctx = fsa.nsa_forward(q, k, v, torch.from_numpy(tau).to("cuda", torch.float32), cfg, keep_scores=True)
    idx = O.select_topk(host(ctx.scores).astype(np.float64), c)
    np.testing.assert_array_equal(host(ctx.sel.idx), idx)
    cmp = O.compress_kv(K, V, c)
    outs = (O.compressed_forward(Q, cmp, c)[0], O.selected_forward(Q, K, V, idx, c)[0],
            O.sliding_forward(Q, K, V, c)[0])
    want, _ = O.gated_combine(outs, tau, c)
    assert_close(host(out.permute(0, 2, 1)), want, "bf16", "combined")
    fQ, fK, fV, dtau = fsa.nsa_backward(ctx, do, full=True)
    gs = O.selected_backward(Q, K, V, idx, dO * tau[:, 1][:, None, None], c)
    gl = O.sliding_backward(Q, K, V, dO * tau[:, 2][:, None, None], c)
    gc = O.compressed_backward(Q, K, V, dO * tau[:, 0][:, None, None], c)
    for got, a, b, cc, name in zip((fQ, fK, fV), gs, gl, gc, ("dQ", "dK", "dV")):
        assert_close(host(got.permute(0, 2, 1)), a + b + cc, "bf16", name, grad=True)
    assert_close(host(dtau), O.gate_grad(outs, dO, c), "bf16", "dtau", grad=True)


def test_selection_vs_oracle_fp64_scores_near_ties():
    """SURVEY 8(c) score-path caveat: with the oracle's OWN float64 scores (not
    the GPU's fp32 ones) a few rows may select differently; every such row
    must be a near-tie -- each block in the symmetric difference scores within
    the row's GPU-vs-oracle score error of the T-th best score."""
    kw = dict(N=8192, d_K=128, d_V=128, h=8, h_K=2, B_K=64, T=16, W=512)
    c = O.cfg_of(**kw)
    cfg = _cfg(kw)
    Q, K, V = (round_inputs(x, "bf16") for x in O.make_qkv(c, 1))
    tau = O.make_gates(c, 1)
    q, k, v = (dev(x, torch.bfloat16).permute(0, 2, 1).contiguous() for x in (Q, K, V))
    _, ctx = fsa.nsa_forward(q, k, v, torch.from_numpy(tau).to("cuda", torch.float32), cfg, keep_scores=True)
    got = host(ctx.sel.idx)
    s_gpu = host(ctx.scores).astype(np.float64)
    s64 = O.importance_scores(Q, O.compress_kv(K, V, c).K_cmp, c)
    want = O.select_topk(s64, c)
    rows = np.argwhere((got != want).any(-1))
    print(f"rows selecting differently under fp64 oracle scores: {len(rows)} of {c.h_K * c.N}")
    # hi/lo bf16 scores keep ~fp32 accuracy: 1 row of 16,384 measured (bf16 operands: 293)
    assert len(rows) <= 1e-3 * c.h_K * c.N
    for kh, t in rows:
        own = t // c.B_K
        cand = np.arange(own + 1)
        sc = s64[kh, t, cand].copy()
        sc[own] = np.inf
        s_T = np.sort(sc)[::-1][c.T - 1]
        err = np.abs(s_gpu[kh, t, :own] - s64[kh, t, :own]).max()
        diff = np.setxor1d(got[kh, t][got[kh, t] >= 0], want[kh, t][want[kh, t] >= 0])
        assert np.all(np.abs(s64[kh, t, diff] - s_T) <= 2 * err + 1e-12), (kh, t, diff)


def test_tc_window_forward_requires_the_f16_value_copy():
    """The bf16 tensor-core window forward multiplies P by the scaled fp16 copy
    of V (fsa_v_to_f16): called without its scales it refuses with the
    library's error instead of reading bf16 V as fp16."""
    import ctypes

    from paper_2508_18224_b200 import _lib
    cfg = fsa.make_config(N=256, d_K=128, d_V=128, h=4, h_K=2, B_K=64, T=2, W=64)
    s = _lib.shape_of(cfg)
    q = torch.zeros(cfg.N, cfg.h, 128, device="cuda", dtype=torch.bfloat16)
    k = torch.zeros(cfg.N, cfg.h_K, 128, device="cuda", dtype=torch.bfloat16)
    out = torch.empty(cfg.N, cfg.h, 128, device="cuda")
    lse = torch.empty(cfg.h, cfg.N, device="cuda")
    rc = _lib.lib().fsa_slide_fwd(ctypes.byref(s), _lib.DT_BF16, _lib.ptr(q), _lib.ptr(k),
                                  _lib.ptr(k), None, _lib.ptr(out), _lib.ptr(lse), None)
    assert rc != 0 and b"fsa_v_to_f16" in _lib.lib().fsa_last_error()


def test_v_to_f16_scales_per_kv_head():
    """fsa_v_to_f16: V16 = fp16(V * s_kh) with s_kh = 2^(15 - k), max|V_kh| = f 2^k,
    f in [0.5, 1): every head's maximum lands in [2^14, 2^15), exactly (a bf16
    value times a power of two is representable in fp16 in that range), also
    for values far outside fp16's range."""
    from paper_2508_18224_b200 import _lib
    cfg = fsa.make_config(N=512, d_K=128, d_V=128, h=3, h_K=3, B_K=64, T=2, W=64)
    g = torch.Generator(device="cuda").manual_seed(5)
    v = torch.randn(cfg.N, 3, 128, device="cuda", generator=g)
    v[:, 1] *= 1e6     # above fp16's 65504
    v[:, 2] *= 1e-7    # below fp16's normal range
    v = v.to(torch.bfloat16)
    v16, vscale = _lib.v_to_f16(cfg, v)
    vd = v.double()
    for kh in range(3):
        m = float(vd[:, kh].abs().max())
        s = float(vscale[kh])
        assert 2.0 ** 14 <= m * s < 2.0 ** 15
        assert s == 2.0 ** round(np.log2(s))
        big = vd[:, kh].abs() * s >= 2.0 ** -14  # fp16 normal range: exact
        got = v16[:, kh].double()
        assert torch.equal(got[big], (vd[:, kh] * s)[big])


# ---------------------------------------------------------------------------
# selection fixtures (selection.py:201-218): byte-identical with the reference
# ---------------------------------------------------------------------------

@pytest.mark.parametrize("tag", ["sel_n32", "sel_n8"])
def test_selection_fixture_round_trip(tag, tmp_path):
    """GPU top-k of the stored scores, saved, reproduces the reference-written
    file byte for byte; loading that file gives the same device selection
    (test_selection.py:178-196)."""
    import os
    from golden_io import GOLDEN
    z = load("selection_fixtures")
    kw = json.loads(str(z[tag + "__cfg"]))
    cfg = _cfg(kw)
    ref_bytes = open(os.path.join(GOLDEN, tag + ".bin"), "rb").read()
    sel = fsa.select_topk_blocks(torch.from_numpy(z[tag + "__scores"]).cuda(), cfg)
    path = tmp_path / "sel.bin"
    fsa.save_selection(sel, path)
    assert path.read_bytes() == ref_bytes
    loaded = fsa.load_selection(os.path.join(GOLDEN, tag + ".bin"))
    assert loaded.idx.is_cuda
    np.testing.assert_array_equal(host(loaded.idx), host(sel.idx))
    fsa.validate_selection(loaded, cfg)


# Buffer-reusing schedule: kv-head chunks of the step reuse the
# scores / partial buffers; every operator is independent per kv head, so the
# chunked step equals the unchunked one bit for bit (dtau: the per-token sum
# over heads is taken chunk by chunk -> fp32 rounding only).
@pytest.mark.parametrize("kv_chunk", [1, 2])
def test_kv_chunked_step_matches_unchunked(kv_chunk):
    kw = dict(N=4096, d_K=128, d_V=128, h=12, h_K=4, B_K=64, T=8, W=256)
    cfg = _cfg(kw)
    g = torch.Generator(device="cuda").manual_seed(5)
    mk = lambda *s: torch.randn(*s, device="cuda", dtype=torch.bfloat16, generator=g)  # noqa: E731
    q, k, v, do = mk(cfg.N, cfg.h, 128), mk(cfg.N, cfg.h_K, 128), mk(cfg.N, cfg.h_K, 128), mk(cfg.N, cfg.h, 128)
    tau = torch.rand(cfg.N, 3, device="cuda", generator=g)
    out, ctx = fsa.nsa_forward(q, k, v, tau, cfg)
    ref = (out,) + tuple(fsa.nsa_backward(ctx, do, full=True))
    o2, c2 = fsa.nsa_forward(q, k, v, tau, cfg, kv_chunk=kv_chunk, keep_scores=False)
    assert isinstance(c2, fsa.ChunkedNSAContext) and len(c2.chunks) == cfg.h_K // kv_chunk
    got = (o2,) + tuple(fsa.nsa_backward(c2, do, full=True))
    for a, b, name in zip(got[:4], ref[:4], ("out", "dQ", "dK", "dV")):
        assert torch.equal(a, b), name
    assert torch.allclose(got[4], ref[4], rtol=1e-5, atol=1e-6), "dtau"
    for bad in (0, 3):
        with pytest.raises(ValueError, match="does not divide"):
            fsa.nsa_forward(q, k, v, tau, cfg, kv_chunk=bad)
    o3, c3 = fsa.nsa_forward(q, k, v, tau, cfg, kv_chunk="auto")  # fits: one chunk (unchunked)
    assert not isinstance(c3, fsa.ChunkedNSAContext) and torch.equal(o3, out)
    fused = fsa.nsa_forward_backward(q, k, v, tau, do, cfg, full=True, kv_chunk=kv_chunk)
    for a, b in zip(fused[:4], ref[:4]):
        assert torch.equal(a, b)
    assert torch.allclose(fused[4], ref[4], rtol=1e-5, atol=1e-6)


def test_kv_chunk_auto_above_the_tensor_core_limit(monkeypatch):
    """N * h past the 32-bit row-offset limit of the tensor-core kernels is
    chunked by kv head automatically (here with the limit lowered)."""
    from paper_2508_18224_b200 import nsa as nsa_mod
    kw = dict(N=2048, d_K=128, d_V=128, h=8, h_K=4, B_K=64, T=8, W=128)
    cfg = _cfg(kw)
    g = torch.Generator(device="cuda").manual_seed(6)
    mk = lambda *s: torch.randn(*s, device="cuda", dtype=torch.bfloat16, generator=g)  # noqa: E731
    q, k, v = mk(cfg.N, cfg.h, 128), mk(cfg.N, cfg.h_K, 128), mk(cfg.N, cfg.h_K, 128)
    tau = torch.rand(cfg.N, 3, device="cuda", generator=g)
    ref, _ = fsa.nsa_forward(q, k, v, tau, cfg)
    monkeypatch.setattr(nsa_mod, "TC_MAX_TOKEN_HEADS", cfg.N * 5)  # room for 2 kv heads x g = 2
    out, ctx = fsa.nsa_forward(q, k, v, tau, cfg)
    assert isinstance(ctx, fsa.ChunkedNSAContext) and len(ctx.chunks) == 2
    assert torch.equal(out, ref)


def test_keep_scores_default_releases_the_scores():
    kw = dict(N=2048, d_K=128, d_V=128, h=8, h_K=2, B_K=64, T=8, W=128)
    cfg = _cfg(kw)
    g = torch.Generator(device="cuda").manual_seed(3)
    q, k, v = (torch.randn(cfg.N, hh, 128, device="cuda", dtype=torch.bfloat16, generator=g)
               for hh in (cfg.h, cfg.h_K, cfg.h_K))
    tau = torch.full((cfg.N, 3), 1.0 / 3, device="cuda")
    out, ctx = fsa.nsa_forward(q, k, v, tau, cfg)
    out2, ctx2 = fsa.nsa_forward(q, k, v, tau, cfg, keep_scores=True)
    assert ctx.scores is None and ctx2.scores.shape == (cfg.h_K, cfg.N, cfg.b)
    assert torch.equal(out, out2) and torch.equal(ctx.sel.idx, ctx2.sel.idx)
    assert torch.equal(ctx.sel.idx, fsa.select_topk_blocks(ctx2.scores, cfg).idx)

"""Generate golden fixtures by running the REAL reference package.

Run in the build container only (``/root/reference`` does not exist on the GPU
box):

    cp -r /root/reference/pkg /tmp/refpkg && (cd /tmp/refpkg && python setup.py build_ext --inplace)
    python tests/golden/make_golden.py --ref /tmp/refpkg/src

Every fixture is an ``.npz`` holding the inputs (or the seed that regenerates
them through the reference's ``blockattn.rng`` streams) and the reference's
outputs in float64.  ``tests/test_oracle_golden.py`` pins ``oracle/`` against
these files; the GPU parity tests compare the CUDA path against both.
"""

from __future__ import annotations

import argparse
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))


def _meter_dict(meter):
    return {name: dict(bytes_loaded=p.bytes_loaded, bytes_stored=p.bytes_stored, flops=p.flops,
                       task_count=p.task_count, inner_iterations=p.inner_iterations)
            for name, p in meter.phases.items()}


def _inverse_csr(inv, cfg):
    offsets = np.zeros((cfg.h_K, cfg.b + 1), dtype=np.int64)
    toks = []
    for kh in range(cfg.h_K):
        lens = [len(q) for q in inv.queries[kh]]
        offsets[kh, 1:] = np.cumsum(lens)
        toks.append(np.concatenate([np.asarray(q, dtype=np.int64) for q in inv.queries[kh]]))
    return offsets, np.concatenate(toks)


def round_inputs(x, dtype):
    """Round float64 stream values to the GPU run dtype and back (exact on re-read).
    The tests apply the same function to regenerate these inputs from the seed."""
    if dtype is None or dtype == "f64":
        return np.asarray(x, dtype=np.float64)
    if dtype == "f32":
        return np.asarray(x, dtype=np.float32).astype(np.float64)
    if dtype == "bf16":
        import torch
        return torch.from_numpy(np.asarray(x, dtype=np.float64)).to(torch.bfloat16).double().numpy()
    raise ValueError(dtype)


def full_case(ba, name, cfg_kw, seed, *, round_to=None, sel_mode="random_uniform",
              with_dense=True, with_sliding=True, token_stride=1, store=np.float64):
    """Everything on the hot path for one config + seed.  Inputs are not stored:
    they are regenerated from ``seed`` through the rng streams + ``round_inputs``."""
    from blockattn import kv_major
    cfg = ba.make_config(**cfg_kw)
    Q, K, V = ba.rng.make_qkv(cfg, seed)
    dOut = ba.rng.make_dout(cfg, seed)
    tau = ba.rng.make_gates(cfg, seed)
    Q, K, V, dOut = (round_inputs(x, round_to) for x in (Q, K, V, dOut))
    cmp = ba.compress_kv(K, V, cfg)
    scores_cmp = ba.importance_scores_from_compressed(Q, cmp.K_cmp, cfg)
    if sel_mode == "random_uniform":
        scores = ba.rng.make_scores(cfg, seed)
    else:
        scores = scores_cmp
    sel = ba.select_topk_blocks(scores, cfg)
    inv = ba.build_inverse_index(sel, cfg)
    offsets, toks = _inverse_csr(inv, cfg)
    stats = kv_major.compute_softmax_stats(Q, K, sel, cfg)
    stats_sh = kv_major.compute_softmax_stats(Q, K, sel, cfg, shared_max=True)
    fwd, meter_f = kv_major.selected_forward(Q, K, V, sel, cfg)
    fwd_sh, _ = kv_major.selected_forward(Q, K, V, sel, cfg, shared_max=True)
    dQ, dK, dV, meter_b = kv_major.selected_backward(Q, K, V, sel, dOut, cfg)
    comp = ba.compressed_attention_forward(Q, cmp, cfg)
    rec = dict(cfg=json.dumps(cfg_kw), seed=seed, round_to=str(round_to), sel_mode=sel_mode, scores=scores, scores_cmp=scores_cmp,
               K_cmp=cmp.K_cmp, V_cmp=cmp.V_cmp, K_prefix=cmp.K_prefix, V_prefix=cmp.V_prefix,
               idx=sel.idx, inv_offsets=offsets, inv_tok=toks, n_valid=inv.n_valid,
               m=stats.m, l=stats.l, m_sh=stats_sh.m, l_sh=stats_sh.l,
               out=fwd.out, lse=fwd.lse, out_sh=fwd_sh.out,
               dQ=dQ, dK=dK, dV=dV, cmp_out=comp.out, cmp_lse=comp.lse, tau=tau,
               meter_fwd=json.dumps(_meter_dict(meter_f)), meter_bwd=json.dumps(_meter_dict(meter_b)))
    if with_sliding:
        sl = ba.sliding_attention_forward(Q, K, V, cfg)
        rec.update(slide_out=sl.out, slide_lse=sl.lse)
        g = ba.dense_backward(Q, K, V, ba.band_mask(cfg, cfg.W), dOut, cfg)
        rec.update(slide_dQ=g[0], slide_dK=g[1], slide_dV=g[2])
        comb = ba.gated_combine((comp, fwd, sl), tau, cfg)
        rec.update(comb_out=comb.out)
    if with_dense:
        mask = ba.mask_from_selection(sel, cfg)
        dense = ba.masked_attention_forward(Q, K, V, mask, cfg)
        rec.update(dense_out=dense.out, dense_lse=dense.lse)
    if token_stride > 1:   # keep large fixtures small: thin out the (N, ., h) tensors
        for key in ("out", "out_sh", "dQ", "dK", "dV", "cmp_out", "slide_out", "slide_dQ",
                    "slide_dK", "slide_dV", "comb_out", "dense_out"):
            if key in rec:
                rec[key] = rec[key][::token_stride]
        for key in ("scores", "scores_cmp"):
            rec[key] = rec[key][:, ::token_stride]
        rec["token_stride"] = token_stride
    for key, val in list(rec.items()):
        if isinstance(val, np.ndarray) and val.dtype == np.float64:
            rec[key] = val.astype(store)
    np.savez_compressed(os.path.join(HERE, name + ".npz"), **rec)
    return rec


def selection_kats(ba):
    """Tie / special-value vectors for select_topk_blocks (selection.py:78-102)."""
    cases = {}

    def run(tag, cfg_kw, scores, seed=None, f32=False):
        """Large score tensors are not stored: ``seed`` regenerates them from the
        reference's ``scores`` stream (rng.py:34-35), optionally rounded to fp32."""
        cfg = ba.make_config(**cfg_kw)
        sel = ba.select_topk_blocks(scores, cfg)
        cases[tag + "__cfg"] = json.dumps(cfg_kw)
        if seed is None:
            cases[tag + "__scores"] = scores
        else:
            cases[tag + "__seed"] = np.array([seed, int(f32)])
        cases[tag + "__idx"] = sel.idx

    base = dict(N=12, d_K=4, d_V=4, h=2, h_K=1, B_K=4, T=2)
    s = np.zeros((1, 12, 3))
    s[0] = (0.5, 0.5, 0.9)
    run("tie_lower_index", base, s)                                  # test_selection.py:44-50
    s = np.zeros((1, 12, 3))
    s[0, :, 0] = -0.0
    s[0, :, 1] = 0.0
    run("neg_zero_tie", dict(base, T=2), s)
    s = np.random.default_rng(3).uniform(size=(1, 12, 3))
    s[0, 8:, 0] = np.inf                                             # +inf non-own competitor
    run("posinf_competitor_T1", dict(base, T=1), s)
    run("posinf_competitor_T2", dict(base, T=2), s)
    s = np.random.default_rng(4).uniform(size=(1, 12, 3))
    s[0, 8:, 0] = -np.inf
    s[0, 8:, 1] = np.nan
    run("neginf_nan_unselectable", dict(base, T=3), s)
    cfg_kw = dict(N=64, d_K=4, d_V=4, h=4, h_K=2, B_K=4, T=5)
    rng = np.random.default_rng(5)
    s = rng.integers(0, 4, size=(2, 64, 16)).astype(np.float64) / 4.0  # heavy ties
    s[rng.uniform(size=s.shape) < 0.05] = np.nan
    s[rng.uniform(size=s.shape) < 0.05] = -np.inf
    s[rng.uniform(size=s.shape) < 0.02] = np.inf
    s[rng.uniform(size=s.shape) < 0.05] = -0.0
    run("mixed_specials", cfg_kw, s)
    cfg_kw = dict(N=4096, d_K=8, d_V=8, h=1, h_K=1, B_K=64, T=16)
    cfg = ba.make_config(**cfg_kw)
    s = ba.rng.make_scores(cfg, 10)
    run("uniform_4096_T16", cfg_kw, s, seed=10)
    s32 = s.astype(np.float32).astype(np.float64)
    run("uniform_4096_T16_f32", cfg_kw, s32, seed=10, f32=True)
    cfg_kw = dict(N=2048, d_K=8, d_V=8, h=2, h_K=2, B_K=16, T=40)   # T > 32 path
    cfg = ba.make_config(**cfg_kw)
    run("uniform_T40", cfg_kw, ba.rng.make_scores(cfg, 11), seed=11)
    np.savez_compressed(os.path.join(HERE, "selection_kats.npz"), **cases)


def malformed(ba):
    """Error messages of validate_selection (selection.py:49-75)."""
    from blockattn import SelectionError, SelectionTensor
    cfg_kw = dict(N=8, d_K=4, d_V=4, h=2, h_K=1, B_K=2, T=2)
    cfg = ba.make_config(**cfg_kw)
    good = ba.self_block_selection(cfg).idx.copy()
    out = {"cfg": json.dumps(cfg_kw), "good": good}
    edits = {
        "dup": (0, 5, (2, 2)), "noncausal": (0, 1, (0, 3)), "empty": (0, 4, (-1, -1)),
        "decreasing": (0, 6, (3, 1)), "after_sentinel": (0, 6, (-1, 3)), "range": (0, 6, (3, 9)),
        "negative": (0, 6, (-2, 3)),
    }
    msgs = {}
    for tag, (kh, t, row) in edits.items():
        idx = good.copy()
        idx[kh, t, :] = row
        try:
            ba.validate_selection(SelectionTensor(idx), cfg)
            msgs[tag] = ""
        except SelectionError as exc:
            msgs[tag] = str(exc)
        out["idx_" + tag] = idx
    out["messages"] = json.dumps(msgs)
    np.savez_compressed(os.path.join(HERE, "malformed.npz"), **out)


def selection_fixtures(ba):
    """Binary selection fixtures written by the reference's save_selection
    (selection.py:201-206): the files themselves are the golden bytes that
    paper_2508_18224_b200.save_selection must reproduce and load_selection
    must read (test_selection.py:178-206)."""
    meta = {}
    for tag, cfg_kw, seed in (("sel_n32", dict(N=32, d_K=4, d_V=4, h=4, h_K=2, B_K=8, T=3), 8),
                              ("sel_n8", dict(N=8, d_K=4, d_V=4, h=4, h_K=2, B_K=2, T=2), 12)):
        cfg = ba.make_config(**cfg_kw)
        scores = ba.rng.make_scores(cfg, seed)
        sel = ba.select_topk_blocks(scores, cfg)
        ba.save_selection(sel, os.path.join(HERE, tag + ".bin"))
        meta[tag + "__cfg"] = json.dumps(cfg_kw)
        meta[tag + "__scores"] = scores
        meta[tag + "__idx"] = sel.idx
    np.savez_compressed(os.path.join(HERE, "selection_fixtures.npz"), **meta)


def acceptance_sweep(ba):
    """Criterion-3 style random scenarios (tests/helpers.py:75-99): store the
    configs and reference outputs for a size-bounded subset."""
    sys.path.insert(0, os.path.join(os.path.dirname(ba.__file__), "..", "..", "tests"))
    from blockattn import kv_major
    rng = np.random.default_rng(2024)
    recs = {}
    n = 0
    count = 0
    while count < 50:
        N = int(rng.choice([64, 128, 256, 512, 1024]))
        B_K = int(rng.choice([4, 8, 16, 32]))
        if N % B_K:
            continue
        b = N // B_K
        g = int(rng.choice([1, 2, 4, 8]))
        h_K = int(rng.choice([1, 2]))
        d = int(rng.choice([8, 16, 32, 64]))
        T = int(rng.integers(1, min(b, 8) + 1))
        B_Q = int(rng.choice([4, 8, 16]))
        cfg_kw = dict(N=N, d_K=d, d_V=d, h=g * h_K, h_K=h_K, B_K=B_K, T=T, B_Q=B_Q)
        seed = count
        count += 1
        if N * d * g * h_K > 16 * 1024 or n >= 12:
            continue
        cfg = ba.make_config(**cfg_kw)
        Q, K, V = ba.rng.make_qkv(cfg, seed)
        sel = ba.select_topk_blocks(ba.rng.make_scores(cfg, seed), cfg)
        dOut = ba.rng.make_dout(cfg, seed)
        fwd, _ = kv_major.selected_forward(Q, K, V, sel, cfg)
        dQ, dK, dV, _ = kv_major.selected_backward(Q, K, V, sel, dOut, cfg)
        p = f"s{n}__"
        recs.update({p + "cfg": json.dumps(cfg_kw), p + "seed": seed, p + "idx": sel.idx,
                     p + "out": fwd.out, p + "lse": fwd.lse, p + "dQ": dQ, p + "dK": dK, p + "dV": dV})
        n += 1
    recs["count"] = n
    np.savez_compressed(os.path.join(HERE, "acceptance_sweep.npz"), **recs)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ref", required=True, help="src dir of a built copy of the reference pkg")
    ap.add_argument("--only", default=None, help="run one generator (e.g. selection_fixtures)")
    args = ap.parse_args()
    sys.path.insert(0, args.ref)
    import blockattn as ba
    import blockattn.rng  # noqa: F401
    assert ba.get_backend() == "compiled", "build the reference Cython core first"
    if args.only:
        globals()[args.only](ba)
        return
    full_case(ba, "case_kv_small", dict(N=64, d_K=8, d_V=8, h=4, h_K=2, B_K=8, T=2, B_Q=8), 1)
    full_case(ba, "case_rect_dims", dict(N=64, d_K=8, d_V=16, h=4, h_K=2, B_K=8, T=3, B_Q=8), 21)
    full_case(ba, "case_pipeline", dict(N=128, d_K=16, d_V=16, h=8, h_K=2, B_K=16, T=3, W=24), 13,
              sel_mode="from_scores")
    full_case(ba, "case_g8_bk1", dict(N=32, d_K=4, d_V=4, h=8, h_K=1, B_K=1, T=4, W=3), 4)
    full_case(ba, "case_unit", dict(N=1, d_K=1, d_V=1, h=1, h_K=1, B_K=1, T=1), 0)
    full_case(ba, "case_tiny_fp32", dict(N=2048, d_K=64, d_V=64, h=4, h_K=1, B_K=64, T=8, W=128), 0,
              round_to="f32", with_dense=False, token_stride=8, store=np.float32)
    full_case(ba, "case_d128_bf16", dict(N=1024, d_K=128, d_V=128, h=4, h_K=1, B_K=64, T=6, W=256), 3,
              round_to="bf16", with_dense=False, token_stride=8, store=np.float32)
    selection_kats(ba)
    malformed(ba)
    selection_fixtures(ba)
    acceptance_sweep(ba)
    total = sum(os.path.getsize(os.path.join(HERE, f)) for f in os.listdir(HERE) if f.endswith(".npz"))
    print(f"fixtures written: {total / 1e6:.2f} MB")


if __name__ == "__main__":
    main()

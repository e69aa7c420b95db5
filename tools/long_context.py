"""Long-context NSA steps on one B200 with the buffer-reusing kv-head-chunked
schedule (nsa.nsa_forward_backward(kv_chunk=...)).

    python tools/long_context.py [N ...]      (default: Qwen3-14B shape at 128K, 256K, 512K, 1M)

Per N: the chunk plan_kv_chunk picks, device ms per fwd+bwd step (CUDA events,
median of 3 after a warm-up), tokens/s, peak device memory, and -- as a cheap
full-size sanity check -- the per-kv-head identity
sum_s dV[s, kh] = sum_t sum_{j in group kh} (tau1 + tau2)[t] dOut[t, j]
(selected and sliding softmax rows sum to one), relative error printed.
"""
import json
import os
import sys

# one allocation pattern per N: expandable segments keep the 64 GB score
# buffer of a 1M-token chunk from failing on a fragmented cache
os.environ.setdefault("PYTORCH_CUDA_ALLOC_CONF", "expandable_segments:True")
import torch  # noqa: E402

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2508_18224_b200 as fsa  # noqa: E402
from paper_2508_18224_b200 import nsa  # noqa: E402


def run(N, h=40, h_K=8):
    cfg = fsa.make_config(N=N, d_K=128, d_V=128, h=h, h_K=h_K, B_K=64, T=16, W=512)
    chunk = fsa.plan_kv_chunk(cfg)
    g = torch.Generator(device="cuda").manual_seed(0)
    mk = lambda *s: torch.randn(*s, device="cuda", dtype=torch.bfloat16, generator=g)  # noqa: E731
    q, k, v, do = mk(N, h, 128), mk(N, h_K, 128), mk(N, h_K, 128), mk(N, h, 128)
    tau = torch.rand(N, 3, device="cuda", generator=g)
    torch.cuda.synchronize()
    base = torch.cuda.memory_allocated()
    torch.cuda.reset_peak_memory_stats()
    res = nsa.nsa_forward_backward(q, k, v, tau, do, cfg, kv_chunk=chunk)
    torch.cuda.synchronize()
    peak = torch.cuda.max_memory_allocated() - base
    dV = res[3]
    lhs = dV.double().sum(0)  # (h_K, d)
    w = (tau[:, 1] + tau[:, 2]).double()
    rhs = (do.double() * w[:, None, None]).reshape(N, h_K, cfg.g, 128).sum((0, 2))
    ident = float((lhs - rhs).abs().max() / rhs.abs().max())
    del res, dV
    times = []
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        nsa.nsa_forward_backward(q, k, v, tau, do, cfg, kv_chunk=chunk)
        e1.record()
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1))
    ms = sorted(times)[1]
    return {"N": N, "h": h, "h_K": h_K, "kv_chunk": chunk, "ms_per_step": round(ms, 2),
            "tokens_per_s": round(N / ms * 1e3), "peak_transient_GB": round(peak / 1e9, 1),
            "dV_identity_rel_err": ident}


if __name__ == "__main__":
    Ns = [int(x) for x in sys.argv[1:]] or [131072, 262144, 524288, 1048576]
    for N in Ns:
        print(json.dumps(run(N)), flush=True)
        torch.cuda.empty_cache()

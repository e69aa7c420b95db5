"""NSA forward+backward benchmark (BASELINE.json metric) -- one JSON line.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 \
        --master-port P bench.py --gpus N ...

Workload (BASELINE.json configs[1]): Llama-3-8B attention shape, 32 q / 8 kv
heads (GQA 4), d = 128, block 64, top-16, window 512, bf16, seq 32K, NSA
forward + backward.  A step = compress -> compressed attention + scores ->
top-k -> inverse index -> FSA selected forward -> sliding window -> gated
combine, then the selected and sliding backward (the branches the reference
differentiates).  Synthetic N(0,1) inputs, random-init -- no datasets.
Scaling is weak: each rank runs its own sequence (batch sharding, no
collective on the data path); value = all ranks' tokens / max-over-ranks time.

``--impl reference`` times the reference algorithm on the host CPU (the oracle
port, oracle/fsa_oracle.py -- the reference is Python and cannot travel to the
GPU box) on a bounded sample, rank 0 only.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

WORKLOAD = dict(name="llama3-8b-attn-32k", N=32768, d=128, h=32, h_K=8, B_K=64, T=16, W=512)
CPU_SAMPLE_N = int(os.environ.get("FSA_BENCH_CPU_SAMPLE", 8192))  # smaller only in the CPU tests


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            p = json.load(fh)
        return p["hbm_gbs"], p["bf16_tflops"], p.get("bf16_tflops_sustained", p["bf16_tflops"]), "measured"
    except Exception:
        return 6650.0, 1590.0, 1400.0, "fallback"


# ---------------------------------------------------------------------------
# clocks sampled during the timed region
# ---------------------------------------------------------------------------
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        # nvidia-smi numbers the physical GPUs: map the CUDA device through
        # CUDA_VISIBLE_DEVICES when it is set
        vis = [x for x in os.environ.get("CUDA_VISIBLE_DEVICES", "").split(",") if x.strip()]
        self.index = vis[index].strip() if index < len(vis) else index
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "20"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            threading.Thread(target=self._read, daemon=True).start()
            t0 = time.time()
            while not self.rows and time.time() - t0 < 3.0:  # first sample before timing
                time.sleep(0.01)
            self.rows.clear()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) >= 7:
                self.rows.append(parts)

    def stop(self):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        smax = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        reasons = sorted({n for r in self.rows for n, v in zip(names, r[3:7]) if v == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(smax) if smax else None, "reasons": reasons,
                "samples": len(self.rows)}


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------
def run_ours(args, rank, world, local_rank):
    import numpy as np
    import torch

    import paper_2508_18224_b200 as fsa
    from paper_2508_18224_b200 import _lib, kv_major, nsa

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
    w = WORKLOAD
    cfg = fsa.make_config(N=w["N"], d_K=w["d"], d_V=w["d"], h=w["h"], h_K=w["h_K"], B_K=w["B_K"],
                          T=w["T"], W=w["W"])
    gen = torch.Generator(device=dev).manual_seed(1234 + rank)
    bf = torch.bfloat16
    q = torch.randn(cfg.N, cfg.h, cfg.d_K, device=dev, dtype=bf, generator=gen)
    k = torch.randn(cfg.N, cfg.h_K, cfg.d_K, device=dev, dtype=bf, generator=gen)
    v = torch.randn(cfg.N, cfg.h_K, cfg.d_V, device=dev, dtype=bf, generator=gen)
    dout = torch.randn(cfg.N, cfg.h, cfg.d_V, device=dev, dtype=bf, generator=gen)
    tau = torch.rand(cfg.N, 3, device=dev, generator=gen)

    def barrier():
        if world > 1:
            import torch.distributed as dist
            dist.barrier()

    # per-step timing of the dominant kernel (K5) on the launching stream
    def step():
        out, ctx = nsa.nsa_forward(q, k, v, tau, cfg)
        grads = nsa.nsa_backward(ctx, dout)
        return out, grads, ctx

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()

    # kernel launches of our library inside one step (profiler, outside the timed region)
    gpu_launches, kernel_names = None, {}
    try:
        from torch.profiler import ProfilerActivity, profile
        with profile(activities=[ProfilerActivity.CUDA]) as prof:
            step()
            torch.cuda.synchronize()
        kernel_ms = {}
        for e in prof.key_averages():
            if e.device_type is not None and "fsa" in e.key and e.count:
                kernel_names[e.key[:80]] = kernel_names.get(e.key[:80], 0) + e.count
                t_us = getattr(e, "device_time_total", None) or getattr(e, "cuda_time_total", 0)
                kernel_ms[e.key[:80]] = round(t_us / 1e3, 4)
        gpu_launches = sum(kernel_names.values()) * args.steps
        kernel_names = {"launches": kernel_names, "device_ms_profiled": kernel_ms}
    except Exception as exc:  # pragma: no cover
        kernel_names = {"profiler_error": str(exc)[:120]}

    # The tensor-core kernels are timed inside the same loop with CUDA events
    # on the launching stream: the C-ABI entry points are wrapped so that each
    # fsa_sel_fwd (K5) / fsa_sel_bwd (K8, selected branch) launch is bracketed.
    sampler = ClockSampler(local_rank)
    barrier()
    torch.cuda.synchronize()
    sampler.start()
    start = torch.cuda.Event(enable_timing=True)
    stop = torch.cuda.Event(enable_timing=True)
    kev = {"fsa_sel_fwd": [], "fsa_sel_bwd": []}
    orig_call = _lib.call

    def timed_call(name, *a):
        if name not in kev:
            return orig_call(name, *a)
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        r = orig_call(name, *a)
        e1.record()
        kev[name].append((e0, e1))
        return r

    _lib.call = timed_call
    start.record()
    for _ in range(args.steps):
        out_, grads_, ctx_ = step()
    stop.record()
    torch.cuda.synchronize()
    _lib.call = orig_call
    clocks = sampler.stop()
    ms = start.elapsed_time(stop) / args.steps
    if world > 1:
        import torch.distributed as dist
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    k5_ms = statistics.median(e0.elapsed_time(e1) for e0, e1 in kev["fsa_sel_fwd"])
    k8_ms = statistics.median(e0.elapsed_time(e1) for e0, e1 in kev["fsa_sel_bwd"])
    inv = ctx_.inv
    nnz = int(inv.offsets[:, -1].to(torch.int64).sum())
    R = nnz * cfg.g
    k5_flops = 4.0 * cfg.d_K * cfg.B_K * R
    k8_flops = 10.0 * cfg.d_K * cfg.B_K * R

    # ---- end to end through the public API: pinned host inputs in, out + grads
    # (bf16, the input dtype) back to pinned host memory, every step.  Copies
    # run on their own streams, double-buffered, so step i+1's upload and step
    # i-1's download overlap step i's kernels.
    names = ("q", "k", "v", "dout", "tau")
    host_in = {n: t.cpu().pin_memory() for n, t in zip(names, (q, k, v, dout, tau))}
    h2d = sum(t.numel() * t.element_size() for t in host_in.values())
    dev_in = [{n: torch.empty_like(t, device=dev) for n, t in host_in.items()} for _ in range(2)]
    out_shapes = ((cfg.N, cfg.h, cfg.d_V), (cfg.N, cfg.h, cfg.d_K), (cfg.N, cfg.h_K, cfg.d_K),
                  (cfg.N, cfg.h_K, cfg.d_V))
    dev_out = [[torch.empty(s_, dtype=bf, device=dev) for s_ in out_shapes] for _ in range(2)]
    host_out = [[torch.empty(s_, dtype=bf).pin_memory() for s_ in out_shapes] for _ in range(2)]
    d2h = sum(x.numel() * x.element_size() for x in host_out[0])
    comp = torch.cuda.current_stream()
    up, down = torch.cuda.Stream(), torch.cuda.Stream()
    ev = lambda: torch.cuda.Event()  # noqa: E731
    in_ready, in_free, out_ready, out_free = ([ev() for _ in range(2)] for _ in range(4))

    def upload(i):
        s_ = i % 2
        with torch.cuda.stream(up):
            if i >= 2:
                up.wait_event(in_free[s_])
            for n in names:
                dev_in[s_][n].copy_(host_in[n], non_blocking=True)
            in_ready[s_].record(up)

    def e2e_step(i):
        s_ = i % 2
        comp.wait_event(in_ready[s_])
        x = dev_in[s_]
        out, ctx = nsa.nsa_forward(x["q"], x["k"], x["v"], x["tau"], cfg)
        gq, gk, gv = nsa.nsa_backward(ctx, x["dout"])
        in_free[s_].record(comp)
        if i >= 2:
            comp.wait_event(out_free[s_])
        for dst, src in zip(dev_out[s_], (out, gq, gk, gv)):
            dst.copy_(src)
        out_ready[s_].record(comp)
        with torch.cuda.stream(down):
            down.wait_event(out_ready[s_])
            for dst, src in zip(host_out[s_], dev_out[s_]):
                dst.copy_(src, non_blocking=True)
            out_free[s_].record(down)

    # the copy pipeline's fill (first upload) and drain (last download) are
    # one-off costs; time enough steps that the per-step figure is the steady
    # state of a long run (each step still uploads its inputs and downloads
    # its results inside the timed region)
    e2e_steps = max(args.steps, 30)
    for i in range(2):  # warm the copy path
        upload(i)
        e2e_step(i)
    torch.cuda.synchronize()
    barrier()
    torch.cuda.synchronize()
    e_start = torch.cuda.Event(enable_timing=True)
    e_stop = torch.cuda.Event(enable_timing=True)
    e_start.record(comp)
    up.wait_event(e_start)
    upload(0)
    for i in range(e2e_steps):
        if i + 1 < e2e_steps:
            upload(i + 1)
        e2e_step(i)
    comp.wait_stream(down)
    e_stop.record(comp)
    torch.cuda.synchronize()
    e2e_ms = e_start.elapsed_time(e_stop) / e2e_steps
    if world > 1:
        import torch.distributed as dist
        t = torch.tensor([e2e_ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = float(t.item())

    hbm, pk_burst, pk_sus, pk_src = _peaks()
    tokens = world * cfg.N
    value = tokens / (ms / 1e3)
    step_flops = (4.0 + 10.0) * cfg.d_K * cfg.B_K * R  # selected fwd + bwd
    slide_pairs = sum(min(t + 1, cfg.W) for t in range(cfg.N))
    step_flops += (4.0 + 10.0) * cfg.d_K * cfg.h * slide_pairs
    step_flops += 4.0 * cfg.d_K * cfg.h * sum((t + 1) // cfg.B_K for t in range(cfg.N))
    traffic = {}
    try:  # dram__bytes_read.sum + dram__bytes_write.sum per launch, from the committed ncu capture
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as fh:
            traffic = json.load(fh)
    except Exception:
        pass

    def roof(kernel, flops, kms, algo, tkey):
        ach = flops / (kms / 1e3) / 1e12
        return {"kernel": kernel, "bound": "tensor", "achieved": round(ach, 2), "peak": pk_sus,
                "unit": "TFLOP/s", "frac": round(ach / pk_sus, 4),
                "traffic": traffic.get(tkey), "peak_source": f"{pk_src} sustained bf16",
                "kernel_ms": round(kms, 4), "share_of_step": round(kms / ms, 4),
                "algorithmic": algo}
    line = {
        "metric": "NSA fwd+bwd tokens/s (Llama-3-8B attention, 32K, GQA 4)",
        "value": round(value, 1),
        "unit": "tokens/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(ms, 4),
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "bf16",
        "data": "synthetic N(0,1) Q/K/V/dOut, U[0,1) gates, random init",
        "config": arm_config(world),
        "effective_tflops": round(step_flops / (ms / 1e3) / 1e12, 2),
        # dominant kernel: the selected-attention backward (K8)
        "roofline": roof("sel_bwd (K8, tcgen05, selected branch)", k8_flops, k8_ms,
                         "10*d*B_K*R FLOPs, R = (query head, token, block) rows = %d" % R,
                         "tc_sel_bwd_selected"),
        "roofline_sel_fwd": roof("sel_fwd (K5, tcgen05)", k5_flops, k5_ms,
                                 "4*d*B_K*R FLOPs, R = %d" % R, "tc_sel_fwd"),
        "e2e": {"value": round(tokens / (e2e_ms / 1e3), 1), "unit": "tokens/s",
                "ms_per_step": round(e2e_ms, 3), "steps": e2e_steps, "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h},
        "gpu_launches": gpu_launches,
        "kernels_per_step": kernel_names,
        "clocks": clocks,
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:  # rank 0 at N = 1 only
        line["cpu_baseline"] = cpu_baseline(args, sample_n=CPU_SAMPLE_N, steps=1)
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()
    return line


# ---------------------------------------------------------------------------
# CPU reference arm (the oracle port -- the reference itself is Python and is
# not present on the GPU box)
# ---------------------------------------------------------------------------
def _cpu_group(args_tuple):
    n_tok, seed = args_tuple
    os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
    import numpy as np
    from oracle import fsa_oracle as O
    w = WORKLOAD
    c = O.cfg_of(N=n_tok, d_K=w["d"], d_V=w["d"], h=w["h"] // w["h_K"], h_K=1, B_K=w["B_K"],
                 T=w["T"], W=w["W"])
    Q, K, V = O.make_qkv(c, seed)
    dO = O.make_dout(c, seed)
    tau = O.make_gates(c, seed)
    t0 = time.perf_counter()
    O.nsa_forward_backward_group(Q, K, V, dO, tau, c)
    return time.perf_counter() - t0


def cpu_baseline(args, sample_n=CPU_SAMPLE_N, steps=1):
    """The oracle port on the host cores: one process per KV group (bit-exact
    sharding); sample = the first ``sample_n`` tokens of each KV
    group of the workload, fwd+bwd of every branch."""
    import multiprocessing as mp
    w = WORKLOAD
    cores = max(1, min(len(os.sched_getaffinity(0)), w["h_K"]))
    times = []
    with mp.get_context("spawn").Pool(cores) as pool:
        for s in range(steps):
            t0 = time.perf_counter()
            pool.map(_cpu_group, [(sample_n, 100 + s * 16 + kh) for kh in range(w["h_K"])])
            times.append(time.perf_counter() - t0)
    wall = statistics.median(times)
    return {"value": round(sample_n / wall, 2), "unit": "tokens/s", "cores": cores, "kind": "port",
            "sample": f"all {w['h_K']} KV groups of {w['name']}, first {sample_n} tokens "
                      f"(N={sample_n} causal prefix), NSA fwd+bwd in float64 numpy, "
                      f"{cores} processes; {wall:.1f} s wall"}


def arm_config(world):
    """The workload both arms report (the reference arm measures a bounded
    sample of it; cpu_baseline.sample says which)."""
    w = WORKLOAD
    return {"workload": w["name"], "seq_len": w["N"], "batch_per_gpu": 1, "q_heads": w["h"],
            "kv_heads": w["h_K"], "head_dim": w["d"], "block": w["B_K"], "top_k": w["T"],
            "window": w["W"], "parallelism": f"batch{world}", "l2": "inputs exceed L2 "
            "(Q 268 MB, K/V 67 MB each, partial buffer 4.2 GB); no flush"}


def run_reference(args, rank, world):
    if rank != 0:
        return None
    n = CPU_SAMPLE_N
    cb = cpu_baseline(args, sample_n=n, steps=max(1, min(args.steps, 5)))
    return {
        "impl": "reference",
        "metric": "NSA fwd+bwd tokens/s (Llama-3-8B attention, 32K, GQA 4)",
        "value": cb["value"], "unit": "tokens/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic", "config": arm_config(world),
        "cpu_baseline": cb,
        "e2e": {"value": cb["value"], "unit": "tokens/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", args.gpus if args.gpus == 1 else 1))
    local_rank = int(os.environ.get("LOCAL_RANK", 0))
    if args.impl == "reference":
        line = run_reference(args, rank, world)
    else:
        line = run_ours(args, rank, world, local_rank)
    if rank == 0 and line is not None:
        print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()

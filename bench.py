"""NSA forward+backward benchmark (BASELINE.json metric) -- one JSON line.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 \
        --master-port P bench.py --gpus N ...

Headline workload (BASELINE.json configs[4], the config the metric's
"tokens/s at 1/2/4/8 GPU" is quoted on): Qwen3-14B attention shape, 40 q /
8 kv heads (GQA 5), d = 128, block 64, top-16, window 512, bf16, seq 128K,
NSA forward + backward, sharded by kv head.  A step = compress -> compressed
attention + scores -> top-k -> inverse index -> FSA selected forward ->
sliding window -> gated combine, then the selected and sliding backward (the
branches the reference differentiates).  Synthetic N(0,1) inputs, random
init -- no datasets.

Multi-GPU: rank r of N owns kv heads [r h_K / N, (r+1) h_K / N)
of the one sequence and their query heads and runs the unmodified
single-GPU path on them -- no collective on the data path.  Total work is
fixed: "scaling": "strong"; value = the sequence's tokens / max-over-ranks
step time.

The step is captured once in a CUDA graph (static input buffers; the
operator path has no host synchronisation), so the timed region measures the
device, not the host's launch rate.  Extra keys time the Llama-3-8B shape at
32K (configs[1]) and at 64K (the north_star target) the same way.

``--impl reference`` times the reference on the host CPU -- the blockattn
package installed into baseline/_ref (its compiled Cython core), or the
oracle port when that is absent -- on a labelled bounded sample, rank 0 only.
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

WORKLOADS = {
    # BASELINE.json configs[4]: the headline (tokens/s at 1/2/4/8 GPU, kv-head shards)
    "qwen3-14b-attn-128k": dict(N=131072, h=40, h_K=8, d=128, B_K=64, T=16, W=512),
    # configs[1]
    "llama3-8b-attn-32k": dict(N=32768, h=32, h_K=8, d=128, B_K=64, T=16, W=512),
    # the north_star target shape
    "llama3-8b-attn-64k": dict(N=65536, h=32, h_K=8, d=128, B_K=64, T=16, W=512),
}
HEADLINE = "qwen3-14b-attn-128k"
METRIC = "NSA fwd+bwd tokens/s (Qwen3-14B attention, 128K, GQA 5, kv-head sharded)"
# reference-arm / cpu_baseline sample: the causal prefix of every kv group
CPU_SAMPLE_N = int(os.environ.get("FSA_BENCH_CPU_SAMPLE", 16384))


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            p = json.load(fh)
        return (p["hbm_gbs"], p["bf16_tflops"], p.get("bf16_tflops_sustained", p["bf16_tflops"]),
                "MEASURED_PEAKS.json")
    except Exception:
        return 6650.0, 1590.0, 1400.0, "fallback (B200_PROFILING.md)"


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
def full_cfg(w):
    import paper_2508_18224_b200 as fsa
    return fsa.make_config(N=w["N"], d_K=w["d"], d_V=w["d"], h=w["h"], h_K=w["h_K"], B_K=w["B_K"],
                           T=w["T"], W=w["W"])


def rank_inputs(cfg, kv_lo, kv_hi, dev, seed=1234):
    """This rank's slice of the synthetic problem: every kv head's group is
    drawn from its own generator, so a shard is the same data whatever the
    world size.  Q / dOut (N, g*(kv_hi-kv_lo), d), K / V (N, kv_hi-kv_lo, d),
    gates (N, 3) shared by all heads."""
    import torch
    bf = torch.bfloat16
    qs, ks, vs, ds = [], [], [], []
    for kh in range(kv_lo, kv_hi):
        gen = torch.Generator(device=dev).manual_seed(seed + kh)
        qs.append(torch.randn(cfg.N, cfg.g, cfg.d_K, device=dev, dtype=bf, generator=gen))
        ks.append(torch.randn(cfg.N, 1, cfg.d_K, device=dev, dtype=bf, generator=gen))
        vs.append(torch.randn(cfg.N, 1, cfg.d_V, device=dev, dtype=bf, generator=gen))
        ds.append(torch.randn(cfg.N, cfg.g, cfg.d_V, device=dev, dtype=bf, generator=gen))
    gen = torch.Generator(device=dev).manual_seed(seed - 1)
    tau = torch.rand(cfg.N, 3, device=dev, generator=gen)
    cat = lambda xs: torch.cat(xs, 1).contiguous()  # noqa: E731
    return cat(qs), cat(ks), cat(vs), cat(ds), tau


def algorithmic_flops(cfg, R):
    """selected 4 / 10 d B_K R, sliding 4 / 10 d h sum_t min(t+1, W),
    compressed forward 4 d h sum_t floor((t+1)/B_K)."""
    slide = sum(min(t + 1, cfg.W) for t in range(cfg.N))
    formed = sum((t + 1) // cfg.B_K for t in range(cfg.N))
    return ((4.0 + 10.0) * cfg.d_K * cfg.B_K * R + (4.0 + 10.0) * cfg.d_K * cfg.h * slide
            + 4.0 * cfg.d_K * cfg.h * formed)


def measure(name, w, rank, world, dev, steps, warmup, barrier, use_graph=True):
    """Device-timed NSA fwd+bwd of this rank's kv-head shard of workload w.
    Returns per-rank ms/step plus the K5 / K8 launch durations (CUDA events
    on the launching stream inside the timed region)."""
    import torch

    from paper_2508_18224_b200 import _lib, nsa, parallel

    cfg0 = full_cfg(w)
    sh = parallel.shard_kv_heads(cfg0, rank, world)
    cfg = sh.cfg
    q, k, v, dout, tau = rank_inputs(cfg0, sh.kv_lo, sh.kv_hi, dev)
    orig_call = _lib.call
    kev = {"fsa_sel_fwd": [], "fsa_sel_bwd": [], "fsa_merge_combine_fwd": [], "fsa_dq_reduce_add": []}
    capturing = [False]

    def record(e):
        if capturing[0]:
            # inside stream capture a plain record is only a dependency edge;
            # an "external" record becomes a timing node of the graph
            _cu_event_record_external(e, torch.cuda.current_stream())
        else:
            e.record()

    def timed_call(name_, *a):
        if name_ not in kev:
            return orig_call(name_, *a)
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        if capturing[0]:  # create the driver events before capture uses them
            e0.record(side)
            e1.record(side)
        record(e0)
        r = orig_call(name_, *a)
        record(e1)
        kev[name_].append((e0, e1))
        return r

    def step():
        out, ctx = nsa.nsa_forward(q, k, v, tau, cfg)
        grads = nsa.nsa_backward(ctx, dout)
        return out, grads, ctx

    for _ in range(warmup):
        step()
    torch.cuda.synchronize()
    _, _, ctx = step()
    nnz = int(ctx.inv.offsets[:, -1].to(torch.int64).sum())
    R = nnz * cfg.g
    del ctx

    graph = None
    if use_graph:
        # one CUDA graph holding all K timed steps, each with its own K5 / K8
        # events (a replayed single-step graph would overwrite them)
        try:
            side = torch.cuda.Stream()
            side.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(side):
                step()
            torch.cuda.current_stream().wait_stream(side)
            torch.cuda.synchronize()
            graph = torch.cuda.CUDAGraph()
            _lib.call = timed_call
            capturing[0] = True
            with torch.cuda.graph(graph):
                for _ in range(steps):
                    step()
        except Exception as exc:  # pragma: no cover - reported, then the eager loop runs
            graph = None
            print(f"bench: CUDA graph capture failed ({exc!s:.120}); timing eager launches",
                  file=sys.stderr)
        finally:
            _lib.call = orig_call
            capturing[0] = False
        if graph is None:
            kev = {k_: [] for k_ in kev}
        else:
            graph.replay()  # untimed: first replay uploads the graph
            torch.cuda.synchronize()
    barrier()
    torch.cuda.synchronize()
    start = torch.cuda.Event(enable_timing=True)
    stop = torch.cuda.Event(enable_timing=True)
    if graph is not None:
        start.record()
        graph.replay()
        stop.record()
    else:
        _lib.call = timed_call
        start.record()
        for _ in range(steps):
            step()
        stop.record()
        _lib.call = orig_call
    torch.cuda.synchronize()
    ms = start.elapsed_time(stop) / steps
    per = {k_: statistics.mean([e0.elapsed_time(e1) for e0, e1 in ev][-steps:])
           for k_, ev in kev.items() if ev}
    del graph
    torch.cuda.empty_cache()
    return dict(name=name, cfg=cfg, cfg0=cfg0, shard=sh, ms=ms, R=R,
                k5_ms=per["fsa_sel_fwd"], k8_ms=per["fsa_sel_bwd"],
                merge_ms=per.get("fsa_merge_combine_fwd"), dqr_ms=per.get("fsa_dq_reduce_add"),
                graph=use_graph, inputs=(q, k, v, dout, tau))


_LIBCUDA = None


def _cu_event_record_external(ev, stream):
    """cuEventRecordWithFlags(CU_EVENT_RECORD_EXTERNAL): a timing event inside a
    CUDA graph (torch's Event.record during capture is only a dependency)."""
    import ctypes
    global _LIBCUDA
    if _LIBCUDA is None:
        _LIBCUDA = ctypes.CDLL("libcuda.so.1")
    rc = _LIBCUDA.cuEventRecordWithFlags(ctypes.c_void_p(ev.cuda_event),
                                         ctypes.c_void_p(stream.cuda_stream), ctypes.c_uint(1))
    if rc != 0:
        raise RuntimeError(f"cuEventRecordWithFlags failed ({rc})")


def max_over_ranks(x, world, dev):
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], device=dev if dist.get_backend() == "nccl" else "cpu", dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(x, world, dev):
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], device=dev if dist.get_backend() == "nccl" else "cpu", dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


def e2e_run(m, world, dev, steps, barrier):
    """End to end through the public API: pinned host inputs in, out + grads
    (bf16, the input dtype) back to pinned host memory, every step.  Copies
    run on their own streams, double-buffered, so step i+1's upload and step
    i-1's download overlap step i's kernels."""
    import torch

    from paper_2508_18224_b200 import nsa
    cfg = m["cfg"]
    bf = torch.bfloat16
    names = ("q", "k", "v", "dout", "tau")
    host_in = {n: t.cpu().pin_memory() for n, t in zip(names, m["inputs"])}
    h2d = sum(t.numel() * t.element_size() for t in host_in.values())
    dev_in = [{n: torch.empty_like(t, device=dev) for n, t in host_in.items()} for _ in range(2)]
    out_shapes = ((cfg.N, cfg.h, cfg.d_V), (cfg.N, cfg.h, cfg.d_K), (cfg.N, cfg.h_K, cfg.d_K),
                  (cfg.N, cfg.h_K, cfg.d_V))
    dev_out = [[torch.empty(s_, dtype=bf, device=dev) for s_ in out_shapes] for _ in range(2)]
    host_out = [[torch.empty(s_, dtype=bf).pin_memory() for s_ in out_shapes] for _ in range(2)]
    d2h = sum(x.numel() * x.element_size() for x in host_out[0])
    comp = torch.cuda.current_stream()
    up, down = torch.cuda.Stream(), torch.cuda.Stream()
    in_ready, in_free, out_ready, out_free = ([torch.cuda.Event() for _ in range(2)] for _ in range(4))

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
    for i in range(steps):
        if i + 1 < steps:
            upload(i + 1)
        e2e_step(i)
    comp.wait_stream(down)
    e_stop.record(comp)
    torch.cuda.synchronize()
    return e_start.elapsed_time(e_stop) / steps, h2d, d2h


def count_launches(m):
    """Our kernels launched in one step (profiler, outside the timed region)."""
    import torch

    from paper_2508_18224_b200 import nsa
    q, k, v, dout, tau = m["inputs"]
    names, kms = {}, {}
    try:
        from torch.profiler import ProfilerActivity, profile
        with profile(activities=[ProfilerActivity.CUDA]) as prof:
            out, ctx = nsa.nsa_forward(q, k, v, tau, m["cfg"])
            nsa.nsa_backward(ctx, dout)
            torch.cuda.synchronize()
        for e in prof.key_averages():
            if e.device_type is not None and "fsa" in e.key and e.count:
                names[e.key[:80]] = names.get(e.key[:80], 0) + e.count
                t_us = getattr(e, "device_time_total", None) or getattr(e, "cuda_time_total", 0)
                kms[e.key[:80]] = round(t_us / 1e3, 4)
        return sum(names.values()), {"launches": names, "device_ms_profiled": kms}
    except Exception as exc:  # pragma: no cover
        return None, {"profiler_error": str(exc)[:120]}


def run_ours(args, rank, world, local_rank):
    import torch

    # FSA_BENCH_ONE_GPU=1: every rank on cuda:0 with gloo collectives -- a
    # functional check of the N > 1 path on a one-GPU box (timings meaningless)
    one_gpu = os.environ.get("FSA_BENCH_ONE_GPU") == "1"
    if one_gpu:
        local_rank = 0
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    if world > 1:
        import torch.distributed as dist
        if one_gpu:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)

    def barrier():
        if world > 1:
            import torch.distributed as dist
            dist.barrier()

    hbm, pk_burst, pk_sus, pk_src = _peaks()
    traffic = {}
    try:  # dram__bytes_read.sum + dram__bytes_write.sum per launch, committed ncu capture
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as fh:
            traffic = json.load(fh)
    except Exception:
        pass

    sampler = ClockSampler(local_rank)
    sampler.start()
    m = measure(HEADLINE, WORKLOADS[HEADLINE], rank, world, dev, args.steps, args.warmup, barrier,
                use_graph=not args.no_graph)
    clocks = sampler.stop()
    cfg0 = m["cfg0"]
    ms = max_over_ranks(m["ms"], world, dev)
    k5_ms = max_over_ranks(m["k5_ms"], world, dev)
    k8_ms = max_over_ranks(m["k8_ms"], world, dev)
    merge_ms = max_over_ranks(m["merge_ms"] or 0.0, world, dev)
    dqr_ms = max_over_ranks(m["dqr_ms"] or 0.0, world, dev)
    R_rank = m["R"]
    R_all = sum_over_ranks(R_rank, world, dev)
    gpu_launches, kernel_names = count_launches(m)
    if gpu_launches is not None:
        gpu_launches *= args.steps
    e2e_ms, h2d, d2h = e2e_run(m, world, dev, max(args.steps, 10), barrier)
    e2e_ms = max_over_ranks(e2e_ms, world, dev)
    h2d, d2h = sum_over_ranks(h2d, world, dev), sum_over_ranks(d2h, world, dev)
    del m

    step_flops = algorithmic_flops(cfg0, R_all)

    def roof(kernel, flops, kms, algo, tkey):
        # burst peak: a kernel timed alone inside a 20-step loop at full clocks
        ach = flops / (kms / 1e3) / 1e12
        return {"kernel": kernel, "bound": "tensor", "achieved": round(ach, 2), "peak": pk_burst,
                "unit": "TFLOP/s", "frac": round(ach / pk_burst, 4),
                "traffic": traffic.get(tkey), "peak_source": f"{pk_src} bf16 burst",
                "kernel_ms": round(kms, 4), "share_of_step": round(kms / ms, 4),
                "algorithmic": algo}

    def hbm_roof(nbytes, kms, peak, algo):
        if not kms:
            return None
        ach = nbytes / (kms / 1e3) / 1e9
        return {"bound": "hbm", "achieved": round(ach, 1), "peak": peak, "unit": "GB/s",
                "frac": round(ach / peak, 4), "kernel_ms": round(kms, 4), "algorithmic": algo}

    nhd = cfg0.N * (cfg0.h // world) * cfg0.d_V
    merge_bytes = R_rank * (2 * cfg0.d_V + 8) + 2 * nhd * 4 + nhd * 4 + nhd * 2
    dqr_bytes = R_rank * (2 * cfg0.d_K + 4) + nhd * 4 + nhd * 4
    # per-rank FLOPs of the selected kernels (R of the rank's shard)
    k5_flops = 4.0 * cfg0.d_K * cfg0.B_K * R_rank
    k8_flops = 10.0 * cfg0.d_K * cfg0.B_K * R_rank
    line = {
        "metric": METRIC,
        "value": round(cfg0.N / (ms / 1e3), 1),
        "unit": "tokens/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(ms, 4),
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "bf16",
        "data": "synthetic N(0,1) Q/K/V/dOut, U[0,1) gates, random init",
        "config": arm_config(world, HEADLINE),
        "timing": "CUDA graph of the K timed steps, one replay between CUDA events"
                  if not args.no_graph else "eager launches between CUDA events",
        "effective_tflops": round(step_flops / (ms / 1e3) / 1e12, 2),
        # dominant kernel: the selected-attention backward (K8)
        "roofline": roof("sel_bwd (K8, tcgen05, selected branch)", k8_flops, k8_ms,
                         "10*d*B_K*R FLOPs per launch, R = (query head, token, block) rows = %d "
                         "on this rank" % R_rank, "tc_sel_bwd_selected"),
        "roofline_sel_fwd": roof("sel_fwd (K5, tcgen05)", k5_flops, k5_ms,
                                 "4*d*B_K*R FLOPs per launch, R = %d on this rank" % R_rank,
                                 "tc_sel_fwd"),
        # the two HBM-bound kernels around the FSA partial buffers
        "roofline_hbm": {
            "merge (K6+K12)": hbm_roof(merge_bytes, merge_ms, hbm,
                                       "R*(2d+8) partial rows + 2 N h d*4 (out_cmp, out_slide) read, "
                                       "N h d*4 (out_sel) + N h d*2 (out) written"),
            "dq_reduce (K9)": hbm_roof(dqr_bytes, dqr_ms, hbm,
                                       "R*(2d+4) dq partial rows + N h d*4 (sliding dQ) read, "
                                       "N h d*4 (dQ) written"),
        },
        "e2e": {"value": round(cfg0.N / (e2e_ms / 1e3), 1), "unit": "tokens/s",
                "ms_per_step": round(e2e_ms, 3), "steps": max(args.steps, 10),
                "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h)},
        "gpu_launches": gpu_launches,
        "kernels_per_step": kernel_names,
        "clocks": clocks,
    }
    if not args.no_extras:
        extras = {}
        for name in ("llama3-8b-attn-32k", "llama3-8b-attn-64k"):
            x = measure(name, WORKLOADS[name], rank, world, dev, args.steps, args.warmup, barrier,
                        use_graph=not args.no_graph)
            xms = max_over_ranks(x["ms"], world, dev)
            xk5 = max_over_ranks(x["k5_ms"], world, dev)
            xk8 = max_over_ranks(x["k8_ms"], world, dev)
            xR = sum_over_ranks(x["R"], world, dev)
            c0 = x["cfg0"]
            extras[name] = {
                "tokens_per_s": round(c0.N / (xms / 1e3), 1), "ms_per_step": round(xms, 4),
                "effective_tflops": round(algorithmic_flops(c0, xR) / (xms / 1e3) / 1e12, 2),
                "k5_ms": round(xk5, 4), "k8_ms": round(xk8, 4),
                "k5_frac_burst": round(4.0 * c0.d_K * c0.B_K * x["R"] / (xk5 / 1e3) / 1e12 / pk_burst, 4),
                "k8_frac_burst": round(10.0 * c0.d_K * c0.B_K * x["R"] / (xk8 / 1e3) / 1e12 / pk_burst, 4),
                "config": arm_config(world, name)}
            del x
        line["extra_workloads"] = extras
    if rank == 0 and world == 1 and not args.no_cpu_baseline:  # rank 0 at N = 1 only
        line["cpu_baseline"] = cpu_baseline(sample_n=CPU_SAMPLE_N, steps=1)
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()
    return line


# ---------------------------------------------------------------------------
# CPU reference arm: the reference package itself (blockattn, installed
# offline into baseline/_ref with its compiled Cython core; it travels to the
# GPU box with the snapshot), through its own public API.  Its sliding branch
# is dense O(N^2) (oracle.py:39-44, 64-74, 102-131) -- 2 GB of float64 per head
# at 16K -- so that one branch runs the oracle's banded restatement.  Without
# baseline/_ref the whole step is the oracle port.
# ---------------------------------------------------------------------------
REF_PATH = os.path.join(ROOT, "baseline", "_ref")


def _reference_importable():
    if not os.path.isdir(os.path.join(REF_PATH, "blockattn")):
        return False
    sys.path.insert(0, REF_PATH)
    try:
        import blockattn  # noqa: F401
        return blockattn.get_backend() == "compiled"
    except Exception:
        return False


def _ref_group(args_tuple):
    """One KV group of the headline workload on its first n_tok tokens, through
    blockattn's public API: compress_kv -> importance scores -> top-k ->
    compressed / selected (kv_major) / sliding forward -> gated combine, then
    the selected backward (kv_major.selected_backward) and the sliding
    backward -- the reference's differentiable branches."""
    n_tok, seed = args_tuple
    os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
    sys.path.insert(0, REF_PATH)
    import blockattn as ba
    import blockattn.rng as brng
    from blockattn import kv_major
    from oracle import fsa_oracle as O
    w = WORKLOADS[HEADLINE]
    g = w["h"] // w["h_K"]
    cfg = ba.make_config(N=n_tok, d_K=w["d"], d_V=w["d"], h=g, h_K=1, B_K=w["B_K"], T=w["T"], W=w["W"])
    Q, K, V = brng.make_qkv(cfg, seed)
    dO = brng.make_dout(cfg, seed)
    tau = brng.make_gates(cfg, seed)
    c = O.cfg_of(N=n_tok, d_K=w["d"], d_V=w["d"], h=g, h_K=1, B_K=w["B_K"], T=w["T"], W=w["W"])
    t0 = time.perf_counter()
    cmp = ba.compress_kv(K, V, cfg)
    sel = ba.select_topk_blocks(ba.importance_scores_from_compressed(Q, cmp.K_cmp, cfg), cfg)
    o_cmp = ba.compressed_attention_forward(Q, cmp, cfg)
    o_sel, _ = kv_major.selected_forward(Q, K, V, sel, cfg)
    o_sl, _ = O.sliding_forward(Q, K, V, c)  # banded (the reference's is dense O(N^2))
    ba.gated_combine([o_cmp, o_sel, ba.AttentionOutput(o_sl, None)], tau, cfg)
    kv_major.selected_backward(Q, K, V, sel, dO * tau[:, 1][:, None, None], cfg)
    O.sliding_backward(Q, K, V, dO * tau[:, 2][:, None, None], c)
    return time.perf_counter() - t0


def _cpu_group(args_tuple):
    n_tok, seed = args_tuple
    os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
    from oracle import fsa_oracle as O
    w = WORKLOADS[HEADLINE]
    c = O.cfg_of(N=n_tok, d_K=w["d"], d_V=w["d"], h=w["h"] // w["h_K"], h_K=1, B_K=w["B_K"],
                 T=w["T"], W=w["W"])
    Q, K, V = O.make_qkv(c, seed)
    dO = O.make_dout(c, seed)
    tau = O.make_gates(c, seed)
    t0 = time.perf_counter()
    O.nsa_forward_backward_group(Q, K, V, dO, tau, c)
    return time.perf_counter() - t0


def cpu_baseline(sample_n=CPU_SAMPLE_N, steps=1):
    """The reference (or, without baseline/_ref, the oracle port) on the host
    cores: one process per KV group (bit-exact sharding); sample =
    the first ``sample_n`` tokens of each KV group of the headline workload."""
    import multiprocessing as mp
    w = WORKLOADS[HEADLINE]
    cores = max(1, min(len(os.sched_getaffinity(0)), w["h_K"]))
    real = _reference_importable()
    fn = _ref_group if real else _cpu_group
    times = []
    with mp.get_context("spawn").Pool(cores) as pool:
        for s in range(steps):
            t0 = time.perf_counter()
            pool.map(fn, [(sample_n, 100 + s * 16 + kh) for kh in range(w["h_K"])])
            times.append(time.perf_counter() - t0)
    wall = statistics.median(times)
    what = ("blockattn (baseline/_ref, compiled Cython core) public API; the sliding branch "
            "as the oracle's banded restatement (the reference's is dense O(N^2))" if real
            else "the oracle port (float64 numpy)")
    return {"value": round(sample_n / wall, 2), "unit": "tokens/s", "cores": cores,
            "kind": "reference" if real else "port",
            "sample": f"all {w['h_K']} KV groups of {HEADLINE}, first {sample_n} tokens "
                      f"(N={sample_n} causal prefix of the 131072-token sequence), NSA fwd+bwd "
                      f"via {what}, {cores} processes; {wall:.1f} s wall"}


def arm_config(world, name=HEADLINE, seq_len=None, sample=None):
    """The workload an arm reports."""
    w = WORKLOADS[name]
    c = {"workload": name, "seq_len": w["N"] if seq_len is None else seq_len, "batch": 1,
         "q_heads": w["h"], "kv_heads": w["h_K"], "head_dim": w["d"], "block": w["B_K"],
         "top_k": w["T"], "window": w["W"], "parallelism": f"kv-head shards x{world}",
         "l2": "inputs exceed L2 (Q and dOut 1.3 GB each at 128K, slot-partial buffers "
               "21 GB); no flush"}
    if sample:
        c["sample"] = sample
    return c


def run_reference(args, rank, world):
    if rank != 0:
        return None
    n = CPU_SAMPLE_N
    cb = cpu_baseline(sample_n=n, steps=max(1, min(args.steps, 3)))
    return {
        "impl": "reference",
        "metric": METRIC,
        "value": cb["value"], "unit": "tokens/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic",
        "config": arm_config(world, HEADLINE, seq_len=n,
                             sample=f"first {n} tokens (causal prefix) of every kv group of the "
                                    f"{WORKLOADS[HEADLINE]['N']}-token workload"),
        "cpu_baseline": cb,
        "e2e": {"value": cb["value"], "unit": "tokens/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extras", action="store_true", help="skip the Llama 32K / 64K extra keys")
    ap.add_argument("--no-graph", action="store_true", help="time eager launches (no CUDA graph)")
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

"""Kernel timeline of one CUDA-graph replay of the NSA step (torch.profiler /
CUPTI): per-kernel start, duration and the idle gap before it, to locate the
device time between the graph-timed step and the sum of kernel durations.

    python tools/graph_gaps.py [N h h_K]
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2508_18224_b200 as fsa  # noqa: E402
from paper_2508_18224_b200 import nsa  # noqa: E402

N, h, hk = (int(x) for x in sys.argv[1:4]) if len(sys.argv) > 3 else (131072, 40, 8)
cfg = fsa.make_config(N=N, d_K=128, d_V=128, h=h, h_K=hk, B_K=64, T=16, W=512)
g = torch.Generator(device="cuda").manual_seed(0)
mk = lambda *s: torch.randn(*s, device="cuda", dtype=torch.bfloat16, generator=g)  # noqa: E731
q, k, v, do = mk(N, h, 128), mk(N, hk, 128), mk(N, hk, 128), mk(N, h, 128)
tau = torch.rand(N, 3, device="cuda", generator=g)


def step():
    out, ctx = nsa.nsa_forward(q, k, v, tau, cfg)
    return nsa.nsa_backward(ctx, do)


for _ in range(3):
    step()
torch.cuda.synchronize()
side = torch.cuda.Stream()
side.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(side):
    step()
torch.cuda.current_stream().wait_stream(side)
torch.cuda.synchronize()
graph = torch.cuda.CUDAGraph()
with torch.cuda.graph(graph):
    step()
graph.replay()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
graph.replay()
e1.record()
torch.cuda.synchronize()
print(f"graph step {e0.elapsed_time(e1):.3f} ms (events)")
from torch.profiler import ProfilerActivity, profile  # noqa: E402
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    graph.replay()
    torch.cuda.synchronize()
evs = [e for e in prof.events() if e.device_type is not None and str(e.device_type).endswith("CUDA")]
evs = sorted(evs, key=lambda e: e.time_range.start)
t0 = evs[0].time_range.start
prev_end = t0
busy = gaps = 0.0
rows = []
for e in evs:
    s, d = e.time_range.start, e.time_range.end - e.time_range.start
    gap = max(0.0, s - prev_end)
    rows.append((s - t0, d, gap, e.name[:70]))
    busy += d
    gaps += gap
    prev_end = max(prev_end, e.time_range.end)
span = prev_end - t0
print(f"span {span / 1e3:.3f} ms  kernels {busy / 1e3:.3f} ms  gaps {gaps / 1e3:.3f} ms  ({len(evs)} ops)")
for s, d, gap, name in rows:
    print(f"{s / 1e3:9.3f} {d / 1e3:8.3f} gap {gap:7.1f} us  {name}")

"""Per-entry-point device time of the NSA step (warm, CUDA events around every
C-ABI call on the launching stream).  python tools/kernel_times.py [N h h_K] [--full]"""
import collections
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2508_18224_b200 as fsa  # noqa: E402
from paper_2508_18224_b200 import _lib, nsa  # noqa: E402


def main():
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    N, h, hk = (int(a) for a in args) if args else (32768, 32, 8)
    full = "--full" in sys.argv
    cfg = fsa.make_config(N=N, d_K=128, d_V=128, h=h, h_K=hk, B_K=64, T=16, W=512)
    g = torch.Generator(device="cuda").manual_seed(0)
    mk = lambda *s: torch.randn(*s, device="cuda", dtype=torch.bfloat16, generator=g)  # noqa: E731
    q, k, v, do = mk(N, h, 128), mk(N, hk, 128), mk(N, hk, 128), mk(N, h, 128)
    tau = torch.rand(N, 3, device="cuda", generator=g)

    def step():
        _, ctx = nsa.nsa_forward(q, k, v, tau, cfg)
        nsa.nsa_backward(ctx, do, full=full)

    for _ in range(3):
        step()
    torch.cuda.synchronize()
    ev = collections.defaultdict(list)
    orig = _lib.call

    def timed(name, *a):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        r = orig(name, *a)
        e1.record()
        ev[name].append((e0, e1))
        return r

    steps = 5
    s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    _lib.call = timed
    s0.record()
    for _ in range(steps):
        step()
    s1.record()
    _lib.call = orig
    torch.cuda.synchronize()
    tot = s0.elapsed_time(s1) / steps
    rows = []
    for name, lst in ev.items():
        per = len(lst) // steps
        ms = [e0.elapsed_time(e1) for e0, e1 in lst]
        rows.append((statistics.median(ms) * per, per, name))
    rows.sort(reverse=True)
    print(f"N={N} h={h} h_K={hk} full={full}: step {tot:.3f} ms (with event overhead)")
    for ms, per, name in rows:
        print(f"  {ms:7.3f} ms  {100 * ms / tot:5.1f}%  x{per}  {name}")
    print(f"  {sum(r[0] for r in rows):7.3f} ms  sum of C-ABI calls")


if __name__ == "__main__":
    main()

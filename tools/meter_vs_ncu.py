"""the reference's value-independent TrafficMeter (meter.py
closed forms, kv_major.py:89-102, :186-203, :229-241, :285-354) against the
DRAM traffic ncu measured for the kernels that implement each phase.

    python tools/meter_vs_ncu.py        (GPU: needs the inverse index of a real selection)

Reads profiles/traffic.json (dram__bytes_read.sum + dram__bytes_write.sum per
launch) and prints a markdown table.  The meter counts LOGICAL bytes at
bytes_per_elem = 2 (bf16); ncu counts DRAM bytes after L2 -- gathered query
rows hit L2 (head-major task order), so loads are expected far below the
meter, stores (the partial rows, streamed past L2) close to it."""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2508_18224_b200 as fsa  # noqa: E402
from paper_2508_18224_b200 import meter, nsa  # noqa: E402


def main():
    cfg = fsa.make_config(N=32768, d_K=128, d_V=128, h=32, h_K=8, B_K=64, T=16, W=512)
    g = torch.Generator(device="cuda").manual_seed(0)
    mk = lambda *s: torch.randn(*s, device="cuda", dtype=torch.bfloat16, generator=g)  # noqa: E731
    q, k, v = mk(cfg.N, 32, 128), mk(cfg.N, 8, 128), mk(cfg.N, 8, 128)
    tau = torch.rand(cfg.N, 3, device="cuda", generator=g)
    _, ctx = nsa.nsa_forward(q, k, v, tau, cfg)
    nv = ctx.inv.n_valid
    fwd = meter.forward_meter(nv, cfg)
    bwd = meter.backward_meter(nv, cfg)
    bp_f = fwd.phases["block_pass"]
    bp_b = bwd.phases["block_pass"]
    bwd_only_loaded = bp_b.bytes_loaded - bp_f.bytes_loaded
    bwd_only_stored = bp_b.bytes_stored - bp_f.bytes_stored
    tr = json.load(open(os.path.join(ROOT, "profiles", "traffic.json")))
    rows = [
        ("forward block pass (K5, tc_sel_fwd)", bp_f.bytes_loaded, bp_f.bytes_stored, tr.get("tc_sel_fwd")),
        ("backward block tasks (K8 selected)", bwd_only_loaded, bwd_only_stored, tr.get("tc_sel_bwd_selected")),
    ]
    print("| phase (meter.py) -> kernel | meter loaded GB | meter stored GB | meter total GB | ncu DRAM GB | ncu / meter |")
    print("|---|---|---|---|---|---|")
    for name, ld, stv, dram in rows:
        tot = ld + stv
        print(f"| {name} | {ld / 1e9:.2f} | {stv / 1e9:.2f} | {tot / 1e9:.2f} | "
              f"{(dram or 0) / 1e9:.2f} | {(dram or 0) / tot:.2f} |")
    print()
    print(f"n_valid total = {int(nv.sum())}; R = {int(nv.sum()) * cfg.g}")
    print("stores: meter forward block_pass stored = partial rows R*d_V*2 B;",
          f"{bp_f.bytes_stored / 1e9:.3f} GB vs the K5 DRAM write in profiles/r1_ncu_summary_final.md")


if __name__ == "__main__":
    main()

"""the reference's value-independent TrafficMeter (meter.py
closed forms, kv_major.py:89-102, :186-203, :229-241, :285-354) against what
ncu counts for the kernels that implement each phase -- loads, stores and
FLOPs (meter.py:1-28 says the meter models a kernel's traffic and work).

    # GPU: the meter of the profiled problem (tools/prof_k8.py's inputs)
    python tools/meter_vs_ncu.py dump N h h_K > meter.json
    # anywhere with ncu: compare with `ncu --set full` reports of K5 and K8
    python tools/meter_vs_ncu.py compare meter.json k5.ncu-rep k8.ncu-rep

Counters:
* loads  -> lts__t_sectors_srcunit_tex_op_read.sum x 32 B: every byte the SMs
  read through L2 (gathered Q / dOut rows, K / V tiles, statistics), before
  L2 hits are taken out -- the meter's logical loads are a model of exactly this;
* stores -> lts__t_sectors_srcunit_tex_op_write.sum x 32 B;
* DRAM   -> dram__bytes_read.sum + dram__bytes_write.sum (after L2);
* FLOPs  -> smsp__sass_inst_executed_op_utcmma.sum (tcgen05.mma instructions)
  x the kernel's FLOPs per instruction: K5 issues per 128-row item 8 M128xN64xK16
  (S) and 4 M128xN128xK16 (P.V) MMAs; K8 32 M128xN64xK16 (S, dP, dV^T, dK^T)
  and 4 M128xN128xK16 (dQ).
"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

MMA_N64, MMA_N128 = 2 * 128 * 64 * 16, 2 * 128 * 128 * 16
FLOP_PER_MMA = {"k5": (8 * MMA_N64 + 4 * MMA_N128) / 12, "k8": (32 * MMA_N64 + 4 * MMA_N128) / 36}


def dump(N, h, hk):
    import torch
    import paper_2508_18224_b200 as fsa
    from paper_2508_18224_b200 import meter, nsa

    cfg = fsa.make_config(N=N, d_K=128, d_V=128, h=h, h_K=hk, B_K=64, T=16, W=512)
    g = torch.Generator(device="cuda").manual_seed(0)  # the inputs of tools/prof_k8.py
    mk = lambda *s: torch.randn(*s, device="cuda", dtype=torch.bfloat16, generator=g)  # noqa: E731
    q, k, v = mk(N, h, 128), mk(N, hk, 128), mk(N, hk, 128)
    tau = torch.rand(N, 3, device="cuda", generator=g)
    _, ctx = nsa.nsa_forward(q, k, v, tau, cfg)
    nv = ctx.inv.n_valid
    fwd = meter.forward_meter(nv, cfg)
    bwd = meter.backward_meter(nv, cfg)
    ph = lambda m, n: {a: int(getattr(m.phases[n], a)) for a in ("bytes_loaded", "bytes_stored", "flops")}  # noqa: E731
    out = {"N": N, "h": h, "h_K": hk, "nnz": int(nv.sum()), "R": int(nv.sum()) * cfg.g,
           "forward": {n: ph(fwd, n) for n in fwd.phases}, "backward": {n: ph(bwd, n) for n in bwd.phases}}
    print(json.dumps(out))


def _raw(rep):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr, units, data = rows[0], rows[1], rows[2]
    scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}

    def val(k):
        if k not in hdr:
            return float("nan")
        i = hdr.index(k)
        return float(data[i].replace(",", "")) * scale.get(units[i], 1.0)
    return {"l2_read": 32 * val("lts__t_sectors_srcunit_tex_op_read.sum"),
            "l2_write": 32 * val("lts__t_sectors_srcunit_tex_op_write.sum"),
            "dram": val("dram__bytes_read.sum") + val("dram__bytes_write.sum"),
            "mma": val("smsp__sass_inst_executed_op_utcmma.sum"),
            "ms": val("gpu__time_duration.sum") * 1e-6}


def compare(meter_json, k5_rep, k8_rep):
    m = json.load(open(meter_json))
    f = m["forward"]
    b = m["backward"]
    # the fused path has no stats pre-pass: K5 = the block pass; K8 = the
    # backward's block tasks (its meter recomputes the forward: subtract it)
    fb = f["block_pass"]
    bb = {a: b["block_pass"][a] - fb[a] for a in fb}
    rows = [("K5 tc_sel_fwd <- forward block_pass (kv_major.py:186-203)", fb, _raw(k5_rep), "k5"),
            ("K8 tc_sel_bwd <- backward block tasks (kv_major.py:285-324)", bb, _raw(k8_rep), "k8")]
    print(f"Problem: N={m['N']}, h={m['h']}, h_K={m['h_K']}; nnz = {m['nnz']}, R = {m['R']} "
          "(bytes_per_elem = 2)\n")
    print("| kernel <- meter phase | meter loads GB | L2 reads GB | ratio | meter stores GB | L2 writes GB "
          "| ratio | DRAM GB | meter GFLOP | tcgen05.mma GFLOP | ratio |")
    print("|---|---|---|---|---|---|---|---|---|---|---|")
    for name, mt, nc, kk in rows:
        fl = nc["mma"] * FLOP_PER_MMA[kk]
        print(f"| {name} | {mt['bytes_loaded'] / 1e9:.2f} | {nc['l2_read'] / 1e9:.2f} | "
              f"{nc['l2_read'] / mt['bytes_loaded']:.2f} | {mt['bytes_stored'] / 1e9:.2f} | "
              f"{nc['l2_write'] / 1e9:.2f} | {nc['l2_write'] / mt['bytes_stored']:.2f} | "
              f"{nc['dram'] / 1e9:.2f} | {mt['flops'] / 1e9:.0f} | {fl / 1e9:.0f} | {fl / mt['flops']:.3f} |")


if __name__ == "__main__":
    if sys.argv[1] == "dump":
        dump(*(int(x) for x in sys.argv[2:5]))
    else:
        compare(*sys.argv[2:5])

"""Print a bench.py JSON line as a per-kernel table (read here, no GPU).

    python tools/bench_summary.py gpurun_out/bench.json
"""
import json
import sys


def main():
    d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    print(f"value {d['value']:.0f} {d['unit']}  ms/step {d['ms_per_step']:.3f}  e2e ms {d['e2e']['ms_per_step']:.2f}"
          f"  clocks {d['clocks']}")
    for key in ("roofline", "roofline_sel_fwd"):
        r = d[key]
        print(f"{key}: {r['kernel']} {r['kernel_ms']:.3f} ms frac {r['frac']:.3f} share {r['share_of_step']:.3f}")
    k = d["kernels_per_step"]["device_ms_profiled"]
    for n, v in sorted(k.items(), key=lambda x: -x[1]):
        print(f"{v:8.3f}  {n[:100]}")
    print(f"{sum(k.values()):8.3f}  (sum)")
    for w, x in d.get("extra_workloads", {}).items():
        print(w, {a: x[a] for a in ("ms_per_step", "k5_ms", "k8_ms", "k5_frac_burst", "k8_frac_burst")})


if __name__ == "__main__":
    main()

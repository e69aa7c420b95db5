"""Compact per-launch summary of an ncu report (read here, no GPU needed).

    python tools/ncu_summary.py gpurun_out/prof.ncu-rep [--source]

Prints duration, DRAM bytes / throughput, tensor-pipe activity, L2 hit rate,
issue activity and registers per launch; --source adds the top stall lines.
"""

import csv
import io
import subprocess
import sys

METRICS = [
    ("ms", "gpu__time_duration.sum", 1e-6),
    ("dram_rd_GB", "dram__bytes_read.sum", 1e-9),
    ("dram_wr_GB", "dram__bytes_write.sum", 1e-9),
    ("dram_%", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", 1),
    ("tensor_%", "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed", 1),
    ("L2hit_%", "lts__t_sector_hit_rate.pct", 1),
    ("L2_%", "lts__throughput.avg.pct_of_peak_sustained_elapsed", 1),
    ("issue_%", "smsp__issue_active.avg.pct_of_peak_sustained_active", 1),
    ("regs", "launch__registers_per_thread", 1),
]


def _csv(args):
    out = subprocess.run(["ncu"] + args, capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


def main():
    rep = sys.argv[1]
    rows = _csv(["-i", rep, "--page", "raw", "--csv"])
    hdr, units, data = rows[0], rows[1], rows[2:]
    col = {h: i for i, h in enumerate(hdr)}
    name_i = col.get("Kernel Name")
    print("  ".join(f"{m[0]:>10}" for m in METRICS) + "  kernel")
    for r in data:
        vals = []
        for label, key, scale in METRICS:
            i = col.get(key)
            if i is None:
                vals.append(f"{'-':>10}")
                continue
            try:
                v = float(r[i].replace(",", "")) if r[i] else 0.0
            except ValueError:  # "no data" (metric not collected for this launch)
                v = float("nan")
            u = units[i]
            if key.startswith("gpu__time"):
                v *= {"ns": 1, "nsecond": 1, "us": 1e3, "usecond": 1e3, "ms": 1e6, "msecond": 1e6}.get(u, 1)
            if key.startswith("dram__bytes") and u in ("Mbyte", "MB"):
                v *= 1e6
            elif key.startswith("dram__bytes") and u in ("Gbyte", "GB"):
                v *= 1e9
            elif key.startswith("dram__bytes") and u in ("Kbyte", "KB"):
                v *= 1e3
            vals.append(f"{v * scale:>10.3f}")
        print("  ".join(vals) + "  " + (r[name_i][:60] if name_i is not None else ""))
    if "--source" in sys.argv:
        which = 0
        for a in sys.argv:
            if a.startswith("--kernel="):
                which = int(a.split("=")[1])
        src = _csv(["-i", rep, "--page", "source", "--csv", "--print-source", "sass"])
        sections, cur = [], None
        for r in src:
            if r and r[0] == "Kernel Name":
                cur = {"hdr": None, "rows": []}
                sections.append(cur)
            elif cur is not None and r and r[0] == "Address":
                cur["hdr"] = r
            elif cur is not None and cur["hdr"] and len(r) == len(cur["hdr"]):
                cur["rows"].append(r)
        if not sections:
            print("no source page")
            return
        sec = sections[min(which, len(sections) - 1)]
        h = sec["hdr"]
        ci = {x: i for i, x in enumerate(h)}
        key = "Warp Stall Sampling (All Samples)"
        body = [r for r in sec["rows"] if r[ci[key]].replace(".", "").isdigit()]
        tot = sum(float(r[ci[key]]) for r in body) or 1.0
        order = sorted(range(len(body)), key=lambda k: -float(body[k][ci[key]]))
        print(f"stall samples: {tot:.0f} ({len(sections)} kernel sections, showing #{which})")
        for k in order[:int(dict(a.split("=") for a in sys.argv if a.startswith("--top=")).get("--top", 30))]:
            r = body[k]
            print(f"{100 * float(r[ci[key]]) / tot:6.2f}%  [{k:5d}] {r[ci['Source']].strip()[:100]}")


if __name__ == "__main__":
    main()

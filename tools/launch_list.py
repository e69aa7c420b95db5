"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch log.

    python tools/launch_list.py gpurun_out/launches.csv [--last-half | --last=K]

Groups launches by kernel name and prints ms, share and launch count; with
--last-half only the second half of the launches is used (the second of two
identical steps, i.e. warm code paths).
"""

import collections
import csv
import sys


def main():
    rows = list(csv.reader(open(sys.argv[1])))
    hdr, data = None, []
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    if "--last-half" in sys.argv:
        data = data[len(data) // 2:]
    for a in sys.argv:
        if a.startswith("--last="):
            data = data[-int(a.split("=")[1]):]
    scale = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0}
    ms, cnt = collections.defaultdict(float), collections.Counter()
    for d in data:
        name = d["Kernel Name"]
        name = name.split("(")[0] if "(" in name else name
        ms[name] += float(d["Metric Value"].replace(",", "")) * scale.get(d["Metric Unit"], 1.0)
        cnt[name] += 1
    tot = sum(ms.values())
    print("#   ms      share  launches  kernel")
    for name, v in sorted(ms.items(), key=lambda x: -x[1]):
        print(f"{v:8.3f}  {100 * v / tot:5.1f}%  {cnt[name]:4d}      {name[:80]}")
    print(f"{tot:8.3f}  total ({sum(cnt.values())} launches)")


if __name__ == "__main__":
    main()

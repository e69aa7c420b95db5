"""Top CUDA source lines by warp-stall samples of an ncu report (--import-source on, -lineinfo).

    python tools/ncu_lines.py report.ncu-rep [--top N]
"""
import csv
import io
import subprocess
import sys


def main():
    rep = sys.argv[1]
    top = int(sys.argv[sys.argv.index("--top") + 1]) if "--top" in sys.argv else 40
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass,cuda"],
                         capture_output=True, text=True).stdout
    f, hdr, rows = "?", None, []
    for r in csv.reader(io.StringIO(out)):
        if len(r) == 2 and r[0] == "File Path":
            f = r[1].split("/")[-1]
            continue
        if r and r[0] == "Line No":
            hdr = r
            continue
        if hdr and len(r) == len(hdr) and r[0]:
            try:
                v = float(r[4] or 0)
                ni = float(r[5] or 0)
            except ValueError:
                continue
            rows.append((v, ni, f, r[0], r[1][:100]))
    tot = sum(x[0] for x in rows) or 1
    rows.sort(reverse=True)
    print(f"stall samples {int(tot)} (all / not-issued)")
    for v, ni, f, ln, src in rows[:top]:
        print(f"{100 * v / tot:5.1f}% {100 * ni / tot:5.1f}%  {f}:{ln}  {src}")


if __name__ == "__main__":
    main()

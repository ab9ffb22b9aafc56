#!/usr/bin/env python
"""Per-source-line instructions executed and stall samples from an ncu report
(`--page source --print-source=cuda,sass`), hottest first.

    python tools/ncu_lines.py report.ncu-rep [--top N]
"""
import csv
import io
import subprocess
import sys


def main():
    rep = sys.argv[1]
    top = int(sys.argv[sys.argv.index("--top") + 1]) if "--top" in sys.argv else 40
    txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"],
                         capture_output=True, text=True).stdout
    fname, rows, tot_i, tot_s = "?", [], 0.0, 0.0
    for r in csv.reader(io.StringIO(txt)):
        if not r:
            continue
        if r[0] == "File Path":
            fname = r[1].split("/")[-1]
            continue
        if r[0] and r[0].isdigit() and len(r) > 8:
            try:
                inst, samp = float(r[7]), float(r[4])
            except ValueError:
                continue
            rows.append((inst, samp, f"{fname}:{r[0]}", r[1].strip()[:70]))
            tot_i += inst
            tot_s += samp
    rows.sort(key=lambda x: -x[0])
    print(f"total warp-instructions {tot_i:.4g}, stall samples {tot_s:.0f}")
    print(f"{'inst%':>6} {'stall%':>6}  line  source")
    for inst, samp, loc, src in rows[:top]:
        print(f"{100 * inst / tot_i:6.2f} {100 * samp / max(tot_s, 1):6.2f}  {loc:28s} {src}")


if __name__ == "__main__":
    main()

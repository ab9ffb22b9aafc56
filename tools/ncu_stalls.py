#!/usr/bin/env python
"""Stall reasons per source-line group from an ncu report (cuda,sass source page).

    python tools/ncu_stalls.py report.ncu-rep [--top N]
Prints, for the hottest source lines by stall samples, the split by reason.
"""
import csv
import io
import subprocess
import sys

REASONS = ["stall_wait", "stall_short_sb", "stall_math", "stall_barrier", "stall_not_selected", "stall_selected",
           "stall_dispatch", "stall_no_inst", "stall_long_sb", "stall_mio", "stall_branch_resolving", "stall_lg"]


def main():
    rep = sys.argv[1]
    top = int(sys.argv[sys.argv.index("--top") + 1]) if "--top" in sys.argv else 30
    txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"],
                         capture_output=True, text=True).stdout
    fname, hdr, rows = "?", None, []
    tot = {r: 0.0 for r in REASONS}
    for r in csv.reader(io.StringIO(txt)):
        if not r:
            continue
        if r[0] == "File Path":
            fname = r[1].split("/")[-1]
        elif r[0] == "Line No":
            hdr = r
        elif hdr and r[0].isdigit():
            d = dict(zip(hdr, r))
            vals = {}
            for k in REASONS:
                try:
                    vals[k] = float(d.get(k, 0) or 0)
                except ValueError:
                    vals[k] = 0.0
                tot[k] += vals[k]
            rows.append((sum(vals.values()), f"{fname}:{r[0]}", r[1].strip()[:50], vals))
    rows.sort(key=lambda x: -x[0])
    T = sum(tot.values()) or 1
    print("total by reason:", ", ".join(f"{k[6:]} {100 * v / T:.1f}%" for k, v in sorted(tot.items(), key=lambda x: -x[1])))
    short = [k[6:] for k in REASONS]
    print(f"{'all%':>5}  " + " ".join(f"{s[:7]:>7}" for s in short) + "  line")
    for s, loc, src, vals in rows[:top]:
        print(f"{100 * s / T:5.1f}  " + " ".join(f"{100 * vals[k] / T:7.2f}" for k in REASONS) + f"  {loc} {src}")


if __name__ == "__main__":
    main()

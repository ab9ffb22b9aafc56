#!/usr/bin/env python
"""Summarise an ncu report's SASS source page: instructions executed and warp-stall
samples per opcode, plus the hottest instructions.

    python tools/ncu_sass_summary.py report.ncu-rep [kernel-regex] [--top N]
"""
import collections
import csv
import io
import re
import subprocess
import sys


def load(rep, kernel=None):
    cmd = ["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"]
    if kernel:
        cmd += ["-k", f"regex:{kernel}"]
    txt = subprocess.run(cmd, capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr, out = None, []
    for r in rows:
        if r and r[0] == "Address":
            hdr = r
            continue
        if hdr and len(r) >= len(hdr) - 1 and r[0].startswith("0x"):
            out.append(dict(zip(hdr, r)))
    return out


def num(x):
    try:
        return float(x)
    except (TypeError, ValueError):
        return 0.0


def main():
    argv = sys.argv[1:]
    top = 25
    if "--top" in argv:
        k = argv.index("--top")
        top = int(argv[k + 1])
        del argv[k:k + 2]
    args = argv
    rows = load(args[0], args[1] if len(args) > 1 else None)
    by_op = collections.defaultdict(lambda: [0.0, 0.0])
    tot_i = tot_s = 0.0
    for r in rows:
        op = re.sub(r"^@!?U?P\d+\s+", "", r["Source"].strip()).split(" ")[0]
        i, s = num(r["Instructions Executed"]), num(r["Warp Stall Sampling (All Samples)"])
        by_op[op][0] += i
        by_op[op][1] += s
        tot_i += i
        tot_s += s
    print(f"total warp-instructions {tot_i:.3e}, stall samples {tot_s:.0f}")
    print(f"{'opcode':24s} {'instr%':>8s} {'stall%':>8s}")
    for op, (i, s) in sorted(by_op.items(), key=lambda kv: -kv[1][1])[:30]:
        print(f"{op:24s} {100 * i / tot_i:8.2f} {100 * s / max(tot_s, 1):8.2f}")
    print("\nhottest instructions (stall samples):")
    for r in sorted(rows, key=lambda r: -num(r["Warp Stall Sampling (All Samples)"]))[:top]:
        print(f"{r['Address'][-5:]} {num(r['Warp Stall Sampling (All Samples)']):7.0f} "
              f"{num(r['Instructions Executed']):10.0f}  {r['Source'].strip()[:90]}")


if __name__ == "__main__":
    main()

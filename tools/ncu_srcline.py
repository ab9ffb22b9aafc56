"""Stall samples / executed instructions of an ncu source page (--print-source=sass csv) per
CUDA source line, via the line table of the kernel's cubin (nvdisasm -g output of the same build).
    python tools/ncu_srcline.py page.csv kernel_g.sass source.cu [top]"""
import collections
import csv
import re
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr, data = rows[1], rows[2:]
iS, iE = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
base = int(data[0][0], 16)
line, off2line = None, {}
src_name = sys.argv[3].split("/")[-1]
for l in open(sys.argv[2]):
    m = re.search(r'line (\d+)', l)
    if m:
        line = int(m.group(1)) if src_name in l else None
    m = re.match(r'\s*/\*([0-9a-f]{4,})\*/', l)
    if m:
        off2line[int(m.group(1), 16)] = line
tot = sum(float(r[iS]) for r in data)
by, byE, byR = collections.Counter(), collections.Counter(), collections.defaultdict(collections.Counter)
for r in data:
    ln = off2line.get(int(r[0], 16) - base)
    by[ln] += float(r[iS])
    byE[ln] += float(r[iE])
    for h in reasons:
        byR[ln][h] += float(r[hdr.index(h)] or 0)
src = open(sys.argv[3]).read().split("\n")
for ln, v in by.most_common(int(sys.argv[4]) if len(sys.argv) > 4 else 40):
    top = ", ".join(f"{k[6:]}={100 * x / tot:.1f}" for k, x in byR[ln].most_common(3))
    text = src[ln - 1].strip()[:70] if ln else "(other)"
    print(f"{100 * v / tot:5.1f}% {byE[ln] / 1e6:8.1f}M  {ln}: {text:70s} [{top}]")

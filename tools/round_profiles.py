#!/usr/bin/env python
"""Summarise a tools/capture_profiles.sh run into profiles/ (round tag, e.g. r01):

  profiles/<tag>_<cfg>_launches.csv   per-launch time and DRAM bytes of one bench step
                                      (the launches after the last L2-flush fill)
  profiles/<tag>_launch_summary.txt   per config: libga kernels of the step, their share
  profiles/traffic.json               "<cfg>:auto" -> DRAM bytes (read + write) of the step's
                                      libga launches (bench.py roofline.traffic)

    python tools/round_profiles.py r01 [gpurun_out]
"""
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def launches(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    h = rows[0]
    ki, mi, vi, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
    out = {}
    for r in rows[1:]:
        d = out.setdefault(int(r[ii]), {"name": r[ki]})
        d[r[mi]] = float(r[vi].replace(",", ""))
    return [out[k] for k in sorted(out)]


def ours(name):
    return any(s in name for s in ("ga::", "lnet", "band_kernel", "edge_kernel", "heavy_", "longnet", "scan_",
                                   "window_tc", "csr_mma", "csr_tma", "full_rows", "full_merge", "coo_", "bb::", "bwd::"))


def main():
    tag = sys.argv[1]
    src = sys.argv[2] if len(sys.argv) > 2 else os.path.join(ROOT, "gpurun_out")
    prof = os.path.join(ROOT, "profiles")
    tp = os.path.join(prof, "traffic.json")
    traffic = json.load(open(tp)) if os.path.exists(tp) else {}
    summary = [f"{tag}: one bench.py step per config under `ncu --metrics gpu__time_duration.sum,"
               "dram__bytes_read.sum,dram__bytes_write.sum --clock-control none` (cold caches, serialised;",
               "shares, not absolute times, are comparable with the bench's CUDA-event timing)", ""]
    for cfg in ("cfg1", "cfg2", "cfg3", "cfg3i", "cfg4", "cfg5"):
        p = os.path.join(src, f"launches_{cfg}.csv")
        if not os.path.exists(p):
            continue
        L = launches(p)
        last_fill = max(i for i, d in enumerate(L) if "FillFunctor" in d["name"])
        step = [d for d in L[last_fill + 1:] if ours(d["name"])]
        with open(os.path.join(prof, f"{tag}_{cfg}_launches.csv"), "w", newline="") as f:
            w = csv.writer(f)
            w.writerow(["kernel", "duration_us", "dram_read_bytes", "dram_write_bytes"])
            for d in step:
                w.writerow([d["name"][:120], round(d.get("gpu__time_duration.sum", 0) / 1e3, 2),
                            int(d.get("dram__bytes_read.sum", 0)), int(d.get("dram__bytes_write.sum", 0))])
        tot = sum(d.get("gpu__time_duration.sum", 0) for d in step)
        byts = sum(d.get("dram__bytes_read.sum", 0) + d.get("dram__bytes_write.sum", 0) for d in step)
        traffic[f"{cfg}:auto"] = int(byts)
        summary.append(f"{cfg}: {len(step)} libga launches, {tot / 1e6:.3f} ms, DRAM {byts / 1e9:.3f} GB")
        for d in step:
            t = d.get("gpu__time_duration.sum", 0)
            summary.append(f"    {100 * t / max(tot, 1):5.1f}%  {t / 1e3:10.1f} us  {d['name'][:90]}")
    json.dump(traffic, open(tp, "w"), indent=1, sort_keys=True)
    open(os.path.join(prof, f"{tag}_launch_summary.txt"), "w").write("\n".join(summary) + "\n")
    print("\n".join(summary))


if __name__ == "__main__":
    main()

#!/usr/bin/env python
"""Write a text summary of an ncu --set full report (key metrics + SASS opcode mix) and
update profiles/traffic.json with the kernel's DRAM bytes per launch.

    python tools/profile_summary.py REPORT.ncu-rep OUT.txt [--key cfg2:auto] [--kernel REGEX]
"""
import csv
import io
import json
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from ncu_sass_summary import load, num  # noqa: E402

METRICS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
    "sm__cycles_active.avg", "sm__cycles_elapsed.avg", "smsp__inst_executed.sum",
    "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "launch__registers_per_thread",
    "launch__shared_mem_per_block_dynamic", "launch__occupancy_limit_registers",
    "launch__occupancy_limit_shared_mem", "launch__grid_size", "launch__block_size",
    "sm__ops_path_tensor_op_hmma_src_bf16_dst_fp32_sparsity_off.avg.pct_of_peak_sustained_elapsed",
    "sm__ops_path_tensor_op_utchmma_src_bf16_dst_fp32_sparsity_off.avg.pct_of_peak_sustained_elapsed",
]


def raw(rep, kernel=None):
    cmd = ["ncu", "-i", rep, "--page", "raw", "--csv"]
    if kernel:
        cmd += ["-k", f"regex:{kernel}"]
    rows = list(csv.reader(io.StringIO(subprocess.run(cmd, capture_output=True, text=True).stdout)))
    h, u, v = rows[0], rows[1], rows[2]
    return {n: (v[i], u[i]) for i, n in enumerate(h)}, v[h.index("Kernel Name")] if "Kernel Name" in h else "?"


def main():
    a = sys.argv[1:]
    key = kernel = None
    if "--key" in a:
        k = a.index("--key"); key = a[k + 1]; del a[k:k + 2]
    if "--kernel" in a:
        k = a.index("--kernel"); kernel = a[k + 1]; del a[k:k + 2]
    rep, out = a[0], a[1]
    m, name = raw(rep, kernel)
    lines = [f"ncu --set full summary of {os.path.basename(rep)}", f"kernel: {name}", ""]
    for n in METRICS:
        if n in m:
            lines.append(f"{n:92s} {m[n][0]:>16s} {m[n][1]}")
    rows = load(rep, kernel)
    import collections
    by = collections.defaultdict(lambda: [0.0, 0.0])
    ti = ts = 0.0
    for r in rows:
        op = r["Source"].strip()
        op = op.split(" ")[1] if op.startswith("@") else op.split(" ")[0]
        i, s = num(r["Instructions Executed"]), num(r["Warp Stall Sampling (All Samples)"])
        by[op][0] += i; by[op][1] += s; ti += i; ts += s
    lines += ["", f"SASS opcode mix (warp-instructions {ti:.4g}, stall samples {ts:.0f}):",
              f"{'opcode':28s} {'instr%':>8s} {'stall%':>8s}"]
    for op, (i, s) in sorted(by.items(), key=lambda kv: -kv[1][0])[:28]:
        lines.append(f"{op:28s} {100 * i / max(ti, 1):8.2f} {100 * s / max(ts, 1):8.2f}")
    os.makedirs(os.path.dirname(os.path.abspath(out)), exist_ok=True)
    with open(out, "w") as f:
        f.write("\n".join(lines) + "\n")
    if key:
        tp = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "traffic.json")
        d = json.load(open(tp)) if os.path.exists(tp) else {}
        rd = num(m["dram__bytes_read.sum"][0]) * (1e6 if m["dram__bytes_read.sum"][1] == "Mbyte" else
                                                  1e9 if m["dram__bytes_read.sum"][1] == "Gbyte" else 1e3 if
                                                  m["dram__bytes_read.sum"][1] == "Kbyte" else 1)
        wr = num(m["dram__bytes_write.sum"][0]) * (1e6 if m["dram__bytes_write.sum"][1] == "Mbyte" else
                                                   1e9 if m["dram__bytes_write.sum"][1] == "Gbyte" else 1e3 if
                                                   m["dram__bytes_write.sum"][1] == "Kbyte" else 1)
        d[key] = int(rd + wr)
        json.dump(d, open(tp, "w"), indent=1, sort_keys=True)
    print("\n".join(lines[:30]))


if __name__ == "__main__":
    main()

#!/usr/bin/env python
"""bench.py — graph-view masked attention (arXiv 2502.01659) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config cfg4]
                    [--scaling weak|strong] [--no-per-config] [--max-context]

One "step" is one pass of the whole hot path (neighbour enumeration, scores, online
softmax, aggregation — one ga_attention call, or one ga_attention_sharded call per rank at N>1)
over the configuration's full synthetic input.  Default workload: the largest single-GPU
configuration of BASELINE.json, configs[3] (cfg4: L=2^24, d=64, bf16, LongNet(w0=2048,
alpha=2) implicit).  At N=1 the line also carries `per_config`: cfg2, cfg3 (explicit CSR, as
BASELINE.json names it), cfg3i (the same BigBird mask as an implicit descriptor) and cfg5
(L=160M, Window(128)), each with its own time, edges/s and roofline.

N>1 (torchrun, one process per GPU): --scaling weak (default) gives every rank L query rows
of an N*L-token sequence; --scaling strong cuts one L-token sequence into N shards.  K/V
shards sit in symmetric CUDA-IPC buffers and the kernels read the halo / long-range rows they
need from the other ranks' HBM over NVLink (CSR / BigBird: K/V all-gather).

metric: attention edges/s = (mask nnz x heads) / step time, whole job.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "attention edges/sec (graph-view masked attention; edges = mask nnz x heads)"
CONFIGS = {
    "cfg1": dict(L=1024, H=1, d=64, dtype="f32", mask=("window", 32, 1)),
    "cfg2": dict(L=65536, H=8, d=64, dtype="bf16", mask=("window", 256, 2)),
    "cfg3": dict(L=2 ** 20, H=1, d=64, dtype="bf16", mask=("bigbird", 128, 64, 64)),
    "cfg3i": dict(L=2 ** 20, H=1, d=64, dtype="bf16", mask=("bigbird_implicit", 128, 64, 64)),
    "cfg4": dict(L=2 ** 24, H=1, d=64, dtype="bf16", mask=("longnet", 2048, 2)),
    "cfg5": dict(L=160_000_000, H=1, d=64, dtype="bf16", mask=("window", 128, 1)),
}
SEEDS = {"cfg1": 0x5EED0001, "cfg2": 0x5EED0002, "cfg3": 0x5EED0003, "cfg3i": 0x5EED0003, "cfg4": 0x5EED0004,
         "cfg5": 0x5EED0005}
PER_CONFIG = ("cfg2", "cfg3", "cfg3i", "cfg5")  # extra N=1 lines next to the headline
BIGBIRD_SEED = 0xB16B12D
L2_FLUSH_BYTES = 256 << 20  # > 126 MB L2


def mask_desc(cfg):
    kind, *a = cfg["mask"]
    if kind == "window":
        return f"Window(w={a[0]}, r={a[1]})"
    if kind == "bigbird":
        return f"BigBird(window={a[0]}, globals={a[1]} evenly spaced, random={a[2]}/row) as explicit CSR"
    if kind == "bigbird_implicit":
        return f"BigBird(window={a[0]}, globals={a[1]} evenly spaced, random={a[2]}/row) implicit descriptor"
    return f"LongNet(w0={a[0]}, alpha={a[1]}) implicit"


def eb(dtype):
    return 4 if dtype == "f32" else 2


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            return json.load(f), "measured"
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0, "sm_max_mhz": 1965.0}, "fallback"


# ------------------------------------------------------------------ clocks sampler
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.lines:
            f = [x.strip() for x in line.split(",")]
            if len(f) < 8:
                continue
            try:
                sm.append(float(f[0]))
                mx.append(float(f[1]))
            except ValueError:
                continue
            for n, v in zip(names, f[4:8]):
                if v.lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ------------------------------------------------------------------ oracle arm
_ORACLE_INPUTS = {}


def oracle_rate(cfg_name, budget_s=15.0, max_rows=None):
    """Time the fp64 oracle (as it stands) on a bounded row sample of the workload.
    Returns (edges/s, threads, sample description, edges, seconds)."""
    import numpy as np

    import oracle

    cfg = CONFIGS[cfg_name]
    L, H, d = cfg["L"], cfg["H"], cfg["d"]
    seed = SEEDS[cfg_name]
    kind, *a = cfg["mask"]
    om = {"window": lambda: oracle.window(L, a[0], a[1]),
          "bigbird": lambda: oracle.bigbird(L, a[0], a[1], a[2], BIGBIRD_SEED),
          "bigbird_implicit": lambda: oracle.bigbird(L, a[0], a[1], a[2], BIGBIRD_SEED),
          "longnet": lambda: oracle.longnet(L, a[0], a[1])}[kind]()
    arrays = 3 * L * H * d * 8 <= 4 << 30
    if arrays:
        if cfg_name not in _ORACLE_INPUTS:
            _ORACLE_INPUTS[cfg_name] = oracle.inputs(seed, L, H, d, cfg["dtype"])
        qkv = _ORACLE_INPUTS[cfg_name]

    def run(rows):
        t0 = time.perf_counter()
        if arrays:
            _, e = oracle.attention(*qkv, om, rows=rows)
        else:
            _, e = oracle.attention_seeded(seed, cfg["dtype"], om, H, d, rows=rows)
        return e, time.perf_counter() - t0

    rng = np.random.default_rng(0)
    n = 32
    e, t = run(np.sort(rng.choice(L, n, replace=False)))
    while t < budget_s / 8 and n < L:
        n = min(L, n * 4)
        e, t = run(np.sort(rng.choice(L, n, replace=False)))
    target = int(n * budget_s / max(t, 1e-3))
    n = max(32, min(L, target, max_rows or L))
    rows = np.sort(rng.choice(L, n, replace=False))
    e, t = run(rows)
    sample = (f"{n} uniformly sampled query rows of {L} ({'fp64 arrays' if arrays else 'rows regenerated from the seed'}"
              f", all {H} heads), {e} edges")
    return e / t, oracle.num_threads(), sample, e, t


def backward_line(ga, torch, dist, dev, flush, args):
    """The backward pass (ga_attention_backward) on cfg2's workload: dQ, dK,
    dV of out = attention(Q, K, V, Window(256, 2)) for a seeded dO, lse recomputed (the whole
    backward: row pass lse + D + dQ, column pass dK + dV, on the tensor cores).  Algorithmic
    flops per head-edge: 2d for s, 2d for dP, 2d for dQ in the row pass plus 2d for the lse
    sweep, and 2d s + 2d dP + 2d dK + 2d dV in the column pass = 16d."""
    cfg = CONFIGS["cfg2"]
    L, H, d = cfg["L"], cfg["H"], cfg["d"]
    seed = SEEDS["cfg2"]
    mask = ga.Window(*cfg["mask"][1:])
    q, k, v = ga.qkv_device(seed, L, H, d, torch.bfloat16)
    g = ga.qkv_device(seed + 7, L, H, d, torch.bfloat16, shift=-0.5)[0]
    out = ga.attention(q, k, v, mask)

    class W:  # the time_steps interface
        pass
    w = W()
    w.ga = ga
    w.step = lambda: ga.attention_backward(q, k, v, out, g, mask)
    steps = max(3, min(args.steps, 10))
    ms, ps, launches, _ = time_steps(torch, dist, 1, w, steps, 3, flush)
    nnz = ga.mask_count(mask, L)
    he = nnz * H
    peaks, src = load_peaks()
    s = statistics.median(ps) / 1e3
    # the band backward runs on the tensor cores (mma.sync, bf16 in, fp32 accumulate):
    # flops against the measured dense bf16 peak; 3 exp2 per head-edge (lse sweep, row and
    # column passes) on MUFU; Q, K, V, O, dO read and dQ, dK, dV (fp32) written once on HBM
    flops = 16 * d * he
    t_f = flops / (peaks["bf16_tflops"] * 1e12)
    t_m = (5 * L * H * d * 2 + 3 * L * H * d * 4) / (peaks["hbm_gbs"] * 1e9)
    t_x = 3 * he / (MUFU_EX2_PER_CLK_SM * SMS * peaks.get("sm_max_mhz", 1965.0) * 1e6)
    byts = 5 * L * H * d * 2 + 3 * L * H * d * 4
    bound = max((t_m, "hbm"), (t_f, "tensor"), (t_x, "alu"))[1]
    if bound == "hbm":
        roof = {"bound": "hbm", "achieved": round(byts / s / 1e9, 1), "peak": peaks["hbm_gbs"], "unit": "GB/s",
                "frac": round(t_m / s, 4), "peak_source": f"hbm_gbs, {src} MEASURED_PEAKS.json"}
    elif bound == "tensor":
        roof = {"bound": "tensor", "achieved": round(flops / s / 1e12, 2), "peak": peaks["bf16_tflops"],
                "unit": "TFLOP/s", "frac": round(t_f / s, 4), "peak_source": f"bf16 dense tensor ({src})"}
    else:
        roof = {"bound": "alu", "achieved": round(3 * he / s / 1e9, 1), "unit": "Gexp2/s", "frac": round(t_x / s, 4),
                "peak_source": "MUFU.EX2 15.7/clk/SM measured x 148 SMs x max clock"}
    roof.update({"algorithmic": f"{byts} B, {flops} flop (16d x {he} head-edges) and {3 * he} exp2 per backward",
                 "lower_bound_us": {"tensor": round(t_f * 1e6, 2), "hbm": round(t_m * 1e6, 2), "mufu": round(t_x * 1e6, 2)},
                 "kernel_ms_median": round(statistics.median(ps), 4),
                 "kernels": "tensor-core band backward (backward_tc.cu): row pass (lse, D, dQ) + column pass (dK, dV)"})
    return {"workload": f"backward (dQ, dK, dV fp32) of cfg2: L={L}, {H} heads, d={d}, bf16, {mask_desc(cfg)}",
            "value": he / (ms / 1e3), "unit": "edges/s", "ms_per_step": ms, "steps": steps, "warmup": 3, "nnz": nnz,
            "gpu_launches": launches, "roofline": roof}


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def cpu_baseline_line(cfg_name, budget_s):
    """The oracle as it stands on the host cores (all threads), plus a 1-thread rate on a
    smaller sample; rows are sampled uniformly, so the full-workload time is extrapolated."""
    import oracle

    rate, cores, sample, e, t = oracle_rate(cfg_name, budget_s)
    nthreads = oracle.num_threads()
    oracle.set_num_threads(1)
    try:
        rate1, _, sample1, e1, t1 = oracle_rate(cfg_name, max(2.0, budget_s / 4))
    finally:
        oracle.set_num_threads(nthreads)
    cfg = CONFIGS[cfg_name]
    return {"value": rate, "unit": "edges/s", "cores": cores, "kind": "oracle", "sample": sample,
            "cpu_model": cpu_model(), "host_logical_cpus": os.cpu_count(),
            "rate_1thread": rate1, "sample_1thread": sample1,
            "full_workload_s_extrapolated": None if not rate else round(
                _nnz_host(cfg_name) * cfg["H"] / rate, 1),
            "note": "fp64 oracle (oracle/oracle.c, OpenMP over rows), timed on sampled query rows; "
                    "full-workload time extrapolated from the per-edge rate"}


def _nnz_host(cfg_name):
    import paper_2502_01659_b200 as ga

    cfg = CONFIGS[cfg_name]
    kind, *a = cfg["mask"]
    m = {"window": lambda: ga.Window(a[0], a[1]), "longnet": lambda: ga.LongNet(a[0], a[1]),
         "bigbird": lambda: ga.BigBird(a[0], a[1], a[2], seed=BIGBIRD_SEED),
         "bigbird_implicit": lambda: ga.BigBird(a[0], a[1], a[2], seed=BIGBIRD_SEED)}[kind]()
    return ga.mask_count(m, cfg["L"])


class Workload:
    """Inputs resident in HBM and the step function of one configuration on this rank."""

    def __init__(self, ga, torch, name, dev, world, rank, kernel, scaling):
        cfg = CONFIGS[name]
        self.name, self.cfg = name, cfg
        self.kind, *a = cfg["mask"]
        self.H, self.d = cfg["H"], cfg["d"]
        L0 = cfg["L"]
        if scaling == "strong" and world > 1:
            self.L = L0
            S = -(-L0 // world)
            self.r0, self.r1 = min(L0, rank * S), min(L0, (rank + 1) * S)
        else:
            self.L = L0 * world
            self.r0, self.r1 = rank * L0, (rank + 1) * L0
        self.L_local = self.r1 - self.r0
        tdt = {"f32": torch.float32, "bf16": torch.bfloat16}[cfg["dtype"]]
        seed = SEEDS[name]
        L, H, d = self.L, self.H, self.d
        self.ws = None
        if self.kind == "window":
            self.mask = ga.Window(a[0], a[1])
            self.nnz = ga.mask_count(self.mask, L)
        elif self.kind == "bigbird":
            self.mask = ga.mask_to_csr(ga.BigBird(a[0], a[1], a[2], seed=BIGBIRD_SEED), L)
            self.nnz = self.mask.nnz
            self.ws = torch.empty(ga.workspace_size(self.mask, L, d, H, tdt, q_begin=self.r0, q_rows=self.L_local),
                                  dtype=torch.uint8, device=dev)
        elif self.kind == "bigbird_implicit":
            self.mask = ga.BigBird(a[0], a[1], a[2], seed=BIGBIRD_SEED)
            self.nnz = ga.mask_count(self.mask, L)
            self.ws = torch.empty(ga.workspace_size(self.mask, L, d, H, tdt, q_begin=self.r0, q_rows=self.L_local),
                                  dtype=torch.uint8, device=dev)
        else:
            self.mask = ga.LongNet(a[0], a[1])
            self.nnz = ga.mask_count(self.mask, L)
            wsb = ga.workspace_size(self.mask, L, d, H, tdt, q_begin=self.r0, q_rows=self.L_local)
            self.ws = torch.empty(wsb, dtype=torch.uint8, device=dev) if wsb else None
        self.q = torch.empty((self.L_local, H, d), dtype=tdt, device=dev)
        ga.fill_inputs(self.q, seed, 0, self.r0 * H * d)
        self.comm = None
        if world > 1:
            from paper_2502_01659_b200.comm import Comm

            self.comm = Comm()
            S = -(-L // world)  # symmetric buffers: every rank allocates the largest shard
            self.k = self.comm.empty((S, H, d), tdt)[:self.L_local]
            self.v = self.comm.empty((S, H, d), tdt)[:self.L_local]
        else:
            self.k = torch.empty((self.L_local, H, d), dtype=tdt, device=dev)
            self.v = torch.empty_like(self.k)
        ga.fill_inputs(self.k, seed, 1, self.r0 * H * d)
        ga.fill_inputs(self.v, seed, 2, self.r0 * H * d)
        self.out = torch.empty_like(self.q)
        self.ga, self.kernel = ga, kernel
        self.edges_total = self.nnz * H  # all ranks together (one global mask)

    def step(self):
        if self.comm is not None:
            self.comm.attention(self.q, self.k, self.v, self.mask, self.L, out=self.out, kernel=self.kernel,
                                workspace=self.ws)
        else:
            self.ga.attention(self.q, self.k, self.v, self.mask, self.out, kernel=self.kernel, workspace=self.ws)

    def close(self):
        if self.comm is not None:
            self.comm.check()
            self.comm.close()
            self.comm = None
        self.q = self.k = self.v = self.out = self.ws = self.mask = None


def time_steps(torch, dist, world, wl, steps, warmup, flush, sampler=None):
    """W untimed steps; K timed steps, each bracketed by CUDA events on the launching stream
    with an L2 flush before it (outside the events); max over ranks."""
    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(warmup):
        wl.step()
    barrier()
    if sampler is not None:
        sampler.start()
    lib = wl.ga._abi.lib()
    launches0 = lib.ga_launch_count()
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
    barrier()
    for s in range(steps):
        flush.zero_()  # L2 flush between timed steps (outside the events)
        if world > 1:
            dist.barrier()
        starts[s].record()
        wl.step()
        ends[s].record()
    barrier()
    launches = lib.ga_launch_count() - launches0
    clocks = sampler.stop() if sampler is not None else None
    per_step = [st.elapsed_time(en) for st, en in zip(starts, ends)]
    total_ms = torch.tensor([sum(per_step)], dtype=torch.float64, device=flush.device)
    if world > 1:
        dist.all_reduce(total_ms, op=dist.ReduceOp.MAX)
    return total_ms.item() / steps, per_step, launches, clocks


def workload_desc(wl, world, scaling):
    cfg = wl.cfg
    shard = (f"L={wl.L_local}x{world}" if scaling == "weak" else f"L={wl.L} over {world} shards") if world > 1 \
        else f"L={wl.L}"
    return f"{wl.name}: {shard} tokens, {wl.H} heads, d={wl.d}, {cfg['dtype']}, {mask_desc(cfg)}"


# ------------------------------------------------------------------ main
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", choices=sorted(CONFIGS), default="cfg4")
    ap.add_argument("--kernel", default="auto", choices=["auto", "edge", "tiled", "window", "tc"])
    ap.add_argument("--scaling", choices=["weak", "strong"], default="weak")
    ap.add_argument("--no-per-config", action="store_true", help="skip the extra per-config lines at N=1")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--cpu-budget", type=float, default=15.0)
    ap.add_argument("--max-context", action="store_true",
                    help="measure the largest Window(128) bf16 sequence that fits (one step + sampled parity)")
    args = ap.parse_args()
    if args.warmup < 3:
        print("warning: --warmup < 3 violates the timing rules; using 3", file=sys.stderr)
        args.warmup = 3

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    cfg = CONFIGS[args.config]

    if args.impl == "reference":
        return reference_arm(args, cfg, world, rank)
    if args.max_context:
        return max_context(args, world, rank, local_rank)

    import torch
    import torch.distributed as dist

    import paper_2502_01659_b200 as ga

    dev = _init_dist(torch, dist, world, local_rank)
    flush = torch.empty(L2_FLUSH_BYTES, dtype=torch.uint8, device=dev)
    wl = Workload(ga, torch, args.config, dev, world, rank, args.kernel, args.scaling)
    sampler = ClockSampler(local_rank)
    ms, per_step, launches, clocks = time_steps(torch, dist, world, wl, args.steps, args.warmup, flush, sampler)
    value = wl.edges_total / (ms / 1e3)
    # ---- roofline for the dominant kernel (per rank's share of the work)
    roofline, gather = roofline_for(args.config, args.kernel, cfg, wl.kind, wl.edges_total * wl.L_local // wl.L,
                                    wl.L_local, wl.H, wl.d, wl.nnz * wl.L_local // wl.L, per_step)
    # ---- end-to-end through the public API with host buffers
    e2e = None
    if not args.no_e2e:
        c_abi = None
        if world == 1 and wl.kind != "bigbird":
            c_abi = (wl.mask, wl.q.cpu().pin_memory(), wl.k.cpu().pin_memory(), wl.v.cpu().pin_memory())
        e2e = measure_e2e(args, ga, world, dev, wl.edges_total, [wl.q, wl.k, wl.v], wl.step, wl.out, c_abi)
        c_abi = None
    workload = workload_desc(wl, world, args.scaling)
    conf = {"workload": workload, "L": wl.L, "heads": wl.H, "d": wl.d, "mask": mask_desc(cfg), "nnz": wl.nnz,
            "kernel": args.kernel,
            "parallelism": f"query-range shards x{world}" + (
                ", ga_attention_sharded (remote K/V rows read over NVLink peer memory"
                + (", K/V all-gather" if wl.kind.startswith("bigbird") else "") + ")" if world > 1 else ""),
            "l2": "flushed between timed steps (256 MiB write outside the events); inputs > L2"}
    wl.close()
    wl = None
    torch.cuda.empty_cache()

    # ---- the other BASELINE.json configurations at N=1
    per_config = None
    if world == 1 and not args.no_per_config:
        per_config = {}
        for name in PER_CONFIG:
            if name == args.config:
                continue
            w2 = Workload(ga, torch, name, dev, 1, 0, "auto", "weak")
            ms2, ps2, _, _ = time_steps(torch, dist, 1, w2, max(3, min(args.steps, 10)), 3, flush)
            roof2, _ = roofline_for(name, "auto", w2.cfg, w2.kind, w2.edges_total, w2.L_local, w2.H, w2.d, w2.nnz, ps2)
            per_config[name] = {"workload": workload_desc(w2, 1, "weak"), "value": w2.edges_total / (ms2 / 1e3),
                                "unit": "edges/s", "ms_per_step": ms2, "steps": max(3, min(args.steps, 10)),
                                "warmup": 3, "nnz": w2.nnz, "roofline": roof2}
            w2.close()
            w2 = None
            torch.cuda.empty_cache()
        per_config["cfg2_backward"] = backward_line(ga, torch, dist, dev, flush, args)
        torch.cuda.empty_cache()

    # ---- CPU oracle baseline (rank 0, N=1 only)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline_line(args.config, args.cpu_budget)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "edges/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "weak" if (world == 1 or args.scaling == "weak") else "strong",
            "vs_baseline": None, "dtype": cfg["dtype"], "accum": "f32", "data": "synthetic",
            "config": conf, "clocks": clocks, "roofline": roofline, "gather_model": gather, "cpu_baseline": cpu,
            "e2e": e2e, "gpu_launches": launches, "per_config": per_config,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


MUFU_EX2_PER_CLK_SM = 15.7  # measured, profiles/r01_microbench.txt (tools/microbench.cu)
SMS = 148


def roofline_for(cfg_name, kernel, cfg, kind, head_edges, L_local, H, d, nnz, per_step):
    """Roofline of the attention step: the binding resource is whichever
    lower-bound time is largest at the measured peaks.

    * HBM: algorithmic bytes per launch = Q, K, V read once + O written once (+ row_ptr and
      col_idx for explicit CSR) — no implementation can move less — at MEASURED_PEAKS hbm_gbs.
    * tensor: algorithmic flops = 4d per head-edge (2d for q.k, 2d for p*v) at the
      measured dense bf16 peak (fp32 inputs: the FP32 FMA pipe, 148 x 128 x 2 x clock).
    * alu (MUFU): one exp2 per head-edge — the online softmax's weight 2^(s - m) — at the
      measured MUFU.EX2 rate (15.7 /clk/SM x 148 SMs x max clock).
    The north-star "gather model" (every edge pulls K_j and V_j) is reported separately."""
    peaks, peak_src = load_peaks()
    kernel_ms = statistics.median(per_step)
    e = eb(cfg["dtype"])
    csr = kind == "bigbird"
    bytes_alg = 4 * L_local * H * d * e + ((L_local + 1) * 8 + nnz * 4 if csr else 0)
    flops_alg = 4 * d * head_edges
    hbm = peaks["hbm_gbs"]
    clk = peaks.get("sm_max_mhz", 1965.0) * 1e6
    if cfg["dtype"] == "f32":
        fpeak, funit = SMS * 128 * 2 * clk / 1e12, "fp32 FMA pipe (derived: 148 SMs x 128 FMA/clk x max clock)"
    else:
        fpeak, funit = peaks["bf16_tflops"], f"bf16 dense tensor ({peak_src} MEASURED_PEAKS.json)"
    xpeak = MUFU_EX2_PER_CLK_SM * SMS * clk  # exp2 / s
    t_mem, t_fl, t_ex = bytes_alg / (hbm * 1e9), flops_alg / (fpeak * 1e12), head_edges / xpeak
    s = kernel_ms / 1e3
    bound = max((t_mem, "hbm"), (t_fl, "tensor"), (t_ex, "alu"))[1]
    if bound == "hbm":
        ach = bytes_alg / s / 1e9
        roof = {"bound": "hbm", "achieved": round(ach, 1), "peak": hbm, "unit": "GB/s", "frac": round(ach / hbm, 4),
                "peak_source": f"hbm_gbs, {peak_src} MEASURED_PEAKS.json (copy bandwidth)"}
    elif bound == "tensor":
        ach = flops_alg / s / 1e12
        roof = {"bound": "tensor" if cfg["dtype"] != "f32" else "alu", "achieved": round(ach, 2), "peak": fpeak,
                "unit": "TFLOP/s", "frac": round(ach / fpeak, 4), "peak_source": funit}
    else:
        ach = head_edges / s / 1e9
        roof = {"bound": "alu", "achieved": round(ach, 1), "peak": round(xpeak / 1e9, 1), "unit": "Gexp2/s",
                "frac": round(ach * 1e9 / xpeak, 4),
                "peak_source": "MUFU.EX2: 15.7/clk/SM measured (profiles/r01_microbench.txt) x 148 SMs x "
                               f"{clk / 1e6:.0f} MHz; one exp2 per head-edge"}
    traffic = None
    tp = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tp):
        with open(tp) as f:
            traffic = json.load(f).get(f"{cfg_name}:{kernel}")
    roof.update({
        "traffic": traffic,
        "algorithmic": f"{bytes_alg} B (Q,K,V,O once{' + CSR' if csr else ''}), {flops_alg} flop "
                       f"(4d x {head_edges} head-edges) and {head_edges} exp2 per launch",
        "lower_bound_us": {"hbm": round(t_mem * 1e6, 2), "tensor": round(t_fl * 1e6, 2), "mufu": round(t_ex * 1e6, 2)},
        "frac_hbm": round(t_mem / s, 4), "frac_tensor": round(t_fl / s, 4), "frac_mufu": round(t_ex / s, 4),
        "kernel_ms_median": round(kernel_ms, 4)})
    if traffic:  # measured DRAM bytes of the step (ncu, profiles/traffic.json) over this run's time
        roof["dram_GBps_measured_traffic"] = round(traffic / s / 1e9, 1)
        roof["dram_frac_measured_traffic"] = round(traffic / s / 1e9 / hbm, 4)
    gbe = 2 * d * e + (4 if csr else 0)
    ggbs = head_edges * gbe / s / 1e9
    gather = {"bytes_per_edge": gbe, "GBps": round(ggbs, 1), "frac_of_8TBps": round(ggbs / 8000.0, 3),
              "frac_of_measured_hbm": round(ggbs / hbm, 3),
              "note": "north-star gather model (every edge pulls K_j and V_j); window/LongNet masks reuse K/V "
                      "on chip, so it can exceed 1 — the roofline above is the binding bound"}
    return roof, gather


def measure_e2e(args, ga, world, dev, edges_total, targets, run_step, out, c_abi=None):
    """The same metric end to end with pinned HOST buffers: every step copies this step's
    inputs host -> device (`targets`: the device tensors the step reads), runs the step, and
    copies the output device -> host, all inside the timed region.  At N=1 with an implicit
    mask (`c_abi` = (mask, host q, k, v)) the step is one ga_attention_host call (C ABI with
    host buffers, copies inside libga)."""
    import torch
    import torch.distributed as dist

    steps = max(3, min(args.steps, 5))
    if c_abi is not None:
        mask, hq, hk, hv = c_abi
        hout = torch.empty_like(hq).pin_memory()
        s = torch.cuda.current_stream()

        def step():
            ga.attention_host(hq, hk, hv, mask, hout, stream=s)
        h2d = 3 * hq.numel() * hq.element_size()
        path = "ga_attention_host (C ABI, pinned host buffers, copies inside libga)"
    else:
        hosts = [t.detach().cpu().pin_memory() for t in targets]
        hout = torch.empty(out.shape, dtype=out.dtype).pin_memory()

        def step():
            for t, h in zip(targets, hosts):
                t.copy_(h, non_blocking=True)
            run_step()
            hout.copy_(out, non_blocking=True)
        h2d = sum(h.numel() * h.element_size() for h in hosts)
        path = "pinned host -> device copies + ga_attention_ex step + device -> host copy"
    d2h = hout.numel() * hout.element_size()
    for _ in range(2):
        step()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        step()
    e1.record()
    torch.cuda.synchronize()
    t = torch.tensor([e0.elapsed_time(e1) / steps], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = t.item()
    return {"value": edges_total / (ms / 1e3), "unit": "edges/s", "h2d_bytes_per_step": h2d * world,
            "d2h_bytes_per_step": d2h * world, "ms_per_step": ms, "steps": steps, "path": path}


def _init_dist(torch, dist, world, local_rank):
    """One process per GPU over NCCL.  GA_DIST_BACKEND=gloo with GA_FORCE_DEVICE=0 lets
    several ranks share one GPU for a functional check of the N>1 code (not a timing)."""
    dev_index = int(os.environ.get("GA_FORCE_DEVICE", local_rank))
    torch.cuda.set_device(dev_index)
    dev = torch.device("cuda", dev_index)
    if world > 1:
        backend = os.environ.get("GA_DIST_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
    return dev


def max_context(args, world, rank, local_rank):
    """Largest Window(128) bf16 d=64 sequence that fits in HBM: Q, K, V
    resident and the output written over Q (one launch owns each row, so the band and edge
    kernels allow it for implicit masks).  At N>1 every rank holds L tokens (no halo copy).
    One step runs; rows at the start, the end and the shard boundaries are checked against
    the oracle (which regenerates them from the seed)."""
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2502_01659_b200 as ga

    dev = _init_dist(torch, dist, world, local_rank)
    H, d, w, seed = 1, 64, 128, 0x5EED0005
    mask = ga.Window(w)
    free, total = torch.cuda.mem_get_info(dev)
    row = H * d * 2
    reserve = 2 << 30  # context, runtime workspace, clocks
    L_local = int((free - reserve) // (3 * row))
    L_local = (L_local // 256) * 256  # tcgen05 window-kernel tile pairs (2 x 128 rows), shard-aligned
    L = L_local * world
    r0, r1 = rank * L_local, (rank + 1) * L_local
    comm = None
    if world > 1:  # K/V shards in symmetric buffers; halo rows read from the neighbours
        from paper_2502_01659_b200.comm import Comm

        comm = Comm()
        k = comm.empty((L_local, H, d), torch.bfloat16)
        v = comm.empty((L_local, H, d), torch.bfloat16)
    else:
        k = torch.empty((L_local, H, d), dtype=torch.bfloat16, device=dev)
        v = torch.empty_like(k)
    q = torch.empty((L_local, H, d), dtype=torch.bfloat16, device=dev)
    ga.fill_inputs(q, seed, 0, r0 * H * d)
    ga.fill_inputs(k, seed, 1, r0 * H * d)
    ga.fill_inputs(v, seed, 2, r0 * H * d)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    if comm is not None:
        comm.attention(q, k, v, mask, L, out=q)
    else:
        ga.attention(q, k, v, mask, q)
    e1.record()
    torch.cuda.synchronize()
    ms = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    import oracle

    local = np.unique(np.clip(np.concatenate([np.arange(r0, r0 + 64), np.arange(r1 - 64, r1),
                                              np.random.default_rng(rank).integers(r0, r1, 64)]), r0, r1 - 1))
    got = q[torch.from_numpy(local - r0).to(dev)].double().cpu().numpy()
    want, _ = oracle.attention_seeded(seed, "bf16", oracle.window(L, w), H, d, rows=local)
    err = torch.tensor([float(np.abs(got - want).max())], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(err, op=dist.ReduceOp.MAX)
    if rank == 0:
        print(json.dumps({
            "metric": "max context length (Window(128), bf16, d=64, 1 head; out aliased on Q)", "value": L,
            "unit": "tokens", "n_gpus": world, "higher_is_better": True, "scaling": "weak",
            "per_gpu_tokens": L_local, "hbm_total_bytes": total, "bytes_per_token": 3 * row,
            "step_ms": ms.item(), "edges": ga.mask_count(mask, L),
            "parity_max_abs_err_sampled": err.item(), "parity_ok": err.item() <= 2e-2,
            "paper_context": "160,000,000 tokens on one A100 80GB (PAPER.md:22, :452)"}), flush=True)
    if comm is not None:
        comm.close()
    if world > 1:
        dist.destroy_process_group()


def reference_arm(args, cfg, world, rank):
    """The reference arm for this tier is the fp64 CPU oracle, timed as it stands on the
    host cores; each step is a bounded row sample of the same workload."""
    if rank != 0:
        return
    budget = max(1.0, min(10.0, 120.0 / max(1, args.steps + args.warmup)))
    rates, edges, secs = [], 0, 0.0
    sample = None
    cores = None
    for s in range(args.warmup + args.steps):
        rate, cores, sample, e, t = oracle_rate(args.config, budget_s=budget)
        if s >= args.warmup:
            rates.append(rate)
            edges += e
            secs += t
    value = edges / secs
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "edges/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": secs / args.steps * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        # the same workload keys as the GPU arm's line (N = 1: the reference arm runs on rank 0 only)
        "config": {"workload": f"{args.config}: L={cfg['L']} tokens, {cfg['H']} heads, d={cfg['d']}, {cfg['dtype']}, "
                               f"{mask_desc(cfg)}", "L": cfg["L"], "heads": cfg["H"], "d": cfg["d"], "mask": mask_desc(cfg),
                   "note": "fp64 CPU oracle (oracle/oracle.c), OpenMP over rows, on sampled query rows"},
        "cpu_baseline": {"value": value, "unit": "edges/s", "cores": cores, "kind": "oracle", "sample": sample},
        "e2e": {"value": value, "unit": "edges/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()

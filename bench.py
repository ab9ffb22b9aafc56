#!/usr/bin/env python
"""bench.py — graph-view masked attention (arXiv 2502.01659) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config cfg2]

One "step" is one pass of the whole hot path (neighbour enumeration, scores, online
softmax, aggregation — one ga_attention call, or one ga_attention_sharded call per rank at N>1)
over the configuration's full synthetic input.  Default workload: BASELINE.json configs[1]
(L=65536, 8 heads, d=64, bf16, dilated window w=256 r=2) on one B200.  N>1 (torchrun,
one process per GPU) is weak scaling: every rank owns L query rows of an N*L-token
sequence; its K/V shard sits in a symmetric CUDA-IPC buffer and the kernels read the halo /
long-range rows they need from the other ranks' HBM over NVLink (CSR: K/V all-gather).

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
    "cfg4": dict(L=2 ** 24, H=1, d=64, dtype="bf16", mask=("longnet", 2048, 2)),
    "cfg5": dict(L=160_000_000, H=1, d=64, dtype="bf16", mask=("window", 128, 1)),
}
SEEDS = {"cfg1": 0x5EED0001, "cfg2": 0x5EED0002, "cfg3": 0x5EED0003, "cfg4": 0x5EED0004, "cfg5": 0x5EED0005}
BIGBIRD_SEED = 0xB16B12D
L2_FLUSH_BYTES = 256 << 20  # > 126 MB L2


def mask_desc(cfg):
    kind, *a = cfg["mask"]
    if kind == "window":
        return f"Window(w={a[0]}, r={a[1]})"
    if kind == "bigbird":
        return f"BigBird(window={a[0]}, globals={a[1]} evenly spaced, random={a[2]}/row) as explicit CSR"
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


# ------------------------------------------------------------------ main
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", choices=sorted(CONFIGS), default="cfg2")
    ap.add_argument("--kernel", default="auto", choices=["auto", "edge", "tiled", "window", "tc"])
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
    L_local, H, d = cfg["L"], cfg["H"], cfg["d"]
    L = L_local * world
    tdt = {"f32": torch.float32, "bf16": torch.bfloat16}[cfg["dtype"]]
    seed = SEEDS[args.config]
    kind, *a = cfg["mask"]
    r0, r1 = rank * L_local, (rank + 1) * L_local

    # ---- inputs (resident in HBM before timing) and the step function
    ws = None
    if kind == "window":
        mask = ga.Window(a[0], a[1])
        nnz = ga.mask_count(mask, L)
    elif kind == "bigbird":
        mask = ga.mask_to_csr(ga.BigBird(a[0], a[1], a[2], seed=BIGBIRD_SEED), L)
        nnz = mask.nnz
        ws = torch.empty(ga.workspace_size(mask, L, d, H, tdt, q_begin=r0, q_rows=L_local), dtype=torch.uint8,
                         device=dev)
    else:
        mask = ga.LongNet(a[0], a[1])
        nnz = ga.mask_count(mask, L)
        wsb = ga.workspace_size(mask, L, d, H, tdt, q_begin=r0, q_rows=L_local)  # tcgen05 block partials
        ws = torch.empty(wsb, dtype=torch.uint8, device=dev) if wsb else None
    q = torch.empty((L_local, H, d), dtype=tdt, device=dev)
    ga.fill_inputs(q, seed, 0, r0 * H * d)
    comm = None
    if world > 1:
        # weak scaling: rank owns rows [r0, r1) of an N*L sequence; its K/V shard lives in a
        # symmetric buffer the other ranks read over NVLink (ga_attention_sharded)
        from paper_2502_01659_b200.comm import Comm

        comm = Comm()
        k = comm.empty((L_local, H, d), tdt)
        v = comm.empty((L_local, H, d), tdt)
    else:
        k = torch.empty((L_local, H, d), dtype=tdt, device=dev)
        v = torch.empty_like(k)
    ga.fill_inputs(k, seed, 1, r0 * H * d)
    ga.fill_inputs(v, seed, 2, r0 * H * d)
    out = torch.empty_like(q)

    def step():
        if comm is not None:
            comm.attention(q, k, v, mask, L, out=out, kernel=args.kernel, workspace=ws)
        else:
            ga.attention(q, k, v, mask, out, kernel=args.kernel, workspace=ws)
    e2e_targets = [q, k, v]

    edges_total = nnz * H  # all ranks together (global mask over the N*L sequence)
    flush = torch.empty(L2_FLUSH_BYTES, dtype=torch.uint8, device=dev)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        step()
    barrier()

    sampler = ClockSampler(local_rank)
    sampler.start()
    lib = ga._abi.lib()
    launches0 = lib.ga_launch_count()
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    barrier()
    for s in range(args.steps):
        flush.zero_()  # L2 flush between timed steps (outside the events)
        if world > 1:
            dist.barrier()
        starts[s].record()
        step()
        ends[s].record()
    barrier()
    launches = lib.ga_launch_count() - launches0
    clocks = sampler.stop()
    per_step = [st.elapsed_time(en) for st, en in zip(starts, ends)]
    total_ms = torch.tensor([sum(per_step)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(total_ms, op=dist.ReduceOp.MAX)
    ms = total_ms.item() / args.steps
    value = edges_total / (ms / 1e3)

    # ---- roofline for the dominant kernel (the attention kernel; one launch per step at N=1)
    roofline, gather = roofline_for(args, cfg, kind, edges_total // world, L_local, H, d, nnz, per_step)
    # ---- end-to-end through the public API with host buffers
    e2e = None
    if not args.no_e2e:
        c_abi = None
        if world == 1 and kind != "bigbird":
            c_abi = (mask, q.cpu().pin_memory(), e2e_targets[1].cpu().pin_memory(), e2e_targets[2].cpu().pin_memory())
        e2e = measure_e2e(args, ga, world, dev, edges_total, e2e_targets, step, out, c_abi)

    # ---- CPU oracle baseline (rank 0, N=1 only)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        rate, cores, sample, _, _ = oracle_rate(args.config, args.cpu_budget)
        cpu = {"value": rate, "unit": "edges/s", "cores": cores, "kind": "oracle", "sample": sample}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "edges/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": cfg["dtype"], "accum": "f32", "data": "synthetic",
            "config": {"workload": f"{args.config}: L={L_local}{'x' + str(world) if world > 1 else ''} tokens, "
                                   f"{H} heads, d={d}, {cfg['dtype']}, {mask_desc(cfg)}",
                       "L": L, "heads": H, "d": d, "mask": mask_desc(cfg), "nnz": nnz,
                       "kernel": args.kernel, "parallelism": f"query-range shards x{world}" + (
                           ", ga_attention_sharded (remote K/V rows read over NVLink peer memory"
                           + (", CSR K/V all-gather" if kind == "bigbird" else "") + ")" if world > 1 else ""),
                       "l2": "flushed between timed steps (256 MiB write outside the events); inputs > L2"},
            "clocks": clocks, "roofline": roofline, "gather_model": gather, "cpu_baseline": cpu, "e2e": e2e,
            "gpu_launches": launches,
        }
        print(json.dumps(line), flush=True)
    if comm is not None:
        comm.close()
    if world > 1:
        dist.destroy_process_group()


def roofline_for(args, cfg, kind, head_edges, L_local, H, d, nnz, per_step):
    """Roofline of the attention kernel.

    Algorithmic bytes per launch = Q, K, V read once + O written once (+ row_ptr and col_idx
    for explicit CSR): no implementation can move less.  Algorithmic flops = 4d per
    head-edge (2d for q.k, 2d for p*v).  The bound is whichever resource's
    lower-bound time is larger at the measured peaks (HBM copy GB/s vs bf16 tensor TFLOP/s;
    fp32 inputs use the FP32 FMA pipe).  The north-star "gather model" (every edge pulls
    K_j and V_j from memory) is reported separately."""
    peaks, peak_src = load_peaks()
    kernel_ms = statistics.median(per_step)
    e = eb(cfg["dtype"])
    bytes_alg = 4 * L_local * H * d * e + ((L_local + 1) * 8 + nnz * 4 if kind == "bigbird" else 0)
    flops_alg = 4 * d * head_edges
    hbm = peaks["hbm_gbs"]
    if cfg["dtype"] == "f32":
        fpeak, funit = 148 * 128 * 2 * peaks.get("sm_max_mhz", 1965.0) * 1e6 / 1e12, "fp32 FMA pipe (derived)"
    else:
        fpeak, funit = peaks["bf16_tflops"], f"bf16 dense tensor ({peak_src})"
    t_mem, t_fl = bytes_alg / (hbm * 1e9), flops_alg / (fpeak * 1e12)
    s = kernel_ms / 1e3
    if t_mem >= t_fl:
        ach = bytes_alg / s / 1e9
        roof = {"bound": "hbm", "achieved": round(ach, 1), "peak": hbm, "unit": "GB/s", "frac": round(ach / hbm, 4),
                "peak_source": f"hbm_gbs, {peak_src} MEASURED_PEAKS.json (copy bandwidth)"}
    else:
        ach = flops_alg / s / 1e12
        roof = {"bound": "tensor" if cfg["dtype"] != "f32" else "alu", "achieved": round(ach, 2), "peak": fpeak,
                "unit": "TFLOP/s", "frac": round(ach / fpeak, 4), "peak_source": funit}
    traffic = None
    tp = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tp):
        with open(tp) as f:
            traffic = json.load(f).get(f"{args.config}:{args.kernel}")
    roof.update({
        "traffic": traffic,
        "algorithmic": f"{bytes_alg} B (Q,K,V,O once{' + CSR' if kind == 'bigbird' else ''}) and {flops_alg} flop "
                       f"(4d x {head_edges} head-edges) per launch",
        "lower_bound_us": {"hbm": round(t_mem * 1e6, 2), "flops": round(t_fl * 1e6, 2)},
        "tensor_tflops_achieved": round(flops_alg / s / 1e12, 2),
        "kernel_ms_median": round(kernel_ms, 4)})
    if traffic:  # measured DRAM bytes of the step (ncu, profiles/traffic.json) over this run's time
        roof["dram_GBps_measured_traffic"] = round(traffic / s / 1e9, 1)
        roof["dram_frac_measured_traffic"] = round(traffic / s / 1e9 / hbm, 4)
    gbe = 2 * d * e + (4 if kind == "bigbird" else 0)
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
    L_local = (L_local // 224) * 224  # band-kernel tile multiple (112 rows x r=1) x 2
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
        "config": {"workload": f"{args.config}: L={cfg['L']}, {cfg['H']} heads, d={cfg['d']}, {cfg['dtype']} inputs, "
                               f"{mask_desc(cfg)}", "note": "fp64 CPU oracle (oracle/oracle.c), OpenMP over rows"},
        "cpu_baseline": {"value": value, "unit": "edges/s", "cores": cores, "kind": "oracle", "sample": sample},
        "e2e": {"value": value, "unit": "edges/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()

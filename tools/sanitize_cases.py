"""One small invocation of every production kernel, for compute-sanitizer (T8 of SURVEY §4):
    compute-sanitizer --tool memcheck|racecheck|synccheck python tools/sanitize_cases.py [case ...]
Each case checks its output against the fp64 oracle so a sanitizer-clean run is also a
correct one."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
import paper_2502_01659_b200 as ga  # noqa: E402
import synth  # noqa: E402


def run(name, mask, om, L, H, d, dt, **kw):
    cpu = synth.qkv(5, L, H, d, dt, centred=True)
    q, k, v = (x.cuda() for x in cpu)
    out = ga.attention(q, k, v, mask, **kw)
    torch.cuda.synchronize()
    want, _ = oracle.attention(*(synth.as_f64(x) for x in cpu), om)
    err = float(np.abs(out.double().cpu().numpy() - want).max())
    tol = 1e-4 if dt == "f32" else 2e-2
    print(f"{name}: max err {err:.2e}", "OK" if err <= tol else "FAIL", flush=True)
    assert err <= tol


def run_env(env, *a, **kw):
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    try:
        run(*a, **kw)
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


def main(cases):
    L = 2048
    bb = ga.mask_to_csr(ga.BigBird(64, 4, 16, seed=3), L)
    all_cases = {
        "window_tc": lambda: run("window_tc", ga.Window(256, 2), oracle.window(L, 256, 2), L, 2, 64, "bf16", kernel="tc"),
        # many items per CTA (GA_WTC_GRID caps the persistent grid): cursor, ring reuse, S prefetch
        "window_tc_run": lambda: run_env({"GA_WTC_GRID": "3"}, "window_tc_run", ga.Window(200, 2),
                                         oracle.window(4 * L, 200, 2), 4 * L, 2, 64, "bf16", kernel="tc"),
        "band": lambda: run("band", ga.Window(64, 1), oracle.window(L, 64, 1), L, 2, 64, "bf16", kernel="tiled"),
        "edge": lambda: run("edge", ga.Window(40, 3), oracle.window(L, 40, 3), L, 2, 64, "f32", kernel="edge"),
        "longnet_umma": lambda: run("longnet_umma", ga.LongNet(512, 2), oracle.longnet(8192, 512, 2), 8192, 1, 64,
                                    "bf16"),
        "longnet_tiled": lambda: run("longnet_tiled", ga.LongNet(256, 2), oracle.longnet(4096, 256, 2), 4096, 1, 64,
                                     "bf16", kernel="tiled"),
        "csr_tma": lambda: run("csr_tma", bb, oracle.bigbird(L, 64, 4, 16, 3), L, 1, 64, "bf16",
                               workspace=torch.empty(ga.workspace_size(bb, L, 64, 1, heavy_threshold=1024), dtype=torch.uint8,
                                                        device="cuda"),
                               heavy_threshold=1024),
        "bigbird_implicit": lambda: run("bigbird_implicit", ga.BigBird(128, 4, 16, seed=3),
                                        oracle.bigbird(L, 128, 4, 16, 3), L, 2, 64, "bf16"),
        "maskgen": lambda: maskgen(L),
        "backward": lambda: backward(L),
    }
    for c in cases or list(all_cases):
        all_cases[c]()


def maskgen(L):
    m = ga.mask_to_csr(ga.LongNet(64, 2), L)
    rp, ci, _ = oracle.mask_to_csr(oracle.longnet(L, 64, 2))
    assert np.array_equal(m.col_idx.cpu().numpy(), ci)
    coo = ga.coo_to_csr(torch.randint(0, L, (5000,), device="cuda"), torch.randint(0, L, (5000,), device="cuda"), L)
    torch.cuda.synchronize()
    print("maskgen/coo: OK", flush=True)


def backward(L):
    q, k, v = ga.qkv_device(3, L, 2, 64, torch.bfloat16, shift=-0.5)
    m = ga.mask_to_csr(ga.BigBird(16, 2, 8, seed=3), L)
    out = ga.attention(q, k, v, m)
    ga.attention_backward(q, k, v, out, q, m)
    ga.attention_backward(q, k, v, ga.attention(q, k, v, ga.Window(33)), q, ga.Window(33))
    torch.cuda.synchronize()
    print("backward: OK", flush=True)


if __name__ == "__main__":
    main(sys.argv[1:])

"""Backward pass (ga_attention_backward) against the fp64 oracle backward
(oracle.c orc_attention_backward, pinned by finite differences and torch autograd in
tests/test_oracle_pins.py) on identical inputs.

The kernels compute in fp32 on the exact stored input values; the only lower-precision
input is the forward output O (D_i = dO_i . O_i), so bf16/fp16 runs carry O's rounding
(2^-9 relative) into dS.  Tolerance: max |err| <= tol * max |ref| per gradient, tol = 1e-4
(fp32) and 2e-2 (bf16/fp16, BASELINE.json's forward tolerance).
"""
import math

import numpy as np
import pytest
import torch

import synth

pytestmark = pytest.mark.gpu

TDT = {"f32": torch.float32, "bf16": torch.bfloat16, "f16": torch.float16}
TOL = {"f32": 1e-4, "bf16": 2e-2, "f16": 2e-2}


@pytest.fixture(scope="module")
def ga():
    import paper_2502_01659_b200 as ga

    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    return ga


def _random_csr(L, seed, max_deg=60):
    rng = np.random.default_rng(seed)
    deg = rng.integers(0, max_deg, L)
    deg[::13] = 0
    cols = [np.sort(rng.choice(L, n, replace=False)) for n in deg]
    rp = np.concatenate([[0], np.cumsum(deg)]).astype(np.int64)
    ci = np.concatenate(cols).astype(np.int32)
    return rp, ci


def _masks(ga, orc, fam, L):
    if fam == "window":
        return ga.Window(40, 1), orc.window(L, 40, 1)
    if fam == "dilated":
        return ga.Window(100, 3), orc.window(L, 100, 3)
    if fam == "longnet":
        return ga.LongNet(64, 2), orc.longnet(L, 64, 2)
    if fam == "longnet_multiset":
        return ga.LongNet(32, 2, multiset=True), orc.longnet(L, 32, 2, multiset=True)
    if fam == "block":
        return ga.BlockDilated(96, 3), orc.block_dilated(L, 96, 3)
    if fam == "csr":
        rp, ci = _random_csr(L, 5)
        return ga.CSR(torch.from_numpy(rp).cuda(), torch.from_numpy(ci).cuda()), orc.csr(L, rp, ci)
    if fam == "bigbird_csr":  # not symmetric: the column pass needs the transposed CSR
        m = ga.mask_to_csr(ga.BigBird(16, 3, 8, seed=9), L)
        return m, orc.bigbird(L, 16, 3, 8, 9)
    raise ValueError(fam)


def _check(got, want, tol, what):
    ref = np.abs(want).max()
    err = np.abs(got - want).max()
    assert err <= tol * ref, f"{what}: max err {err:.3e} vs {tol} x {ref:.3e}"


@pytest.mark.parametrize("fam", ["window", "dilated", "longnet", "longnet_multiset", "block", "csr", "bigbird_csr"])
@pytest.mark.parametrize("dt,d", [("f32", 64), ("bf16", 64), ("f16", 32), ("bf16", 128)])
def test_backward_vs_oracle(ga, orc, fam, dt, d):
    L, H = 1200, 2
    q, k, v = synth.qkv(500 + d, L, H, d, dt, centred=True)
    g = synth.qkv(900 + d, L, H, d, dt, centred=True)[0]
    m, om = _masks(ga, orc, fam, L)
    qd, kd, vd, gd = (x.cuda() for x in (q, k, v, g))
    out = ga.attention(qd, kd, vd, m)
    dq, dk, dv = ga.attention_backward(qd, kd, vd, out, gd, m)
    torch.cuda.synchronize()
    wq, wk, wv, edges = orc.attention_backward(*(synth.as_f64(x) for x in (q, k, v)), om, synth.as_f64(g))
    for name, a, b in (("dQ", dq, wq), ("dK", dk, wk), ("dV", dv, wv)):
        _check(a.double().cpu().numpy(), b, TOL[dt], f"{fam} {dt} d={d} {name}")


def test_backward_lse_passthrough(ga):
    """lse from a carried state (lse = m + log2 l) gives the gradients of the recomputing call
    (within the bf16 rounding of P and dS on the tensor-core band path: both are 2e-3-close to
    the oracle, tests below)."""
    L, H, d = 3000, 2, 64
    q, k, v = ga.qkv_device(3, L, H, d, torch.bfloat16, shift=-0.5)
    g = ga.qkv_device(4, L, H, d, torch.bfloat16, shift=-0.5)[0]
    m = ga.Window(128)
    st = ga.State.empty(L, H, d)
    out = ga.attention(q, k, v, m, torch.empty_like(q), state=st)
    lse = st.m + torch.log2(st.l)
    a = ga.attention_backward(q, k, v, out, g, m)
    b = ga.attention_backward(q, k, v, out, g, m, lse=lse)
    torch.cuda.synchronize()
    for x, y in zip(a, b):
        assert (x - y).abs().max().item() <= 5e-3 * x.abs().max().item()


def test_autograd_function_matches_torch_dense(ga):
    """GraphAttention (torch.autograd.Function) against torch autograd through a dense masked
    softmax on the GPU in fp32 (library routine)."""
    L, H, d = 512, 2, 64
    torch.manual_seed(0)
    q, k, v = (torch.randn(L, H, d, device="cuda", requires_grad=True) for _ in range(3))
    g = torch.randn(L, H, d, device="cuda")
    out = ga.GraphAttention.apply(q, k, v, ga.Window(33, 2))
    (out * g).sum().backward()
    got = [x.grad.clone() for x in (q, k, v)]
    i = torch.arange(L, device="cuda")
    dist = (i[:, None] - i[None, :]).abs()
    mask = (dist < 33) & (dist % 2 == 0)
    q2, k2, v2 = (x.detach().clone().requires_grad_(True) for x in (q, k, v))
    s = torch.einsum("ihc,jhc->hij", q2, k2) / math.sqrt(d)
    p = torch.softmax(s.masked_fill(~mask, float("-inf")), dim=-1)
    o = torch.einsum("hij,jhc->ihc", p, v2)
    (o * g).sum().backward()
    for a, b in zip(got, (q2.grad, k2.grad, v2.grad)):
        assert (a - b).abs().max().item() <= 1e-4 * b.abs().max().item()


def test_backward_rejects(ga):
    L = 256
    q, k, v = ga.qkv_device(1, L, 1, 64, torch.bfloat16)
    with pytest.raises(ga.GaError, match="UNSUPPORTED"):
        ga.attention_backward(q, k, v, q, q, ga.BigBird(8, 2, 2))


@pytest.mark.parametrize("L,w,r,dt", [(3000, 256, 2, "bf16"), (2049, 128, 1, "f16"), (1500, 17, 1, "bf16"),
                                      (4000, 400, 4, "bf16"), (700, 600, 1, "f16"),
                                      (2500, 256, 1, "bf16")])  # m = 255: the widest band (592 staged rows)
def test_backward_tensor_core_band_vs_oracle(ga, orc, L, w, r, dt):
    """The tensor-core band backward (backward_tc.cu: Window masks, bf16/fp16, d = 64, m <=
    255) against the fp64 oracle backward, ragged class lengths and sequences shorter than
    the band included; and against the CUDA-core kernels (GA_BWD_CUDACORE=1)."""
    import os

    H, d = 2, 64
    q, k, v = synth.qkv(600 + w, L, H, d, dt, centred=True)
    g = synth.qkv(700 + w, L, H, d, dt, centred=True)[0]
    m = ga.Window(w, r)
    qd, kd, vd, gd = (x.cuda() for x in (q, k, v, g))
    out = ga.attention(qd, kd, vd, m)
    got = ga.attention_backward(qd, kd, vd, out, gd, m)
    os.environ["GA_BWD_CUDACORE"] = "1"
    try:
        ref = ga.attention_backward(qd, kd, vd, out, gd, m)
    finally:
        del os.environ["GA_BWD_CUDACORE"]
    torch.cuda.synchronize()
    want = orc.attention_backward(*(synth.as_f64(x) for x in (q, k, v)), orc.window(L, w, r), synth.as_f64(g))
    for name, a, b, c in zip(("dQ", "dK", "dV"), got, want[:3], ref):
        _check(a.double().cpu().numpy(), b, TOL[dt], f"tc {name}")
        _check(c.double().cpu().numpy(), b, TOL[dt], f"cuda-core {name}")

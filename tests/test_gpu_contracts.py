"""Boundary contracts of include/ga.h that parity tests do not exercise.

* Aliasing (SURVEY §8(b) "Aliasing"): `out` may be `Q` itself.  Every AUTO path — including
  the multi-launch ones (LongNet tcgen05 group + block + merge, CSR light rows + heavy split
  + full-row tiles) — reads a row's Q before any launch writes that row's O, so out=Q must
  give the same bits as a separate output; a shifted overlap of out and Q is rejected.
* Host-buffer pipeline: a chunk's launch must not read K/V rows that its
  copies have not delivered (whole 64-key TMA chunks reach past the band).  Stale NaN in the
  recycled scratch pool must not reach the output (0 x NaN = NaN).
"""
import numpy as np
import pytest
import torch

import synth

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ga():
    import paper_2502_01659_b200 as ga

    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    return ga


def _alias_case(ga, q, k, v, mask, **kw):
    ref = ga.attention(q, k, v, mask, **kw)
    qa = q.clone()
    got = ga.attention(qa, k, v, mask, out=qa, **kw)
    torch.cuda.synchronize()
    assert got.data_ptr() == qa.data_ptr()
    assert torch.equal(qa, ref), f"{mask} {kw}: out=Q differs from a separate output"


@pytest.mark.parametrize("kernel", ["auto", "tc", "tiled", "edge"])
def test_alias_out_is_q_window(ga, kernel):
    L, H, d = 20011, 2, 64
    q, k, v = ga.qkv_device(31, L, H, d, torch.bfloat16, shift=-0.5)
    _alias_case(ga, q, k, v, ga.Window(200, 2), kernel=kernel)


@pytest.mark.parametrize("kernel,d", [("auto", 64), ("tiled", 64), ("auto", 32), ("edge", 64)])
def test_alias_out_is_q_longnet(ga, kernel, d):
    """AUTO at d=64 is the multi-launch tcgen05 path (group, block partials, merge)."""
    L = 65536
    q, k, v = ga.qkv_device(32, L, 1, d, torch.bfloat16, shift=-0.5)
    _alias_case(ga, q, k, v, ga.LongNet(2048, 2), kernel=kernel)


@pytest.mark.parametrize("dt", [torch.bfloat16, torch.float32])
def test_alias_out_is_q_csr_heavy_split(ga, dt):
    """Light rows (csr_tma / edge), heavy-row chunks + merge and full-row tiles + merge."""
    L, H, d = 16384, 1, 64
    q, k, v = ga.qkv_device(33, L, H, d, dt, shift=-0.5)
    csr = ga.mask_to_csr(ga.BigBird(128, 16, 64, seed=0xB16B12D), L)
    ws = torch.empty(ga.workspace_size(csr, L, d, H, dt), dtype=torch.uint8, device="cuda")
    _alias_case(ga, q, k, v, csr, workspace=ws)


def test_shifted_overlap_rejected(ga):
    L, H, d = 4096, 1, 64
    buf = torch.zeros(2 * L, H, d, dtype=torch.bfloat16, device="cuda")
    q = buf[:L]
    k, v = (x.cuda() for x in synth.qkv(3, L, H, d, "bf16")[1:])
    with pytest.raises(ga.GaError, match="INVALID_ARG"):
        ga.attention(q, k, v, ga.Window(128), out=buf[1:L + 1])
    with pytest.raises(ga.GaError, match="INVALID_ARG"):
        ga.attention(q, k, v, ga.Window(128), out=k)


@pytest.mark.parametrize("win", [(101, 1), (200, 2), (128, 1), (65, 1)])
def test_host_pipeline_ignores_stale_nan_scratch(ga, win):
    """run the host path once on NaN inputs (the scratch pool then holds NaN in
    the recycled K/V blocks), then on real inputs: bit-identical to the device call."""
    L, H, d = 40000, 2, 64
    cpu = synth.qkv(41, L, H, d, "bf16", centred=True)
    m = ga.Window(*win)
    pinned = [x.pin_memory() for x in cpu]
    nan = [torch.full_like(x, float("nan")).pin_memory() for x in cpu]
    out = torch.empty_like(pinned[0]).pin_memory()
    for _ in range(2):
        ga.attention_host(*nan, m, out)
        torch.cuda.synchronize()
        ga.attention_host(*pinned, m, out)
        torch.cuda.synchronize()
    dev = ga.attention(*(x.cuda() for x in cpu), m)
    torch.cuda.synchronize()
    assert not torch.isnan(out.float()).any()
    assert torch.equal(out, dev.cpu())

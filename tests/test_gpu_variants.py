"""LongNet per-head offsets (reading R11c: LongNet's s_j = j mod r — head h
keeps, at level k, the in-segment offsets congruent to h mod alpha^k) on the GPU: forward and
backward against the fp64 oracle (per-head neighbour sets from the definition), and the exact
per-head edge multiset with the one-hot count test of test_gpu_edgesets.py."""
import numpy as np
import pytest
import torch

import synth
from tests.test_gpu_edgesets import check_counts, classes, onehot_inputs

pytestmark = pytest.mark.gpu

TOL = {"f32": 1e-4, "bf16": 2e-2, "f16": 2e-2}


@pytest.fixture(scope="module")
def ga():
    import paper_2502_01659_b200 as ga

    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    return ga


@pytest.mark.parametrize("L,w0,alpha,multiset", [(4096, 64, 2, False), (3000, 27, 3, False), (2048, 32, 2, True)])
@pytest.mark.parametrize("dt", ["f32", "bf16"])
def test_longnet_head_offsets_forward(ga, orc, L, w0, alpha, multiset, dt):
    H, d = 5, 64
    cpu = synth.qkv(31 + L, L, H, d, dt, centred=True)
    out = ga.attention(*(x.cuda() for x in cpu), ga.LongNet(w0, alpha, multiset=multiset, head_offsets=True))
    torch.cuda.synchronize()
    want, _ = orc.attention(*(synth.as_f64(x) for x in cpu),
                            orc.longnet(L, w0, alpha, multiset=multiset, head_offsets=True))
    assert np.abs(out.double().cpu().numpy() - want).max() <= TOL[dt]


@pytest.mark.parametrize("L,w0,alpha", [(8192, 128, 2), (5000, 100, 3)])
def test_longnet_head_offsets_exact_edges(ga, orc, L, w0, alpha):
    H, d = 4, 64
    q, k, v = (x.cuda() for x in onehot_inputs(L, H, d, "f16"))
    out = ga.attention(q, k, v, ga.LongNet(w0, alpha, head_offsets=True))
    torch.cuda.synchronize()
    got = out.double().cpu().numpy()
    deg = np.zeros((L, H), dtype=np.int64)
    cnt = np.zeros((L, H, d), dtype=np.int64)
    for h in range(H):
        rp, ci, _ = orc.mask_to_csr(orc.longnet(L, w0, alpha, head_offsets=True, head=h))
        deg[:, h] = np.diff(rp)
        row_of = np.repeat(np.arange(L), deg[:, h])
        cnt[:, h, :] = np.bincount(row_of * d + classes(ci.astype(np.int64), h, d), minlength=L * d).reshape(L, d)
    for h in range(H):
        check_counts(got[:, h:h + 1], deg[:, h], cnt[:, h:h + 1], "f16", f"head {h}")


def test_longnet_head_offsets_backward(ga, orc):
    L, H, d = 1000, 3, 64
    q, k, v = synth.qkv(7, L, H, d, "f32", centred=True)
    g = synth.qkv(8, L, H, d, "f32", centred=True)[0]
    m = ga.LongNet(16, 2, head_offsets=True)
    qd, kd, vd, gd = (x.cuda() for x in (q, k, v, g))
    out = ga.attention(qd, kd, vd, m)
    grads = ga.attention_backward(qd, kd, vd, out, gd, m)
    torch.cuda.synchronize()
    want = orc.attention_backward(*(synth.as_f64(x) for x in (q, k, v)), orc.longnet(L, 16, 2, head_offsets=True),
                                  synth.as_f64(g))
    for a, b in zip(grads, want[:3]):
        assert np.abs(a.double().cpu().numpy() - b).max() <= 1e-4 * np.abs(b).max()


def test_longnet_head_offsets_rejects_single_csr(ga):
    with pytest.raises(ga.GaError, match="UNSUPPORTED"):
        ga.mask_count(ga.LongNet(64, 2, head_offsets=True), 4096)
    with pytest.raises(ga.GaError, match="UNSUPPORTED"):
        ga.mask_to_csr(ga.LongNet(64, 2, head_offsets=True), 4096)

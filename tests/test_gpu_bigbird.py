"""Implicit BigBird / Longformer descriptors in ga_attention (bigbird.cu).

Window part on the window kernels into a carried state, the global columns and R10's random
columns enumerated on the fly and merged, global rows as dense full-row tiles — checked
against the fp64 oracle (mask definitions; readings R8-R10)
within BJ's tolerances, and edge-exactly with the one-hot count test.
"""
import numpy as np
import pytest
import torch

import synth
from tests.test_gpu_edgesets import run_counts

pytestmark = pytest.mark.gpu

TOL = {"f32": 1e-4, "bf16": 2e-2, "f16": 2e-2}


@pytest.fixture(scope="module")
def ga():
    import paper_2502_01659_b200 as ga

    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    return ga


# (L, w, n_global, n_random, r, parts): window_tc window (w=128 / (200, 2)), edge-kernel window
# (w=51), no globals, no random, exhausted complements (L=300), ragged L (no full-row tiles),
# Longformer (parts = window | global), dilated Longformer
CASES = [
    (4096, 128, 16, 64, 1, 0), (3000, 128, 3, 64, 1, 0), (20000, 128, 64, 64, 1, 0), (4096, 51, 3, 8, 1, 0),
    (4096, 200, 5, 20, 2, 0), (300, 128, 8, 64, 1, 0), (4096, 128, 0, 64, 1, 0), (4096, 128, 16, 0, 1, 0),
    (4096, 51, 3, 0, 1, 3), (4096, 101, 3, 0, 2, 3), (5000, 128, 7, 30, 1, 5),
]


@pytest.mark.parametrize("case", CASES, ids=lambda c: "L{}w{}g{}n{}r{}p{}".format(*c))
@pytest.mark.parametrize("dt", ["bf16", "f32"])
def test_bigbird_implicit_vs_oracle(ga, orc, case, dt):
    L, w, g, nr, r, parts = case
    H, d, seed = 2, 64, 0xB16B12D
    cpu = synth.qkv(77 + L, L, H, d, dt, centred=True)
    q, k, v = (x.cuda() for x in cpu)
    out = ga.attention(q, k, v, ga.BigBird(w, g, nr, seed=seed, r=r, parts=parts))
    torch.cuda.synchronize()
    want, _ = orc.attention(*(synth.as_f64(x) for x in cpu), orc.bigbird(L, w, g, nr, seed, r=r, parts=parts))
    err = np.abs(out.double().cpu().numpy() - want).max()
    assert err <= TOL[dt], err


@pytest.mark.parametrize("d,dt", [(32, "f16"), (128, "bf16"), (64, "f16")])
def test_bigbird_implicit_dims(ga, orc, d, dt):
    L, w, g, nr, seed = 4096, 128, 8, 32, 5
    cpu = synth.qkv(3, L, 1, d, dt, centred=True)
    out = ga.attention(*(x.cuda() for x in cpu), ga.BigBird(w, g, nr, seed=seed))
    torch.cuda.synchronize()
    want, _ = orc.attention(*(synth.as_f64(x) for x in cpu), orc.bigbird(L, w, g, nr, seed))
    assert np.abs(out.double().cpu().numpy() - want).max() <= TOL[dt]


@pytest.mark.parametrize("case", [(4096, 128, 16, 64, 1, 0), (3000, 51, 3, 64, 1, 0), (300, 128, 8, 64, 1, 0),
                                  (8192, 200, 5, 20, 2, 0), (4096, 101, 3, 0, 2, 3)],
                         ids=lambda c: "L{}w{}g{}n{}r{}p{}".format(*c))
def test_bigbird_implicit_exact_edges(ga, orc, case):
    """Every row's visited multiset equals the oracle's BigBird neighbour set: the on-the-fly
    random columns are R10's, globals are not double counted, global rows see every column."""
    L, w, g, nr, r, parts = case
    seed = 0xB16B12D
    run_counts(ga, orc, ga.BigBird(w, g, nr, seed=seed, r=r, parts=parts),
               orc.bigbird(L, w, g, nr, seed, r=r, parts=parts), L, 2, 64, "f16")


def test_bigbird_implicit_matches_csr(ga):
    """Same mask through the CSR kernels (materialised by ga_mask_to_csr): close agreement
    (different kernels: rounding differs, the edge set does not)."""
    L, H, d = 16384, 1, 64
    q, k, v = ga.qkv_device(9, L, H, d, torch.bfloat16, shift=-0.5)
    m = ga.BigBird(128, 16, 64, seed=0xB16B12D)
    a = ga.attention(q, k, v, m)
    csr = ga.mask_to_csr(m, L)
    ws = torch.empty(ga.workspace_size(csr, L, d, H, torch.bfloat16), dtype=torch.uint8, device="cuda")
    b = ga.attention(q, k, v, csr, workspace=ws)
    torch.cuda.synchronize()
    assert (a.float() - b.float()).abs().max().item() <= 1e-2


def test_bigbird_implicit_workspace_and_alias(ga):
    L, H, d = 8192, 2, 64
    q, k, v = ga.qkv_device(10, L, H, d, torch.bfloat16, shift=-0.5)
    m = ga.BigBird(128, 8, 16, seed=1)
    ref = ga.attention(q, k, v, m)
    ws = torch.empty(ga.workspace_size(m, L, d, H, torch.bfloat16), dtype=torch.uint8, device="cuda")
    a = ga.attention(q, k, v, m, workspace=ws)
    qa = q.clone()
    ga.attention(qa, k, v, m, out=qa)
    torch.cuda.synchronize()
    assert torch.equal(a, ref) and torch.equal(qa, ref)


def test_bigbird_implicit_unsupported(ga):
    L = 1024
    q, k, v = ga.qkv_device(1, L, 1, 64, torch.bfloat16)
    with pytest.raises(ga.GaError, match="UNSUPPORTED"):
        ga.attention(q, k, v, ga.BigBird(8, 2, 2, parts=ga.BB_GLOBAL))  # no window component
    with pytest.raises(ga.GaError, match="UNSUPPORTED"):
        ga.attention(q, k, v, ga.BigBird(8, 900, 200))  # n_global + n_random > 1024


def test_cfg3_bigbird_implicit_full_size_sampled(ga, orc):
    """BASELINE cfg3 as an implicit descriptor: L=2^20, bf16, 64 evenly spaced globals,
    Window(128), 64 random per row — sampled rows incl. every global row and its neighbours."""
    L, H, d, seed = 2 ** 20, 1, 64, 0x5EED0003
    q, k, v = ga.qkv_device(seed, L, H, d, torch.bfloat16)
    m = ga.BigBird(128, 64, 64, seed=0xB16B12D)
    out = ga.attention(q, k, v, m).double().cpu().numpy()
    G = [(kk * L) // 64 for kk in range(64)]
    rng = np.random.default_rng(3)
    rows = sorted(set(G) | {x + 1 for x in G if x + 1 < L} | set(range(0, 64)) | set(range(L - 64, L))
                  | set(int(x) for x in rng.integers(0, L, 256)))
    rows = np.array(rows, dtype=np.int64)
    want, _ = orc.attention_seeded(seed, "bf16", orc.bigbird(L, 128, 64, 64, 0xB16B12D), H, d, rows=rows)
    assert np.abs(out[rows] - want).max() <= 2e-2


@pytest.mark.parametrize("with_out", [False, True])
def test_window_tc_carried_state(ga, orc, with_out):
    """The tcgen05 window kernel's state epilogue (ga_opts.state): WRITE gives the row's
    (m, l, o~) — same softmax mass l 2^m as the edge kernel's state — and ACCUMULATE (+)s
    into a state from another component: window (tcgen05) + CSR(global | random) composed
    equals the BigBird oracle (PAPER.md:521 sequential composition)."""
    L, H, d, seed = 5000, 2, 64, 0xB16B12D
    cpu = synth.qkv(12, L, H, d, "bf16", centred=True)
    q, k, v = (x.cuda() for x in cpu)
    f64 = tuple(synth.as_f64(x) for x in cpu)
    st_tc = ga.State.empty(L, H, d)
    st_ed = ga.State.empty(L, H, d)
    out = torch.empty_like(q) if with_out else None
    ga.attention(q, k, v, ga.Window(128), out, state=st_tc, kernel="tc")
    ga.attention(q, k, v, ga.Window(128), state=st_ed, kernel="edge")
    torch.cuda.synchronize()
    z_tc = st_tc.l.double() * torch.exp2(st_tc.m.double())
    z_ed = st_ed.l.double() * torch.exp2(st_ed.m.double())
    assert ((z_tc - z_ed).abs() / z_ed).max().item() < 5e-3
    want_w, _ = orc.attention(*f64, orc.window(L, 128))
    fin = ga.state_finalize(st_tc, torch.bfloat16).double().cpu().numpy()
    assert np.abs(fin - want_w).max() <= 2e-2
    if with_out:
        assert np.abs(out.double().cpu().numpy() - want_w).max() <= 2e-2
    # composition: CSR of the global + random components first (edge kernel), then the window
    rest = ga.mask_to_csr(ga.BigBird(128, 5, 16, seed=seed, parts=ga.BB_GLOBAL | ga.BB_RANDOM), L)
    st = ga.State.empty(L, H, d)
    ga.attention(q, k, v, rest, state=st, accumulate=True)
    ga.attention(q, k, v, ga.Window(128), state=st, accumulate=True, kernel="tc")
    got = ga.state_finalize(st, torch.bfloat16).double().cpu().numpy()
    want, _ = orc.attention(*f64, orc.bigbird(L, 128, 5, 16, seed))
    assert np.abs(got - want).max() <= 2e-2


@pytest.mark.parametrize("d,variant", [(64, ""), (64, "GA_CSR_LDG"), (32, ""), (128, "")])
def test_csr_tensor_core_carried_state(ga, orc, d, variant, monkeypatch):
    """The explicit-CSR mma.sync kernels (csr_tma at d = 64, the LDG variant otherwise) write /
    (+)-combine a carried state: BigBird = CSR(global | random) WRITE, then CSR(window)
    ACCUMULATE with an output — equal to the oracle; the state's mass l 2^m matches the edge
    kernel's."""
    if variant:
        monkeypatch.setenv(variant, "1")
    L, H, seed = 3000, 2, 0xB16B12D
    cpu = synth.qkv(13, L, H, d, "bf16", centred=True)
    q, k, v = (x.cuda() for x in cpu)
    rest = ga.mask_to_csr(ga.BigBird(64, 5, 16, seed=seed, parts=ga.BB_GLOBAL | ga.BB_RANDOM), L)
    win = ga.mask_to_csr(ga.BigBird(64, 5, 16, seed=seed, parts=ga.BB_WINDOW), L)
    st, st_e = ga.State.empty(L, H, d), ga.State.empty(L, H, d)
    ga.attention(q, k, v, rest, state=st)
    ga.attention(q, k, v, rest, state=st_e, kernel="edge")
    torch.cuda.synchronize()
    z = st.l.double() * torch.exp2(st.m.double())
    ze = st_e.l.double() * torch.exp2(st_e.m.double())
    ok = st_e.l > 0
    assert torch.equal(st.l > 0, ok)
    assert ((z - ze).abs()[ok] / ze[ok]).max().item() < 5e-3
    out = torch.empty_like(q)
    ga.attention(q, k, v, win, out, state=st, accumulate=True)
    torch.cuda.synchronize()
    want, _ = orc.attention(*(synth.as_f64(x) for x in cpu), orc.bigbird(L, 64, 5, 16, seed))
    assert np.abs(out.double().cpu().numpy() - want).max() <= 2e-2
    assert np.abs(ga.state_finalize(st, torch.bfloat16).double().cpu().numpy() - want).max() <= 2e-2

"""Pins for the CPU oracle (oracle/): checked against things OTHER than itself.

Each test names what pins it: a value printed in PAPER.md / SPEC.md, a closed form, a
library routine (torch SDPA in fp64), an invariant, or brute force on tiny inputs
(oracle/dense.py, which shares no code with oracle.c).
"""
import math

import numpy as np
import pytest
import torch

import synth
from tests.conftest import golden

pytestmark = pytest.mark.filterwarnings("ignore")


def _kv(rows):
    return {r.split()[0]: r.split()[1] for r in rows}


# ------------------------------------------------------------------ generator
def test_rng_golden(orc):
    g = _kv(golden("rng.txt"))
    assert orc.splitmix64(0) == int(g["splitmix64_0"], 16)
    assert orc.splitmix64(1) == int(g["splitmix64_1"], 16)
    assert synth.splitmix64(0) == int(g["splitmix64_0"], 16)
    seed = int(g["seed"], 16)
    for t, name in enumerate("QKV"):
        want = float(g[f"{name}_e0_f32"])
        assert orc.input_value(seed, t, 0, "f32") == want
        assert float(synth.uniform_f32(seed, t, 1, 0)[0]) == want
        q = synth.qkv(seed, 1, 8, 64, "bf16")[t]
        assert (q.view(torch.int16)[0, 0, 0].item() & 0xFFFF) == int(g[f"{name}_e0_bf16"], 16)
        # oracle's bf16 rounding equals torch's RNE
        assert orc.input_value(seed, t, 0, "bf16") == q[0, 0, 0].double().item()
    assert orc.input_value(seed, 0, 512, "f32") == float(g["Q_e512_f32"])


def test_rng_dtypes_match_torch(orc):
    """oracle.c RNE to bf16/fp16 == torch's conversion, on 4096 values incl. tiny ones."""
    seed = 1234
    a = synth.uniform_f32(seed, 2, 4096)
    for dt, tdt in (("bf16", torch.bfloat16), ("f16", torch.float16)):
        ref = torch.from_numpy(a).to(tdt).double().numpy()
        got = np.array([orc.input_value(seed, 2, e, dt) for e in range(4096)])
        assert np.array_equal(ref, got)


# ------------------------------------------------------------------ masks
def test_spec_examples(orc):
    """SPEC.md worked examples."""
    from oracle import dense

    for row in golden("spec_examples.txt"):
        lhs, rhs = row.split("->")
        want = rhs.split(";")[0].strip()
        kind, *args = lhs.split()
        a = [int(x) for x in args]
        if kind == "window_pred":
            i, j, w = a
            L = max(i, j) + 1
            assert int(dense.window_mask(L, w)[i, j]) == int(want)
            assert (j in orc.neighbors(orc.window(L, w), i)) == bool(int(want))
        elif kind == "dil1d_pred":
            i, j, w, r = a
            L = max(i, j) + 1
            assert int(dense.window_mask(L, w, r)[i, j]) == int(want)
            assert (j in orc.neighbors(orc.window(L, w, r), i)) == bool(int(want))
        elif kind == "dil2d_pred":
            i, j, L, b, r = a
            assert int(dense.block_dilated_mask(L, b, r)[i, j]) == int(want)
            assert (j in orc.neighbors(orc.block_dilated(L, b, r), i)) == bool(int(want))
        elif kind == "local_nnz":
            L, w = a
            assert orc.mask_to_csr(orc.window(L, w), False)[2] == int(want)
            assert dense.window_mask(L, w).sum() == int(want)
        elif kind == "local_neighbors":
            L, w, i = a
            assert list(orc.neighbors(orc.window(L, w), i)) == [int(x) for x in want.split(",")]
        elif kind == "global_minus_local_nnz":
            L, g, w = a
            m = dense.global_window_mask(L, w, [g]) & ~dense.window_mask(L, w)
            assert m.sum() == int(want)
        else:
            raise AssertionError(kind)


def window_nnz_closed_form(L, w, r):
    """nnz = L + 2 * sum_{t=1}^{m'} (L - t r), m' = min(floor((w-1)/r), floor((L-1)/r))."""
    mp = min((w - 1) // r, (L - 1) // r)
    return L + 2 * sum(L - t * r for t in range(1, mp + 1))


@pytest.mark.parametrize("L,w,r", [(1024, 32, 1), (1000, 256, 2), (77, 5, 3), (64, 200, 1), (300, 17, 4),
                                   (1, 1, 1), (5, 1, 2)])
def test_window_nnz_and_degrees_closed_form(orc, L, w, r):
    rp, ci, nnz = orc.mask_to_csr(orc.window(L, w, r))
    assert nnz == window_nnz_closed_form(L, w, r)
    m = (w - 1) // r
    i = np.arange(L)
    deg = 1 + np.minimum(i // r, m) + np.minimum((L - 1 - i) // r, m)
    assert np.array_equal(np.diff(rp), deg)
    # CSR invariants: sorted strictly increasing per row, in range
    for row in range(0, L, max(1, L // 13)):
        c = ci[rp[row]:rp[row + 1]]
        assert np.all(np.diff(c) > 0) and c.min() >= 0 and c.max() < L


def test_cfg1_nnz(orc):
    """Window(32) on L=1024 has 63,520 edges."""
    assert orc.mask_to_csr(orc.window(1024, 32), False)[2] == 63520


def _valuation(x, a, K):
    if x == 0:
        return K
    v = 0
    while x % a == 0:
        x //= a
        v += 1
    return v


@pytest.mark.parametrize("L,w0,alpha", [(256, 16, 2), (243, 9, 3), (200, 16, 2), (64, 64, 2), (50, 64, 2),
                                        (1024, 8, 4)])
def test_longnet_definition_vs_closed_predicate(orc, L, w0, alpha):
    """Union-of-levels enumerator == closed predicate floor(i/w_t)==floor(j/w_t),
    t = min(nu(i), nu(j), K) [derived, SURVEY §8(c) item 11] == dense grid union."""
    from oracle import dense

    K = orc.longnet_levels(w0, alpha, L)
    Kp = 0
    while w0 * alpha ** (Kp + 1) <= L:
        Kp += 1
    assert K == (Kp if w0 <= L else 0)
    dm = dense.longnet_mask(L, w0, alpha)
    rp, ci, nnz = orc.mask_to_csr(orc.longnet(L, w0, alpha))
    assert nnz == dm.sum()
    for i in range(L):
        row = ci[rp[i]:rp[i + 1]]
        assert np.array_equal(row, np.nonzero(dm[i])[0])
        nu_i = _valuation(i, alpha, K)
        pred = [j for j in range(L)
                if (i // (w0 * alpha ** min(nu_i, _valuation(j, alpha, K), K)))
                == (j // (w0 * alpha ** min(nu_i, _valuation(j, alpha, K), K)))]
        assert list(row) == pred


def test_longnet_nnz_closed_form(orc):
    """For alpha^K w0 | L: nnz = L w0 + w0 (1 - 1/alpha) sum_{s=1}^{K} L/alpha^s; per-row
    degree w0 + min(nu(i),K) w0 (1-1/alpha) (SURVEY §8(c) closed forms)."""
    for L, w0, alpha in [(4096, 64, 2), (8192, 128, 2), (2187, 27, 3)]:
        K = orc.longnet_levels(w0, alpha, L)
        rp, _, nnz = orc.mask_to_csr(orc.longnet(L, w0, alpha), False)
        want = L * w0 + sum(w0 * (alpha - 1) * (L // alpha ** s) // alpha for s in range(1, K + 1))
        assert nnz == want
        deg = np.diff(rp)
        for i in range(0, L, 7):
            assert deg[i] == w0 + min(_valuation(i, alpha, K), K) * w0 * (alpha - 1) // alpha


def test_bigbird_golden_and_structure(orc):
    G = [0, 256, 512, 768]
    m = orc.bigbird(1024, 8, 4, 4, 0xB16B12D)
    for row in golden("bigbird_random.txt"):
        i, deg, *rnd = [int(x) for x in row.split()]
        nb = orc.neighbors(m, i)
        assert len(nb) == deg
        got = [j for j in nb if abs(j - i) >= 8 and j not in G]
        assert got == rnd
    # structure: global rows full; others = window U G U exactly n_random others
    L, w, nr = 1024, 8, 4
    for i in range(L):
        nb = set(orc.neighbors(m, i).tolist())
        if i in G:
            assert len(nb) == L
            continue
        win = {j for j in range(max(0, i - w + 1), min(L, i + w))}
        assert win <= nb and set(G) <= nb
        assert len(nb - win - set(G)) == nr


def test_bigbird_nnz_closed_form(orc):
    """nnz = g L + sum_{i not in G} (|W_i U G| + min(n_random, L - |W_i U G|))."""
    for L, w, g, nr in [(1024, 8, 4, 4), (300, 20, 3, 7), (64, 30, 2, 50)]:
        m = orc.bigbird(L, w, g, nr, 99)
        G = [k * L // g for k in range(g)]
        want = g * L
        for i in range(L):
            if i in G:
                continue
            win = set(range(max(0, i - w + 1), min(L, i + w)))
            u = len(win | set(G))
            want += u + min(nr, L - u)
        assert orc.mask_to_csr(m, False)[2] == want


# ------------------------------------------------------------------ attention
def _rand(L, H, d, seed, centred=False):
    q, k, v = synth.qkv(seed, L, H, d, "f32", centred=centred)
    return synth.as_f64(q), synth.as_f64(k), synth.as_f64(v)


@pytest.mark.parametrize("fam", ["window", "dilated", "block", "longnet", "bigbird_nornd", "longnet3"])
def test_oracle_vs_dense_bruteforce(orc, fam):
    from oracle import dense

    L, H, d = 200, 2, 16
    q, k, v = _rand(L, H, d, 7, centred=True)
    q *= 4.0  # sharpen softmax so a wrong weight shows
    if fam == "window":
        m, dm = orc.window(L, 9), dense.window_mask(L, 9)
    elif fam == "dilated":
        m, dm = orc.window(L, 20, 3), dense.window_mask(L, 20, 3)
    elif fam == "block":
        m, dm = orc.block_dilated(L, 25, 2), dense.block_dilated_mask(L, 25, 2)
    elif fam == "longnet":
        m, dm = orc.longnet(L, 8, 2), dense.longnet_mask(L, 8, 2)
    elif fam == "longnet3":
        m, dm = orc.longnet(L, 5, 3), dense.longnet_mask(L, 5, 3)
    else:
        m = orc.bigbird(L, 6, 3, 0, 1)
        dm = dense.global_window_mask(L, 6, [0, L // 3, 2 * L // 3])
    got, edges = orc.attention(q, k, v, m)
    want = dense.masked_attention(q, k, v, dm)
    assert edges == dm.sum() * H  # work == nnz (per head)
    np.testing.assert_allclose(got, want, rtol=0, atol=1e-12)


def test_empty_rows_are_zero(orc):
    from oracle import dense

    L, H, d = 64, 1, 8
    q, k, v = _rand(L, H, d, 3)
    m, dm = orc.block_dilated(L, 16, 3), dense.block_dilated_mask(L, 16, 3)
    got, _ = orc.attention(q, k, v, m)
    empty = dm.sum(1) == 0
    assert empty.any()
    assert np.all(got[empty] == 0)
    np.testing.assert_allclose(got, dense.masked_attention(q, k, v, dm), atol=1e-12, rtol=0)
    # explicit CSR with empty rows
    rp = np.array([0, 0, 2, 2, 3], np.int64)
    ci = np.array([0, 3, 1], np.int32)
    q4, k4, v4 = q[:4], k[:4], v[:4]
    got, e = orc.attention(q4, k4, v4, orc.csr(4, rp, ci))
    assert e == 3 and np.all(got[0] == 0) and np.all(got[2] == 0)
    np.testing.assert_array_equal(got[3], v4[1])


def test_full_window_equals_sdpa(orc):
    """Window(w >= L) is full attention: library routine torch SDPA (fp64, no mask)."""
    L, H, d = 96, 3, 32
    q, k, v = _rand(L, H, d, 11)
    got, edges = orc.attention(q, k, v, orc.window(L, L + 5))
    assert edges == L * L * H
    t = lambda a: torch.from_numpy(a).permute(1, 0, 2)  # [H, L, d]
    ref = torch.nn.functional.scaled_dot_product_attention(t(q), t(k), t(v)).permute(1, 0, 2).numpy()
    np.testing.assert_allclose(got, ref, rtol=0, atol=1e-13)


def test_longnet_K0_is_block_diagonal_sdpa(orc):
    """LongNet with L < alpha*w0 has one level: block-diagonal full attention (SDPA per block)."""
    L, H, d, w0 = 100, 2, 16, 64
    q, k, v = _rand(L, H, d, 5)
    got, _ = orc.attention(q, k, v, orc.longnet(L, w0, 2))
    t = lambda a: torch.from_numpy(a).permute(1, 0, 2)
    for b0 in (0, 64):
        b1 = min(L, b0 + w0)
        ref = torch.nn.functional.scaled_dot_product_attention(
            t(q[b0:b1]), t(k[b0:b1]), t(v[b0:b1])).permute(1, 0, 2).numpy()
        np.testing.assert_allclose(got[b0:b1], ref, rtol=0, atol=1e-13)


def test_identity_mask_gives_v(orc):
    """Window(1): each row attends only to itself -> O = V exactly."""
    L, H, d = 50, 2, 8
    q, k, v = _rand(L, H, d, 9)
    got, edges = orc.attention(q, k, v, orc.window(L, 1))
    assert edges == L * H
    assert np.array_equal(got, v)


def test_zero_q_gives_neighbour_mean(orc):
    L, H, d = 80, 1, 16
    q, k, v = _rand(L, H, d, 13)
    q[:] = 0.0
    m = orc.window(L, 7, 2)
    got, _ = orc.attention(q, k, v, m)
    for i in range(L):
        nb = orc.neighbors(m, i)
        np.testing.assert_allclose(got[i, 0], v[nb, 0].mean(0), rtol=0, atol=1e-14)


def test_constant_v_and_key_shift_invariance(orc):
    L, H, d = 90, 2, 16
    q, k, v = _rand(L, H, d, 17)
    m = orc.longnet(L, 8, 2)
    vc = np.full_like(v, 0.375)
    got, _ = orc.attention(q, k, vc, m)
    np.testing.assert_allclose(got, vc, rtol=0, atol=1e-15)
    base, _ = orc.attention(q, k, v, m)
    c = np.linspace(-3, 5, d)
    shifted, _ = orc.attention(q, k + c[None, None, :] * 50.0, v, m)  # large shift: overflow-safe
    np.testing.assert_allclose(shifted, base, rtol=0, atol=1e-10)


def test_equal_scores_average(orc):
    """Two neighbours with equal scores -> plain average of their V."""
    L, H, d = 2, 1, 4
    q = np.ones((L, H, d))
    k = np.ones((L, H, d))
    v = np.array([[[1.0, 2, 3, 4]], [[3.0, 2, 1, 0]]])
    got, _ = orc.attention(q, k, v, orc.window(L, 2))
    np.testing.assert_array_equal(got[0, 0], [2.0, 2.0, 2.0, 2.0])


def test_safe_softmax_large_q(orc):
    """Q + 1000 stays finite: all exponents <= 0 after max subtraction."""
    L, H, d = 64, 1, 16
    q, k, v = _rand(L, H, d, 19)
    got, _ = orc.attention(q + 1000.0, k, v, orc.window(L, 5))
    assert np.all(np.isfinite(got))


def test_alg1_equals_two_pass(orc):
    """Literal Algorithm 1 (per-step division) == two-pass softmax within 1e-12."""
    L, H, d = 160, 2, 32
    q, k, v = _rand(L, H, d, 23, centred=True)
    for m in (orc.window(L, 40, 3), orc.longnet(L, 8, 2), orc.bigbird(L, 5, 2, 4, 3)):
        a, e1 = orc.attention(q * 3, k, v, m)
        b, e2 = orc.attention_alg1(q * 3, k, v, m)
        assert e1 == e2
        np.testing.assert_allclose(a, b, rtol=0, atol=1e-12)


def test_seeded_rows_match_arrays(orc):
    """Row regeneration from the counter hash equals the full-array path."""
    L, H, d = 300, 2, 32
    for dt in ("f32", "bf16", "f16"):
        q, k, v = synth.qkv(77, L, H, d, dt)
        Q, Kt, V = (synth.as_f64(x) for x in (q, k, v))
        m = orc.window(L, 20, 2)
        rows = [0, 1, 150, 299]
        a, _ = orc.attention(Q, Kt, V, m, rows=rows)
        b, _ = orc.attention_seeded(77, dt, m, H, d, rows=rows)
        np.testing.assert_array_equal(a, b)


def test_sparsity_schedule_paper_values():
    """S_f = 2730/L reproduces the printed values with decimal k."""
    for row in golden("paper_values.txt"):
        key, *vals = row.split()
        if key != "sf":
            continue
        L, want = int(vals[0]), float(vals[1])
        got = 2730.0 / L
        assert float(f"{got:.2g}") == pytest.approx(want, rel=1e-9), (L, got, want)


# ------------------------------------------------------------ composition components (f1)
@pytest.mark.parametrize("L,w,ng,nr,r,gidx", [(300, 9, 3, 5, 1, None), (500, 21, 4, 6, 2, None),
                                             (200, 15, 3, 2, 3, [0, 77, 199]), (40, 8, 2, 60, 1, None)])
def test_bigbird_components_are_disjoint_and_cover_the_mask(orc, L, w, ng, nr, r, gidx):
    """Window, global-minus-window and random parts partition the BigBird
    mask: pairwise disjoint, union = the full definition, window part = WINDOW(w, r), and
    the global part is exactly {(i, j) : (i in G or j in G) and j not in W_i}."""
    full = orc.bigbird(L, w, ng, nr, 7, global_idx=gidx, r=r)
    parts = {p: orc.bigbird(L, w, ng, nr, 7, global_idx=gidx, r=r, parts=p) for p in (1, 2, 4)}
    G = set(gidx) if gidx is not None else {(k * L) // ng for k in range(ng)}
    win = orc.window(L, w, r)
    for i in range(L):
        rows = {p: set(orc.neighbors(m, i).tolist()) for p, m in parts.items()}
        assert not (rows[1] & rows[2]) and not (rows[1] & rows[4]) and not (rows[2] & rows[4])
        assert rows[1] | rows[2] | rows[4] == set(orc.neighbors(full, i).tolist())
        assert rows[1] == set(orc.neighbors(win, i).tolist())
        W = rows[1]
        want_g = {j for j in range(L) if (i in G or j in G) and j not in W}
        assert rows[2] == want_g
        if i in G:
            assert not rows[4]


@pytest.mark.parametrize("seed", range(4))
def test_coo_to_csr_matches_dense_brute_force(orc, seed):
    """oracle.coo_to_csr (sets) against a dense 0-1 matrix built from the edge list and read
    back row-major by np.nonzero — an independent route to the same unique sorted CSR.
    Duplicates, shuffled order, empty rows and a full row are present."""
    rng = np.random.default_rng(seed)
    L = [1, 7, 64, 300][seed]
    n = [3, 40, 900, 5000][seed]
    rows = rng.integers(0, L, n)
    cols = rng.integers(0, L, n)
    if L > 2:
        rows = np.concatenate([rows, np.full(L, L - 1), rows[: n // 3]])  # full last row + duplicates
        cols = np.concatenate([cols, np.arange(L), cols[: n // 3]])
    perm = rng.permutation(len(rows))
    rows, cols = rows[perm], cols[perm]
    rp, ci = orc.coo_to_csr(L, rows, cols)
    dense = np.zeros((L, L), dtype=bool)
    dense[rows, cols] = True
    r2, c2 = np.nonzero(dense)
    assert np.array_equal(ci, c2.astype(np.int32))
    assert np.array_equal(rp, np.concatenate([[0], np.cumsum(dense.sum(1))]))
    if L > 2:
        assert rp[L] - rp[L - 1] == L


def test_coo_to_csr_rejects_out_of_range(orc):
    with pytest.raises(ValueError):
        orc.coo_to_csr(4, [0, 4], [1, 1])


@pytest.mark.parametrize("L,w0,alpha", [(256, 16, 2), (300, 7, 3), (512, 64, 2), (100, 200, 2)])
def test_longnet_multiset_against_weighted_dense(orc, L, w0, alpha):
    """LongNet's multiset mixture (reading R11b): the oracle's neighbour lists with repeats
    reproduce the dense multiplicity matrix (each level's BlockDilated block added), and its
    attention equals the weighted dense softmax within 1e-12; with one level (w0 >= L) it is
    the set version."""
    from oracle import dense

    om = orc.longnet(L, w0, alpha, multiset=True)
    C = dense.longnet_multiplicity(L, w0, alpha)
    rp, ci, nnz = orc.mask_to_csr(om)
    assert nnz == C.sum()
    for i in range(0, L, max(1, L // 37)):
        want = np.repeat(np.arange(L), C[i])
        assert np.array_equal(ci[rp[i]:rp[i + 1]], want)
    q, k, v = orc.inputs(0x5EED0004, L, 1, 16, "f32")
    got, _ = orc.attention(q, k, v, om)
    assert np.abs(got - dense.weighted_attention(q, k, v, C)).max() < 1e-12
    if w0 >= L:
        want_set, _ = orc.attention(q, k, v, orc.longnet(L, w0, alpha))
        assert np.abs(got - want_set).max() < 1e-12
    else:  # repeats exist and change the result
        assert C.max() > 1
        want_set, _ = orc.attention(q, k, v, orc.longnet(L, w0, alpha))
        assert np.abs(got - want_set).max() > 1e-6


def test_longnet_multiset_closed_form_count(orc):
    """Full segments: level k holds L / alpha^k lattice points, each meeting w0 of them, so
    nnz = L w0 sum_k alpha^-k — at L = 2^12, w0 = 16: 16 * 4096 * (2 - 2^-8) = 130,816."""
    rp, _, nnz = orc.mask_to_csr(orc.longnet(4096, 16, 2, multiset=True), with_cols=False)
    assert nnz == 130_816


# ---------------------------------------------------------------- backward
def _bwd_inputs(L, H, d, seed):
    rng = np.random.default_rng(seed)
    return tuple(rng.standard_normal((L, H, d)) for _ in range(4))  # q, k, v, dO


@pytest.mark.parametrize("fam", ["window", "longnet_multiset", "csr_empty_rows", "bigbird"])
def test_backward_matches_finite_differences(orc, fam):
    """orc_attention_backward against central differences of orc_attention (an independent
    route: only the forward definition is used) for the scalar loss sum(dO * O)."""
    L, H, d = 12, 2, 4
    q, k, v, g = _bwd_inputs(L, H, d, 7)
    if fam == "window":
        om = orc.window(L, 3, 1)
    elif fam == "longnet_multiset":
        om = orc.longnet(L, 2, 2, multiset=True)  # repeated columns: weights count twice
    elif fam == "bigbird":
        om = orc.bigbird(L, 2, 1, 2, 5)
    else:
        rp = np.array([0, 2, 2, 5, 6, 6, 8, 9, 9, 12, 13, 13, 16], dtype=np.int64)  # rows 1, 4, 7, 10 empty
        ci = np.array([0, 5, 1, 2, 11, 3, 4, 9, 6, 7, 8, 10, 11, 0, 5, 11], dtype=np.int32)
        om = orc.csr(L, rp, ci)
    dq, dk, dv, _ = orc.attention_backward(q, k, v, om, g)

    def loss(q_, k_, v_):
        return float((orc.attention(q_, k_, v_, om)[0] * g).sum())

    h = 1e-6
    for name, x, grad in (("q", q, dq), ("k", k, dk), ("v", v, dv)):
        num = np.zeros_like(x)
        for idx in np.ndindex(*x.shape):
            xp, xm = x.copy(), x.copy()
            xp[idx] += h
            xm[idx] -= h
            args_p = {"q": q, "k": k, "v": v}
            args_m = dict(args_p)
            args_p[name], args_m[name] = xp, xm
            num[idx] = (loss(**{a + "_": b for a, b in args_p.items()}) -
                        loss(**{a + "_": b for a, b in args_m.items()})) / (2 * h)
        np.testing.assert_allclose(grad, num, rtol=1e-6, atol=1e-8, err_msg=f"d{name} ({fam})")


@pytest.mark.parametrize("fam,L,args", [("window", 64, (9, 2)), ("longnet", 64, (8, 2)), ("block", 60, (12, 3))])
def test_backward_matches_torch_autograd_dense(orc, fam, L, args):
    """Library routine: torch.autograd (fp64) through the dense masked softmax of
    oracle/dense.py's predicate grid (shares no code with oracle.c)."""
    from oracle import dense

    H, d = 2, 8
    q, k, v, g = _bwd_inputs(L, H, d, 11)
    grid = {"window": dense.window_mask, "longnet": dense.longnet_mask, "block": dense.block_dilated_mask}[fam](L, *args)
    om = {"window": orc.window, "longnet": orc.longnet, "block": orc.block_dilated}[fam](L, *args)
    tq, tk, tv = (torch.tensor(x, requires_grad=True) for x in (q, k, v))
    mask = torch.tensor(grid)
    s = torch.einsum("ihc,jhc->hij", tq, tk) / math.sqrt(d)
    s = s.masked_fill(~mask, float("-inf"))
    p = torch.softmax(s, dim=-1)
    p = torch.nan_to_num(p, nan=0.0)  # empty rows (none here)
    o = torch.einsum("hij,jhc->ihc", p, tv)
    (o * torch.tensor(g)).sum().backward()
    dq, dk, dv, edges = orc.attention_backward(q, k, v, om, g)
    assert edges == int(grid.sum()) * H
    for got, want in ((dq, tq.grad), (dk, tk.grad), (dv, tv.grad)):
        np.testing.assert_allclose(got, want.numpy(), rtol=1e-10, atol=1e-12)


@pytest.mark.parametrize("L,w0,alpha", [(300, 8, 2), (250, 5, 3), (128, 16, 2)])
def test_longnet_head_offsets_vs_dense(orc, L, w0, alpha):
    """Per-head offsets (f4, reading R11c): the oracle's per-head attention equals the dense
    brute force over each head's own predicate grid; head 0 equals plain LongNet."""
    from oracle import dense

    H, d = 6, 8
    rng = np.random.default_rng(L)
    q, k, v = (rng.random((L, H, d)) for _ in range(3))
    got, edges = orc.attention(q, k, v, orc.longnet(L, w0, alpha, head_offsets=True))
    total = 0
    for h in range(H):
        grid = dense.longnet_mask(L, w0, alpha, head=h)
        total += int(grid.sum())
        want = dense.masked_attention(q[:, h:h + 1], k[:, h:h + 1], v[:, h:h + 1], grid)
        np.testing.assert_allclose(got[:, h:h + 1], want, rtol=0, atol=1e-12)
    assert edges == total
    plain, _ = orc.attention(q, k, v, orc.longnet(L, w0, alpha))
    np.testing.assert_array_equal(got[:, 0], plain[:, 0])
    assert np.array_equal(dense.longnet_mask(L, w0, alpha, head=0), dense.longnet_mask(L, w0, alpha))

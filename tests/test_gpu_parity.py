"""GPU parity: the CUDA path (through the C ABI) against the fp64 oracle.

Tolerances (BASELINE.json north_star): max abs error 1e-4 for fp32 and 2e-2 for
bf16/fp16 against the oracle on identical inputs; the paper's own protocol (PAPER.md:302:
L=256, d=32, U[0,1), atol 1e-8 + rtol 1e-5) additionally at fp32.  CSR construction and
the work counters are compared bit for bit.
"""
import numpy as np
import pytest
import torch

import synth

pytestmark = pytest.mark.gpu

TOL = {"f32": 1e-4, "bf16": 2e-2, "f16": 2e-2}
TDT = {"f32": torch.float32, "bf16": torch.bfloat16, "f16": torch.float16}


@pytest.fixture(scope="module")
def ga():
    import paper_2502_01659_b200 as ga

    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    return ga


def _pair(ga, orc, fam, L, args):
    """(product mask, oracle mask) for a family."""
    if fam == "window":
        return ga.Window(*args), orc.window(L, *args)
    if fam == "block":
        return ga.BlockDilated(*args), orc.block_dilated(L, *args)
    if fam == "longnet":
        return ga.LongNet(*args), orc.longnet(L, *args)
    if fam == "bigbird":
        return ga.BigBird(*args), orc.bigbird(L, *args)
    raise ValueError(fam)


def _inputs(L, H, d, dt, seed, centred=False):
    q, k, v = synth.qkv(seed, L, H, d, dt, centred=centred)
    return (q, k, v), tuple(synth.as_f64(x) for x in (q, k, v))


def _run(ga, cpu_qkv, mask, **kw):
    q, k, v = (x.cuda() for x in cpu_qkv)
    out = ga.attention(q, k, v, mask, **kw)
    torch.cuda.synchronize()
    return out.double().cpu().numpy()


def _csr_from_oracle(ga, orc_mask):
    import oracle

    rp, ci, nnz = oracle.mask_to_csr(orc_mask)
    return ga.CSR(torch.from_numpy(rp).cuda(), torch.from_numpy(ci.astype(np.int32)).cuda()), (rp, ci)


# ---------------------------------------------------------------- paper protocol E0
@pytest.mark.parametrize("fam,args", [("window", (9, 1)), ("window", (40, 3)), ("block", (32, 2)),
                                      ("longnet", (16, 2)), ("window", (300, 1))])
def test_paper_protocol_fp32(ga, orc, fam, args):
    """L=256, d_k=32, U[0,1), allclose(atol=1e-8, rtol=1e-5) at fp32."""
    L, H, d = 256, 1, 32
    cpu, f64 = _inputs(L, H, d, "f32", 302)
    m, om = _pair(ga, orc, fam, L, args)
    want, _ = orc.attention(*f64, om)
    got = _run(ga, cpu, m, kernel="edge")
    np.testing.assert_allclose(got, want, rtol=1e-5, atol=1e-8)


@pytest.mark.parametrize("seed", range(20))
def test_paper_protocol_random_csr(ga, orc, seed):
    """20 seeded random masks of varied sparsity, explicit CSR (S:492 acceptance 1)."""
    L, H, d = 256, 1, 32
    rng = np.random.default_rng(seed)
    dense = rng.random((L, L)) < [0.001, 0.01, 0.1, 0.5][seed % 4]
    rp = np.concatenate([[0], np.cumsum(dense.sum(1))]).astype(np.int64)
    ci = np.nonzero(dense)[1].astype(np.int32)
    om = orc.csr(L, rp, ci)
    cpu, f64 = _inputs(L, H, d, "f32", 1000 + seed)
    want, _ = orc.attention(*f64, om)
    m = ga.CSR(torch.from_numpy(rp).cuda(), torch.from_numpy(ci).cuda())
    got = _run(ga, cpu, m)
    np.testing.assert_allclose(got, want, rtol=1e-5, atol=1e-8)


# ---------------------------------------------------------------- families x dtypes x d
CASES = [
    ("window", 1031, (33, 1)), ("window", 1500, (64, 2)), ("window", 777, (200, 3)),
    ("block", 1000, (64, 2)), ("longnet", 2048, (64, 2)), ("longnet", 1800, (27, 3)),
    ("longnet", 3000, (100, 3)),
]


@pytest.mark.parametrize("dt", ["f32", "bf16", "f16"])
@pytest.mark.parametrize("d", [32, 64, 128])
@pytest.mark.parametrize("case", CASES, ids=lambda c: f"{c[0]}{c[1]}")
def test_families_dtypes_dims(ga, orc, dt, d, case):
    fam, L, args = case
    H = 2
    cpu, f64 = _inputs(L, H, d, dt, 11 + d, centred=True)
    m, om = _pair(ga, orc, fam, L, args)
    want, _ = orc.attention(*f64, om)
    for kernel in ("edge", "auto"):
        got = _run(ga, cpu, m, kernel=kernel)
        err = np.abs(got - want).max()
        assert err <= TOL[dt], (kernel, err)


@pytest.mark.parametrize("w,r", [(16, 1), (17, 1), (41, 2), (64, 1), (128, 1), (256, 2), (262, 1), (300, 3)])
@pytest.mark.parametrize("dt,d", [("bf16", 64), ("f16", 64), ("bf16", 32), ("bf16", 128)])
def test_band_kernel_vs_oracle(ga, orc, w, r, dt, d):
    """Tensor-core band kernel (forced) against the oracle: m = floor((w-1)/r) covers the
    exact-16 dense case (m=127), ragged dense remainders, m=15 (smallest), dilation r>1."""
    L, H = 3000, 2
    cpu, f64 = _inputs(L, H, d, dt, w * 7 + r, centred=True)
    want, _ = orc.attention(*f64, orc.window(L, w, r))
    m = (w - 1) // r
    if 112 * 2 * d + 2 * (112 + 2 * m) * 2 * d > 227 * 1024:  # Q tile + K/V band do not fit SMEM
        with pytest.raises(ga.GaError, match="UNSUPPORTED"):
            _run(ga, cpu, ga.Window(w, r), kernel="window")
        got = _run(ga, cpu, ga.Window(w, r), kernel="auto")  # falls back to the edge kernel
        assert np.abs(got - want).max() <= TOL[dt]
        return
    got = _run(ga, cpu, ga.Window(w, r), kernel="window")
    assert np.abs(got - want).max() <= TOL[dt]


@pytest.mark.parametrize("L,w,r", [(3000, 65, 1), (3000, 128, 1), (3000, 129, 1), (3000, 256, 2), (3001, 200, 2),
                                   (3000, 300, 3), (2999, 400, 4), (5000, 512, 4), (100, 128, 1), (1, 128, 1),
                                   (700, 256, 2), (20000, 256, 2)])
@pytest.mark.parametrize("dt", ["bf16", "f16"])
def test_window_tc_vs_oracle(ga, orc, L, w, r, dt):
    """tcgen05 window kernel (forced) against the oracle: m = floor((w-1)/r) from 64 to 128,
    dilation 1-4, ragged L (partial tiles, partial chunks, sequences shorter than one tile),
    tile pairs with one tile, several pairs per CTA run (L=20000)."""
    H, d = 2, 64
    cpu, f64 = _inputs(L, H, d, dt, w * 11 + r + L, centred=True)
    want, _ = orc.attention(*f64, orc.window(L, w, r))
    got = _run(ga, cpu, ga.Window(w, r), kernel="tc")
    assert np.abs(got - want).max() <= TOL[dt]
    # uncentred U[0,1) inputs (the paper's distribution): flat softmax, all weights alive
    cpu2, f642 = _inputs(L, H, d, dt, w * 13 + r + L)
    want2, _ = orc.attention(*f642, orc.window(L, w, r))
    got2 = _run(ga, cpu2, ga.Window(w, r), kernel="tc")
    assert np.abs(got2 - want2).max() <= TOL[dt]


def test_window_tc_scaled_queries(ga, orc):
    """Sharp softmax (queries x 8): the lazy rescale fires often; tcgen05 kernel vs oracle."""
    L, H, d = 4096, 2, 64
    q, k, v = synth.qkv(77, L, H, d, "bf16", centred=True)
    q = (q.float() * 8).bfloat16()
    f64 = tuple(synth.as_f64(x) for x in (q, k, v))
    want, _ = orc.attention(*f64, orc.window(L, 256, 2))
    got = _run(ga, (q, k, v), ga.Window(256, 2), kernel="tc")
    assert np.abs(got - want).max() <= 2e-2


def test_window_tc_unsupported(ga):
    """The tcgen05 window kernel refuses what it does not implement (d != 64, fp32, m outside
    [64, 128], r > 4) instead of computing something else."""
    for shape, dt, mask in (((300, 1, 32), torch.bfloat16, ga.Window(128)), ((300, 1, 64), torch.float32, ga.Window(128)),
                            ((300, 1, 64), torch.bfloat16, ga.Window(300)), ((300, 1, 64), torch.bfloat16, ga.Window(40)),
                            ((3000, 1, 64), torch.bfloat16, ga.Window(600, 5))):
        x = torch.zeros(shape, dtype=dt, device="cuda")
        with pytest.raises(ga.GaError, match="UNSUPPORTED"):
            ga.attention(x, x.clone(), x.clone(), mask, kernel="tc")


def test_band_kernel_cfg2_shape(ga, orc):
    """cfg2 geometry (8 heads, Window(256, r=2), bf16) at L=8192: every row vs the oracle."""
    L, H, d = 8192, 8, 64
    cpu, f64 = _inputs(L, H, d, "bf16", 0x5EED0002)
    want, _ = orc.attention(*f64, orc.window(L, 256, 2))
    for kernel in ("window", "tc", "edge"):
        got = _run(ga, cpu, ga.Window(256, 2), kernel=kernel)
        assert np.abs(got - want).max() <= 2e-2, kernel
    with pytest.raises(ga.GaError, match="UNSUPPORTED"):
        q32 = torch.zeros(64, 1, 64, device="cuda")
        ga.attention(q32, q32.clone(), q32.clone(), ga.Window(32), kernel="window")


@pytest.mark.parametrize("L,w0,alpha", [(8192, 64, 2), (5000, 100, 3), (4096, 16, 2), (3000, 2048, 2),
                                         (6561, 27, 3), (10000, 40, 4)])
@pytest.mark.parametrize("dt,d", [("bf16", 64), ("f16", 64), ("bf16", 32), ("bf16", 128)])
def test_longnet_tiled_vs_oracle(ga, orc, L, w0, alpha, dt, d):
    """LongNet dense-group tensor-core kernel (forced) vs the oracle; covers ragged key
    tails (w0 not a multiple of 16), alpha in {2,3,4}, a single partial segment, and a
    query-range shard (q_begin > 0 with the full K/V)."""
    H = 2
    cpu, f64 = _inputs(L, H, d, dt, L + w0, centred=True)
    om = orc.longnet(L, w0, alpha)
    want, _ = orc.attention(*f64, om)
    got = _run(ga, cpu, ga.LongNet(w0, alpha), kernel="tiled")
    assert np.abs(got - want).max() <= TOL[dt]
    q, k, v = (x.cuda() for x in cpu)
    r0, r1 = L // 3, L // 3 + L // 4
    part = ga.attention(q[r0:r1].contiguous(), k, v, ga.LongNet(w0, alpha), L=L, q_begin=r0, kernel="tiled")
    assert np.abs(part.double().cpu().numpy() - want[r0:r1]).max() <= TOL[dt]


@pytest.mark.parametrize("L,w0,alpha,dt", [(32768, 2048, 2, "bf16"), (4096, 256, 2, "bf16"), (8192, 512, 2, "f16"),
                                            (20000, 1000, 3, "bf16"), (5000, 300, 2, "bf16")])
def test_longnet_tcgen05_vs_oracle(ga, orc, L, w0, alpha, dt):
    """tcgen05/TMEM path (groups of >= 128 rows: S and P V on tcgen05.mma, softmax from
    TMEM) + mma.sync for the small groups, against the oracle; full and query-shard runs.
    (1000, alpha 3) and 300 give ragged key tails and partial 128-row tiles."""
    H, d = 1, 64
    cpu, f64 = _inputs(L, H, d, dt, w0 + L, centred=True)
    want, _ = orc.attention(*f64, orc.longnet(L, w0, alpha))
    got = _run(ga, cpu, ga.LongNet(w0, alpha), kernel="tc")
    assert np.abs(got - want).max() <= TOL[dt]
    q, k, v = (x.cuda() for x in cpu)
    r0, r1 = L // 4, L // 4 + L // 3
    part = ga.attention(q[r0:r1].contiguous(), k, v, ga.LongNet(w0, alpha), L=L, q_begin=r0, kernel="tc")
    assert np.abs(part.double().cpu().numpy() - want[r0:r1]).max() <= TOL[dt]


@pytest.mark.parametrize("dt", ["f32", "bf16"])
def test_csr_bigbird_with_heavy_split(ga, orc, dt):
    """BigBird via device CSR; heavy global rows through the split+merge path (a7)."""
    L, H, d = 4096, 2, 64
    m = ga.BigBird(32, 8, 16, seed=77)
    om = orc.bigbird(L, 32, 8, 16, 77)
    csr = ga.mask_to_csr(m, L)
    cpu, f64 = _inputs(L, H, d, dt, 5)
    want, _ = orc.attention(*f64, om)
    q, k, v = (x.cuda() for x in cpu)
    for C in (256, 1000, 0):
        ws = torch.empty(ga.workspace_size(csr, L, d, H, TDT[dt], heavy_threshold=C), dtype=torch.uint8,
                         device="cuda")
        out = ga.attention(q, k, v, csr, workspace=ws, heavy_threshold=C)
        err = (out.double().cpu().numpy() - want).__abs__().max()
        assert err <= TOL[dt], (C, err)
    out = ga.attention(q, k, v, csr)  # no workspace: unsplit rows
    assert np.abs(out.double().cpu().numpy() - want).max() <= TOL[dt]


def test_empty_rows_and_ragged_csr(ga, orc):
    L, H, d = 300, 1, 64
    rng = np.random.default_rng(3)
    deg = rng.integers(0, 5, L)
    deg[::7] = 0
    deg[5] = 300
    rows = [np.sort(rng.choice(L, k, replace=False)) for k in deg]
    rp = np.concatenate([[0], np.cumsum(deg)]).astype(np.int64)
    ci = np.concatenate(rows).astype(np.int32)
    cpu, f64 = _inputs(L, H, d, "f32", 8)
    want, _ = orc.attention(*f64, orc.csr(L, rp, ci))
    m = ga.CSR(torch.from_numpy(rp).cuda(), torch.from_numpy(ci).cuda())
    got = _run(ga, cpu, m)
    assert np.all(got[deg == 0] == 0)
    assert np.abs(got - want).max() <= 1e-4


@pytest.mark.parametrize("variant", ["", "GA_CSR_CPASYNC", "GA_CSR_LDG"])
@pytest.mark.parametrize("dt", ["bf16", "f16"])
@pytest.mark.parametrize("d", [32, 64, 128])
def test_csr_mma_ragged_degrees(ga, orc, dt, d, variant, monkeypatch):
    """Explicit CSR on the mma.sync path (csr_mma.cu; d = 64 staged by TMA gather4, or the
    cp.async ring / direct loads when the variant flag is set): degrees 0, 1, 15, 16, 17,
    31..33, 47, 48, 200 and a full row cover every 16-edge block tail, the stage ring and the
    index ring; random sorted columns; centred inputs.  Same bar for the edge kernel."""
    if variant:
        monkeypatch.setenv(variant, "1")
    L, H = 700, 2
    rng = np.random.default_rng(d + (0 if dt == "bf16" else 1))
    pattern = [0, 1, 15, 16, 17, 31, 32, 33, 47, 48, 200, 5, 64, 65, 700]
    deg = np.array([pattern[i % len(pattern)] for i in range(L)])
    rows = [np.sort(rng.choice(L, k, replace=False)) for k in deg]
    rp = np.concatenate([[0], np.cumsum(deg)]).astype(np.int64)
    ci = np.concatenate(rows).astype(np.int32)
    cpu, f64 = _inputs(L, H, d, dt, 21 + d, centred=True)
    want, _ = orc.attention(*f64, orc.csr(L, rp, ci))
    m = ga.CSR(torch.from_numpy(rp).cuda(), torch.from_numpy(ci).cuda())
    for kernel in ("auto", "edge"):
        got = _run(ga, cpu, m, kernel=kernel)
        assert np.all(got[deg == 0] == 0), kernel
        err = np.abs(got - want).max()
        assert err <= TOL[dt], (kernel, err)


def test_csr_mma_large_scores_rescale(ga, orc):
    """Scores spanning many 2^8 rescale thresholds (queries scaled x40) on the mma CSR path."""
    L, H, d = 512, 1, 64
    rng = np.random.default_rng(5)
    deg = rng.integers(1, 300, L)
    rows = [np.sort(rng.choice(L, k, replace=False)) for k in deg]
    rp = np.concatenate([[0], np.cumsum(deg)]).astype(np.int64)
    ci = np.concatenate(rows).astype(np.int32)
    (q, k, v), _ = _inputs(L, H, d, "bf16", 99, centred=True)
    q = (q.float() * 40).bfloat16()
    f64 = tuple(synth.as_f64(x) for x in (q, k, v))
    want, _ = orc.attention(*f64, orc.csr(L, rp, ci))
    m = ga.CSR(torch.from_numpy(rp).cuda(), torch.from_numpy(ci).cuda())
    got = _run(ga, (q, k, v), m)
    assert np.abs(got - want).max() <= 2e-2


@pytest.mark.parametrize("L,n", [(1, 0), (1, 5), (97, 2000), (5000, 200_000)])
def test_coo_to_csr_bit_exact(ga, orc, L, n):
    """ga_coo_to_csr (device sort + unique) == the oracle's set-based conversion, bit for bit,
    for shuffled edge lists with duplicates; attention over the result equals attention over
    the same CSR built on the host."""
    rng = np.random.default_rng(L + n)
    rows = rng.integers(0, L, n).astype(np.int32)
    cols = rng.integers(0, L, n).astype(np.int32)
    rows = np.concatenate([rows, rows[: n // 4]])
    cols = np.concatenate([cols, cols[: n // 4]])
    perm = rng.permutation(len(rows))
    rows, cols = rows[perm], cols[perm]
    rp, ci = orc.coo_to_csr(L, rows, cols)
    csr = ga.coo_to_csr(torch.from_numpy(rows).cuda(), torch.from_numpy(cols).cuda(), L)
    assert np.array_equal(csr.row_ptr.cpu().numpy(), rp)
    assert np.array_equal(csr.col_idx.cpu().numpy(), ci)
    if 0 < n <= 2000:
        H, d = 1, 64
        cpu, f64 = _inputs(L, H, d, "bf16", 31)
        want, _ = orc.attention(*f64, orc.csr(L, rp, ci))
        got = _run(ga, cpu, csr)
        assert np.abs(got - want).max() <= 2e-2


def test_coo_to_csr_errors(ga):
    r = torch.tensor([0, 5], dtype=torch.int32, device="cuda")
    c = torch.tensor([1, 1], dtype=torch.int32, device="cuda")
    with pytest.raises(ga.GaError):
        ga.coo_to_csr(r, c, 4)
    with pytest.raises(ga.GaError):
        ga.coo_to_csr(r, -c, 8)


@pytest.mark.parametrize("L,w0,alpha", [(2048, 64, 2), (1800, 27, 3)])
@pytest.mark.parametrize("dt", ["f32", "bf16"])
def test_longnet_multiset_vs_oracle(ga, orc, L, w0, alpha, dt):
    """LongNet multiset mixture (reading R11b): implicit (edge kernel) and
    as device CSR with repeated columns (bit-exact with the oracle's CSR; CSR kernels)."""
    H, d = 2, 64
    cpu, f64 = _inputs(L, H, d, dt, 41, centred=True)
    m = ga.LongNet(w0, alpha, multiset=True)
    om = orc.longnet(L, w0, alpha, multiset=True)
    want, _ = orc.attention(*f64, om)
    got = _run(ga, cpu, m)
    assert np.abs(got - want).max() <= TOL[dt]
    rp, ci, nnz = orc.mask_to_csr(om)
    assert ga.mask_count(m, L) == nnz
    csr = ga.mask_to_csr(m, L)
    assert np.array_equal(csr.row_ptr.cpu().numpy(), rp)
    assert np.array_equal(csr.col_idx.cpu().numpy(), ci)
    got2 = _run(ga, cpu, csr)
    assert np.abs(got2 - want).max() <= TOL[dt]
    # differs from the set union (repeats weigh twice)
    want_set, _ = orc.attention(*f64, orc.longnet(L, w0, alpha))
    assert np.abs(want - want_set).max() > 1e-4


@pytest.mark.parametrize("L,w0", [(65536, 2048), (5000, 300), (8192, 256)])
def test_longnet_tma_lattice_loader_bitwise(ga, L, w0, monkeypatch):
    """The LongNet tcgen05 kernel's two K/V loaders — TMA boxes from per-level lattice tensor
    maps (alpha = 2, default) and per-row cp.async (GA_LNET_CPASYNC=1) — stage the same bytes,
    so the outputs are bit-identical, for a whole run and a query sub-range, repeated (the
    repeats also catch races such as the TMEM WAR hazard of DESIGN.md K5)."""
    H, d = 2, 64
    q, k, v = ga.qkv_device(L + 3, L, H, d, torch.bfloat16)
    m = ga.LongNet(w0, 2)
    r0 = (L // 3 // w0) * w0
    monkeypatch.setenv("GA_LNET_CPASYNC", "1")
    ref = ga.attention(q, k, v, m, kernel="tc")
    ref_part = ga.attention(q[r0:].contiguous(), k, v, m, L=L, q_begin=r0, kernel="tc")
    monkeypatch.delenv("GA_LNET_CPASYNC")
    for _ in range(5):
        assert torch.equal(ga.attention(q, k, v, m, kernel="tc"), ref)
        assert torch.equal(ga.attention(q[r0:].contiguous(), k, v, m, L=L, q_begin=r0, kernel="tc"), ref_part)


@pytest.mark.parametrize("variant", ["", "GA_CSR_CPASYNC"])
def test_csr_contiguous_blocks_and_duplicate_traps(ga, orc, variant, monkeypatch):
    """Explicit CSR rows made of 16-column runs (loaded as one 16-row TMA box each) next to
    blocks that only look like runs: repeated columns spanning exactly 15 (a multiset row),
    a run shifted by one, a run cut by the row end.  Repeats weigh twice, as in the oracle."""
    if variant:
        monkeypatch.setenv(variant, "1")
    L, H, d = 600, 2, 64
    rows = []
    for i in range(L):
        b = (i * 7) % (L - 64)
        k = i % 5
        if k == 0:
            r = list(range(b, b + 48))                                  # three whole runs
        elif k == 1:
            r = [b, b + 1, b + 1] + list(range(b + 3, b + 16))           # span 15, one column repeated
        elif k == 2:
            r = list(range(b, b + 16)) + [b + 20] + list(range(b + 21, b + 37))  # run, then shifted run
        elif k == 3:
            r = list(range(b, b + 23))                                  # run + ragged tail
        else:
            r = sorted(set(range(b, b + 40, 2)))                        # strided: never a run
        rows.append(np.array(sorted(r), dtype=np.int32))
    deg = np.array([len(r) for r in rows])
    rp = np.concatenate([[0], np.cumsum(deg)]).astype(np.int64)
    ci = np.concatenate(rows).astype(np.int32)
    cpu, f64 = _inputs(L, H, d, "bf16", 77, centred=True)
    want, _ = orc.attention(*f64, orc.csr(L, rp, ci))
    m = ga.CSR(torch.from_numpy(rp).cuda(), torch.from_numpy(ci).cuda())
    got = _run(ga, cpu, m)
    assert np.abs(got - want).max() <= 2e-2


# ---------------------------------------------------------------- work optimality (T4)
@pytest.mark.parametrize("fam,L,args", [("window", 2000, (100, 3)), ("longnet", 4096, (64, 2)),
                                        ("block", 1000, (50, 4))])
def test_edge_counter_and_fingerprints(ga, orc, fam, L, args):
    """Dot products computed == nnz(mask) x heads exactly; per-row (deg, sum j,
    sum splitmix64(j)) fingerprints equal the oracle's neighbour lists (S:281 probe build)."""
    H, d = 3, 64
    m, om = _pair(ga, orc, fam, L, args)
    rp, ci, nnz = orc.mask_to_csr(om)
    q, k, v = ga.qkv_device(1, L, H, d, torch.bfloat16)
    cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
    fp = torch.zeros(L * 3, dtype=torch.int64, device="cuda")
    ga.attention(q, k, v, m, edge_counter=cnt, row_fingerprint=fp)
    assert int(cnt.item()) == nnz * H
    fp = fp.cpu().numpy().view(np.uint64).reshape(L, 3)
    deg = np.diff(rp).astype(np.uint64)
    assert np.array_equal(fp[:, 0], deg)
    with np.errstate(over="ignore"):  # per-row sums mod 2^64 via wrapping prefix sums
        z = np.zeros(1, np.uint64)
        cj = np.concatenate([z, np.cumsum(ci.astype(np.uint64), dtype=np.uint64)])
        ch = np.concatenate([z, np.cumsum(synth.splitmix64_np(ci.astype(np.uint64)), dtype=np.uint64)])
        sj = cj[rp[1:]] - cj[rp[:-1]]
        sh = ch[rp[1:]] - ch[rp[:-1]]
    assert np.array_equal(fp[:, 1], sj)
    assert np.array_equal(fp[:, 2], sh)


# ---------------------------------------------------------------- CSR generator (T5)
@pytest.mark.parametrize("fam,L,args", [
    ("window", 3000, (128, 1)), ("window", 4097, (256, 2)), ("block", 3000, (100, 3)),
    ("longnet", 8192, (64, 2)), ("longnet", 5000, (27, 3)), ("bigbird", 1024, (8, 4, 4, 0xB16B12D)),
    ("bigbird", 5000, (64, 16, 64, 99)), ("bigbird", 300, (20, 3, 300, 1)),
])
def test_csr_generator_bit_exact(ga, orc, fam, L, args):
    m, om = _pair(ga, orc, fam, L, args)
    csr = ga.mask_to_csr(m, L)
    rp, ci, nnz = orc.mask_to_csr(om)
    assert np.array_equal(csr.row_ptr.cpu().numpy(), rp)
    assert np.array_equal(csr.col_idx.cpu().numpy(), ci)
    assert ga.mask_validate(csr, L)


def test_mask_validate_rejects_malformed(ga):
    L = 10
    rp = torch.tensor([0, 2, 2, 2, 2, 2, 2, 2, 2, 2, 2], dtype=torch.int64, device="cuda")
    bad = ga.CSR(rp, torch.tensor([3, 3], dtype=torch.int32, device="cuda"))  # not strictly increasing
    assert not ga.mask_validate(bad, L)
    bad2 = ga.CSR(rp, torch.tensor([1, 10], dtype=torch.int32, device="cuda"))  # out of range
    assert not ga.mask_validate(bad2, L)


# ---------------------------------------------------------------- inputs (a0)
def test_device_input_generator_matches_golden_and_numpy(ga):
    from tests.conftest import golden

    g = {r.split()[0]: r.split()[1] for r in golden("rng.txt")}
    seed = int(g["seed"], 16)
    for dt in ("f32", "bf16", "f16"):
        q, k, v = ga.qkv_device(seed, 64, 8, 64, TDT[dt])
        ref = synth.qkv(seed, 64, 8, 64, dt)
        for a, b in zip((q, k, v), ref):
            assert torch.equal(a.cpu(), b)
    q, _, _ = ga.qkv_device(seed, 2, 8, 64, torch.float32)
    assert q[0, 0, 0].item() == float(g["Q_e0_f32"])
    assert q[1, 0, 0].item() == float(g["Q_e512_f32"])


# ---------------------------------------------------------------- properties (T3)
def test_properties(ga, orc):
    L, H, d = 513, 2, 64
    q, k, v = ga.qkv_device(4, L, H, d, torch.float32)
    out = ga.attention(q, k, v, ga.Window(1))
    assert torch.equal(out, v)  # identity mask -> O = V exactly
    vc = torch.full_like(v, 0.375)
    out = ga.attention(q, k, vc, ga.LongNet(16, 2))
    assert (out - 0.375).abs().max().item() < 1e-6
    full = ga.attention(q, k, v, ga.Window(L + 10))
    ref = torch.nn.functional.scaled_dot_product_attention(q.transpose(0, 1).double(), k.transpose(0, 1).double(),
                                                           v.transpose(0, 1).double()).transpose(0, 1)
    assert (full.double() - ref).abs().max().item() < 1e-5
    r1 = ga.attention(q, k, v, ga.Window(40, 1))
    r2 = ga.attention(q, k, v, ga.mask_to_csr(ga.Window(40), L))
    assert (r1 - r2).abs().max().item() < 1e-6
    shifted = ga.attention(q + 1000.0, k, v, ga.Window(7))
    assert torch.isfinite(shifted).all()


def test_sharded_offsets_bitwise(ga):
    """Query-range shards with halo'd K/V buffers reproduce the 1-GPU rows bit for bit
    (T7-i logical shards on one GPU)."""
    L, H, d = 8192, 4, 64
    q, k, v = ga.qkv_device(9, L, H, d, torch.bfloat16)
    m = ga.Window(256, 2)
    halo = 127 * 2
    for kernel in ("edge", "window", "tc", "auto"):
        full = ga.attention(q, k, v, m, kernel=kernel)
        # shard boundaries aligned to the kernel's tile (band kernel: 112 class rows x r tokens,
        # tcgen05 kernel: 128 x r; auto: ga.query_alignment)
        al = {"edge": 1, "window": 224, "tc": 256, "auto": ga.query_alignment(m, L, d, torch.bfloat16)}[kernel]
        for r0, r1 in ((0, 10 * al), (10 * al, 20 * al), (20 * al, 8192)):
            k0, k1 = max(0, r0 - halo), min(L, r1 + halo)
            part = ga.attention(q[r0:r1].contiguous(), k[k0:k1].contiguous(), v[k0:k1].contiguous(), m, L=L,
                                q_begin=r0, kv_begin=k0, kernel=kernel)
            assert torch.equal(part, full[r0:r1]), kernel
    # unaligned shards still agree within tolerance
    r0, r1 = 1000, 3000
    part = ga.attention(q[r0:r1].contiguous(), k[r0 - halo:r1 + halo].contiguous(), v[r0 - halo:r1 + halo].contiguous(),
                        m, L=L, q_begin=r0, kv_begin=r0 - halo)
    assert (part.float() - full[r0:r1].float()).abs().max().item() < 2e-2


@pytest.mark.parametrize("fam,args,kernel", [("longnet", (256, 2), "tiled"), ("longnet", (256, 2), "tc"),
                                             ("longnet", (100, 3), "auto"), ("window", (256, 2), "auto"),
                                             ("window", (100, 1), "auto"), ("bigbird", (64, 8, 6, 5), "auto")])
def test_repeat_launches_bitwise(ga, fam, args, kernel):
    """Every kernel is deterministic: the same launch repeated, with other kernels run in
    between to leave different data in shared memory, gives identical bytes.  (Pad rows of
    partial tiles used to take part in the rescale vote uninitialised.)"""
    L, H, d = 10000, 2, 64
    q, k, v = ga.qkv_device(31, L, H, d, torch.bfloat16)
    mask = {"window": ga.Window, "longnet": ga.LongNet, "bigbird": ga.BigBird}[fam](*args)
    if fam == "bigbird":
        mask = ga.mask_to_csr(mask, L)
    ref = ga.attention(q, k, v, mask, kernel=kernel)
    dirt = [ga.Window(300, 3), ga.LongNet(64, 2), ga.Window(40, 1)]
    for dm in dirt:
        ga.attention(q * 7.0, k * -3.0, v, dm)
        again = ga.attention(q, k, v, mask, kernel=kernel)
        assert torch.equal(again, ref), (fam, args, kernel, dm)
    # a query sub-range computes the same rows (tiles are anchored absolutely)
    al = ga.query_alignment(mask, L, d, torch.bfloat16)
    r0 = (L // 3 // al) * al
    part = ga.attention(q[r0:].contiguous(), k, v, mask, L=L, q_begin=r0, kv_begin=0, kernel=kernel)
    assert torch.equal(part, ref[r0:])


@pytest.mark.parametrize("L,w0,alpha", [(65536, 2048, 2), (20000, 1000, 3), (5000, 300, 2)])
def test_longnet_block_partials_workspace(ga, orc, L, w0, alpha):
    """High-valuation rows run block-wise on tcgen05 with partial states merged at the end;
    the partials live in the caller's workspace or in stream-ordered scratch: identical
    bytes either way, and a query sub-range computes the same rows."""
    H, d = 2, 64
    q, k, v = ga.qkv_device(L + 3, L, H, d, torch.bfloat16)
    m = ga.LongNet(w0, alpha)
    nbytes = ga.workspace_size(m, L, d, H, torch.bfloat16)
    assert nbytes > 0
    ws = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    a = ga.attention(q, k, v, m, kernel="tc")
    b = ga.attention(q, k, v, m, kernel="tc", workspace=ws)
    assert torch.equal(a, b)
    r0 = (L // 3 // w0) * w0
    part = ga.attention(q[r0:].contiguous(), k, v, m, L=L, q_begin=r0, kernel="tc")
    assert torch.equal(part, a[r0:])
    cpu = tuple(x.cpu() for x in (q, k, v))
    want, _ = orc.attention(*(synth.as_f64(x) for x in cpu), orc.longnet(L, w0, alpha))
    assert np.abs(a.double().cpu().numpy() - want).max() <= TOL["bf16"]


@pytest.mark.parametrize("fam,L,args,kernel", [
    ("longnet", 10000, (256, 2), "tc"), ("longnet", 5000, (300, 2), "tc"), ("longnet", 20000, (1000, 3), "tc"),
    ("longnet", 10000, (100, 3), "tiled"), ("longnet", 10000, (256, 2), "edge"),
    ("window", 3001, (256, 2), "window"), ("window", 3001, (41, 1), "window"), ("bigbird", 3000, (64, 8, 6, 5), "auto")])
def test_uniform_attention_is_neighbour_mean(ga, orc, fam, L, args, kernel):
    """q = 0 makes every softmax weight exactly 1 (no rounding of P), so each row must be the
    plain mean of V over N(i).  The tight tolerance (bf16 output rounding of |mean| <= 0.2)
    catches a missing, duplicated or extra key that the general 2e-2 bound can hide."""
    H, d = 2, 64
    cpu, f64 = _inputs(L, H, d, "bf16", 77 + L, centred=True)
    q0 = torch.zeros_like(cpu[0])
    m, om = _pair(ga, orc, fam, L, args)
    if fam == "bigbird":
        m = ga.mask_to_csr(m, L)
    want, _ = orc.attention(np.zeros_like(f64[0]), f64[1], f64[2], om)
    got = _run(ga, (q0, cpu[1], cpu[2]), m, kernel=kernel)
    assert np.abs(got - want).max() <= 1e-3


@pytest.mark.parametrize("L,H,dt,win", [
    (2048, 8, "bf16", (256, 2)),      # below the pipelining threshold: one launch
    (65536, 8, "bf16", (256, 2)),     # cfg2 shape: 8 aligned chunks, copies overlapped
    (20011, 2, "bf16", (128, 1)),     # ragged last chunk
    (9000, 1, "f32", (33, 3)),        # fp32 edge kernel, chunked
    (12289, 3, "f16", (1, 1)),        # w = 1: no halo
    (20011, 2, "bf16", "csr"),        # CSR (BigBird without globals): K/V with chunk 0
])
def test_host_entry_point_matches_device(ga, L, H, dt, win):
    d = 64
    cpu = synth.qkv(21, L, H, d, dt)
    q, k, v = (x.cuda() for x in cpu)
    m = ga.mask_to_csr(ga.BigBird(64, 0, 8, seed=3), L) if win == "csr" else ga.Window(*win)
    dev = ga.attention(q, k, v, m)
    pinned = [x.pin_memory() for x in cpu]
    out = torch.empty_like(pinned[0]).pin_memory()
    ga.attention_host(*pinned, m, out)
    torch.cuda.synchronize()
    assert torch.equal(out, dev.cpu())


def test_errors_are_reported(ga):
    L, H, d = 128, 1, 64
    q, k, v = ga.qkv_device(1, L, H, d, torch.bfloat16)
    with pytest.raises(ga.GaError, match="INVALID_ARG"):
        ga.attention(q, k, v, ga.Window(8), out=k)
    with pytest.raises(ga.GaError, match="UNSUPPORTED"):  # implicit BigBird needs its window part
        ga.attention(q, k, v, ga.BigBird(8, 2, 2, parts=ga.BB_GLOBAL))
    q48 = torch.zeros(L, 1, 48, dtype=torch.bfloat16, device="cuda")
    with pytest.raises(ga.GaError, match="UNSUPPORTED"):
        ga.attention(q48, q48.clone(), q48.clone(), ga.Window(8))


# ---------------------------------------------------------------- full-size sampled parity
def _sample_rows(L, extra=(), n=256, seed=0):
    rng = np.random.default_rng(seed)
    rows = set(range(0, min(L, 64))) | set(range(max(0, L - 64), L)) | set(int(x) for x in rng.integers(0, L, n))
    rows |= {int(x) for x in extra if 0 <= x < L}
    return np.array(sorted(rows), dtype=np.int64)


def test_cfg2_full_size_sampled(ga, orc):
    """BASELINE cfg2 (bench workload): L=65536, H=8, d=64, bf16, Window(256, r=2)."""
    L, H, d, seed = 65536, 8, 64, 0x5EED0002
    q, k, v = ga.qkv_device(seed, L, H, d, torch.bfloat16)
    m = ga.Window(256, 2)
    out = ga.attention(q, k, v, m).double().cpu().numpy()
    rows = _sample_rows(L, extra=range(32000, 33000, 7))
    want, edges = orc.attention_seeded(seed, "bf16", orc.window(L, 256, 2), H, d, rows=rows)
    assert np.abs(out[rows] - want).max() <= 2e-2


def test_cfg3_bigbird_full_size_sampled(ga, orc):
    """BASELINE cfg3: L=2^20, BigBird (64 global, Window(128), 64 random) explicit CSR.
    CSR rows bit-exact on samples (incl. all global rows); attention sampled."""
    L, H, d, seed = 2 ** 20, 1, 64, 0x5EED0003
    m = ga.BigBird(128, 64, 64, seed=0xB16B12D)
    om = orc.bigbird(L, 128, 64, 64, 0xB16B12D)
    csr = ga.mask_to_csr(m, L)
    assert csr.nnz == 468_656_702
    rp = csr.row_ptr.cpu().numpy()
    G = [kk * L // 64 for kk in range(64)]
    rows = _sample_rows(L, extra=G[:4] + [g + 1 for g in G] + [g - 1 for g in G], n=128)
    for i in rows:
        nb = orc.neighbors(om, int(i))
        assert np.array_equal(csr.col_idx[rp[i]:rp[i + 1]].cpu().numpy(), nb)
    q, k, v = ga.qkv_device(seed, L, H, d, torch.bfloat16)
    ws = torch.empty(ga.workspace_size(csr, L, d, H, torch.bfloat16), dtype=torch.uint8, device="cuda")
    out = ga.attention(q, k, v, csr, workspace=ws).double().cpu().numpy()
    want, _ = orc.attention_seeded(seed, "bf16", om, H, d, rows=rows)
    assert np.abs(out[rows] - want).max() <= 2e-2


def test_cfg4_longnet_full_size_sampled(ga, orc):
    """BASELINE cfg4: L=2^24, LongNet(w0=2048, alpha=2), implicit, sampled rows incl. high-nu rows."""
    L, H, d, seed = 2 ** 24, 1, 64, 0x5EED0004
    q, k, v = ga.qkv_device(seed, L, H, d, torch.bfloat16)
    out = ga.attention(q, k, v, ga.LongNet(2048, 2))
    rows = _sample_rows(L, extra=[0, 2 ** 13, 2 ** 23, 3 * 2 ** 22, 2 ** 24 - 2 ** 12, 12345 * 64], n=64)
    got = out[torch.from_numpy(rows).cuda()].double().cpu().numpy()
    want, _ = orc.attention_seeded(seed, "bf16", orc.longnet(L, 2048, 2), H, d, rows=rows)
    assert np.abs(got - want).max() <= 2e-2


def test_cfg5_160M_window_sampled(ga, orc):
    """BASELINE cfg5 on one GPU: L=160,000,000, Window(128), bf16, sampled rows incl. the
    8-way shard boundaries."""
    L, H, d, seed = 160_000_000, 1, 64, 0x5EED0005
    free, _ = torch.cuda.mem_get_info()
    need = 4 * L * H * d * 2
    assert free > need * 1.05, f"needs {need / 1e9:.1f} GB"
    q, k, v = ga.qkv_device(seed, L, H, d, torch.bfloat16)
    out = ga.attention(q, k, v, ga.Window(128))
    del k, v
    bounds = [s * (L // 8) + o for s in range(1, 8) for o in (-300, -128, -1, 0, 1, 127, 300)]
    rows = _sample_rows(L, extra=bounds, n=256)
    got = out[torch.from_numpy(rows).cuda()].double().cpu().numpy()
    want, _ = orc.attention_seeded(seed, "bf16", orc.window(L, 128), H, d, rows=rows)
    assert np.abs(got - want).max() <= 2e-2


# ---------------------------------------------------------------- composition API (f1)
@pytest.mark.parametrize("L,w,ng,nr,r,parts", [(3000, 51, 3, 3, 1, 2), (3000, 51, 3, 3, 1, 4), (3000, 101, 3, 0, 2, 2),
                                               (3000, 101, 3, 0, 2, 0), (2000, 51, 5, 7, 3, 1), (64, 30, 2, 50, 2, 4)])
def test_bigbird_parts_csr_bit_exact(ga, orc, L, w, ng, nr, r, parts):
    """ga_mask_to_csr of the BigBird components (and a dilated window) equals the oracle's
    enumeration from the definitions, bit for bit."""
    m = ga.mask_to_csr(ga.BigBird(w, ng, nr, seed=9, r=r, parts=parts), L)
    rp, ci, _ = orc.mask_to_csr(orc.bigbird(L, w, ng, nr, 9, r=r, parts=parts))
    assert np.array_equal(m.row_ptr.cpu().numpy(), rp)
    assert np.array_equal(m.col_idx.cpu().numpy(), ci.astype(np.int32))


@pytest.mark.parametrize("name", ["longformer", "longformer_dilated", "bigbird"])
@pytest.mark.parametrize("dt", ["f32", "bf16"])
def test_presets_compose_equals_union(ga, orc, name, dt):
    """The paper's Fig. 5 patterns run as sequential component calls carrying
    one (m, l, o) state equal one call over the union CSR, and the oracle."""
    L, H, d = 4096, 2, 64
    pre = getattr(ga.presets, name)(L)
    cpu, f64 = _inputs(L, H, d, dt, 521, centred=True)
    q, k, v = (x.cuda() for x in cpu)
    comp = ga.compose(q, k, v, pre.components)
    one = ga.attention(q, k, v, pre.union)
    pm = pre.pattern
    want, _ = orc.attention(*f64, orc.bigbird(L, pm.w, pm.n_global, pm.n_random, pm.seed, r=pm.r))
    tol = TOL[dt]
    assert np.abs(comp.double().cpu().numpy() - want).max() <= tol
    assert np.abs(one.double().cpu().numpy() - want).max() <= tol
    assert (comp.float() - one.float()).abs().max().item() <= (1e-5 if dt == "f32" else 2e-2)


def test_state_api_semantics(ga, orc):
    """WRITE overwrites, ACCUMULATE (+)-combines, an empty edge set leaves the state
    unchanged, zero buffers are an empty state, and state + out are produced together."""
    L, H, d = 1500, 2, 32
    cpu, f64 = _inputs(L, H, d, "f32", 77, centred=True)
    q, k, v = (x.cuda() for x in cpu)
    st = ga.State.empty(L, H, d)
    w = ga.Window(20)
    ref = ga.attention(q, k, v, w)
    ga.attention(q, k, v, w, state=st)  # write
    assert torch.allclose(ga.state_finalize(st, torch.float32), ref, atol=1e-6)
    ga.attention(q, k, v, w, state=st)  # write again: unchanged, not doubled
    assert torch.allclose(ga.state_finalize(st, torch.float32), ref, atol=1e-6)
    # split Window(20) into the band |i-j| < 5 and the rest (global-free BigBird parts)
    st2 = ga.State.empty(L, H, d)
    near = ga.Window(5)
    far = ga.mask_to_csr(ga.BigBird(20, 0, 0, parts=ga.BB_WINDOW), L)  # = Window(20) as CSR
    # far minus near as an explicit CSR built on the host from the two CSRs
    near_csr = ga.mask_to_csr(ga.BigBird(5, 0, 0, parts=ga.BB_WINDOW), L)
    rp_f, ci_f = far.row_ptr.cpu().numpy(), far.col_idx.cpu().numpy()
    rp_n, ci_n = near_csr.row_ptr.cpu().numpy(), near_csr.col_idx.cpu().numpy()
    rows = [np.setdiff1d(ci_f[rp_f[i]:rp_f[i + 1]], ci_n[rp_n[i]:rp_n[i + 1]]) for i in range(L)]
    rp = np.concatenate([[0], np.cumsum([len(x) for x in rows])]).astype(np.int64)
    ring = ga.CSR(torch.from_numpy(rp).cuda(), torch.from_numpy(np.concatenate(rows).astype(np.int32)).cuda())
    out_near = ga.attention(q, k, v, near, state=st2, out=torch.empty_like(q))  # state + out together
    assert torch.allclose(out_near, ga.attention(q, k, v, near), atol=1e-6)
    ga.attention(q, k, v, ring, state=st2, accumulate=True)
    assert torch.allclose(ga.state_finalize(st2, torch.float32), ref, atol=2e-6)
    # an empty component (rows without edges) leaves the state as it was
    empty = ga.CSR(torch.zeros(L + 1, dtype=torch.int64, device="cuda"), torch.zeros(0, dtype=torch.int32, device="cuda"))
    before = ga.state_finalize(st2, torch.float32)
    ga.attention(q, k, v, empty, state=st2, accumulate=True)
    assert torch.equal(ga.state_finalize(st2, torch.float32), before)
    # state needs the edge kernel
    with pytest.raises(ga.GaError, match="UNSUPPORTED"):
        ga.attention(q.bfloat16(), k.bfloat16(), v.bfloat16(), ga.Window(64), state=ga.State.empty(L, H, d), kernel="tiled")

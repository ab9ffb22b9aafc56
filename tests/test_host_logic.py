"""CPU tests of the product's host-side logic (no GPU): the neighbour enumerator built
with g++, the C-ABI exports, and the host closed-form edge counts, against the oracle."""
import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CSRC = os.path.join(ROOT, "paper_2502_01659_b200", "csrc")


@pytest.fixture(scope="module")
def enum_bin(tmp_path_factory):
    out = str(tmp_path_factory.mktemp("enum") / "enum_host")
    subprocess.check_call(["g++", "-O1", "-std=c++17", "-I", CSRC, "-o", out,
                           os.path.join(ROOT, "tests", "host", "enum_host.cpp")])
    return out


def _run_enum(binary, kind, L, a, b, parts=0, head=0):
    txt = subprocess.check_output([binary, str(kind), str(L), str(a), str(b), str(parts), str(head)], text=True)
    rows = []
    for line in txt.splitlines():
        f = [int(x) for x in line.split()]
        rows.append((f[1], np.array(f[2:], dtype=np.int64)))
    return rows


@pytest.mark.parametrize("kind,L,a,b", [
    (1, 300, 17, 1), (1, 300, 40, 3), (1, 50, 200, 2), (1, 1, 1, 1),
    (4, 257, 16, 3), (4, 100, 100, 1),
    (2, 256, 16, 2), (2, 243, 9, 3), (2, 200, 16, 2), (2, 1000, 8, 4), (2, 50, 64, 2), (2, 4096, 64, 2),
    # alpha does not divide w0: level-t segment starts are not multiples of alpha^(t+1)
    (2, 5000, 100, 3), (2, 999, 7, 2), (2, 3000, 10, 4), (2, 4000, 5, 3),
])
def test_enumerator_matches_oracle(orc, enum_bin, kind, L, a, b):
    if kind == 1:
        m = orc.window(L, a, b)
    elif kind == 4:
        m = orc.block_dilated(L, a, b)
    else:
        m = orc.longnet(L, a, b)
    rp, ci, nnz = orc.mask_to_csr(m)
    rows = _run_enum(enum_bin, kind, L, a, b)
    assert len(rows) == L
    for i, (disjoint, nb) in enumerate(rows):
        assert disjoint == 1, f"row {i}: pieces overlap or degree() disagrees"
        assert np.array_equal(nb, ci[rp[i]:rp[i + 1]]), f"row {i}"


@pytest.mark.parametrize("L,w0,alpha", [(256, 16, 2), (243, 9, 3), (5000, 100, 3), (999, 7, 2)])
def test_enumerator_multiset_matches_oracle(orc, enum_bin, L, w0, alpha):
    """LongNet multiset mixture (f4): the product's pieces (all multiples at every level)
    list exactly the oracle's neighbour multiset, repeats included."""
    rp, ci, nnz = orc.mask_to_csr(orc.longnet(L, w0, alpha, multiset=True))
    rows = _run_enum(enum_bin, 2, L, w0, alpha, parts=1)
    assert len(rows) == L
    for i, (_, nb) in enumerate(rows):
        assert np.array_equal(nb, ci[rp[i]:rp[i + 1]]), f"row {i}"


def test_abi_exports_every_declared_symbol():
    """libga.so loads (no GPU needed) and exports every function include/ga.h declares."""
    import paper_2502_01659_b200._abi as abi

    hdr = open(os.path.join(ROOT, "include", "ga.h")).read()
    declared = set(re.findall(r"\b(ga_[a-z_]+)\s*\(", hdr))
    assert declared, "no declarations parsed"
    lib = abi.lib()
    for name in declared:
        assert hasattr(lib, name), name
    assert declared == {n for n, _, _ in abi.SIGNATURES}
    assert b"sm_100a" in lib.ga_version()


def test_abi_struct_layout_matches_header():
    """ctypes mirrors of ga_mask / ga_opts have the C layout (checked with g++ offsetof)."""
    import paper_2502_01659_b200._abi as abi

    structs = ((abi.GaMask, "ga_mask"), (abi.GaOpts, "ga_opts"), (abi.GaState, "ga_state"))
    probes = " ".join(f"P({c}, {f})" for cls, c in structs for f, _ in cls._fields_ if not f.startswith("reserved"))
    sizes = " ".join(f'printf("sizeof.{c} %zu\\n", sizeof({c}));' for _, c in structs)
    src = ('#include <cstdio>\n#include <cstddef>\n#include "ga.h"\n'
           '#define P(T, f) printf(#T "." #f " %zu\\n", offsetof(T, f));\n'
           f"int main() {{ {probes} {sizes} }}\n")
    import tempfile
    with tempfile.TemporaryDirectory() as td:
        p = os.path.join(td, "l.cpp")
        open(p, "w").write(src)
        subprocess.check_call(["g++", "-I", os.path.join(ROOT, "include"), "-o", p + ".bin", p])
        out = subprocess.check_output([p + ".bin"], text=True)
    got = dict(line.split() for line in out.splitlines())
    for cls, cname in structs:
        for f, _ in cls._fields_:
            if f.startswith("reserved"):
                continue
            assert int(got[f"{cname}.{f}"]) == getattr(cls, f).offset, (cname, f)
        assert int(got[f"sizeof.{cname}"]) == ctypes.sizeof(cls)


@pytest.mark.parametrize("spec", [
    ("window", 1024, (32, 1)), ("window", 65536, (256, 2)), ("window", 777, (100, 7)), ("window", 10, (50, 1)),
    ("block", 1000, (64, 3)), ("block", 999, (10, 1)),
    ("longnet", 4096, (64, 2)), ("longnet", 5000, (64, 2)), ("longnet", 2187, (27, 3)), ("longnet", 300, (512, 2)),
    ("longnet", 12345, (16, 4)), ("longnet", 5000, (100, 3)), ("longnet", 999, (7, 2)), ("longnet", 3000, (10, 4)),
    ("bigbird", 1024, (8, 4, 4)), ("bigbird", 3000, (64, 7, 20)), ("bigbird", 64, (30, 2, 50)),
    # dilated window and single components (the composition API's parts)
    ("bigbird", 3000, (101, 3, 0, 2, 0)), ("bigbird", 3000, (101, 3, 0, 2, 2)), ("bigbird", 3000, (51, 3, 3, 1, 4)),
    ("bigbird", 2000, (51, 5, 7, 3, 1)), ("bigbird", 2000, (51, 5, 7, 3, 6)), ("bigbird", 64, (30, 2, 50, 2, 4)),
])
def test_host_mask_count_equals_oracle(orc, spec):
    import paper_2502_01659_b200 as ga

    fam, L, a = spec
    if fam == "window":
        m, om = ga.Window(*a), orc.window(L, *a)
    elif fam == "block":
        m, om = ga.BlockDilated(*a), orc.block_dilated(L, *a)
    elif fam == "longnet":
        m, om = ga.LongNet(*a), orc.longnet(L, *a)
    else:
        r, parts = (a[3], a[4]) if len(a) > 3 else (1, 0)
        m = ga.BigBird(a[0], a[1], a[2], seed=5, r=r, parts=parts)
        om = orc.bigbird(L, a[0], a[1], a[2], 5, r=r, parts=parts)
    assert ga.mask_count(m, L) == orc.mask_to_csr(om, False)[2]


def test_closed_form_counts_at_bench_sizes():
    """Host counts at the BASELINE.json configurations equal SURVEY §8(c)'s exact values."""
    import paper_2502_01659_b200 as ga

    assert ga.mask_count(ga.Window(32), 1024) == 63_520
    assert ga.mask_count(ga.Window(256, 2), 65536) * 8 == 133_433_344
    assert ga.mask_count(ga.Window(128), 160_000_000) == 40_799_983_744
    assert ga.mask_count(ga.LongNet(2048, 2), 2 ** 24) == 51_537_510_400
    # multiset mixture (f4): w0 L (2 - 2^-13) = 68,715,282,432
    assert ga.mask_count(ga.LongNet(2048, 2, multiset=True), 2 ** 24) == 68_715_282_432
    assert ga.mask_count(ga.BigBird(128, 64, 64), 2 ** 20) == 468_656_702


def test_invalid_arguments_rejected_without_gpu():
    import paper_2502_01659_b200 as ga

    with pytest.raises(ga.GaError, match="INVALID_ARG"):
        ga.mask_count(ga.Window(0), 10)
    with pytest.raises(ga.GaError, match="INVALID_ARG"):
        ga.mask_count(ga.LongNet(16, 1), 10)


def test_bench_roofline_picks_binding_bound():
    """bench.py reports the resource with the largest lower-bound time: HBM for
    the window configs and explicit CSR, MUFU exp2 for LongNet and implicit BigBird (cfg4: 5.15e10 exp2 ~ 11 ms
    against 7.8 ms of tensor flops and 1.3 ms of compulsory HBM traffic)."""
    import bench

    cases = {"cfg2": (133433344, 65536 * 8, "hbm"), "cfg4": (51537510400, 2 ** 24, "alu"),
             "cfg5": (40799983744, 160_000_000, "hbm"), "cfg3": (468656702, 2 ** 20, "hbm"),
             "cfg3i": (468656702, 2 ** 20, "alu")}  # implicit: no CSR bytes, 4.7e8 exp2 > 0.54 GB of QKVO
    for name, (edges, rows, bound) in cases.items():
        cfg = bench.CONFIGS[name]
        roof, _ = bench.roofline_for(name, "auto", cfg, cfg["mask"][0], edges, cfg["L"], cfg["H"], cfg["d"],
                                     edges // cfg["H"], [50.0])
        assert roof["bound"] == bound, (name, roof)
        assert 0 < roof["frac"] < 1


@pytest.mark.parametrize("L,w0,alpha,parts", [(256, 16, 2, 2), (243, 9, 3, 2), (999, 7, 2, 2), (5000, 100, 3, 2),
                                              (256, 16, 2, 3), (3000, 10, 4, 2)])
@pytest.mark.parametrize("head", [0, 1, 2, 3, 5, 13])
def test_enumerator_head_offsets_matches_oracle(orc, enum_bin, L, w0, alpha, parts, head):
    """LongNet per-head offsets (f4, reading R11c): the product's shifted-valuation pieces list
    exactly the oracle's per-head neighbour set (definition: offsets == h mod alpha^k), and
    the set-union pieces are disjoint."""
    om = orc.longnet(L, w0, alpha, multiset=bool(parts & 1), head_offsets=True, head=head)
    rp, ci, nnz = orc.mask_to_csr(om)
    rows = _run_enum(enum_bin, 2, L, w0, alpha, parts=parts, head=head)
    assert len(rows) == L
    for i, (disjoint, nb) in enumerate(rows):
        if not parts & 1:
            assert disjoint == 1, f"row {i}: pieces overlap"
        assert np.array_equal(nb, ci[rp[i]:rp[i + 1]]), f"row {i} head {head}"

"""Multi-process (world_size 2 and 3, gloo, CPU) tests of the sharding host logic:
shard ranges, halo exchange and the K/V all-gather produce exactly the rows the sharded
kernels need (the kernels themselves are covered by the GPU tests)."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2502_01659_b200 import dist as gdist
from paper_2502_01659_b200.masks import Window


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, fn, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        fn(rank, world)
        q.put((rank, None))
    except Exception as e:  # pragma: no cover - reported to the parent
        import traceback
        q.put((rank, traceback.format_exc()))
    finally:
        dist.destroy_process_group()


def _spawn(fn, world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, world, port, fn, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = [q.get(timeout=120) for _ in ps]
    for p in ps:
        p.join(timeout=60)
    errs = [e for _, e in res if e]
    assert not errs, errs[0]


def _global(L, H, d):
    g = torch.Generator().manual_seed(0)
    return torch.rand((L, H, d), generator=g), torch.rand((L, H, d), generator=g)


def _halo_case(rank, world):
    L, H, d = 1000, 2, 8
    mask = Window(40, 3)
    halo = gdist.window_halo(mask)
    assert halo == 39
    K, V = _global(L, H, d)
    r0, r1 = gdist.shard_range(L, world, rank)
    buf = gdist.alloc_halo(L, r0, r1, halo, H, d, torch.float32, "cpu")
    buf.k.fill_(-1)
    buf.v.fill_(-1)
    buf.local_k.copy_(K[r0:r1])
    buf.local_v.copy_(V[r0:r1])
    gdist.exchange_halo(buf)
    assert torch.equal(buf.k, K[buf.kv_begin:buf.kv_end])
    assert torch.equal(buf.v, V[buf.kv_begin:buf.kv_end])
    # every neighbour of every local row lies inside the halo'd buffer
    for i in (r0, r1 - 1):
        lo, hi = i - ((mask.w - 1) // mask.r) * mask.r, i + ((mask.w - 1) // mask.r) * mask.r
        assert buf.kv_begin <= max(0, lo) and min(L - 1, hi) < buf.kv_end


def _allgather_case(rank, world):
    L, H, d = 999, 1, 4
    K, _ = _global(L, H, d)
    per = -(-L // world)
    local = torch.zeros((per, H, d))
    r0, r1 = rank * per, min(L, (rank + 1) * per)
    local[:r1 - r0] = K[r0:r1]
    full = gdist.allgather_rows(local, L)
    assert torch.equal(full, K)


@pytest.mark.parametrize("world", [2, 3])
def test_halo_exchange_gloo(world):
    _spawn(_halo_case, world)


def test_allgather_gloo():
    _spawn(_allgather_case, 2)


def test_shard_ranges_cover_exactly():
    for L, world, align in [(65536, 8, 128), (1000, 3, 1), (160_000_000, 8, 128), (10, 4, 1), (7, 8, 1)]:
        got = [gdist.shard_range(L, world, r, align) for r in range(world)]
        assert got[0][0] == 0 and got[-1][1] == L
        for (a0, a1), (b0, b1) in zip(got, got[1:]):
            assert a1 == b0 and a0 <= a1
        if L >= world * align:
            assert all((r1 - r0) % align == 0 for r0, r1 in got[:-1])


def _longnet_case(rank, world):
    """Each rank keeps only its shard + the gathered strided rows; every neighbour of every
    local row (oracle enumeration) must then hold the true value."""
    import oracle

    L, H, d, w0, alpha = 4096, 1, 4, 64, 2
    K, V = _global(L, H, d)
    per = L // world
    r0, r1 = rank * per, (rank + 1) * per
    stride = gdist.longnet_exchange_stride(L, w0, alpha, per)
    assert stride == 2 ** {2: 6, 3: 6}.get(world, 6) or stride > 0
    kf = torch.full_like(K, float("nan"))
    vf = torch.full_like(V, float("nan"))
    kf[r0:r1] = K[r0:r1]
    vf[r0:r1] = V[r0:r1]
    gdist.exchange_longnet(kf, vf, r0, r1, stride)
    om = oracle.longnet(L, w0, alpha)
    for i in range(r0, r1, 7):
        nb = oracle.neighbors(om, i)
        assert torch.equal(kf[nb], K[nb]), i
        assert torch.equal(vf[nb], V[nb]), i


def test_longnet_strided_allgather_gloo():
    _spawn(_longnet_case, 2)


def test_longnet_exchange_stride_cfg4():
    """cfg4 (L=2^24, w0=2048, alpha=2): k0 = 13/12/11 for 2/4/8 shards;
    the gathered volume L/alpha^k0 rows x 256 B (K and V, bf16, d=64) is 0.52/1.05/2.10 MB."""
    L = 2 ** 24
    for world, k0 in ((2, 13), (4, 12), (8, 11)):
        st = gdist.longnet_exchange_stride(L, 2048, 2, L // world)
        assert st == 2 ** k0
        assert round(L // st * 256 / 1e6, 2) == {2: 0.52, 4: 1.05, 8: 2.10}[world]


# ---------------------------------------------------------------- C-ABI comm bootstrap
def _comm_bootstrap_case(rank, world):
    import ctypes

    from paper_2502_01659_b200 import _abi
    from paper_2502_01659_b200.comm import Comm

    c = Comm(device=-1)  # host-only: TCP bootstrap through the libga C ABI
    assert (c.rank, c.world) == (rank, world)
    got = c.host_allgather(bytes([rank] * 5) + b"xyz")
    assert got == [bytes([q] * 5) + b"xyz" for q in range(world)]
    for _ in range(3):  # repeated exchanges stay in step
        got = c.host_allgather(rank.to_bytes(8, "little"))
        assert [int.from_bytes(g, "little") for g in got] == list(range(world))
    # a host-only comm refuses device work
    with pytest.raises(_abi.GaError, match="INVALID_ARG"):
        c.empty((4,), torch.float32)
    c.close()


@pytest.mark.parametrize("world", [2, 3])
def test_comm_bootstrap_host_allgather(world):
    _spawn(_comm_bootstrap_case, world)


def test_comm_create_errors():
    import ctypes

    from paper_2502_01659_b200 import _abi

    lib = _abi.lib()
    h = ctypes.c_void_p()
    bad = ctypes.create_string_buffer(128)  # no magic
    assert lib.ga_comm_create(2, 0, bad, -1, ctypes.byref(h)) == _abi.GA_ERR_INVALID_ARG
    idb = ctypes.create_string_buffer(128)
    assert lib.ga_comm_get_unique_id(idb) == _abi.GA_OK
    assert lib.ga_comm_create(2, 2, idb, -1, ctypes.byref(h)) == _abi.GA_ERR_INVALID_ARG  # rank >= world
    # world 1 needs no peers
    assert lib.ga_comm_create(1, 0, idb, -1, ctypes.byref(h)) == _abi.GA_OK
    out = ctypes.create_string_buffer(4)
    assert lib.ga_comm_host_allgather(h, b"abcd", 4, out) == _abi.GA_OK and out.raw == b"abcd"
    assert lib.ga_comm_destroy(h) == _abi.GA_OK
    # sharded attention validates its comm before touching the device
    m = _abi.GaMask()
    m.kind, m.L, m.w, m.r = _abi.GA_MASK_WINDOW, 100, 8, 1
    assert lib.ga_attention_sharded(None, None, None, ctypes.byref(m), None, 100, 0, 100, 64, 1, 1, None, None,
                                    None) == _abi.GA_ERR_INVALID_ARG


def test_comm_shard_rows():
    from paper_2502_01659_b200.comm import shard_rows

    for L in (1, 7, 100, 2 ** 20 + 3):
        for world in (1, 2, 3, 8):
            spans = [shard_rows(L, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == L
            for (a, b), (c, _) in zip(spans, spans[1:]):
                assert b == c and a <= b

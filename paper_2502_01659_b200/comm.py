"""Multi-GPU binding: argument marshalling onto the ga_comm_* / ga_attention_sharded C ABI.

One process per GPU.  Rank 0 creates the 128-byte bootstrap id (ga_comm_get_unique_id),
torch.distributed broadcasts it, every rank joins with ga_comm_create.  K/V shards live in
symmetric buffers (Comm.empty) that all ranks map with CUDA IPC, so the attention kernels
read halo / long-range rows from the owning rank over NVLink while computing
(include/ga.h).
"""
from __future__ import annotations

import ctypes
from typing import Optional

import torch
import torch.distributed as dist

from . import _abi
from .attention import _opts, _stream, dtype_code
from .masks import Mask

_CAI_TYPESTR = {torch.float32: "<f4", torch.bfloat16: "<i2", torch.float16: "<f2", torch.uint8: "|u1",
                torch.int64: "<i8", torch.int32: "<i4"}


class _DevBuf:
    """__cuda_array_interface__ view of comm-owned device memory (zero copy)."""

    def __init__(self, ptr: int, shape, typestr: str):
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": typestr, "data": (ptr, False),
                                         "version": 3, "strides": None}


def shard_rows(L: int, world: int, rank: int):
    """[row_begin, row_end) of `rank` (equal contiguous shards of ceil(L / world) rows)."""
    S = -(-L // world)
    b = min(L, rank * S)
    return b, min(L, b + S)


class Comm:
    """A ga_comm over the ranks of a torch.distributed group (any backend: it is only used
    to broadcast the bootstrap id).  device=-1 makes a host-only comm (bootstrap tests)."""

    def __init__(self, group=None, device: Optional[int] = None):
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        lib = _abi.lib()
        idbuf = ctypes.create_string_buffer(_abi.GA_COMM_ID_BYTES)
        if self.rank == 0:
            _abi.check(lib.ga_comm_get_unique_id(idbuf))
        obj = [idbuf.raw]
        src = dist.get_global_rank(group, 0) if group is not None else 0
        dist.broadcast_object_list(obj, src=src, group=group)
        idbuf = ctypes.create_string_buffer(obj[0], _abi.GA_COMM_ID_BYTES)
        self.device = torch.cuda.current_device() if device is None else device
        h = ctypes.c_void_p()
        _abi.check(lib.ga_comm_create(self.world, self.rank, idbuf, self.device, ctypes.byref(h)))
        self._h = h
        self._bufs = {}

    # ---------------------------------------------------------------- buffers
    def empty(self, shape, dtype: torch.dtype) -> torch.Tensor:
        """Collective: a symmetric DEVICE tensor (same shape on every rank)."""
        n = 1
        for s in shape:
            n *= int(s)
        nbytes = n * torch.empty((), dtype=dtype).element_size()
        p = ctypes.c_void_p()
        _abi.check(_abi.lib().ga_comm_alloc(self._h, nbytes, ctypes.byref(p)))
        base = torch.as_tensor(_DevBuf(p.value, shape, _CAI_TYPESTR[dtype]), device=f"cuda:{self.device}")
        t = base.view(dtype) if dtype == torch.bfloat16 else base
        self._bufs[p.value] = t
        return t

    def free(self, t: torch.Tensor) -> None:
        """Collective: release a tensor from empty()."""
        ptr = t.data_ptr()
        self._bufs.pop(ptr, None)
        _abi.check(_abi.lib().ga_comm_free(self._h, ctypes.c_void_p(ptr)))

    # ---------------------------------------------------------------- sync
    def barrier(self) -> None:
        """Device-side barrier on the current stream."""
        _abi.check(_abi.lib().ga_comm_barrier(self._h, _stream(self.device)))

    def host_allgather(self, data: bytes) -> list:
        n = len(data)
        out = ctypes.create_string_buffer(n * self.world)
        _abi.check(_abi.lib().ga_comm_host_allgather(self._h, data, n, out))
        return [out.raw[i * n:(i + 1) * n] for i in range(self.world)]

    def timed_out(self) -> bool:
        """True if a device barrier gave up waiting for a peer (reflects barriers that have
        executed: synchronise first for a definite answer)."""
        t = ctypes.c_int()
        _abi.check(_abi.lib().ga_comm_status(self._h, ctypes.byref(t)))
        return bool(t.value)

    # ---------------------------------------------------------------- attention
    def attention(self, q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, mask: Mask, L: int,
                  out: Optional[torch.Tensor] = None, *, kernel: str = "auto",
                  workspace: Optional[torch.Tensor] = None, heavy_threshold: int = 0,
                  exchange: str = "allgather") -> torch.Tensor:
        """This rank's rows of attention over the whole sequence (ga_attention_sharded).
        q: local query rows [rows, H, d]; k, v: this rank's shard, views of empty() tensors.
        exchange (explicit CSR only): "allgather" (full-length K/V per rank) or "ring" (K/V
        shards streamed through two staging buffers, partial states merged)."""
        rows, H, d = q.shape
        b, e = shard_rows(L, self.world, self.rank)
        if rows != e - b:
            raise ValueError(f"rank {self.rank} owns {e - b} rows of L={L}, q has {rows}")
        if out is None:
            out = torch.empty_like(q)
        cm = mask.to_c(L)
        o = _opts(0, 0, 0, 0, workspace, None, None, kernel, heavy_threshold)
        o.exchange = {"allgather": _abi.GA_EXCHANGE_ALLGATHER, "ring": _abi.GA_EXCHANGE_RING}[exchange]
        _abi.check(_abi.lib().ga_attention_sharded(q.data_ptr(), k.data_ptr(), v.data_ptr(), ctypes.byref(cm),
                                                   out.data_ptr(), L, b, e, d, H, dtype_code(q.dtype),
                                                   ctypes.byref(o), self._h, _stream(q.device)))
        return out

    def check(self) -> None:
        """Synchronise this rank's device and raise if any barrier timed out (the sharded
        output was then poisoned with NaN)."""
        torch.cuda.synchronize(self.device)
        if self.timed_out():
            raise _abi.GaError(_abi.GA_ERR_COMM, "a device barrier timed out: a peer stalled; outputs are NaN")

    def close(self) -> None:
        if self._h is not None:
            self._bufs.clear()
            _abi.check(_abi.lib().ga_comm_destroy(self._h))
            self._h = None

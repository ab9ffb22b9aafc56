"""Query-range sequence sharding across GPUs; one process per GPU.

The paper is single-GPU and names distributed versions as future work.
Rows are independent units of Algorithm 1's parallel outer loop, so the
path shards by contiguous query ranges; the one real exchange step is bringing each
shard the K/V rows its neighbour sets reach:

* Window / dilated masks: a halo of m*r rows (m = floor((w-1)/r)) from each adjacent
  rank, exchanged with point-to-point send/recv (torch.distributed: NCCL over NVLink on
  the GPU box, gloo in the CPU tests), overlapped with the interior rows' compute.
* LongNet / explicit CSR masks: K/V all-gather (all_gather_into_tensor).

torch.distributed is plumbing only; all attention arithmetic runs in libga.so.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Optional, Tuple

import torch
import torch.distributed as dist

from .masks import Mask, Window


def shard_range(L: int, world: int, rank: int, align: int = 1) -> Tuple[int, int]:
    """Contiguous query range [r0, r1) of `rank`: equal shards rounded to `align` rows,
    the last rank takes the remainder."""
    per = L // world
    per = (per // align) * align if per >= align else max(per, 1)
    r0 = min(L, rank * per)
    r1 = L if rank == world - 1 else min(L, r0 + per)
    return r0, r1


def window_halo(mask: Window) -> int:
    """Rows a Window(w, r) query can reach on each side: m*r, m = floor((w-1)/r)."""
    return ((mask.w - 1) // mask.r) * mask.r


@dataclass
class HaloBuffers:
    """K/V of this shard plus `halo` rows on each side (global rows kv_begin..kv_end)."""
    k: torch.Tensor
    v: torch.Tensor
    r0: int
    r1: int
    kv_begin: int
    kv_end: int
    halo: int

    @property
    def local_k(self):
        return self.k[self.r0 - self.kv_begin:self.r1 - self.kv_begin]

    @property
    def local_v(self):
        return self.v[self.r0 - self.kv_begin:self.r1 - self.kv_begin]


def alloc_halo(L: int, r0: int, r1: int, halo: int, H: int, d: int, dtype, device) -> HaloBuffers:
    kb, ke = max(0, r0 - halo), min(L, r1 + halo)
    k = torch.empty((ke - kb, H, d), dtype=dtype, device=device)
    v = torch.empty_like(k)
    return HaloBuffers(k, v, r0, r1, kb, ke, halo)


def exchange_halo(buf: HaloBuffers, group=None) -> None:
    """Fill the halo rows of `buf` from the neighbouring ranks (send/recv in one batch).

    Rank p sends its first `h` local rows to p-1 and its last `h` rows to p+1, and
    receives p-1's last rows into its left halo and p+1's first rows into its right halo.
    Requires every shard to hold at least `halo` rows.
    """
    world, rank = dist.get_world_size(group), dist.get_rank(group)
    staged = dist.get_backend(group) == "gloo" and buf.k.is_cuda  # gloo p2p moves host memory only
    if staged:
        host = HaloBuffers(buf.k.cpu(), buf.v.cpu(), buf.r0, buf.r1, buf.kv_begin, buf.kv_end, buf.halo)
        exchange_halo(host, group)
        buf.k.copy_(host.k)
        buf.v.copy_(host.v)
        return
    ops = []
    left = buf.r0 - buf.kv_begin          # rows of left halo present in the buffer
    right = buf.kv_end - buf.r1
    n_local = buf.r1 - buf.r0
    for t in (buf.k, buf.v):
        if rank > 0 and left > 0:
            ops.append(dist.P2POp(dist.irecv, t[:left], rank - 1, group))
            ops.append(dist.P2POp(dist.isend, t[left:left + left], rank - 1, group))
        if rank < world - 1 and right > 0:
            ops.append(dist.P2POp(dist.isend, t[left + n_local - right:left + n_local], rank + 1, group))
            ops.append(dist.P2POp(dist.irecv, t[left + n_local:], rank + 1, group))
    if ops:
        for r in dist.batch_isend_irecv(ops):
            r.wait()


def longnet_exchange_stride(L: int, w0: int, alpha: int, shard: int) -> int:
    """alpha^k0 for LongNet query shards of `shard` rows.

    Levels whose segment w0*alpha^t fits a shard (and the shards are aligned to it) only
    reach keys inside the shard.  The first level k0 with w0*alpha^k0 > shard reaches
    across shards, and every key a level t >= k0 piece contains is a multiple of alpha^t,
    hence of alpha^k0.  So the exchange is an all-gather of the rows j with alpha^k0 | j.
    Returns 0 when no level crosses a shard (no exchange)."""
    K = 0
    if w0 <= L:
        while w0 * alpha ** (K + 1) <= L:
            K += 1
    for t in range(K + 1):
        if w0 * alpha ** t > shard:
            return alpha ** t
    return 0


def exchange_longnet(k_full: torch.Tensor, v_full: torch.Tensor, r0: int, r1: int, stride: int,
                     group=None) -> None:
    """Fill, in the full-length K/V buffers, the rows j = multiple of `stride` owned by the
    other ranks (this rank's rows [r0, r1) are already in place).  Equal, stride-aligned
    shards: every rank contributes (r1 - r0) / stride rows to one all_gather_into_tensor."""
    if stride == 0:
        return
    world = dist.get_world_size(group)
    n = (r1 - r0) // stride
    mine = torch.stack([k_full[r0:r1:stride], v_full[r0:r1:stride]])  # [2, n, H, d]
    flat = torch.empty((world * 2,) + tuple(mine.shape[1:]), dtype=mine.dtype, device=mine.device)
    dist.all_gather_into_tensor(flat, mine.contiguous(), group=group)
    gathered = flat.view((world, 2) + tuple(mine.shape[1:]))
    L = k_full.shape[0]
    per = r1 - r0
    for p in range(world):
        a = p * per
        k_full[a:a + per:stride] = gathered[p, 0, :n]
        v_full[a:a + per:stride] = gathered[p, 1, :n]
    assert world * per == L, "LongNet exchange assumes equal shards covering the sequence"


def allgather_rows(local: torch.Tensor, L: int, group=None) -> torch.Tensor:
    """All-gather equal-size row shards into a full [L, ...] tensor (LongNet / CSR masks)."""
    world = dist.get_world_size(group)
    full = torch.empty((local.shape[0] * world,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
    dist.all_gather_into_tensor(full, local.contiguous(), group=group)
    return full[:L]


def sharded_window_attention(q_local: torch.Tensor, buf: HaloBuffers, mask: Window, L: int,
                             out: Optional[torch.Tensor] = None, comm_stream: Optional[torch.cuda.Stream] = None,
                             group=None) -> torch.Tensor:
    """One sharded step: interior rows start while the halo is exchanged on a side stream;
    the boundary rows run once it has landed.  Returns this rank's output rows."""
    from .attention import attention, query_alignment

    if out is None:
        out = torch.empty_like(q_local)
    n = buf.r1 - buf.r0
    h = buf.halo
    # interior/boundary split points on the kernel's tile grid, so every row is computed as
    # in a single launch over the whole sequence
    al = query_alignment(mask, L, q_local.shape[2], q_local.dtype)
    up = lambda x: -(-x // al) * al
    h_lo = min(n, up(buf.r0 + h) - buf.r0)
    h_hi = min(n, buf.r1 - (buf.r1 - h) // al * al)
    main = torch.cuda.current_stream()
    comm = comm_stream or torch.cuda.Stream()
    comm.wait_stream(main)
    with torch.cuda.stream(comm):
        exchange_halo(buf, group)
    a, b = h_lo, max(h_lo, n - h_hi)  # interior rows [a, b) need no halo
    if b > a:
        attention(q_local[a:b], buf.k, buf.v, mask, out[a:b], L=L, q_begin=buf.r0 + a, kv_begin=buf.kv_begin)
    main.wait_stream(comm)
    if a > 0:
        attention(q_local[:a], buf.k, buf.v, mask, out[:a], L=L, q_begin=buf.r0, kv_begin=buf.kv_begin)
    if n > b:
        attention(q_local[b:], buf.k, buf.v, mask, out[b:], L=L, q_begin=buf.r0 + b, kv_begin=buf.kv_begin)
    return out

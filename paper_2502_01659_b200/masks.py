"""Mask descriptors: the paper's attention-specific parameters P_a or an explicit graph G
(Algorithm 1 inputs).  Each descriptor marshals into a ga_mask.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass, field
from typing import Optional

from . import _abi


class Mask:
    kind: int

    def to_c(self, L: int) -> _abi.GaMask:  # pragma: no cover - abstract
        raise NotImplementedError

    def _base(self, L):
        m = _abi.GaMask()
        m.kind = self.kind
        m.L = int(L)
        return m


@dataclass(frozen=True)
class Window(Mask):
    """|i-j| < w and |i-j| mod r == 0 (local: r=1; 1D dilated)."""
    w: int
    r: int = 1
    kind = _abi.GA_MASK_WINDOW

    def to_c(self, L):
        m = self._base(L)
        m.w, m.r = self.w, self.r
        return m


@dataclass(frozen=True)
class BlockDilated(Mask):
    """2D dilation (reading R3): same segment of length `seg`, both
    in-segment offsets divisible by r."""
    seg: int
    r: int = 1
    kind = _abi.GA_MASK_BLOCK_DILATED

    def to_c(self, L):
        m = self._base(L)
        m.seg, m.r = self.seg, self.r
        return m


@dataclass(frozen=True)
class LongNet(Mask):
    """Union over k = 0..K of BlockDilated(w0 alpha^k, alpha^k), K = max{k: w0 alpha^k <= L}
    ("alpha = 2 and w0 = 2048"; reading R11); multiset=True keeps repeats
    (reading R11b)."""
    w0: int
    alpha: int = 2
    multiset: bool = False  # LongNet's mixture: a pair in n levels' blocks weighs n times (f4)
    head_offsets: bool = False  # LongNet's per-head offsets s_h = h mod alpha^k (f4, reading R11c)
    kind = _abi.GA_MASK_LONGNET

    def to_c(self, L):
        m = self._base(L)
        m.w0, m.alpha = self.w0, self.alpha
        m.parts = (_abi.GA_LONGNET_MULTISET if self.multiset else 0) | (
            _abi.GA_LONGNET_HEAD_OFFSETS if self.head_offsets else 0)
        return m


BB_WINDOW, BB_GLOBAL, BB_RANDOM = _abi.GA_BB_WINDOW, _abi.GA_BB_GLOBAL, _abi.GA_BB_RANDOM


@dataclass(frozen=True)
class BigBird(Mask):
    """Window(w, r) UNION global rows/cols UNION n_random random columns per non-global row
    (readings R8-R10).  `global_idx`: sorted int64 CUDA tensor or
    None for the evenly spaced set {floor(k L / n_global)}.  `parts` keeps only some of the
    three disjoint components (BB_WINDOW | BB_GLOBAL | BB_RANDOM; 0 = all) — e.g. the
    paper's "global minus local" kernel is parts=BB_GLOBAL."""
    w: int
    n_global: int
    n_random: int
    seed: int = 0xB16B12D
    global_idx: Optional[object] = None
    r: int = 1
    parts: int = 0
    kind = _abi.GA_MASK_BIGBIRD

    def to_c(self, L):
        m = self._base(L)
        m.w, m.r, m.parts = self.w, self.r, self.parts
        m.n_global, m.n_random, m.seed = self.n_global, self.n_random, self.seed & (2**64 - 1)
        if self.global_idx is not None:
            m.global_idx = self.global_idx.data_ptr()
            m.n_global = self.global_idx.numel()
        return m


@dataclass
class CSR(Mask):
    """Explicit binary CSR graph (reading R7): row_ptr int64 [L+1] and
    col_idx int32 [nnz], CUDA tensors, columns strictly increasing per row."""
    row_ptr: object
    col_idx: object
    kind = _abi.GA_MASK_CSR

    @property
    def nnz(self) -> int:
        return int(self.col_idx.numel())

    def to_c(self, L):
        m = self._base(L)
        m.row_ptr = self.row_ptr.data_ptr()
        m.col_idx = self.col_idx.data_ptr() if self.col_idx.numel() else None
        m.nnz = self.nnz
        return m

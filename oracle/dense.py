"""NumPy dense brute force for tiny L (TEST INFRASTRUCTURE ONLY; see oracle/__init__.py).

Materialises the L x L 0-1 mask from vectorised predicates over the full index grid
(PAPER.md:126-136 1D dilation, :138-154 2D dilation, :156 global, LongNet union of
2D-dilated levels per PAPER.md:138/181 and reading R11), then computes
softmax(QK^T / sqrt(d)) with masked entries at -inf, times V (Eq. 1),
the way the paper's SDPA verification does, mapping all -inf (NaN)
rows to 0 (reading R6).  Shares no code with oracle.c.
"""
from __future__ import annotations

import numpy as np


def _grid(L):
    i = np.arange(L, dtype=np.int64)[:, None]
    j = np.arange(L, dtype=np.int64)[None, :]
    return i, j


def window_mask(L, w, r=1):
    i, j = _grid(L)
    a = np.abs(i - j)
    return (a < w) & (a % r == 0)


def block_dilated_mask(L, seg, r=1):
    i, j = _grid(L)
    return (i // seg == j // seg) & ((i % seg) % r == 0) & ((j % seg) % r == 0)


def longnet_mask(L, w0, alpha=2, head=None):
    """Union of BlockDilated(w0 alpha^k, alpha^k) levels; head given: LongNet's per-head
    offsets (reading R11c), in-segment offsets congruent to head mod alpha^k."""
    K = 0
    while w0 * alpha ** (K + 1) <= L:
        K += 1
    m = np.zeros((L, L), dtype=bool)
    i, j = _grid(L)
    for k in range(K + 1):
        seg, r = w0 * alpha ** k, alpha ** k
        off = 0 if head is None else head % r
        m |= (i // seg == j // seg) & ((i % seg) % r == off) & ((j % seg) % r == off)
    return m


def global_window_mask(L, w, globals_):
    """Window(w) UNION global rows UNION global columns (BigBird/Longformer without random)."""
    m = window_mask(L, w, 1)
    g = np.asarray(globals_, dtype=np.int64)
    m[g, :] = True
    m[:, g] = True
    return m


def masked_attention(q, k, v, mask):
    """q,k,v float64 [L,H,d]; mask bool [L,L]. Returns float64 [L,H,d]."""
    L, H, d = q.shape
    out = np.zeros((L, H, d), dtype=np.float64)
    for h in range(H):
        s = (q[:, h, :] @ k[:, h, :].T) / np.sqrt(d)
        s = np.where(mask, s, -np.inf)
        mx = s.max(axis=1, keepdims=True)
        empty = ~np.isfinite(mx[:, 0])
        mx = np.where(np.isfinite(mx), mx, 0.0)
        p = np.exp(s - mx)
        z = p.sum(axis=1, keepdims=True)
        z = np.where(z > 0, z, 1.0)
        o = (p / z) @ v[:, h, :]
        o[empty] = 0.0
        out[:, h, :] = o
    return out


def longnet_multiplicity(L, w0, alpha=2):
    """LongNet's multiset mixture (reading R11b): C[i, j] = number of levels k whose
    BlockDilated(w0 alpha^k, alpha^k) block contains (i, j)."""
    K = 0
    while w0 * alpha ** (K + 1) <= L:
        K += 1
    c = np.zeros((L, L), dtype=np.int64)
    for k in range(K + 1):
        c += block_dilated_mask(L, w0 * alpha ** k, alpha ** k)
    return c


def weighted_attention(q, k, v, mult):
    """Softmax over a multiset of neighbours: O_i = sum_j C_ij e^{s_ij} v_j / sum_j C_ij e^{s_ij}
    (C = multiplicities; C = 0 masks the pair; rows with no neighbour -> 0)."""
    L, H, d = q.shape
    out = np.zeros((L, H, d), dtype=np.float64)
    for h in range(H):
        s = (q[:, h, :] @ k[:, h, :].T) / np.sqrt(d)
        s = np.where(mult > 0, s, -np.inf)
        mx = s.max(axis=1, keepdims=True)
        empty = ~np.isfinite(mx[:, 0])
        mx = np.where(np.isfinite(mx), mx, 0.0)
        p = mult * np.exp(s - mx)
        z = p.sum(axis=1, keepdims=True)
        z = np.where(z > 0, z, 1.0)
        o = (p / z) @ v[:, h, :]
        o[empty] = 0.0
        out[:, h, :] = o
    return out

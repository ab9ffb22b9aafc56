"""CPU oracle for graph-view masked attention (arXiv 2502.01659).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` leg may import this package.
The product package ``paper_2502_01659_b200`` never imports it, and this package never
imports the product: the two share no code.

Contents
--------
* ``oracle.c`` — fp64 two-pass masked softmax attention over neighbour sets enumerated
  from the mask definitions (PAPER.md:71 Eq. 1, :124-158, :232-235, :241-269), plus a
  literal Algorithm 1 replay, the CSR builder and the counter-based input generator.
* ``dense.py`` — NumPy dense brute force (mask from vectorised predicates over the full
  L x L grid, masked softmax, rows with no neighbour -> 0).  Shares nothing with oracle.c.

Parity status per function is listed in DESIGN.md §3 ("Oracle pins").
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB_PATH = os.path.join(_HERE, "liboracle.so")

CSR, WINDOW, LONGNET, BIGBIRD, BLOCK_DILATED = 0, 1, 2, 3, 4
F32, BF16, F16, F64 = 0, 1, 2, 3
_DTYPE_CODE = {"f32": F32, "fp32": F32, "float32": F32, "bf16": BF16, "bfloat16": BF16,
               "f16": F16, "fp16": F16, "float16": F16, "f64": F64}


def build(force: bool = False) -> str:
    """Compile oracle.c -> liboracle.so with gcc (-O2, no fast-math, OpenMP)."""
    if (not force and os.path.exists(_LIB_PATH)
            and os.path.getmtime(_LIB_PATH) >= os.path.getmtime(_SRC)):
        return _LIB_PATH
    tmp = _LIB_PATH + f".tmp{os.getpid()}"
    cmd = ["gcc", "-O2", "-std=gnu11", "-fopenmp", "-fPIC", "-shared", "-o", tmp, _SRC, "-lm"]
    subprocess.check_call(cmd)
    os.replace(tmp, _LIB_PATH)
    return _LIB_PATH


class _OrcMask(ctypes.Structure):
    _fields_ = [
        ("kind", ctypes.c_int64), ("L", ctypes.c_int64),
        ("row_ptr", ctypes.c_void_p), ("col_idx", ctypes.c_void_p),
        ("w", ctypes.c_int64), ("r", ctypes.c_int64),
        ("w0", ctypes.c_int64), ("alpha", ctypes.c_int64),
        ("seg", ctypes.c_int64),
        ("global_idx", ctypes.c_void_p), ("n_global", ctypes.c_int64),
        ("n_random", ctypes.c_int64), ("seed", ctypes.c_uint64), ("parts", ctypes.c_int64),
        ("head", ctypes.c_int64),
    ]


class _OrcInputs(ctypes.Structure):
    _fields_ = [("q", ctypes.c_void_p), ("k", ctypes.c_void_p), ("v", ctypes.c_void_p),
                ("seed", ctypes.c_uint64), ("dtype", ctypes.c_int64), ("kv_rows", ctypes.c_int64)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB_PATH)
        L.orc_splitmix64.restype = ctypes.c_uint64
        L.orc_splitmix64.argtypes = [ctypes.c_uint64]
        L.orc_input_value.restype = ctypes.c_double
        L.orc_input_value.argtypes = [ctypes.c_uint64, ctypes.c_int, ctypes.c_uint64, ctypes.c_int]
        L.orc_fill_inputs.restype = None
        L.orc_fill_inputs.argtypes = [ctypes.c_uint64, ctypes.c_int, ctypes.c_uint64, ctypes.c_int64,
                                      ctypes.c_int, ctypes.c_void_p]
        L.orc_longnet_levels.restype = ctypes.c_int64
        L.orc_longnet_levels.argtypes = [ctypes.c_int64, ctypes.c_int64, ctypes.c_int64]
        L.orc_max_degree.restype = ctypes.c_int64
        L.orc_max_degree.argtypes = [ctypes.POINTER(_OrcMask)]
        L.orc_row_neighbors.restype = ctypes.c_int64
        L.orc_row_neighbors.argtypes = [ctypes.POINTER(_OrcMask), ctypes.c_int64, ctypes.c_void_p]
        L.orc_mask_to_csr.restype = ctypes.c_int64
        L.orc_mask_to_csr.argtypes = [ctypes.POINTER(_OrcMask), ctypes.c_void_p, ctypes.c_void_p]
        for fn in (L.orc_attention, L.orc_attention_alg1):
            fn.restype = ctypes.c_int64
            fn.argtypes = [ctypes.POINTER(_OrcInputs), ctypes.POINTER(_OrcMask), ctypes.c_int64,
                           ctypes.c_int64, ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p]
        L.orc_attention_backward.restype = ctypes.c_int64
        L.orc_attention_backward.argtypes = [ctypes.POINTER(_OrcInputs), ctypes.POINTER(_OrcMask), ctypes.c_int64,
                                             ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                             ctypes.c_void_p]
        L.orc_num_threads.restype = ctypes.c_int
        L.orc_set_num_threads.argtypes = [ctypes.c_int]
        _lib = L
    return _lib


@dataclass
class Mask:
    """Oracle-side mask description ("P_a" parameters or explicit CSR)."""
    kind: int
    L: int
    w: int = 1
    r: int = 1
    w0: int = 0
    alpha: int = 2
    seg: int = 1
    global_idx: Optional[np.ndarray] = None   # int64 sorted; None -> evenly spaced
    n_global: int = 0
    n_random: int = 0
    seed: int = 0
    parts: int = 0                             # BigBird components (0 = all); LongNet variant bits
    head: int = 0                              # LongNet per-head offsets: head of neighbors()
    row_ptr: Optional[np.ndarray] = None       # int64 [L+1]
    col_idx: Optional[np.ndarray] = None       # int32 [nnz]
    _keep: list = field(default_factory=list, repr=False)

    def c(self) -> _OrcMask:
        m = _OrcMask()
        m.kind, m.L, m.w, m.r = self.kind, self.L, self.w, self.r
        m.w0, m.alpha, m.seg = self.w0, self.alpha, self.seg
        m.n_global, m.n_random, m.seed = self.n_global, self.n_random, self.seed & (2**64 - 1)
        m.parts = self.parts
        m.head = self.head
        self._keep = []
        if self.global_idx is not None:
            g = np.ascontiguousarray(self.global_idx, dtype=np.int64)
            self._keep.append(g)
            m.global_idx = g.ctypes.data
            m.n_global = len(g)
        if self.kind == CSR:
            rp = np.ascontiguousarray(self.row_ptr, dtype=np.int64)
            ci = np.ascontiguousarray(self.col_idx, dtype=np.int32)
            self._keep += [rp, ci]
            m.row_ptr, m.col_idx = rp.ctypes.data, ci.ctypes.data
        return m


def window(L, w, r=1):
    return Mask(WINDOW, L, w=w, r=r)


def block_dilated(L, seg, r=1):
    return Mask(BLOCK_DILATED, L, seg=seg, r=r)


def longnet(L, w0, alpha=2, multiset=False, head_offsets=False, head=0):
    """LongNet (reading R11); multiset=True: LongNet's own mixture, the multiset union of the
    levels' blocks (reading R11b); head_offsets=True: head h keeps the
    in-segment offsets congruent to h mod alpha^k at level k (reading R11c) — attention()
    uses each head's own set, neighbors()/mask_to_csr() that of `head`."""
    return Mask(LONGNET, L, w0=w0, alpha=alpha, parts=(1 if multiset else 0) | (2 if head_offsets else 0), head=head)


BB_WINDOW, BB_GLOBAL, BB_RANDOM = 1, 2, 4  # BigBird components (disjoint; union = full mask)


def bigbird(L, w, n_global, n_random, seed, global_idx=None, r=1, parts=0):
    """BigBird / Longformer (readings R8-R10), window optionally dilated
    by r; `parts` selects components (BB_* bits, 0 = all)."""
    return Mask(BIGBIRD, L, w=w, r=r, n_global=n_global, n_random=n_random, seed=seed, parts=parts,
                global_idx=None if global_idx is None else np.asarray(global_idx, np.int64))


def csr(L, row_ptr, col_idx):
    return Mask(CSR, L, row_ptr=np.asarray(row_ptr, np.int64), col_idx=np.asarray(col_idx, np.int32))


def coo_to_csr(L: int, rows, cols):
    """COO edge list -> binary CSR by the plain definition (reading R7: a 0-1
    mask, so a repeated (i, j) is one edge): N(i) = sorted {cols[e] : rows[e] = i}.
    Pure-Python sets: small cases only.  Returns (row_ptr int64 [L+1], col_idx int32)."""
    nbrs = [set() for _ in range(L)]
    for i, j in zip(np.asarray(rows).tolist(), np.asarray(cols).tolist()):
        if not (0 <= i < L and 0 <= j < L):
            raise ValueError(f"edge ({i}, {j}) outside [0, {L})")
        nbrs[i].add(j)
    row_ptr = np.zeros(L + 1, dtype=np.int64)
    col_idx = []
    for i in range(L):
        cs = sorted(nbrs[i])
        col_idx.extend(cs)
        row_ptr[i + 1] = row_ptr[i] + len(cs)
    return row_ptr, np.asarray(col_idx, dtype=np.int32)


def splitmix64(x: int) -> int:
    return lib().orc_splitmix64(x & (2**64 - 1))


def input_value(seed: int, tensor: int, e: int, dtype: str = "f32") -> float:
    return lib().orc_input_value(seed, tensor, e, _DTYPE_CODE[dtype])


def inputs(seed: int, L: int, H: int, d: int, dtype: str = "f32"):
    """Seeded Q, K, V as fp64 arrays [L,H,d] holding the exact stored dtype values."""
    out = []
    for t in range(3):
        a = np.empty((L, H, d), dtype=np.float64)
        lib().orc_fill_inputs(seed, t, 0, a.size, _DTYPE_CODE[dtype], a.ctypes.data)
        out.append(a)
    return tuple(out)


def longnet_levels(w0, alpha, L):
    return lib().orc_longnet_levels(w0, alpha, L)


def neighbors(mask: Mask, i: int) -> np.ndarray:
    cm = mask.c()
    cap = lib().orc_max_degree(ctypes.byref(cm))
    buf = np.empty(cap + 1, dtype=np.int64)
    n = lib().orc_row_neighbors(ctypes.byref(cm), i, buf.ctypes.data)
    return buf[:n].copy()


def mask_to_csr(mask: Mask, with_cols: bool = True):
    """(row_ptr int64 [L+1], col_idx int32 [nnz] or None, nnz) from the definitions."""
    cm = mask.c()
    rp = np.empty(mask.L + 1, dtype=np.int64)
    nnz = lib().orc_mask_to_csr(ctypes.byref(cm), rp.ctypes.data, None)
    if not with_cols:
        return rp, None, nnz
    ci = np.empty(max(nnz, 1), dtype=np.int32)
    lib().orc_mask_to_csr(ctypes.byref(cm), rp.ctypes.data, ci.ctypes.data)
    return rp, ci[:nnz], nnz


def _run(fn, q, k, v, mask, H, d, rows, seed, dtype):
    cm = mask.c()
    inp = _OrcInputs()
    keep = []
    if q is not None:
        for name, a in (("q", q), ("k", k), ("v", v)):
            a = np.ascontiguousarray(a, dtype=np.float64)
            keep.append(a)
            setattr(inp, name, a.ctypes.data)
    else:
        inp.seed = seed & (2**64 - 1)
        inp.dtype = _DTYPE_CODE[dtype]
    if rows is None:
        nrows, rptr = mask.L, None
    else:
        rows = np.ascontiguousarray(rows, dtype=np.int64)
        keep.append(rows)
        nrows, rptr = len(rows), rows.ctypes.data
    out = np.zeros((nrows, H, d), dtype=np.float64)
    edges = fn(ctypes.byref(inp), ctypes.byref(cm), H, d, rptr, nrows, out.ctypes.data)
    return out, edges


def attention(q, k, v, mask: Mask, rows: Optional[Sequence[int]] = None):
    """Two-pass fp64 oracle on explicit arrays q,k,v [L,H,d].  Returns (out, edges)."""
    L, H, d = q.shape
    return _run(lib().orc_attention, q, k, v, mask, H, d, rows, 0, "f64")


def attention_seeded(seed, dtype, mask: Mask, H, d, rows: Optional[Sequence[int]] = None):
    """Two-pass fp64 oracle regenerating Q/K/V rows from the counter hash (reading R22)."""
    return _run(lib().orc_attention, None, None, None, mask, H, d, rows, seed, dtype)


def attention_backward(q, k, v, mask: Mask, dout):
    """fp64 gradients (dQ, dK, dV) of the masked attention for upstream dO (oracle.c
    orc_attention_backward: the chain rule per edge, serial).  Returns (dq, dk, dv, edges)."""
    L, H, d = q.shape
    cm = mask.c()
    inp = _OrcInputs()
    keep = []
    for name, a in (("q", q), ("k", k), ("v", v)):
        a = np.ascontiguousarray(a, dtype=np.float64)
        keep.append(a)
        setattr(inp, name, a.ctypes.data)
    g = np.ascontiguousarray(dout, dtype=np.float64)
    dq, dk, dv = (np.empty((L, H, d), dtype=np.float64) for _ in range(3))
    edges = lib().orc_attention_backward(ctypes.byref(inp), ctypes.byref(cm), H, d, g.ctypes.data, dq.ctypes.data,
                                         dk.ctypes.data, dv.ctypes.data)
    return dq, dk, dv, edges


def attention_alg1(q, k, v, mask: Mask, rows=None):
    """Literal Algorithm 1 replay (per-step division), fp64."""
    L, H, d = q.shape
    return _run(lib().orc_attention_alg1, q, k, v, mask, H, d, rows, 0, "f64")


def num_threads() -> int:
    return lib().orc_num_threads()


def set_num_threads(n: int) -> None:
    lib().orc_set_num_threads(n)

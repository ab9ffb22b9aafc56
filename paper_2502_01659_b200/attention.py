"""Python entry points: argument marshalling onto the C ABI (include/ga.h) only.

Every step of the path runs in libga.so's CUDA kernels; torch provides device memory
and the current stream.
"""
from __future__ import annotations

import ctypes
from typing import Optional

import torch

from . import _abi
from .masks import CSR, Mask

_DT = {torch.float32: _abi.GA_F32, torch.bfloat16: _abi.GA_BF16, torch.float16: _abi.GA_F16}
_KERNELS = {"auto": _abi.GA_KERNEL_AUTO, "edge": _abi.GA_KERNEL_EDGE, "tiled": _abi.GA_KERNEL_TILED, "window": _abi.GA_KERNEL_TILED,
            "tc": _abi.GA_KERNEL_TC}


def _stream(device=None):
    return ctypes.c_void_p(torch.cuda.current_stream(device).cuda_stream)


def dtype_code(t: torch.dtype) -> int:
    if t not in _DT:
        raise TypeError(f"unsupported dtype {t}; use float32, bfloat16 or float16")
    return _DT[t]


class State:
    """Carried online-softmax state (m, l, o) of `rows` query rows x `heads` (include/ga.h
    ga_state): fp32 CUDA tensors m, l [rows, heads] and o [rows, heads, d].
    Zero-filled = empty (l == 0)."""

    def __init__(self, m: torch.Tensor, l: torch.Tensor, o: torch.Tensor):
        self.m, self.l, self.o = m, l, o

    @classmethod
    def empty(cls, rows: int, heads: int, d: int, device="cuda") -> "State":
        z = lambda *s: torch.zeros(s, dtype=torch.float32, device=device)
        return cls(z(rows, heads), z(rows, heads), z(rows, heads, d))

    def c(self) -> _abi.GaState:
        st = _abi.GaState()
        st.m, st.l, st.o = self.m.data_ptr(), self.l.data_ptr(), self.o.data_ptr()
        return st


def _opts(q_begin, q_rows, kv_begin, kv_rows, workspace, edge_counter, row_fingerprint, kernel, heavy,
          state: Optional[State] = None, accumulate: bool = False, tensor_counter=None):
    o = _abi.GaOpts()
    if state is not None:
        o.state = state.c()
        o.state_mode = _abi.GA_STATE_ACCUMULATE if accumulate else _abi.GA_STATE_WRITE
    o.q_begin, o.q_rows, o.kv_begin, o.kv_rows = q_begin, q_rows, kv_begin, kv_rows
    if workspace is not None:
        o.workspace = workspace.data_ptr()
        o.workspace_bytes = workspace.numel() * workspace.element_size()
    if edge_counter is not None:
        o.edge_counter = edge_counter.data_ptr()
    if row_fingerprint is not None:
        o.row_fingerprint = row_fingerprint.data_ptr()
    if tensor_counter is not None:
        o.tensor_counter = tensor_counter.data_ptr()
    o.kernel = _KERNELS[kernel]
    o.heavy_threshold = heavy
    return o


def workspace_size(mask: Mask, L: int, d: int, heads: int, dtype=torch.bfloat16, q_begin=0, q_rows=0,
                   heavy_threshold: int = 0) -> int:
    cm = mask.to_c(L)
    o = _opts(q_begin, q_rows, 0, 0, None, None, None, "auto", heavy_threshold)
    n = ctypes.c_size_t()
    _abi.check(_abi.lib().ga_workspace_size(ctypes.byref(cm), L, d, heads, dtype_code(dtype), ctypes.byref(o),
                                            ctypes.byref(n)))
    return n.value


def attention(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, mask: Mask, out: Optional[torch.Tensor] = None, *,
              L: Optional[int] = None, q_begin: int = 0, kv_begin: int = 0, kernel: str = "auto",
              workspace: Optional[torch.Tensor] = None, edge_counter: Optional[torch.Tensor] = None,
              row_fingerprint: Optional[torch.Tensor] = None, heavy_threshold: int = 0,
              state: Optional[State] = None, accumulate: bool = False,
              tensor_counter: Optional[torch.Tensor] = None) -> Optional[torch.Tensor]:
    """Graph-view masked attention (Algorithm 1) via ga_attention_ex.

    q: [q_rows, H, d] rows q_begin.. of the global sequence; k, v: [kv_rows, H, d] rows
    kv_begin..; L: global length (default q.shape[0]).  CSR masks with heavy rows should
    pass `workspace` (uint8 CUDA tensor of workspace_size(...) bytes) to use the split path.
    With `state` (a State of q's rows) the call also writes — or with accumulate=True
    (+)-combines into — the carried (m, l, o) of its edges; `out` is then only produced when
    given (returns out, or None).  Probes (int64 CUDA tensors of one element, added to):
    edge_counter — q.k products that received a weight (with row_fingerprint, or outside the
    tcgen05 window kernel's range, on the instrumented edge kernel); tensor_counter — products
    the tcgen05 window kernel's MMA tiles computed (masked pairs included, reading R23).
    """
    if not (q.is_cuda and k.is_cuda and v.is_cuda):
        raise ValueError("q, k, v must be CUDA tensors (no CPU path)")
    if q.dtype != k.dtype or q.dtype != v.dtype:
        raise TypeError("q, k, v must share a dtype")
    if q.dim() != 3 or k.dim() != 3 or v.dim() != 3:
        raise ValueError("expected [tokens, heads, d] tensors")
    for t in (q, k, v):
        if not t.is_contiguous():
            raise ValueError("q, k, v must be contiguous")
    rows, H, d = q.shape
    L = rows if L is None else L
    if out is None and state is None:
        out = torch.empty_like(q)
    cm = mask.to_c(L)
    o = _opts(q_begin, rows, kv_begin, k.shape[0], workspace, edge_counter, row_fingerprint, kernel, heavy_threshold,
              state, accumulate, tensor_counter)
    _abi.check(_abi.lib().ga_attention_ex(q.data_ptr(), k.data_ptr(), v.data_ptr(), ctypes.byref(cm),
                                          out.data_ptr() if out is not None else None, L, d, H, dtype_code(q.dtype),
                                          ctypes.byref(o), _stream(q.device)))
    return out


def attention_backward(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, out: torch.Tensor, dout: torch.Tensor,
                       mask: Mask, lse: Optional[torch.Tensor] = None):
    """Gradients (dq, dk, dv) — fp32 CUDA tensors [L, H, d] — of out = attention(q, k, v, mask)
    for the upstream gradient dout (ga_attention_backward).  lse: optional
    fp32 [L, H] log2-sum-exp2 of the forward's row scores (recomputed when None)."""
    for t in (q, k, v, out, dout):
        if not t.is_cuda or not t.is_contiguous() or t.dtype != q.dtype or t.shape != q.shape:
            raise ValueError("q, k, v, out, dout: contiguous CUDA tensors of one shape and dtype")
    L, H, d = q.shape
    dq, dk, dv = (torch.empty((L, H, d), dtype=torch.float32, device=q.device) for _ in range(3))
    cm = mask.to_c(L)
    _abi.check(_abi.lib().ga_attention_backward(q.data_ptr(), k.data_ptr(), v.data_ptr(), out.data_ptr(),
                                                dout.data_ptr(), ctypes.byref(cm),
                                                lse.data_ptr() if lse is not None else None, dq.data_ptr(),
                                                dk.data_ptr(), dv.data_ptr(), L, d, H, dtype_code(q.dtype),
                                                _stream(q.device)))
    return dq, dk, dv


class GraphAttention(torch.autograd.Function):
    """torch.autograd wrapper: forward = ga_attention_ex, backward = ga_attention_backward
    (gradients returned in the input dtype)."""

    @staticmethod
    def forward(ctx, q, k, v, mask):
        out = attention(q.contiguous(), k.contiguous(), v.contiguous(), mask)
        ctx.save_for_backward(q, k, v, out)
        ctx.mask = mask
        return out

    @staticmethod
    def backward(ctx, dout):
        q, k, v, out = ctx.saved_tensors
        dq, dk, dv = attention_backward(q.contiguous(), k.contiguous(), v.contiguous(), out,
                                        dout.contiguous().to(q.dtype), ctx.mask)
        return dq.to(q.dtype), dk.to(k.dtype), dv.to(v.dtype), None


def state_finalize(state: State, dtype=torch.bfloat16, out: Optional[torch.Tensor] = None) -> torch.Tensor:
    """out = o / l of a carried state (ga_state_finalize)."""
    rows, H, d = state.o.shape
    if out is None:
        out = torch.empty((rows, H, d), dtype=dtype, device=state.o.device)
    st = state.c()
    _abi.check(_abi.lib().ga_state_finalize(ctypes.byref(st), rows, H, d, dtype_code(out.dtype), out.data_ptr(),
                                            _stream(out.device)))
    return out


def compose(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, components, *, L: Optional[int] = None,
            q_begin: int = 0, kv_begin: int = 0) -> torch.Tensor:
    """Attention over the union of DISJOINT component masks as sequential calls carrying one
    state (the paper composes its kernels this way)."""
    rows, H, d = q.shape
    st = State.empty(rows, H, d, device=q.device)
    for c in components:
        attention(q, k, v, c, L=L, q_begin=q_begin, kv_begin=kv_begin, state=st, accumulate=True)
    return state_finalize(st, q.dtype)


def attention_host(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, mask: Mask, out: torch.Tensor,
                   stream: Optional[torch.cuda.Stream] = None) -> torch.Tensor:
    """End-to-end call on HOST tensors (pinned for async copies) through ga_attention_host:
    H2D copies, attention, D2H copy, all inside libga on `stream`.  Synchronise the stream
    before reading `out`."""
    L, H, d = q.shape
    cm = mask.to_c(L)
    s = ctypes.c_void_p((stream or torch.cuda.current_stream()).cuda_stream)
    _abi.check(_abi.lib().ga_attention_host(q.data_ptr(), k.data_ptr(), v.data_ptr(), ctypes.byref(cm),
                                            out.data_ptr(), L, d, H, dtype_code(q.dtype), s))
    return out


def mask_count(mask: Mask, L: int) -> int:
    """Exact edge count of a pattern (host closed forms)."""
    cm = mask.to_c(L)
    n = ctypes.c_int64()
    _abi.check(_abi.lib().ga_mask_count(ctypes.byref(cm), ctypes.byref(n)))
    return n.value


def query_alignment(mask: Mask, L: int, d: int, dtype=torch.bfloat16) -> int:
    """Token alignment under which sharded launches are bit-identical to one launch."""
    cm = mask.to_c(L)
    n = ctypes.c_int64()
    _abi.check(_abi.lib().ga_query_alignment(ctypes.byref(cm), d, dtype_code(dtype), ctypes.byref(n)))
    return n.value


def mask_to_csr(mask: Mask, L: int, device="cuda") -> CSR:
    """Materialise an implicit pattern as device CSR (degrees -> scan -> fill)."""
    nnz = mask_count(mask, L)
    row_ptr = torch.empty(L + 1, dtype=torch.int64, device=device)
    col_idx = torch.empty(max(nnz, 1), dtype=torch.int32, device=device)
    cm = mask.to_c(L)
    _abi.check(_abi.lib().ga_mask_to_csr(ctypes.byref(cm), row_ptr.data_ptr(), col_idx.data_ptr(),
                                         _stream(row_ptr.device)))
    return CSR(row_ptr, col_idx[:nnz])


def coo_to_csr(rows: torch.Tensor, cols: torch.Tensor, L: int) -> CSR:
    """COO edge list (int32 CUDA tensors, any order, duplicates counted once) -> device CSR
    (sort + unique on the GPU; PAPER.md:227 COO storage)."""
    n = rows.numel()
    if cols.numel() != n:
        raise ValueError("rows and cols must have the same length")
    rows = rows.to(torch.int32).contiguous()
    cols = cols.to(torch.int32).contiguous()
    row_ptr = torch.empty(L + 1, dtype=torch.int64, device=rows.device)
    col_idx = torch.empty(max(n, 1), dtype=torch.int32, device=rows.device)
    nnz = ctypes.c_int64()
    _abi.check(_abi.lib().ga_coo_to_csr(int(L), rows.data_ptr() if n else None, cols.data_ptr() if n else None, n,
                                        row_ptr.data_ptr(), col_idx.data_ptr(), ctypes.byref(nnz),
                                        _stream(rows.device)))
    return CSR(row_ptr, col_idx[:nnz.value])


def mask_validate(mask: CSR, L: int) -> bool:
    cm = mask.to_c(L)
    ok = ctypes.c_int()
    st = _abi.lib().ga_mask_validate(ctypes.byref(cm), _stream(mask.row_ptr.device), ctypes.byref(ok))
    if st == _abi.GA_ERR_MASK:
        return False
    _abi.check(st)
    return bool(ok.value)


def fill_inputs(dst: torch.Tensor, seed: int, tensor: int, e0: int = 0, shift: float = 0.0) -> torch.Tensor:
    """Seeded U[0,1) (+shift) values on the device (reading R22), in dst's dtype."""
    _abi.check(_abi.lib().ga_fill_inputs(dst.data_ptr(), dtype_code(dst.dtype), dst.numel(), seed & (2**64 - 1),
                                         tensor, e0, shift, _stream(dst.device)))
    return dst


def qkv_device(seed: int, L: int, H: int, d: int, dtype=torch.bfloat16, device="cuda", shift: float = 0.0,
               token0: int = 0):
    """Allocate and fill seeded Q, K, V [L, H, d] (tokens token0.. of the global stream)."""
    out = []
    for t in range(3):
        x = torch.empty((L, H, d), dtype=dtype, device=device)
        fill_inputs(x, seed, t, token0 * H * d, shift)
        out.append(x)
    return tuple(out)


def version() -> str:
    return _abi.lib().ga_version().decode()

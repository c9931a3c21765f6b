"""Stateless device ops over torch CUDA tensors (C ABI family 1).

    route_topk        dataplane::route_topk       (dataplane.hpp:72-106)
    build_index       dataplane::permute, index form (dataplane.hpp:118-140)
    permute_rows      gather-permute of rows (or a hidden_shard column slice)
    unpermute_combine weighted un-permute (dataplane.hpp:325-342)
    combine_backward / dispatch_backward / route_backward   their adjoints
    host_empty        page-locked host tensor (moe_host_alloc) for forward_host

All run on the current CUDA stream; nothing here synchronises unless
`check=True` asks for the device-side validation result.
"""
from __future__ import annotations

import ctypes as C
import math
import weakref
from dataclasses import dataclass

import torch

from . import _lib
from ._lib import check


def _stream() -> int:
    return torch.cuda.current_stream().cuda_stream


def host_empty(shape, dtype: torch.dtype) -> torch.Tensor:
    """Page-locked host tensor allocated by moe_host_alloc (cudaHostAlloc,
    portable), for forward_host buffers.  Freed when the last view dies."""
    lib = _lib.load()
    shape = tuple(shape) if not isinstance(shape, int) else (shape,)
    nbytes = math.prod(shape) * torch.empty((), dtype=dtype).element_size()
    if nbytes == 0:
        return torch.empty(shape, dtype=dtype)
    ptr = C.c_void_p()
    check(lib.moe_host_alloc(nbytes, C.byref(ptr)))
    buf = (C.c_uint8 * nbytes).from_address(ptr.value)
    weakref.finalize(buf, lib.moe_host_free, ptr)  # torch.frombuffer keeps `buf` alive with the storage
    return torch.frombuffer(buf, dtype=torch.uint8).view(dtype).view(shape)


def route_topk(logits: torch.Tensor, k: int):
    """logits [T, E] fp32/fp64 (CUDA) -> (experts int32 [T, k] ascending, probs [T, k] logit dtype)."""
    if logits.dim() != 2:
        raise ValueError("route_topk: logits must be [T, E]")
    logits = logits.contiguous()
    T, E = logits.shape
    experts = torch.empty((T, max(k, 0)), dtype=torch.int32, device=logits.device)
    probs = torch.empty((T, max(k, 0)), dtype=logits.dtype, device=logits.device)
    lib = _lib.load()
    check(lib.moe_route_topk(logits.data_ptr(), _lib.dtype_code(logits.dtype), T, E, k, experts.data_ptr(),
                             probs.data_ptr(), _stream()))
    return experts, probs


@dataclass
class Index:
    perm_src: torch.Tensor       # [T*k] int32 source token of permuted row r
    expert_of: torch.Tensor      # [T*k] int32
    slot_pos: torch.Tensor       # [T, k] int32 permuted row of (token, slot)
    counts: torch.Tensor         # [n, E] int32 rows per (chunk, expert)
    expert_offsets: torch.Tensor  # [E+1] int32


def build_index(experts: torch.Tensor, num_experts: int, n_chunks: int = 1, check_range: bool = False,
                check: bool | None = None) -> Index:
    """Stable expert-major counting sort of the (token, slot) pairs."""
    if check is not None:
        check_range = check
    experts = experts.contiguous().to(torch.int32)
    T, k = experts.shape
    dev = experts.device
    R = T * k
    # rows past expert_offsets[E] (empty slots / out-of-range ids) keep -1:
    # permute_rows zero-fills them instead of gathering garbage
    idx = Index(torch.full((R,), -1, dtype=torch.int32, device=dev), torch.full((R,), -1, dtype=torch.int32, device=dev),
                torch.empty((T, k), dtype=torch.int32, device=dev),
                torch.empty((n_chunks, num_experts), dtype=torch.int32, device=dev),
                torch.empty(num_experts + 1, dtype=torch.int32, device=dev))
    err = torch.zeros(1, dtype=torch.int32, device=dev)
    lib = _lib.load()
    _lib.check(lib.moe_build_index(experts.data_ptr(), T, k, num_experts, n_chunks, idx.perm_src.data_ptr(),
                                   idx.expert_of.data_ptr(), idx.slot_pos.data_ptr(), idx.counts.data_ptr(),
                                   idx.expert_offsets.data_ptr(), err.data_ptr(), _stream()))
    if check_range and int(err.item()) != 0:
        raise _lib.InvalidArgument(int(err.item()), "build_index: expert id out of range")
    return idx


def permute_rows(x: torch.Tensor, perm_src: torch.Tensor, col_off: int = 0, width: int | None = None,
                 out: torch.Tensor | None = None) -> torch.Tensor:
    """out[r] = x[perm_src[r], col_off:col_off+width] (elements)."""
    x = x.contiguous()
    T, h = x.shape
    width = h - col_off if width is None else width
    R = perm_src.numel()
    if out is None:
        out = torch.empty((R, width), dtype=x.dtype, device=x.device)
    es = x.element_size()
    check(_lib.load().moe_permute_rows(x.data_ptr(), h * es, col_off * es, width * es,
                                       perm_src.contiguous().data_ptr(), R, out.data_ptr(), out.stride(0) * es,
                                       _stream()))
    return out


def unpermute_combine(y: torch.Tensor, slot_pos: torch.Tensor, probs: torch.Tensor,
                      out_dtype: torch.dtype | None = None, out: torch.Tensor | None = None) -> torch.Tensor:
    """out[i] = sum_s probs[i, s] * y[slot_pos[i, s]]  (fp32 acc; fp64 for f64/i64)."""
    y = y.contiguous()
    R, h = y.shape
    T, k = slot_pos.shape
    if out_dtype is None:
        out_dtype = torch.float64 if y.dtype in (torch.float64, torch.int64) else y.dtype
    if out is None:
        out = torch.empty((T, h), dtype=out_dtype, device=y.device)
    probs = probs.contiguous()
    check(_lib.load().moe_unpermute_combine(y.data_ptr(), _lib.dtype_code(y.dtype), h, h,
                                            slot_pos.contiguous().data_ptr(), probs.data_ptr(),
                                            _lib.dtype_code(probs.dtype), T, k, out.data_ptr(),
                                            _lib.dtype_code(out.dtype), out.stride(0), _stream()))
    return out


# ---------------------------------------------------------------------------
# Backward of the stateless ops (include/monta.h section 1b).

def combine_backward(grad_out: torch.Tensor, y: torch.Tensor | None, slot_pos: torch.Tensor, probs: torch.Tensor,
                     need_grad_y: bool = True, need_grad_probs: bool = True, num_rows: int | None = None):
    """Adjoint of unpermute_combine.  Returns (grad_y [R, h] in y's dtype or
    None, grad_probs [T, k] in probs' dtype or None)."""
    grad_out = grad_out.contiguous()
    T, h = grad_out.shape
    k = slot_pos.shape[1]
    slot_pos = slot_pos.contiguous()
    if y is not None:
        y = y.contiguous()
        R, ydt = y.shape[0], y.dtype
    else:
        if need_grad_probs:
            raise ValueError("combine_backward: grad_probs needs y")
        R, ydt = (T * k if num_rows is None else num_rows), grad_out.dtype
    probs = probs.contiguous()
    # rows no slot references (empty slots, padding) get no store: start from zero
    grad_y = torch.zeros((R, h), dtype=ydt, device=grad_out.device) if need_grad_y else None
    grad_probs = torch.empty_like(probs) if need_grad_probs else None
    check(_lib.load().moe_combine_backward(
        grad_out.data_ptr(), _lib.dtype_code(grad_out.dtype), h,
        y.data_ptr() if y is not None else None, _lib.dtype_code(ydt), h, h,
        slot_pos.data_ptr(), probs.data_ptr(), _lib.dtype_code(probs.dtype), T, k,
        grad_y.data_ptr() if grad_y is not None else None, h,
        grad_probs.data_ptr() if grad_probs is not None else None, _stream()))
    return grad_y, grad_probs


def dispatch_backward(grad_rows: torch.Tensor, slot_pos: torch.Tensor, out_dtype: torch.dtype | None = None,
                      out: torch.Tensor | None = None) -> torch.Tensor:
    """Adjoint of the dispatch gather: grad_x[i] = sum_s grad_rows[slot_pos[i, s]]."""
    grad_rows = grad_rows.contiguous()
    R, h = grad_rows.shape
    T, k = slot_pos.shape
    slot_pos = slot_pos.contiguous()
    if out is None:
        out = torch.empty((T, h), dtype=out_dtype or grad_rows.dtype, device=grad_rows.device)
    check(_lib.load().moe_dispatch_backward(grad_rows.data_ptr(), _lib.dtype_code(grad_rows.dtype), h, h,
                                            slot_pos.data_ptr(), T, k, out.data_ptr(),
                                            _lib.dtype_code(out.dtype), out.stride(0), _stream()))
    return out


def route_backward(logits: torch.Tensor, experts: torch.Tensor, grad_probs: torch.Tensor) -> torch.Tensor:
    """Adjoint of route_topk with respect to the logits."""
    logits = logits.contiguous()
    T, E = logits.shape
    k = experts.shape[1]
    grad_logits = torch.empty_like(logits)
    experts = experts.contiguous().to(torch.int32)
    grad_probs = grad_probs.contiguous().to(logits.dtype)
    check(_lib.load().moe_route_backward(logits.data_ptr(), _lib.dtype_code(logits.dtype), T, E, k,
                                         experts.data_ptr(), grad_probs.data_ptr(), grad_logits.data_ptr(),
                                         _stream()))
    return grad_logits


# ---------------------------------------------------------------------------
# Expert compute (include/monta.h section 1c): tcgen05 grouped GEMM / SwiGLU FFN.

def grouped_gemm(x: torch.Tensor, w: torch.Tensor, expert_offsets: torch.Tensor, act: int = _lib.ACT_NONE,
                 out: torch.Tensor | None = None) -> torch.Tensor:
    """y[r] = x[r] . w[l]^T for r in [offs[l], offs[l+1]); x [rows, K] bf16,
    w [L, N, K] bf16; act=ACT_SWIGLU -> y has N/2 columns silu(gate)*up
    (w from interleave_w13)."""
    L, N, K = w.shape
    rows = x.shape[0]
    ncol = N // 2 if act == _lib.ACT_SWIGLU else N
    if out is None:
        out = torch.empty((rows, ncol), dtype=torch.bfloat16, device=x.device)
    check(_lib.load().moe_grouped_gemm(x.data_ptr(), x.stride(0), rows, w.contiguous().data_ptr(),
                                       expert_offsets.contiguous().data_ptr(), L, N, K, out.data_ptr(),
                                       out.stride(0), act, _stream()))
    return out


def interleave_w13(w_gate: torch.Tensor, w_up: torch.Tensor) -> torch.Tensor:
    """[L, F, h] gate + up -> [L, 2F, h] in the grouped GEMM's SwiGLU tile order."""
    L, F, h = w_gate.shape
    w13 = torch.empty((L, 2 * F, h), dtype=w_gate.dtype, device=w_gate.device)
    check(_lib.load().moe_interleave_w13(w_gate.contiguous().data_ptr(), w_up.contiguous().data_ptr(), L, F, h,
                                         w13.data_ptr(), _stream()))
    return w13


def expert_ffn(x: torch.Tensor, w13: torch.Tensor, w2: torch.Tensor, expert_offsets: torch.Tensor,
               out: torch.Tensor | None = None, workspace: torch.Tensor | None = None) -> torch.Tensor:
    """SwiGLU experts over expert-major rows: (silu(x Wg^T) * x Wu^T) W2^T per segment."""
    L, F2, h = w13.shape
    F = F2 // 2
    rows = x.shape[0]
    if out is None:
        out = torch.empty((rows, h), dtype=torch.bfloat16, device=x.device)
    if workspace is None:
        workspace = torch.empty((rows, F), dtype=torch.bfloat16, device=x.device)
    check(_lib.load().moe_expert_ffn(x.data_ptr(), x.stride(0), rows, w13.data_ptr(), w2.contiguous().data_ptr(),
                                     expert_offsets.contiguous().data_ptr(), L, h, F, workspace.data_ptr(),
                                     out.data_ptr(), out.stride(0), _stream()))
    return out


# ---------------------------------------------------------------------------
# Communication priorities (include/monta.h section 1d): EP > PP > CP > DP.

def comm_priority(group: int) -> int:
    """The reference's resolution priority of a communication group (conflict.hpp:40-50)."""
    return int(_lib.load().moe_comm_priority(group))


def comm_stream_priority(group: int, device: int | None = None) -> int:
    """CUDA stream priority the library assigns to a group on `device`."""
    dev = torch.cuda.current_device() if device is None else device
    out = C.c_int()
    check(_lib.load().moe_comm_stream_priority(group, dev, C.byref(out)))
    return int(out.value)


def comm_stream(group: int) -> torch.cuda.Stream:
    """A torch stream carrying `group`'s priority (e.g. the stream a caller
    issues its DP gradient all-reduce on, below this library's EP exchange)."""
    return torch.cuda.Stream(priority=comm_stream_priority(group))

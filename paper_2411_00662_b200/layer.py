"""Device-level API: one MoE layer's dispatch + combine over e x t cards.

`MoeLayer` owns a `moe_ctx` from the C ABI.  Every buffer lives in the
context's per-card HBM slab; the properties below are zero-copy torch views
of it (via __cuda_array_interface__) so callers fill inputs and read outputs
in place.  Views must not outlive the layer.

    world_size == 1      : all e*t cards on one GPU (virtual mode — the
                           reference's single-process emulation)
    world_size == e*t    : one card per process/GPU; `connect()` exchanges
                           CUDA IPC handles through torch.distributed so every
                           card can store into its peers over NVLink.

Reference mapping (dataplane.hpp):  route -> route_topk,  permute -> permute,
dispatch(BASELINE) -> dispatch_monolithic,  dispatch(O1/O2/O3, n) ->
dispatch_chunked,  combine -> combine_unpermute.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import torch

from . import _lib
from ._lib import BASELINE, O1, O2, O3, LAND_FINAL, LAND_STAGED, check

_TYPESTR = {torch.float32: "<f4", torch.float64: "<f8", torch.int64: "<i8", torch.int32: "<i4",
            torch.bfloat16: "<i2", torch.float16: "<f2", torch.uint8: "|u1"}


class _CudaArray:
    def __init__(self, ptr: int, shape, typestr: str):
        self.__cuda_array_interface__ = {"shape": tuple(int(s) for s in shape), "typestr": typestr,
                                         "data": (int(ptr), False), "version": 2, "strides": None}


def device_view(ptr: int, shape, dtype: torch.dtype, device: int) -> torch.Tensor:
    """Zero-copy torch view of device memory owned elsewhere."""
    n = 1
    for s in shape:
        n *= int(s)
    if n == 0:
        return torch.empty(tuple(shape), dtype=dtype, device=f"cuda:{device}")
    with torch.cuda.device(device):
        t = torch.as_tensor(_CudaArray(ptr, shape, _TYPESTR[dtype]), device=f"cuda:{device}")
    return t.view(dtype) if dtype is torch.bfloat16 else t


@dataclass
class CardTensors:
    card: int
    node: int
    rho: int
    x: torch.Tensor
    logits: torch.Tensor
    token_ids: torch.Tensor
    experts: torch.Tensor
    probs: torch.Tensor
    perm_src: torch.Tensor
    expert_of: torch.Tensor
    slot_pos: torch.Tensor
    counts: torch.Tensor
    expert_offsets: torch.Tensor
    permuted: torch.Tensor
    recv: torch.Tensor
    recv_tags: torch.Tensor
    pre: torch.Tensor
    pre_tags: torch.Tensor
    comb: torch.Tensor
    out: torch.Tensor
    recv_expert_offsets: torch.Tensor
    grad_probs: torch.Tensor
    grad_logits: torch.Tensor


def _stream_ptr(stream) -> int:
    if stream is None:
        return torch.cuda.current_stream().cuda_stream
    return stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream)


class MoeLayer:
    def __init__(self, e: int, t: int, num_experts: int, top_k: int, tokens: int, hidden: int,
                 dtype: torch.dtype = torch.bfloat16, logit_dtype: torch.dtype = torch.float32,
                 out_dtype: torch.dtype | None = None, max_chunks: int = 64, device: int = 0,
                 rank: int = 0, world_size: int = 1):
        self.lib = _lib.load()
        self.e, self.t, self.E, self.k = e, t, num_experts, top_k
        self.T, self.h = tokens, hidden
        self.dtype, self.logit_dtype = dtype, logit_dtype
        self.out_dtype = out_dtype or dtype
        self.max_chunks = max_chunks
        self.device, self.rank, self.world_size = device, rank, world_size
        self.L = num_experts // e if e else 0
        desc = _lib.LayerDesc(e, t, num_experts, top_k, tokens, hidden, _lib.dtype_code(dtype),
                              _lib.dtype_code(logit_dtype), _lib.dtype_code(self.out_dtype), max_chunks)
        self._ctx = C.c_void_p()
        check(self.lib.moe_ctx_create(C.byref(desc), device, rank, world_size, C.byref(self._ctx)))
        n_local = self.lib.moe_ctx_num_local_cards(self._ctx)
        first = self.lib.moe_ctx_first_card(self._ctx)
        self.local_cards = list(range(first, first + n_local))
        self._cards = {c: self._make_card(c) for c in self.local_cards}
        self._experts: dict = {}

    # ------------------------------------------------------------------ views
    def _make_card(self, card: int) -> CardTensors:
        v = _lib.CardView()
        check(self.lib.moe_ctx_card_view(self._ctx, card, C.byref(v)))
        T, h, E, k, dev = self.T, self.h, self.E, self.k, self.device
        R, cap = v.rows_permuted, v.recv_cap
        i32 = torch.int32
        mk = lambda p, shape, dt: device_view(p, shape, dt, dev)  # noqa: E731
        return CardTensors(
            card=card, node=card // self.t, rho=card % self.t,
            x=mk(v.x, (T, h), self.dtype), logits=mk(v.logits, (T, E), self.logit_dtype),
            token_ids=mk(v.token_ids, (T,), i32), experts=mk(v.experts, (T, k), i32),
            probs=mk(v.probs, (T, k), self.logit_dtype), perm_src=mk(v.perm_src, (R,), i32),
            expert_of=mk(v.expert_of, (R,), i32), slot_pos=mk(v.slot_pos, (T, k), i32),
            counts=mk(v.counts, (self.max_chunks, E), i32), expert_offsets=mk(v.expert_offsets, (E + 1,), i32),
            permuted=mk(v.permuted, (R, h), self.dtype), recv=mk(v.recv, (cap, h), self.dtype),
            recv_tags=mk(v.recv_tags, (cap, 4), i32), pre=mk(v.pre, (cap, h), self.dtype),
            pre_tags=mk(v.pre_tags, (cap, 4), i32), comb=mk(v.comb, (R, h), self.dtype),
            out=mk(v.out, (T, h), self.out_dtype),
            recv_expert_offsets=mk(v.recv_expert_offsets, (self.L + 1,), i32),
            grad_probs=mk(v.grad_probs, (T, k), self.logit_dtype),
            grad_logits=mk(v.grad_logits, (T, E), self.logit_dtype))

    def card(self, c: int) -> CardTensors:
        return self._cards[c]

    @property
    def cards(self) -> list[CardTensors]:
        return [self._cards[c] for c in self.local_cards]

    # ------------------------------------------------------------ multi-GPU
    def connect(self, group=None) -> None:
        """Exchange IPC handles with every rank (torch.distributed must be up)."""
        if self.world_size == 1:
            return
        import torch.distributed as dist
        size = self.lib.moe_ctx_ipc_handle_size()
        blob = (C.c_char * size)()
        check(self.lib.moe_ctx_ipc_export(self._ctx, blob))
        mine = bytes(blob)
        allb: list = [None] * self.world_size
        dist.all_gather_object(allb, mine, group=group)
        joined = b"".join(allb)
        buf = (C.c_char * len(joined)).from_buffer_copy(joined)
        check(self.lib.moe_ctx_ipc_connect(self._ctx, buf))

    # ------------------------------------------------------------------ ops
    def route(self, stream=None) -> None:
        check(self.lib.moe_ctx_route(self._ctx, _stream_ptr(stream)))

    def permute(self, n: int = 1, stream=None) -> None:
        check(self.lib.moe_ctx_permute(self._ctx, n, _stream_ptr(stream)))

    def dispatch(self, level: int = O1, n: int = 1, landing: int = LAND_FINAL, stream=None) -> None:
        check(self.lib.moe_ctx_dispatch(self._ctx, level, n, landing, _stream_ptr(stream)))

    def combine(self, level: int = O1, n: int = 1, stream=None) -> None:
        check(self.lib.moe_ctx_combine(self._ctx, level, n, _stream_ptr(stream)))

    def forward(self, level: int = O1, n: int = 1, landing: int = LAND_FINAL, stream=None) -> None:
        check(self.lib.moe_ctx_forward(self._ctx, level, n, landing, _stream_ptr(stream)))

    def forward_host(self, host_x: torch.Tensor, host_logits: torch.Tensor, host_out: torch.Tensor,
                     level: int = O1, n: int = 1, landing: int = LAND_FINAL, stream=None) -> None:
        """End to end from host buffers (pinned for async copies)."""
        check(self.lib.moe_ctx_forward_host(self._ctx, level, n, landing, host_x.data_ptr(),
                                            host_logits.data_ptr(), host_out.data_ptr(), _stream_ptr(stream)))

    def bind_experts(self, card: int, w13: torch.Tensor | None, w2: torch.Tensor | None = None) -> None:
        """SwiGLU experts of this card's L local experts (w13 from ops.interleave_w13,
        [L, 2F, h]; w2 [L, h, F]); they run between dispatch and combine.  None unbinds."""
        if w13 is None:
            check(self.lib.moe_ctx_bind_experts(self._ctx, card, None, None, 0))
            self._experts.pop(card, None)
            return
        self._experts[card] = (w13, w2)  # keep the weights alive while bound
        check(self.lib.moe_ctx_bind_experts(self._ctx, card, w13.data_ptr(), w2.data_ptr(), w13.shape[1] // 2))

    def autotune(self, candidates, steps: int = 5, stream=None):
        """moe_ctx_autotune: time each (level, n, landing) in place (max over ranks);
        returns (index of the fastest, [us/layer per candidate])."""
        arr = (_lib.Schedule * len(candidates))(*[_lib.Schedule(int(lv), int(n), int(ld), 0.0)
                                                   for lv, n, ld in candidates])
        best = C.c_int32()
        check(self.lib.moe_ctx_autotune(self._ctx, arr, len(candidates), steps, _stream_ptr(stream), C.byref(best)))
        return int(best.value), [arr[i].us for i in range(len(candidates))]

    # ------------------------------------------------------------ backward
    def backward_combine(self, level: int = O1, n: int = 1, stream=None) -> None:
        """d loss/d out read from each card's x; leaves d loss/d expert-output in
        each card's pre rows and grad_probs / grad_logits in the card views."""
        check(self.lib.moe_ctx_backward_combine(self._ctx, level, n, _stream_ptr(stream)))

    def backward_dispatch(self, level: int = O1, n: int = 1, stream=None) -> None:
        """d loss/d x into each card's out, from the gradient rows in pre."""
        check(self.lib.moe_ctx_backward_dispatch(self._ctx, level, n, _stream_ptr(stream)))

    def backward(self, level: int = O1, n: int = 1, stream=None) -> None:
        check(self.lib.moe_ctx_backward(self._ctx, level, n, _stream_ptr(stream)))

    def set_link_rate(self, gbps: float) -> None:
        """Emulated inter-node link for the cross-node legs (GB/s per card; 0: off)."""
        check(self.lib.moe_ctx_set_link_rate(self._ctx, float(gbps)))

    def set_wire(self, wire: int) -> None:
        """Cross-node dispatch payload format: _lib.WIRE_BF16 (exact) or _lib.WIRE_FP8."""
        check(self.lib.moe_ctx_set_wire(self._ctx, wire))

    def enable_checks(self, enable: bool = True) -> None:
        """Poison + verify the landed rows' tags every dispatch (CorruptRoutingError on failure)."""
        check(self.lib.moe_ctx_enable_checks(self._ctx, int(enable)))

    def verify(self, stream=None) -> None:
        check(self.lib.moe_ctx_verify(self._ctx, _stream_ptr(stream)))

    def experts(self, stream=None) -> None:
        check(self.lib.moe_ctx_experts(self._ctx, _stream_ptr(stream)))

    def set_node_dedup(self, mode: int) -> None:
        """Cross-node rows once per (token, remote node), fanned out there: 0 off, 1 on, 2 auto (k >= 2e)."""
        check(self.lib.moe_ctx_set_node_dedup(self._ctx, int(mode)))

    def set_expert_overlap(self, enable: bool) -> None:
        """Fuse the reverse AllToAll into the experts' down-projection epilogue (multi-GPU forward)."""
        check(self.lib.moe_ctx_set_expert_overlap(self._ctx, int(bool(enable))))

    def bind_expert_out(self, card: int, tensor: torch.Tensor | None) -> None:
        check(self.lib.moe_ctx_bind_expert_out(self._ctx, card, tensor.data_ptr() if tensor is not None else None))

    def recv_rows(self, card: int) -> int:
        r = C.c_int64()
        check(self.lib.moe_ctx_recv_rows(self._ctx, card, C.byref(r)))
        return int(r.value)

    def sync(self) -> None:
        check(self.lib.moe_ctx_sync(self._ctx))

    def enable_timing(self, on: bool = True) -> None:
        check(self.lib.moe_ctx_enable_timing(self._ctx, int(on)))

    def enable_graphs(self, on: bool = True) -> None:
        """Replay forward()/forward_host() as captured CUDA graphs."""
        check(self.lib.moe_ctx_enable_graphs(self._ctx, int(on)))

    def set_persistent(self, on: bool = True) -> None:
        """Multi-GPU: one persistent exchange kernel per phase (default) vs per-chunk launches."""
        check(self.lib.moe_ctx_set_persistent(self._ctx, int(on)))

    ROLES = (("aa", "aal", "ag", "d2d"), ("caa", "unpermute", "", ""))

    def xchg_trace(self) -> list[tuple[str, int, float, float]]:
        """Role spans of the last persistent dispatch/combine: (role, chunk, start_us, end_us),
        relative to the earliest start (timing must be enabled)."""
        mc = self.max_chunks
        cap = 2 * 4 * mc * 2
        arr = (C.c_uint64 * cap)()
        got = C.c_int32()
        check(self.lib.moe_ctx_xchg_trace(self._ctx, self.local_cards[0], arr, cap, C.byref(got)))
        out = []
        for kern in range(2):
            for role in range(4):
                for j in range(mc):
                    base = ((kern * 4 + role) * mc + j) * 2
                    a, b = arr[base], arr[base + 1]
                    if a == 0xFFFFFFFFFFFFFFFF or b == 0xFFFFFFFFFFFFFFFF or not self.ROLES[kern][role]:
                        continue
                    out.append((self.ROLES[kern][role], j, a, b))
        if not out:
            return []
        t0 = min(a for _, _, a, _ in out)
        return [(r, j, (a - t0) / 1e3, (b - t0) / 1e3) for r, j, a, b in out]

    def spans(self) -> list[tuple[str, int, float, float]]:
        cap = 4096
        arr = (_lib.Span * cap)()
        n = C.c_int32()
        check(self.lib.moe_ctx_spans(self._ctx, arr, cap, C.byref(n)))
        return [(_lib.STAGES[arr[i].stage], arr[i].chunk, arr[i].start_ms, arr[i].end_ms) for i in range(n.value)]

    def set_aa_ctas(self, ctas: int) -> None:
        check(self.lib.moe_ctx_set_aa_ctas(self._ctx, ctas))

    def xfer(self, rows_per_card, row_bytes: int, grid: int = 0, stream=None) -> None:
        """Transport primitive: rows_per_card[c] rows of `row_bytes` stored to card c."""
        arr = (C.c_int64 * len(rows_per_card))(*[int(r) for r in rows_per_card])
        check(self.lib.moe_ctx_xfer(self._ctx, arr, int(row_bytes), int(grid), _stream_ptr(stream)))

    @property
    def launch_count(self) -> int:
        return int(self.lib.moe_ctx_launch_count(self._ctx))

    def close(self) -> None:
        if getattr(self, "_ctx", None) and self._ctx.value:
            self._cards = {}
            self.lib.moe_ctx_destroy(self._ctx)
            self._ctx = C.c_void_p()

    def __del__(self):  # pragma: no cover
        try:
            self.close()
        except Exception:
            pass


__all__ = ["MoeLayer", "CardTensors", "device_view", "BASELINE", "O1", "O2", "O3", "LAND_FINAL", "LAND_STAGED"]

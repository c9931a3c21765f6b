"""Differentiable lone-card MoE data path over the library's kernels.

    experts, probs = route(logits, k)                 route_topk          (dataplane.hpp:72-106)
    index          = ops.build_index(experts, E)      permute, index form (dataplane.hpp:118-140)
    rows           = dispatch(x, index)               expert-major gather
    y              = <the caller's experts on rows>   (expert_of / expert_offsets give the segments)
    out            = combine(y, probs, index)         weighted un-permute (dataplane.hpp:325-342)

Forward and backward both run on libmonta.so (ops.*_backward, include/monta.h
section 1b); torch.autograd only sequences them.  The selection (experts,
index) is piecewise constant and carries no gradient.  The reference has no
backward: this is SURVEY.md §8(f) item 2, built on the same index the forward
uses.
"""
from __future__ import annotations

import torch

from . import ops


class _Route(torch.autograd.Function):
    @staticmethod
    def forward(ctx, logits, k):
        experts, probs = ops.route_topk(logits.detach(), k)
        ctx.save_for_backward(logits, experts)
        ctx.mark_non_differentiable(experts)
        return experts, probs

    @staticmethod
    def backward(ctx, _g_experts, g_probs):
        logits, experts = ctx.saved_tensors
        return ops.route_backward(logits, experts, g_probs), None


class _Dispatch(torch.autograd.Function):
    @staticmethod
    def forward(ctx, x, perm_src, slot_pos):
        ctx.save_for_backward(slot_pos)
        ctx.x_dtype = x.dtype
        return ops.permute_rows(x.detach(), perm_src)

    @staticmethod
    def backward(ctx, g_rows):
        (slot_pos,) = ctx.saved_tensors
        return ops.dispatch_backward(g_rows, slot_pos, out_dtype=ctx.x_dtype), None, None


class _Combine(torch.autograd.Function):
    @staticmethod
    def forward(ctx, y, probs, slot_pos, out_dtype):
        ctx.save_for_backward(y, probs, slot_pos)
        return ops.unpermute_combine(y.detach(), slot_pos, probs.detach(), out_dtype=out_dtype)

    @staticmethod
    def backward(ctx, g_out):
        y, probs, slot_pos = ctx.saved_tensors
        need_y, need_p = ctx.needs_input_grad[0], ctx.needs_input_grad[1]
        if not (need_y or need_p):
            return None, None, None, None
        g_y, g_p = ops.combine_backward(g_out, y, slot_pos, probs, need_grad_y=need_y, need_grad_probs=need_p)
        return g_y, g_p, None, None


def route(logits: torch.Tensor, k: int):
    """(experts int32 [T, k] ascending, probs [T, k]); probs differentiable in logits."""
    return _Route.apply(logits, k)


def dispatch(x: torch.Tensor, index: ops.Index) -> torch.Tensor:
    """Expert-major rows [T*k, h]: rows[r] = x[index.perm_src[r]]."""
    return _Dispatch.apply(x, index.perm_src, index.slot_pos)


def combine(y: torch.Tensor, probs: torch.Tensor, index: ops.Index, out_dtype: torch.dtype | None = None):
    """out[i] = sum_s probs[i, s] * y[index.slot_pos[i, s]]."""
    return _Combine.apply(y, probs, index.slot_pos, out_dtype)


def moe_local(x: torch.Tensor, logits: torch.Tensor, k: int, num_experts: int, expert_fn):
    """One lone-card MoE layer: route, dispatch, expert_fn(rows, index) -> y,
    combine.  Differentiable in x, logits and whatever expert_fn closes over."""
    experts, probs = route(logits, k)
    index = ops.build_index(experts, num_experts)
    rows = dispatch(x, index)
    y = expert_fn(rows, index)
    return combine(y, probs, index, out_dtype=x.dtype)

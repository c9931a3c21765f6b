"""Backward of the multi-card layer composed from
the forward exchanges of the layer context and the per-card adjoint kernels.

The reference has no backward.  With the forward's routing still in the
context (cd.experts / cd.probs / cd.slot_pos untouched):

  combine backward   grad_out (replicated over a node's TP cards, like x)
                     travels to the expert cards through the forward dispatch
                     (same level, chunk count and landing, so the rows land
                     exactly where the forward's did); on every expert card
                     moe_combine_backward gives grad_y[r] = p_r * g[r] over
                     full rows and the partial <g[r], y[r]> over the card's
                     own 1/t column slice; the partials of the t cards of a
                     node sum to the full dot and are returned to the source
                     token's (position, slot) through the row tags
                     {token_id, source_card, source_position, expert}.
  dispatch backward  grad_x[i] = sum_s grad_rows[r(i,s)] is the forward
                     combine with unit weights: the gradient rows are bound
                     as the expert output and the combine exchange (reverse
                     AllToAll + un-permute + output AllGather) runs as is.

Expert outputs are taken to be consistent across the t cards of a node (each
card's combine leg reads its own column slice of them), which is what the
forward combine assumes.  Only the per-row metadata (probabilities, slots,
partial dots: a few bytes per routed pair) moves through torch.distributed
collectives on the device; every row of payload moves through the library's
kernels.
"""
from __future__ import annotations

import ctypes as C

import torch

from . import _lib
from ._lib import check
from .layer import LAND_FINAL, MoeLayer


def _stream() -> int:
    return torch.cuda.current_stream().cuda_stream


def _source_routing(layer: MoeLayer):
    """experts/probs of every card, indexed by card id: [cards, T, k]."""
    if layer.world_size == 1:
        ex = torch.stack([layer.card(c).experts for c in range(layer.e * layer.t)])
        pr = torch.stack([layer.card(c).probs for c in range(layer.e * layer.t)])
        return ex, pr
    import torch.distributed as dist
    cd = layer.cards[0]
    ex = [torch.empty_like(cd.experts) for _ in range(layer.world_size)]
    pr = [torch.empty_like(cd.probs) for _ in range(layer.world_size)]
    dist.all_gather(ex, cd.experts.contiguous())
    dist.all_gather(pr, cd.probs.contiguous())
    return torch.stack(ex), torch.stack(pr)


def combine_backward(layer: MoeLayer, grad_out: dict, expert_out: dict, level: int, n: int = 1,
                     landing: int = LAND_FINAL):
    """grad_out: {card: [T, h]} (equal on a node's TP cards); expert_out:
    {card: [>= rows, h]} the forward's expert outputs.  Returns
    (grad_expert_out {card: [rows, h] in the payload dtype},
     grad_probs {card: [T, k] in the logit dtype}).  Overwrites cd.x and
    cd.recv (the dispatch carries the gradient rows)."""
    t, h = layer.t, layer.h
    for cd in layer.cards:
        cd.x.copy_(grad_out[cd.card])
    layer.dispatch(level, n, landing)
    layer.sync()
    ex_all, pr_all = _source_routing(layer)
    lib = _lib.load()
    pdt = _lib.dtype_code(layer.logit_dtype)
    ydt = _lib.dtype_code(layer.dtype)
    es = torch.empty((), dtype=layer.dtype).element_size()
    grad_y, parts = {}, []
    for cd in layer.cards:
        rows = layer.recv_rows(cd.card)
        tags = cd.recv_tags[:rows].long()
        src, pos, xe = tags[:, 1], tags[:, 2], tags[:, 3]
        slot = (ex_all[src, pos] == xe[:, None]).int().argmax(dim=1)
        p_r = pr_all[src, pos, slot].contiguous()
        ident = torch.arange(rows, dtype=torch.int32, device=p_r.device)
        g = cd.recv[:rows]
        y = expert_out[cd.card][:rows].contiguous()
        gy = torch.empty((rows, h), dtype=layer.dtype, device=g.device)
        dot = torch.empty((rows,), dtype=layer.logit_dtype, device=g.device)
        if rows:
            # grad_y over full rows; the partial dot over this card's column slice
            check(lib.moe_combine_backward(g.data_ptr(), ydt, h, None, ydt, h, h, ident.data_ptr(), p_r.data_ptr(),
                                           pdt, rows, 1, gy.data_ptr(), h, None, C.c_void_p(_stream())))
            w = h // t
            off = cd.rho * w * es
            check(lib.moe_combine_backward(g.data_ptr() + off, ydt, h, y.data_ptr() + off, ydt, h, w,
                                           ident.data_ptr(), p_r.data_ptr(), pdt, rows, 1, None, h,
                                           dot.data_ptr(), C.c_void_p(_stream())))
        grad_y[cd.card] = gy
        parts.append(torch.stack([src.to(dot.dtype), pos.to(dot.dtype), slot.to(dot.dtype), dot], dim=1))
    part = torch.cat(parts) if parts else torch.empty((0, 4), dtype=layer.logit_dtype)
    if layer.world_size > 1:
        # device-side all-gather of the (source, position, slot, partial) rows,
        # padded to the largest card's row count (padding rows carry 0)
        import torch.distributed as dist
        part = part.to(ex_all.device)
        cnt = torch.tensor([part.shape[0]], dtype=torch.int64, device=part.device)
        cnts = [torch.empty_like(cnt) for _ in range(layer.world_size)]
        dist.all_gather(cnts, cnt)
        cnts = [int(v.item()) for v in cnts]
        pad = torch.zeros((max(cnts), 4), dtype=part.dtype, device=part.device)
        pad[:part.shape[0]] = part
        allp = [torch.empty_like(pad) for _ in range(layer.world_size)]
        dist.all_gather(allp, pad)
        part = torch.cat([a[:c] for a, c in zip(allp, cnts)])
    n_src = layer.e * layer.t
    gp_all = torch.zeros((n_src, layer.T, layer.k), dtype=layer.logit_dtype, device=ex_all.device)
    s_, p_, l_ = part[:, 0].long(), part[:, 1].long(), part[:, 2].long()
    gp_all.index_put_((s_, p_, l_), part[:, 3], accumulate=True)
    # rows are tagged with the node's canonical source card (node * t); every
    # TP card of the node shares that routing, hence that gradient
    grad_probs = {cd.card: gp_all[cd.node * t].clone() for cd in layer.cards}
    return grad_y, grad_probs


def dispatch_backward(layer: MoeLayer, grad_rows: dict, level: int, n: int = 1):
    """grad_rows: {card: [>= rows, h]} gradient of the dispatched rows
    (consistent over a node's TP cards), in the layout of the last dispatch
    with this level and n.  The combine exchange mirrors the last dispatch,
    so this follows combine_backward (backprop order: combine, then
    dispatch).  Returns {card: grad_x [T, h]} in the layer's output dtype.  The forward combine with unit weights; cd.probs and the
    expert-output binding are restored afterwards."""
    saved = {cd.card: cd.probs.clone() for cd in layer.cards}
    try:
        for cd in layer.cards:
            cd.probs.fill_(1.0)
            layer.bind_expert_out(cd.card, grad_rows[cd.card])
        layer.combine(level, n)
        layer.sync()
        return {cd.card: cd.out.clone() for cd in layer.cards}
    finally:
        for cd in layer.cards:
            cd.probs.copy_(saved[cd.card])
            layer.bind_expert_out(cd.card, None)

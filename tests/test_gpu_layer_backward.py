"""Multi-card layer backward (paper_2411_00662_b200/layer_backward.py) in the
virtual topology (all e x t cards on cuda:0, the reference's single-process
emulation), against closed forms in fp64.

Experts are per-expert scalings y = c_x * row (consistent across a node's TP
cards, as the forward combine assumes), so with g the output gradient of a
source node:
  grad_probs[i, s]   = c_{x_s} <g_i, x_i>
  grad_y[r]          = p_r g_{tok(r)}
  grad_x[i] (rows'   = sum_s d_{x_s} g_i       for grad_rows[r] = d_x * g_{tok(r)}
             grads)
"""
import pytest
import torch

from paper_2411_00662_b200 import layer_backward as LB
from paper_2411_00662_b200.layer import BASELINE, LAND_FINAL, LAND_STAGED, MoeLayer, O1, O2, O3

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("e,t,E,k,level,n,landing", [
    (2, 2, 8, 2, O1, 1, LAND_FINAL), (2, 2, 8, 2, O2, 2, LAND_FINAL), (2, 2, 8, 2, O3, 2, LAND_STAGED),
    (2, 2, 8, 2, BASELINE, 1, LAND_FINAL), (2, 1, 8, 2, BASELINE, 1, LAND_FINAL), (1, 2, 4, 2, BASELINE, 1, LAND_FINAL),
    (4, 2, 16, 6, O2, 2, LAND_FINAL), (2, 4, 2, 1, O1, 1, LAND_FINAL)])
def test_layer_backward_closed_form(cuda, e, t, E, k, level, n, landing):
    T, h = 128, 256
    dt = torch.bfloat16
    gen = torch.Generator().manual_seed(e * 10 + t + level)
    x = torch.randn(e, T, h, generator=gen).to(dt)
    logits = torch.randn(e, T, E, generator=gen)
    gout = torch.randn(e, T, h, generator=gen).to(dt)
    c = torch.linspace(0.5, 2.0, E, dtype=torch.float64)
    d = torch.linspace(-1.0, 1.0, E, dtype=torch.float64)
    layer = MoeLayer(e, t, E, k, T, h, dtype=dt, logit_dtype=torch.float32, max_chunks=max(n, 1), device=0)
    try:
        for cd in layer.cards:
            cd.x.copy_(x[cd.node])
            cd.logits.copy_(logits[cd.node])
        layer.route()
        layer.dispatch(level, n, landing)
        layer.sync()
        y = {}
        for cd in layer.cards:
            rows = layer.recv_rows(cd.card)
            xe = cd.recv_tags[:rows, 3].long().cpu()
            y[cd.card] = (cd.recv[:rows].double().cpu() * c[xe][:, None]).to(dt).to(cuda)
        experts = {cd.node: cd.experts.long().cpu() for cd in layer.cards}
        probs = {cd.node: cd.probs.double().cpu() for cd in layer.cards}

        grad_y, grad_p = LB.combine_backward(layer, {cd.card: gout[cd.node] for cd in layer.cards}, y, level, n,
                                             landing)
        torch.cuda.synchronize()
        for cd in layer.cards:
            g, xx = gout[cd.node].double(), x[cd.node].double()
            # y rows are bf16-rounded c_x * x: compare against the dot with the rows actually used
            ex = experts[cd.node]
            yx = (xx[:, None, :] * c[ex][:, :, None]).to(dt).double()          # [T, k, h]
            want = (g[:, None, :] * yx).sum(-1)
            mag = (g[:, None, :] * yx).abs().sum(-1)
            err = ((grad_p[cd.card].double().cpu() - want).abs() / mag).max().item()
            assert err < 1e-5, (cd.card, err)
            rows = layer.recv_rows(cd.card)
            tags = cd.recv_tags[:rows].long().cpu()
            src_node, pos, xe = tags[:, 1] // t, tags[:, 2], tags[:, 3]
            ex_all = torch.stack([experts[g_] for g_ in range(e)])
            pr_all = torch.stack([probs[g_] for g_ in range(e)])
            slot = (ex_all[src_node, pos] == xe[:, None]).int().argmax(dim=1)
            p_r = pr_all[src_node, pos, slot]
            want_gy = (p_r[:, None].float() * gout[src_node, pos].float()).to(dt) if rows else None
            if rows:
                assert torch.equal(grad_y[cd.card].cpu(), want_gy), cd.card

        # dispatch backward: rows' gradients d_x * g_tok (cd.recv holds the dispatched g rows now)
        grad_rows = {}
        for cd in layer.cards:
            rows = layer.recv_rows(cd.card)
            xe = cd.recv_tags[:rows, 3].long().cpu()
            grad_rows[cd.card] = (cd.recv[:rows].double().cpu() * d[xe][:, None]).to(dt).to(cuda)
        gx = LB.dispatch_backward(layer, grad_rows, level, n)
        torch.cuda.synchronize()
        for cd in layer.cards:
            ex = experts[cd.node]
            rows_used = (gout[cd.node].double()[:, None, :] * d[ex][:, :, None]).to(dt).double()
            want = rows_used.sum(1)
            err = ((gx[cd.card].double().cpu() - want).abs().max() / want.abs().max()).item()
            assert err < 1e-2, (cd.card, err)
        # the forward state is restored: probs unchanged, expert_out back on recv
        for cd in layer.cards:
            assert torch.equal(cd.probs.double().cpu(), probs[cd.node])
    finally:
        layer.close()


@pytest.mark.parametrize("e,t,E,k,level,n", [
    (2, 2, 8, 2, O1, 1), (2, 2, 8, 2, O2, 2), (2, 2, 8, 2, BASELINE, 1), (2, 1, 8, 2, BASELINE, 1),
    (1, 2, 4, 2, O1, 1), (4, 2, 16, 6, O2, 2), (2, 4, 2, 1, O1, 1), (1, 1, 160, 6, BASELINE, 1)])
def test_ctx_backward_device_side(cuda, e, t, E, k, level, n):
    """moe_ctx_backward_combine / _dispatch (the whole layer backward inside the
    context, no host round trip) against the closed forms of the composed test
    above: grad_y bit-exact, grad_probs 1e-5 of fp64, grad_logits 1e-4, grad_x 1e-2."""
    T, h = 128, 256
    dt = torch.bfloat16
    gen = torch.Generator().manual_seed(e * 10 + t + level + 7)
    x = torch.randn(e, T, h, generator=gen).to(dt)
    logits = torch.randn(e, T, E, generator=gen)
    gout = torch.randn(e, T, h, generator=gen).to(dt)
    c = torch.linspace(0.5, 2.0, E, dtype=torch.float64)
    d = torch.linspace(-1.0, 1.0, E, dtype=torch.float64)
    layer = MoeLayer(e, t, E, k, T, h, dtype=dt, logit_dtype=torch.float32, max_chunks=max(n, 1), device=0)
    try:
        for cd in layer.cards:
            cd.x.copy_(x[cd.node])
            cd.logits.copy_(logits[cd.node])
        layer.route()
        layer.dispatch(level, n)
        layer.sync()
        for cd in layer.cards:  # experts in place: y = c_x * row (bf16)
            rows = layer.recv_rows(cd.card)
            xe = cd.recv_tags[:rows, 3].long()
            cd.recv[:rows].copy_((cd.recv[:rows].double() * c.to(cuda)[xe][:, None]).to(dt))
        layer.combine(level, n)
        layer.sync()
        experts = {cd.node: cd.experts.long().cpu() for cd in layer.cards}
        probs = {cd.node: cd.probs.double().cpu() for cd in layer.cards}
        for cd in layer.cards:
            cd.x.copy_(gout[cd.node])
        layer.backward_combine(level, n)
        layer.sync()
        ex_all = torch.stack([experts[g_] for g_ in range(e)])
        pr_all = torch.stack([probs[g_] for g_ in range(e)])
        for cd in layer.cards:
            g, xx = gout[cd.node].double(), x[cd.node].double()
            ex = experts[cd.node]
            yx = (xx[:, None, :] * c[ex][:, :, None]).to(dt).double()
            want = (g[:, None, :] * yx).sum(-1)
            mag = (g[:, None, :] * yx).abs().sum(-1)
            gp = cd.grad_probs.double().cpu()
            assert ((gp - want).abs() / mag).max().item() < 1e-5, cd.card
            P = torch.softmax(logits[cd.node].double(), -1)
            G = torch.zeros(T, E, dtype=torch.float64)
            G.scatter_(1, ex, want)
            want_z = P * (G - (G * P).sum(-1, keepdim=True))
            assert torch.allclose(cd.grad_logits.double().cpu(), want_z, rtol=1e-4, atol=1e-5), cd.card
            rows = layer.recv_rows(cd.card)
            if rows:
                tags = cd.recv_tags[:rows].long().cpu()
                src_node, pos, xe = tags[:, 1] // t, tags[:, 2], tags[:, 3]
                slot = (ex_all[src_node, pos] == xe[:, None]).int().argmax(dim=1)
                p_r = pr_all[src_node, pos, slot]
                want_gy = (p_r[:, None].float() * gout[src_node, pos].float()).to(dt)
                assert torch.equal(cd.pre[:rows].cpu(), want_gy), cd.card
                # the caller's expert backward: d loss / d expert input = d_x * g_tok (replaces grad_y)
                cd.pre[:rows].copy_((gout[src_node, pos].double() * d[xe][:, None]).to(dt).to(cuda))
        layer.backward_dispatch(level, n)
        layer.sync()
        for cd in layer.cards:
            ex = experts[cd.node]
            want = (gout[cd.node].double()[:, None, :] * d[ex][:, :, None]).to(dt).double().sum(1)
            err = ((cd.out.double().cpu() - want).abs().max() / want.abs().max()).item()
            assert err < 1e-2, (cd.card, err)
        # identity experts end to end: grad_x = g * sum(p)
        for cd in layer.cards:
            cd.x.copy_(x[cd.node])
        layer.forward(level, n)
        layer.sync()
        for cd in layer.cards:
            cd.x.copy_(gout[cd.node])
        layer.backward(level, n)
        layer.sync()
        for cd in layer.cards:
            want = gout[cd.node].double() * probs[cd.node].sum(1, keepdim=True)
            err = ((cd.out.double().cpu() - want).abs().max() / want.abs().max()).item()
            assert err < 1e-2, (cd.card, err)
    finally:
        layer.close()


@pytest.mark.parametrize("e,t,E,k,level,n", [(2, 2, 8, 2, O1, 1), (2, 2, 8, 2, O2, 2), (1, 1, 160, 6, BASELINE, 1)])
def test_ctx_backward_graph_replay(cuda, e, t, E, k, level, n):
    """moe_ctx_backward captured once and replayed as a CUDA graph gives the
    eager result bit for bit (device-resident epochs keep replays in step)."""
    T, h = 128, 256
    dt = torch.bfloat16
    gen = torch.Generator().manual_seed(e + t + E + n)
    x = torch.randn(e, T, h, generator=gen).to(dt)
    logits = torch.randn(e, T, E, generator=gen)
    gout = torch.randn(e, T, h, generator=gen).to(dt)
    outs = []
    for graphs in (False, True):
        layer = MoeLayer(e, t, E, k, T, h, dtype=dt, logit_dtype=torch.float32, max_chunks=max(n, 1), device=0)
        try:
            layer.enable_graphs(graphs)
            res = None
            for _ in range(3):  # graphs: capture, then replays
                for cd in layer.cards:
                    cd.x.copy_(x[cd.node])
                    cd.logits.copy_(logits[cd.node])
                layer.forward(level, n)
                for cd in layer.cards:
                    cd.x.copy_(gout[cd.node])
                layer.backward(level, n)
                layer.sync()
                res = [(cd.out.clone(), cd.grad_probs.clone(), cd.grad_logits.clone()) for cd in layer.cards]
            outs.append(res)
        finally:
            layer.close()
    for (a0, b0, c0), (a1, b1, c1) in zip(*outs):
        assert torch.equal(a0, a1) and torch.equal(b0, b1) and torch.equal(c0, c1)

"""GPU checks of the backward kernels (include/monta.h section 1b, SURVEY.md
§8(f) item 2) against plain PyTorch fp64/fp32 references of the same ops.

The reference has no backward, so there is no oracle row for it; the bar is
the forward's: index-exact placement, bit-exact where the arithmetic is a
single rounding (grad_y = p * g) or a sequential fp32 sum (grad_x), and
relative 1e-5 (fp32 arithmetic) for the dot products and the softmax
adjoint, measured against fp64.
"""
import pytest
import torch

from paper_2411_00662_b200 import _lib
from paper_2411_00662_b200 import autograd as mag
from paper_2411_00662_b200 import ops

pytestmark = pytest.mark.gpu


def _index(T, E, k, seed, dev, logit_dtype=torch.float32):
    g = torch.Generator(device="cpu").manual_seed(seed)
    logits = torch.randn(T, E, generator=g, dtype=torch.float64).to(logit_dtype).to(dev)
    experts, probs = ops.route_topk(logits, k)
    return logits, experts, probs, ops.build_index(experts, E)


def _rand(shape, dtype, seed, dev):
    g = torch.Generator(device="cpu").manual_seed(seed)
    return torch.randn(*shape, generator=g, dtype=torch.float64).to(dtype).to(dev)


@pytest.mark.parametrize("T,h,E,k", [(300, 1000, 8, 2), (257, 1001, 8, 2), (1000, 256, 160, 6), (64, 40, 2, 1),
                                     (33, 8, 4, 4), (5, 4104, 80, 32), (2, 9000, 8, 3)])
@pytest.mark.parametrize("ydt,gdt,pdt", [(torch.float32, torch.float32, torch.float32),
                                         (torch.bfloat16, torch.bfloat16, torch.float32),
                                         (torch.bfloat16, torch.float32, torch.float32),
                                         (torch.float16, torch.float16, torch.float32),
                                         (torch.float64, torch.float64, torch.float64)])
def test_combine_backward(cuda, T, h, E, k, ydt, gdt, pdt):
    _, _, probs, idx = _index(T, E, k, seed=T + h, dev=cuda, logit_dtype=pdt)
    R = T * k
    y = _rand((R, h), ydt, 1, cuda)
    g = _rand((T, h), gdt, 2, cuda)
    gy, gp = ops.combine_backward(g, y, idx.slot_pos, probs)
    torch.cuda.synchronize()
    # grad_y: one multiply in the accumulation precision, one rounding to y's dtype.
    acc = torch.float64 if torch.float64 in (ydt, gdt, pdt) else torch.float32
    want = torch.empty((R, h), dtype=ydt, device=cuda)
    for s in range(k):
        want[idx.slot_pos[:, s].long()] = (probs[:, s:s + 1].to(acc) * g.to(acc)).to(ydt)
    assert torch.equal(gy, want)
    # grad_probs against fp64 dot products, relative to sum |g y|.
    yr = y.double()[idx.slot_pos.long()]                      # [T, k, h]
    ref = (g.double()[:, None, :] * yr).sum(-1)
    mag_ = (g.double()[:, None, :] * yr).abs().sum(-1) + 1e-30
    tol = 1e-12 if acc is torch.float64 else 1e-5
    assert ((gp.double() - ref).abs() / mag_).max().item() < tol


@pytest.mark.parametrize("T,h,E,k", [(300, 1000, 8, 2), (257, 1001, 8, 2), (1000, 256, 160, 6), (100, 64, 64, 32), (3, 4104, 80, 31)])
@pytest.mark.parametrize("idt,odt", [(torch.float32, torch.float32), (torch.bfloat16, torch.bfloat16),
                                     (torch.bfloat16, torch.float32), (torch.float64, torch.float64)])
def test_dispatch_backward_is_sequential_sum(cuda, T, h, E, k, idt, odt):
    _, _, _, idx = _index(T, E, k, seed=7 * T + h, dev=cuda)
    rows = _rand((T * k, h), idt, 3, cuda)
    gx = ops.dispatch_backward(rows, idx.slot_pos, out_dtype=odt)
    torch.cuda.synchronize()
    acc = torch.float64 if torch.float64 in (idt, odt) else torch.float32
    want = torch.zeros((T, h), dtype=acc, device=cuda)
    for s in range(k):                                          # ascending slot order, as the kernel
        want += rows[idx.slot_pos[:, s].long()].to(acc)
    assert torch.equal(gx, want.to(odt))


@pytest.mark.parametrize("T,E,k", [(2048, 8, 2), (8192, 2, 1), (1000, 160, 6), (77, 33, 3), (5, 4, 4)])
@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
def test_route_backward_matches_autograd(cuda, T, E, k, dtype):
    logits, experts, _, _ = _index(T, E, k, seed=T + E, dev=cuda, logit_dtype=dtype)
    gp = _rand((T, k), dtype, 4, cuda)
    gz = ops.route_backward(logits, experts, gp)
    torch.cuda.synchronize()
    z = logits.double().clone().requires_grad_(True)
    p = torch.softmax(z, dim=-1).gather(1, experts.long())
    (p * gp.double()).sum().backward()
    tol = 1e-12 if dtype is torch.float64 else 1e-5
    assert (gz.double() - z.grad).abs().max().item() < tol


def test_backward_empty_and_errors(cuda):
    e = torch.empty((0, 2), dtype=torch.int32, device=cuda)
    g = torch.empty((0, 16), dtype=torch.float32, device=cuda)
    assert ops.dispatch_backward(torch.empty((0, 16), device=cuda), e).shape == (0, 16)
    gy, gp = ops.combine_backward(g, torch.empty((0, 16), device=cuda), e, torch.empty((0, 2), device=cuda))
    assert gy.shape == (0, 16) and gp.shape == (0, 2)
    with pytest.raises(_lib.InvalidArgument):
        ops.dispatch_backward(torch.zeros((65, 16), device=cuda), torch.zeros((1, 65), dtype=torch.int32,
                                                                                 device=cuda))
    with pytest.raises(_lib.InvalidArgument):
        ops.route_backward(torch.zeros((4, 2), device=cuda), torch.zeros((4, 3), dtype=torch.int32, device=cuda),
                           torch.zeros((4, 3), device=cuda))


def _torch_layer(x, logits, k, experts_w):
    """Plain fp64 PyTorch MoE layer with the reference's routing (stable top-k
    on raw scores, unrenormalised softmax probs)."""
    p_all = torch.softmax(logits, dim=-1)
    order = torch.sort(logits.detach(), dim=-1, descending=True, stable=True).indices[:, :k]
    sel = torch.sort(order, dim=-1).values
    probs = p_all.gather(1, sel)
    out = torch.zeros_like(x)
    for s in range(k):
        ys = torch.einsum("th,thd->td", x, experts_w[sel[:, s]])
        out = out + probs[:, s:s + 1] * ys
    return out


@pytest.mark.parametrize("T,h,E,k", [(256, 64, 8, 2), (128, 32, 16, 4)])
def test_layer_gradients_match_torch(cuda, T, h, E, k):
    x0 = _rand((T, h), torch.float32, 10, cuda)
    z0 = _rand((T, E), torch.float32, 11, cuda)
    w0 = _rand((E, h, h), torch.float32, 12, cuda) / h ** 0.5
    gout = _rand((T, h), torch.float32, 13, cuda)

    x, z, w = (t.clone().requires_grad_(True) for t in (x0, z0, w0))

    def experts_fn(rows, index):
        offs = index.expert_offsets.tolist()
        return torch.cat([rows[offs[e]:offs[e + 1]] @ w[e] for e in range(E)])

    out = mag.moe_local(x, z, k, E, experts_fn)
    (out * gout).sum().backward()

    xr, zr, wr = (t.double().clone().requires_grad_(True) for t in (x0, z0, w0))
    ref = _torch_layer(xr, zr, k, wr)
    (ref * gout.double()).sum().backward()
    torch.cuda.synchronize()
    for got, want in ((out, ref), (x.grad, xr.grad), (z.grad, zr.grad), (w.grad, wr.grad)):
        scale = want.abs().max().item() + 1e-30
        assert (got.double() - want).abs().max().item() / scale < 1e-4


def test_full_size_deepseek_adjoint_properties(cuda):
    """DeepSeek-V2 layer size (T=8192, h=5120, E=160, top-6, bf16): dispatch
    backward of the dispatched rows is exactly k*x (small integer multiples
    of a bf16 value are exact in fp32), and combine backward with y = the
    dispatched rows gives grad_probs[i, s] = <g_i, x_i> for every slot."""
    T, h, E, k = 8192, 5120, 160, 6
    _, _, probs, idx = _index(T, E, k, seed=5, dev=cuda)
    x = _rand((T, h), torch.bfloat16, 6, cuda)
    rows = ops.permute_rows(x, idx.perm_src)
    gx = ops.dispatch_backward(rows, idx.slot_pos)
    torch.cuda.synchronize()
    assert torch.equal(gx, (k * x.float()).to(torch.bfloat16))
    g = _rand((T, h), torch.bfloat16, 7, cuda)
    gy, gp = ops.combine_backward(g, rows, idx.slot_pos, probs)
    torch.cuda.synchronize()
    ref = (g.double() * x.double()).sum(-1, keepdim=True).expand(T, k)
    mag_ = (g.double() * x.double()).abs().sum(-1, keepdim=True)
    assert ((gp.double() - ref).abs() / mag_).max().item() < 1e-5
    # grad_y rows land exactly where the forward put the token's rows.
    assert torch.equal(gy[idx.slot_pos[:, 0].long()], (probs[:, :1] * g.float()).to(torch.bfloat16))


@pytest.mark.parametrize("dt", [torch.float32, torch.bfloat16])
def test_backward_skips_empty_slots(cuda, dt):
    """Tokens padded with empty slots (expert -1, as the drop-in pads ragged
    routing): the index gives them slot position -1; the forward skips them and
    so must every adjoint (no store before the allocation, grad_prob 0)."""
    T, h, E, k = 257, 136, 8, 3
    g0 = torch.Generator().manual_seed(3)
    experts = torch.sort(torch.stack([torch.randperm(E, generator=g0)[:k] for _ in range(T)]), dim=1).values
    experts = experts.to(torch.int32)
    experts[::3, 0] = -1                      # one empty slot on every third token
    experts[1::7, :2] = -1                    # two on every seventh
    experts = torch.sort(experts, dim=1).values.to(cuda)
    idx = ops.build_index(experts, E)
    pos = idx.slot_pos
    live = pos >= 0
    assert (~live).any() and torch.equal(~live, experts < 0)
    rows_used = int(idx.expert_offsets[-1].item())
    # permute: the tail past expert_offsets[E] is -1 and gathers zero rows
    x = _rand((T, h), dt, 5, cuda)
    perm = ops.permute_rows(x, idx.perm_src)
    assert torch.all(idx.perm_src[rows_used:] == -1)
    assert torch.all(perm[rows_used:] == 0)
    assert torch.equal(perm[:rows_used], x[idx.perm_src[:rows_used].long()])
    # combine backward
    probs = torch.rand(T, k, generator=g0).to(cuda)
    y = _rand((T * k, h), dt, 6, cuda)
    g = _rand((T, h), dt, 7, cuda)
    gy, gp = ops.combine_backward(g, y, pos, probs)
    torch.cuda.synchronize()
    assert torch.all(gp[~live] == 0)
    want_gy = torch.zeros((T * k, h), dtype=dt, device=cuda)
    for s in range(k):
        m = live[:, s]
        want_gy[pos[m, s].long()] = (probs[m, s:s + 1] * g[m].float()).to(dt)
    assert torch.equal(gy, want_gy)
    ref = torch.zeros(T, k, dtype=torch.float64, device=cuda)
    for s in range(k):
        m = live[:, s]
        ref[m, s] = (g[m].double() * y[pos[m, s].long()].double()).sum(-1)
    assert torch.allclose(gp.double(), ref, rtol=1e-4, atol=1e-3)
    # dispatch backward
    gx = ops.dispatch_backward(y, pos, out_dtype=torch.float32)
    want = torch.zeros((T, h), dtype=torch.float32, device=cuda)
    for s in range(k):
        m = live[:, s]
        want[m] += y[pos[m, s].long()].float()
    assert torch.equal(gx, want)
    # route backward with an empty slot's gradient ignored
    logits = _rand((T, E), torch.float32, 8, cuda)
    gpr = _rand((T, k), torch.float32, 9, cuda)
    gz = ops.route_backward(logits, experts, gpr)
    P = torch.softmax(logits.double(), -1)
    G = torch.zeros(T, E, dtype=torch.float64, device=cuda)
    for s in range(k):
        m = live[:, s]
        G[m, experts[m, s].long()] = gpr[m, s].double()
    want_z = P * (G - (G * P).sum(-1, keepdim=True))
    assert torch.allclose(gz.double(), want_z, rtol=1e-4, atol=1e-6)

"""GPU checks of the expert compute (include/monta.h section 1c, SURVEY.md
§8(f) item 1): the tcgen05 grouped GEMM and the SwiGLU expert FFN against
plain PyTorch fp32 references of the same ops.

Bar: every element within one bf16 rounding of the fp32 reference plus the
fp32-accumulation slack of its dot product,
    |got - ref| <= 2^-8 |ref| + 2^-14 * (|x| . |w|)
(a wrong tile, swizzle or row offset is off by O(|ref|), far outside it), and
rows past an expert's segment are never written.
"""
import pytest
import torch

from paper_2411_00662_b200 import _lib
from paper_2411_00662_b200 import ops

pytestmark = pytest.mark.gpu


def _offsets(sizes, dev):
    return torch.tensor([0] + list(torch.tensor(sizes).cumsum(0).tolist()), dtype=torch.int32, device=dev)


def _check(got, ref, mag, what):
    bound = 2.0 ** -8 * ref.abs() + 2.0 ** -14 * mag + 1e-30
    bad = (got.float() - ref).abs() > bound
    assert not bool(bad.any()), f"{what}: {int(bad.sum())} elements out of bound, worst " \
                                f"{float(((got.float() - ref).abs() / bound).max()):.3g}x"


def _gemm_ref(x, w, offs):
    L = w.shape[0]
    ref = torch.zeros(x.shape[0], w.shape[1], dtype=torch.float32, device=x.device)
    mag = torch.zeros_like(ref)
    o = offs.tolist()
    for l in range(L):
        a, b = o[l], o[l + 1]
        if b > a:
            ref[a:b] = x[a:b].float() @ w[l].float().T
            mag[a:b] = x[a:b].float().abs() @ w[l].float().abs().T
    return ref, mag


@pytest.mark.parametrize("sizes,N,K", [
    ([128], 256, 64),                       # one exact tile
    ([1], 128, 64),                         # one row, BN = 128 path
    ([0, 5, 0, 130, 127, 128, 129, 0], 256, 192),
    ([300, 7, 0, 1000], 384, 512),          # N % 256 != 0 -> BN = 128
    ([257] * 12, 512, 1024),
    ([0, 0, 0], 256, 128),                  # nothing to do
])
def test_grouped_gemm_matches_fp32(cuda, sizes, N, K):
    g = torch.Generator(device="cpu").manual_seed(sum(sizes) + N + K)
    L = len(sizes)
    rows = sum(sizes)
    cap = rows + 64  # addressable rows past the last expert (never written)
    x = torch.randn(cap, K, generator=g).to(torch.bfloat16).to(cuda)
    w = (torch.randn(L, N, K, generator=g) / K ** 0.5).to(torch.bfloat16).to(cuda)
    offs = _offsets(sizes, cuda)
    y = torch.full((cap, N), 7.0, dtype=torch.bfloat16, device=cuda)
    ops.grouped_gemm(x, w, offs, out=y)
    torch.cuda.synchronize()
    ref, mag = _gemm_ref(x[:rows], w, offs)
    _check(y[:rows], ref, mag, "grouped_gemm")
    assert bool((y[rows:] == 7.0).all()), "rows past the last expert were written"


def test_grouped_gemm_strided_rows(cuda):
    """x and y with row strides wider than K / N (a column slice of a wider buffer)."""
    g = torch.Generator(device="cpu").manual_seed(3)
    sizes, N, K = [200, 0, 77], 256, 128
    rows = sum(sizes)
    xb = torch.randn(rows, K + 64, generator=g).to(torch.bfloat16).to(cuda)
    x = xb[:, 32:32 + K]
    w = (torch.randn(3, N, K, generator=g) / K ** 0.5).to(torch.bfloat16).to(cuda)
    yb = torch.zeros(rows, N + 128, dtype=torch.bfloat16, device=cuda)
    y = yb[:, 64:64 + N]
    offs = _offsets(sizes, cuda)
    ops.grouped_gemm(x, w, offs, out=y)
    torch.cuda.synchronize()
    ref, mag = _gemm_ref(x, w, offs)
    _check(y, ref, mag, "strided grouped_gemm")
    assert bool((yb[:, :64] == 0).all()) and bool((yb[:, 64 + N:] == 0).all())


def _swiglu_ref(x, wg, wu, offs):
    L = wg.shape[0]
    out = torch.zeros(x.shape[0], wg.shape[1], dtype=torch.float32, device=x.device)
    mag = torch.zeros_like(out)
    o = offs.tolist()
    for l in range(L):
        a, b = o[l], o[l + 1]
        if b > a:
            gt = x[a:b].float() @ wg[l].float().T
            ut = x[a:b].float() @ wu[l].float().T
            out[a:b] = torch.nn.functional.silu(gt) * ut
            # slack: each factor carries its own accumulation error
            mg = x[a:b].float().abs() @ wg[l].float().abs().T
            mu = x[a:b].float().abs() @ wu[l].float().abs().T
            mag[a:b] = mg * ut.abs() + mu * gt.abs() + mg * mu
    return out, mag


@pytest.mark.parametrize("sizes,F,h", [([130, 0, 64, 300], 128, 256), ([129] * 5, 384, 512)])
def test_swiglu_epilogue(cuda, sizes, F, h):
    g = torch.Generator(device="cpu").manual_seed(F + h)
    L = len(sizes)
    rows = sum(sizes)
    x = torch.randn(rows, h, generator=g).to(torch.bfloat16).to(cuda)
    wg = (torch.randn(L, F, h, generator=g) / h ** 0.5).to(torch.bfloat16).to(cuda)
    wu = (torch.randn(L, F, h, generator=g) / h ** 0.5).to(torch.bfloat16).to(cuda)
    w13 = ops.interleave_w13(wg, wu)
    # the interleave itself: blocks of 128 gate rows then the matching 128 up rows
    B = _lib.W13_BLOCK
    for b in range(F // B):
        assert torch.equal(w13[:, 2 * B * b:2 * B * b + B], wg[:, B * b:B * (b + 1)])
        assert torch.equal(w13[:, 2 * B * b + B:2 * B * (b + 1)], wu[:, B * b:B * (b + 1)])
    offs = _offsets(sizes, cuda)
    hact = ops.grouped_gemm(x, w13, offs, act=_lib.ACT_SWIGLU)
    torch.cuda.synchronize()
    ref, mag = _swiglu_ref(x, wg, wu, offs)
    _check(hact, ref, mag, "swiglu")


@pytest.mark.parametrize("L,F,h,T,k", [(8, 256, 512, 512, 2), (160, 128, 256, 256, 6)])
def test_expert_ffn_on_routed_rows(cuda, L, F, h, T, k):
    """Experts over rows laid out by the router + index (the dispatch's
    expert-major order), compared with an fp32 FFN whose intermediate is
    rounded to bf16 like the kernel's workspace."""
    g = torch.Generator(device="cpu").manual_seed(L + F)
    logits = torch.randn(T, L, generator=g).to(cuda)
    experts, _ = ops.route_topk(logits, k)
    idx = ops.build_index(experts, L)
    x = torch.randn(T, h, generator=g).to(torch.bfloat16).to(cuda)
    rows = ops.permute_rows(x, idx.perm_src)
    wg = (torch.randn(L, F, h, generator=g) / h ** 0.5).to(torch.bfloat16).to(cuda)
    wu = (torch.randn(L, F, h, generator=g) / h ** 0.5).to(torch.bfloat16).to(cuda)
    w2 = (torch.randn(L, h, F, generator=g) / F ** 0.5).to(torch.bfloat16).to(cuda)
    w13 = ops.interleave_w13(wg, wu)
    y = ops.expert_ffn(rows, w13, w2, idx.expert_offsets)
    torch.cuda.synchronize()
    hmid, _ = _swiglu_ref(rows, wg, wu, idx.expert_offsets)
    hmid = hmid.to(torch.bfloat16)
    ref, mag = _gemm_ref(hmid, w2, idx.expert_offsets)
    # the intermediate itself may differ by one bf16 rounding: widen by |h|.|w2| * 2^-8
    _, mag2 = _gemm_ref(hmid, w2.abs(), idx.expert_offsets)
    bound = 2.0 ** -8 * ref.abs() + 2.0 ** -7 * mag2 + 2.0 ** -14 * mag + 1e-30
    assert bool(((y.float() - ref).abs() <= bound).all())
    # in place (y aliases x), as the layer context runs it on recv
    rows2 = rows.clone()
    ops.expert_ffn(rows2, w13, w2, idx.expert_offsets, out=rows2)
    torch.cuda.synchronize()
    assert torch.equal(rows2, y)


def test_grouped_gemm_rejects_bad_shapes(cuda):
    x = torch.zeros(16, 100, dtype=torch.bfloat16, device=cuda)
    w = torch.zeros(1, 128, 100, dtype=torch.bfloat16, device=cuda)
    offs = torch.tensor([0, 16], dtype=torch.int32, device=cuda)
    with pytest.raises(ValueError):
        ops.grouped_gemm(x, w, offs)  # K % 64 != 0
    x = torch.zeros(16, 128, dtype=torch.bfloat16, device=cuda)
    w = torch.zeros(1, 96, 128, dtype=torch.bfloat16, device=cuda)
    with pytest.raises(ValueError):
        ops.grouped_gemm(x, w, offs)  # N % 128 != 0


# ---------------------------------------------------------------------------
# Experts inside the layer context: dispatch -> expert FFN -> combine.
from paper_2411_00662_b200.layer import MoeLayer, BASELINE, O1, O2, O3, LAND_FINAL, LAND_STAGED  # noqa: E402


def _ffn_ref_rows(x, wg, wu, w2):
    """fp32 SwiGLU FFN of rows x through one expert, intermediate and output
    rounded to bf16 like the kernel's workspace and the recv rows.  Also
    returns |hmid| . |w2|^T: the slack one bf16 ulp of the intermediate
    (accumulation order inside the first GEMM) can move the output by."""
    g = x.float() @ wg.float().T
    u = x.float() @ wu.float().T
    hmid = (torch.nn.functional.silu(g) * u).to(torch.bfloat16)
    return (hmid.float() @ w2.float().T).to(torch.bfloat16), hmid.float().abs() @ w2.float().abs().T


@pytest.mark.parametrize("e,t,E,k,level,n,landing", [
    (1, 1, 16, 4, BASELINE, 1, LAND_FINAL),
    (2, 2, 8, 2, O1, 1, LAND_FINAL),
    (2, 2, 8, 2, BASELINE, 1, LAND_FINAL),
    (2, 2, 8, 2, O2, 2, LAND_STAGED),
    (4, 2, 16, 3, O3, 4, LAND_FINAL),
])
def test_layer_with_experts(cuda, e, t, E, k, level, n, landing):
    T, h, F = 256, 256, 128
    gen = torch.Generator(device="cpu").manual_seed(e * 100 + t * 10 + E + n)
    layer = MoeLayer(e, t, E, k, T, h, dtype=torch.bfloat16, max_chunks=max(n, 1))
    try:
        L = E // e
        wg = (torch.randn(E, F, h, generator=gen) / h ** 0.5).to(torch.bfloat16).to(cuda)
        wu = (torch.randn(E, F, h, generator=gen) / h ** 0.5).to(torch.bfloat16).to(cuda)
        w2 = (torch.randn(E, h, F, generator=gen) / F ** 0.5).to(torch.bfloat16).to(cuda)
        w13 = ops.interleave_w13(wg, wu)
        xs = [torch.randn(T, h, generator=gen).to(torch.bfloat16).to(cuda) for _ in range(e)]
        ls = [torch.randn(T, E, generator=gen).to(cuda) for _ in range(e)]
        for cd in layer.cards:
            cd.x.copy_(xs[cd.node])
            cd.logits.copy_(ls[cd.node])
            lo = cd.node * L
            layer.bind_experts(cd.card, w13[lo:lo + L].contiguous(), w2[lo:lo + L].contiguous())
        layer.forward(level, n, landing)
        layer.sync()
        for cd in layer.cards:
            # the experts' segments: this node's local experts in recv order
            offs = cd.recv_expert_offsets.cpu()
            want = torch.zeros(L, dtype=torch.int64)
            for g in range(e):
                ex = layer.card(g * t).experts.cpu().long()
                for l in range(L):
                    want[l] += int((ex == cd.node * L + l).sum())
            assert offs[0] == 0 and torch.equal(offs[1:] - offs[:-1], want.to(offs.dtype))
        for cd in layer.cards:
            ex = cd.experts.long()
            pr = cd.probs.float()
            ref = torch.zeros(T, h, dtype=torch.float32, device=cuda)
            mag = torch.zeros_like(ref)
            for s in range(k):
                for x in range(E):
                    m = ex[:, s] == x
                    if bool(m.any()):
                        y, hw = _ffn_ref_rows(xs[cd.node][m], wg[x], wu[x], w2[x])
                        ref[m] += pr[m, s:s + 1] * y.float()
                        mag[m] += pr[m, s:s + 1] * (2.0 ** -7 * y.float().abs() + 2.0 ** -7 * hw)
            got = cd.out.float()
            # bf16 out (2^-8 |ref|) + per slot: one bf16 ulp of the expert row and one of
            # its intermediate propagated through w2 (accumulation-order differences)
            bound = 2.0 ** -8 * ref.abs() + mag + 1e-6
            bad = (got - ref).abs() > bound
            assert not bool(bad.any()), (cd.card, int(bad.sum()), float(((got - ref).abs() / bound).max()))
        # unbinding restores identity experts: out = x * sum(p)
        for cd in layer.cards:
            layer.bind_experts(cd.card, None)
        layer.forward(level, n, landing)
        layer.sync()
        for cd in layer.cards:
            want = xs[cd.node].double() * cd.probs.double().sum(1, keepdim=True)
            err = ((cd.out.double() - want).abs().max() / want.abs().max()).item()
            assert err <= 1e-2
    finally:
        layer.close()

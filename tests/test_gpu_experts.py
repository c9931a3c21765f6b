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

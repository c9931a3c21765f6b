"""GPU parity of the stateless kernels against the CPU oracle.

Bar (BASELINE.json north_star): routing indices, permutation maps and moved
rows bit-exact; probabilities within 1e-5 relative (fp32 logits) or 1e-12
(fp64 logits, the reference's own precision); combine within 1e-5 (fp32) /
1e-2 (bf16) relative.  Reference: dataplane.hpp:72-140, :317-344.
"""
import ctypes as C

import numpy as np
import pytest
import torch

import oracle
from paper_2411_00662_b200 import _lib
from paper_2411_00662_b200 import ops

pytestmark = pytest.mark.gpu


def _route_case(T, E, k, dtype, seed, ties=False):
    rng = np.random.default_rng(seed)
    if ties:
        logits = rng.integers(0, 4, (T, E)).astype(np.float64)  # many exact ties
    else:
        logits = rng.standard_normal((T, E))
    logits = logits.astype(np.float32 if dtype is torch.float32 else np.float64)
    ex_ref, pr_ref = oracle.route_topk(logits.astype(np.float64), k)
    ex, pr = ops.route_topk(torch.from_numpy(logits).cuda(), k)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(ex.cpu().numpy(), ex_ref)
    rtol = 1e-5 if dtype is torch.float32 else 1e-12
    np.testing.assert_allclose(pr.cpu().double().numpy(), pr_ref, rtol=rtol, atol=0)


@pytest.mark.parametrize("T,E,k", [(1, 1, 1), (7, 2, 1), (2048, 8, 2), (4096, 8, 2), (8192, 2, 1),
                                   (1000, 160, 6), (513, 33, 3), (64, 64, 8), (100, 1024, 4), (5, 4, 4)])
@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
def test_route_topk_matches_oracle(cuda, T, E, k, dtype):
    _route_case(T, E, k, dtype, seed=T * 31 + E)


@pytest.mark.parametrize("E,k", [(4, 2), (8, 2), (160, 6), (2, 1)])
def test_route_topk_ties_break_low(cuda, E, k):
    _route_case(777, E, k, torch.float64, seed=E, ties=True)
    _route_case(777, E, k, torch.float32, seed=E + 1, ties=True)


@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
def test_route_topk_signed_zero_ties(cuda, dtype):
    # -0.0 == +0.0 for the reference's comparator (dataplane.hpp:97-98): lower index wins
    s = torch.tensor([[-0.0, 0.0], [0.0, -0.0], [-0.0, -0.0], [0.0, 0.0]], dtype=dtype, device="cuda")
    ex, _ = ops.route_topk(s, 1)
    assert ex.cpu().flatten().tolist() == [0, 0, 0, 0]
    # a whole warp group (E=32, G=32 redux path) and a sub-warp group (E=5)
    for E in (32, 5, 160):
        row = torch.zeros(3, E, dtype=dtype)
        row[:, ::2] = -0.0
        row[1, E - 1] = 1e-45 if dtype is torch.float32 else 5e-324  # the smallest subnormal beats both zeros
        ex, _ = ops.route_topk(row.cuda(), 3)
        want = oracle.route_topk(row.double().numpy(), 3)[0]
        np.testing.assert_array_equal(ex.cpu().numpy(), want)


@pytest.mark.parametrize("E,k", [(8, 2), (160, 6), (37, 5)])
def test_route_topk_special_values_vs_oracle(cuda, E, k):
    rng = np.random.default_rng(E * 7 + k)
    f = np.finfo(np.float32)
    pool = np.array([-0.0, 0.0, f.smallest_subnormal, -f.smallest_subnormal, f.tiny, 1.0, -1.0, f.max, -f.max,
                     -np.inf], np.float32)
    logits = rng.choice(pool, (513, E))
    ex_ref, pr_ref = oracle.route_topk(logits.astype(np.float64), k)
    ex, pr = ops.route_topk(torch.from_numpy(logits).cuda(), k)
    np.testing.assert_array_equal(ex.cpu().numpy(), ex_ref)
    np.testing.assert_allclose(pr.cpu().double().numpy(), pr_ref, rtol=1e-5, atol=0)


def test_route_topk_known_answers(cuda):
    # dataplane.hpp / test_dataplane.cpp:72-93
    ex, pr = ops.route_topk(torch.tensor([[10.0, 0.0, 0.0, 0.0]], dtype=torch.float64, device="cuda"), 1)
    assert ex.tolist() == [[0]] and abs(pr.item() - 1.0) < 1e-3
    ex, pr = ops.route_topk(torch.tensor([[1.0, 1.0, 1.0, 1.0]], dtype=torch.float64, device="cuda"), 2)
    assert ex.tolist() == [[0, 1]] and np.allclose(pr.cpu().numpy(), 0.25, rtol=1e-12)
    s = [0.1, 0.9, 0.3, 0.5]
    ex, pr = ops.route_topk(torch.tensor([s], dtype=torch.float64, device="cuda"), 2)
    denom = sum(np.exp(v) for v in s)
    assert ex.tolist() == [[1, 3]]
    np.testing.assert_allclose(pr.cpu().numpy()[0], [np.exp(0.9) / denom, np.exp(0.5) / denom], rtol=1e-12)


def test_route_topk_rejects_bad_k(cuda):
    with pytest.raises(ValueError):
        ops.route_topk(torch.tensor([[1.0, 2.0]], device="cuda", dtype=torch.float64), 3)
    with pytest.raises(ValueError):
        ops.route_topk(torch.tensor([[1.0, 2.0]], device="cuda", dtype=torch.float64), 0)


def _index_case(experts: np.ndarray, E: int, n: int):
    T, k = experts.shape
    ps_ref, eo_ref, inv_ref, il_ref = oracle.permute(experts)
    idx = ops.build_index(torch.from_numpy(experts).cuda(), E, n)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(idx.perm_src.cpu().numpy(), ps_ref)
    np.testing.assert_array_equal(idx.expert_of.cpu().numpy(), eo_ref)
    # experts ascend per token -> slot positions == the reference inverse map
    np.testing.assert_array_equal(idx.slot_pos.cpu().numpy(), inv_ref)
    counts = idx.counts.cpu().numpy()
    ct = T // n
    want = np.zeros((n, E), np.int64)
    for i in range(T):
        for x in experts[i]:
            want[i // ct, x] += 1
    np.testing.assert_array_equal(counts, want)
    offs = idx.expert_offsets.cpu().numpy()
    np.testing.assert_array_equal(offs, np.concatenate([[0], np.cumsum(want.sum(0))]))


@pytest.mark.parametrize("T,E,k,n", [(1, 1, 1, 1), (12, 4, 2, 3), (2048, 8, 2, 4), (4096, 8, 2, 1),
                                     (8192, 2, 1, 8), (8192, 160, 6, 8), (3000, 37, 5, 5), (64, 512, 3, 2)])
def test_build_index_matches_oracle(cuda, T, E, k, n):
    rng = np.random.default_rng(T + E + k)
    experts = np.sort(np.argsort(rng.random((T, E)), axis=1)[:, :k], axis=1).astype(np.int32)
    _index_case(experts, E, n)


def test_build_index_skewed_routing(cuda):
    rng = np.random.default_rng(5)
    T, E, k = 8192, 160, 6
    # Zipf-skewed experts, distinct per token
    w = 1.0 / np.arange(1, E + 1) ** 1.2
    experts = np.zeros((T, k), np.int32)
    for i in range(T):
        experts[i] = np.sort(rng.choice(E, k, replace=False, p=w / w.sum()))
    _index_case(experts, E, 4)
    # everything to a single expert
    _index_case(np.zeros((4096, 1), np.int32), 8, 2)


def test_build_index_empty(cuda):
    idx = ops.build_index(torch.zeros((0, 2), dtype=torch.int32, device="cuda"), 4, 1)
    torch.cuda.synchronize()
    assert idx.perm_src.numel() == 0
    assert idx.expert_offsets.cpu().tolist() == [0, 0, 0, 0, 0]


def test_build_index_rejects_out_of_range(cuda):
    with pytest.raises(ValueError):
        ops.build_index(torch.tensor([[0], [5]], dtype=torch.int32, device="cuda"), 4, 1, check=True)


@pytest.mark.parametrize("row_elems,dtype", [(1024, torch.float32), (4096, torch.bfloat16), (3, torch.int64),
                                             (5120, torch.bfloat16), (7, torch.float16)])
def test_permute_rows_bit_exact(cuda, row_elems, dtype):
    rng = np.random.default_rng(row_elems)
    T, E, k = 1536, 8, 2
    experts = np.sort(np.argsort(rng.random((T, E)), axis=1)[:, :k], axis=1).astype(np.int32)
    x = torch.randn(T, row_elems, device="cuda").to(dtype) if dtype.is_floating_point else \
        torch.randint(-2**40, 2**40, (T, row_elems), device="cuda", dtype=dtype)
    idx = ops.build_index(torch.from_numpy(experts).cuda(), E, 1)
    out = ops.permute_rows(x, idx.perm_src)
    torch.cuda.synchronize()
    ps_ref, _, _, _ = oracle.permute(experts)
    want = x.cpu()[torch.from_numpy(ps_ref.astype(np.int64))]
    assert torch.equal(out.cpu().view(torch.uint8), want.view(torch.uint8))


def test_permute_rows_column_slice(cuda):
    T, h, t = 256, 4096, 4
    x = torch.randn(T, h, device="cuda", dtype=torch.bfloat16)
    perm = torch.randperm(T, device="cuda", dtype=torch.int64).to(torch.int32)
    for rho in range(t):
        w = h // t
        out = ops.permute_rows(x, perm, col_off=rho * w, width=w)
        torch.cuda.synchronize()
        assert torch.equal(out.cpu(), x.cpu()[perm.cpu().long(), rho * w:(rho + 1) * w])


@pytest.mark.parametrize("dtype,out_dtype,rtol", [(torch.float32, torch.float32, 1e-5), (torch.bfloat16, torch.bfloat16, 1e-2),
                                                  (torch.bfloat16, torch.float32, 1e-5), (torch.float64, torch.float64, 1e-12),
                                                  (torch.int64, torch.float64, 1e-12), (torch.float16, torch.float16, 1e-2)])
def test_unpermute_combine_matches_oracle(cuda, dtype, out_dtype, rtol):
    rng = np.random.default_rng(11)
    T, E, k, h = 777, 16, 4, 264
    logits = rng.standard_normal((T, E))
    experts, probs = oracle.route_topk(logits, k)
    ps, eo, inv, il = oracle.permute(experts)
    R = T * k
    if dtype.is_floating_point:
        y = torch.randn(R, h, dtype=torch.float64).to(dtype)
    else:
        y = torch.randint(-1000, 1000, (R, h), dtype=dtype)
    pdt = torch.float64 if dtype in (torch.float64, torch.int64) else torch.float32
    out = ops.unpermute_combine(y.cuda(), torch.from_numpy(inv).cuda(), torch.from_numpy(probs).to(pdt).cuda(),
                                out_dtype=out_dtype)
    torch.cuda.synchronize()
    pq = torch.from_numpy(probs).to(pdt).double().numpy()
    yd = y.double().numpy()
    want = np.zeros((T, h))
    for s in range(k):
        want += pq[:, s:s + 1] * yd[inv[:, s]]
    got = out.cpu().double().numpy()
    scale = np.abs(want).max()
    assert np.abs(got - want).max() <= rtol * scale + 1e-300


def test_build_index_empty_slots_are_skipped(cuda):
    """Negative expert ids are empty slots (ragged routing padded with -1):
    like the reference's permute, which only matches experts >= 0."""
    rng = np.random.default_rng(12)
    T, E, k = 777, 16, 4
    experts = np.sort(np.argsort(rng.random((T, E)), axis=1)[:, :k], axis=1).astype(np.int32)
    drop = rng.random((T, k)) < 0.3
    experts[drop] = -1
    ps_ref, eo_ref, inv_ref, il_ref = oracle.permute(experts)
    idx = ops.build_index(torch.from_numpy(experts).cuda(), E, 1, check=True)
    torch.cuda.synchronize()
    valid = int(il_ref.sum())
    np.testing.assert_array_equal(idx.perm_src.cpu().numpy()[:valid], ps_ref[:valid])
    np.testing.assert_array_equal(idx.expert_of.cpu().numpy()[:valid], eo_ref[:valid])
    sp = idx.slot_pos.cpu().numpy()
    assert (sp[drop] == -1).all()
    for i in range(T):
        np.testing.assert_array_equal(np.sort(sp[i][sp[i] >= 0]), inv_ref[i][:il_ref[i]])


@pytest.mark.parametrize("k,h", [(3, 8), (5, 264), (6, 5120), (8, 1032), (16, 256)])
@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float16])
def test_unpermute_any_k_with_empty_slots(cuda, k, h, dtype):
    """The CTA-per-token un-permute (k > 2, 16-bit rows): fp32 accumulation in
    ascending slot order, empty slots (slot_pos < 0) contribute nothing."""
    g = torch.Generator().manual_seed(k * 1000 + h)
    T = 301
    R = T * k
    y = torch.randn(R, h, generator=g).to(dtype)
    pos = torch.randperm(R, generator=g).reshape(T, k).to(torch.int32)
    pos[torch.rand(T, k, generator=g) < 0.2] = -1
    p = torch.rand(T, k, generator=g)
    out = ops.unpermute_combine(y.cuda(), pos.cuda(), p.cuda())
    torch.cuda.synchronize()
    want = torch.zeros(T, h, dtype=torch.float64)
    mag = torch.zeros(T, h, dtype=torch.float64)
    for s in range(k):
        m = pos[:, s] >= 0
        term = p[m, s:s + 1].double() * y[pos[m, s].long()].double()
        want[m] += term
        mag[m] += term.abs()
    # one rounding to the output type (unit roundoff, with slack for fp32 sums
    # landing next to a rounding boundary; fp16 subnormals: absolute) + fp32
    # accumulation over k slots
    ulp = 2.0 ** -8 if dtype == torch.bfloat16 else 2.0 ** -11
    err = (out.cpu().double() - want).abs()
    assert bool((err <= 1.5 * ulp * want.abs() + k * 2.0 ** -23 * mag + 2.0 ** -24).all()), float(err.max())

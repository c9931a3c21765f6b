"""GPU parity of the layer context (virtual mode: every card of the e x t
topology on one GPU, as the reference emulates them in one process) against
the CPU oracle.

Dispatch (dataplane.hpp:145-283): every card's received rows and tags
{token_id, source_card, source_position, expert} bit-exact with the oracle's
monolithic order, for the naive exchange and for O1/O2/O3 at every chunk
count, with direct (final) and staged (pre-copy + reorder) landing; the staged
buffer equals the oracle's pre_copy.  Combine (dataplane.hpp:293-347):
within 1e-5 (fp32) / 1e-2 (bf16) relative of the fp64 oracle.
"""
import numpy as np
import pytest
import torch

import oracle
from paper_2411_00662_b200.ops import host_empty
from paper_2411_00662_b200 import _lib
from paper_2411_00662_b200.layer import MoeLayer, BASELINE, O1, O2, O3, LAND_FINAL, LAND_STAGED

pytestmark = pytest.mark.gpu

_DT = {torch.float32: oracle.F32, torch.bfloat16: oracle.BF16, torch.float16: oracle.F16, torch.float64: oracle.F64,
       torch.int64: oracle.I64}


def _inputs(e, T, h, E, dtype, seed, skew=False):
    g = torch.Generator().manual_seed(seed)
    if dtype.is_floating_point:
        x = torch.randn(e, T, h, generator=g).to(dtype)
    else:
        x = torch.randint(0, 100, (e, T, h), generator=g, dtype=dtype)
    logits = torch.randn(e, T, E, generator=g, dtype=torch.float32)
    if skew:
        logits += torch.linspace(3.0, 0.0, E)[None, None, :]
    return x, logits


_SIGN = {torch.float32: np.uint32(0x7fffffff), torch.bfloat16: np.uint16(0x7fff), torch.float16: np.uint16(0x7fff)}
_UINT = {torch.float32: np.uint32, torch.bfloat16: np.uint16, torch.float16: np.uint16}


def _check_combine(layer, nodes, dtype, fin, probs, want):
    """Per-element relative bound (north_star: 1e-5 fp32 / 1e-2 bf16 relative):
    |got - want| <= rtol * |want| + 8 * eps_acc * sum_s p_s |y_s|.  The second
    term is the conditioning of the k-term sum: fp32 accumulation cannot be
    relative-accurate where the slots cancel, and nothing is allowed beyond
    a few fp32 roundings of the terms' magnitude there.  rtol follows the
    OUTPUT dtype (one final rounding to bf16/f16 is 2^-9 relative)."""
    od = layer.out_dtype
    rtol = 1e-2 if od in (torch.bfloat16, torch.float16) else 1e-5
    if dtype in _SIGN:
        # sum_s p_s |y_s|: the oracle's combine over sign-cleared rows
        absfin = [((r.view(_UINT[dtype]) & _SIGN[dtype]).view(np.uint8), tg) for r, tg in fin]
        mag, _ = nodes.combine(_DT[dtype], absfin, probs)
        eps = 2.0 ** -23  # fp32 accumulation
    else:  # f64 / i64: fp64 accumulation in slot order — the reference's arithmetic
        mag, eps = np.abs(want), 2.0 ** -52
    for cd in layer.cards:
        got = cd.out.cpu().double().numpy()
        w = want[cd.node]
        bound = rtol * np.abs(w) + 8 * eps * mag[cd.node] + 1e-300
        bad = np.abs(got - w) > bound
        assert not bad.any(), (f"card {cd.card}: {int(bad.sum())} combine elements outside "
                               f"rtol={rtol}: worst {float((np.abs(got - w) / bound).max())}x the bound")


def _run(e, t, E, k, T, h, dtype, level, n, landing, seed=0, out_dtype=None, skew=False, check_combine=True):
    x, logits = _inputs(e, T, h, E, dtype, seed, skew)
    layer = MoeLayer(e, t, E, k, T, h, dtype=dtype, logit_dtype=torch.float32, out_dtype=out_dtype, max_chunks=max(n, 1))
    try:
        for cd in layer.cards:
            cd.x.copy_(x[cd.node])
            cd.logits.copy_(logits[cd.node])
        layer.route()
        layer.dispatch(level, n, landing)
        layer.sync()
        experts = np.stack([layer.card(g * t).experts.cpu().numpy() for g in range(e)])
        probs = np.stack([layer.card(g * t).probs.cpu().double().numpy() for g in range(e)])
        # routing is replicated across a node's TP ranks
        for cd in layer.cards:
            np.testing.assert_array_equal(cd.experts.cpu().numpy(), experts[cd.node])
        xb = x.contiguous().view(torch.uint8).numpy().reshape(e, T, -1)
        nodes = oracle.Nodes(e, t, E, xb, experts)
        if level == BASELINE:
            fin, stg = nodes.dispatch_monolithic(), None
        else:
            fin, stg = nodes.dispatch_chunked(level, n, x.element_size())
        for cd in layer.cards:
            rows = layer.recv_rows(cd.card)
            want_rows, want_tags = fin[cd.node]
            assert rows == want_rows.shape[0], (cd.card, rows, want_rows.shape)
            got = cd.recv[:rows].contiguous().view(torch.uint8).cpu().numpy().reshape(rows, -1)
            assert np.array_equal(got, want_rows), f"card {cd.card}: dispatched rows differ"
            np.testing.assert_array_equal(cd.recv_tags[:rows].cpu().numpy(), want_tags)
            if landing == LAND_STAGED and stg is not None:
                pr, pt = stg[cd.node]
                gotp = cd.pre[:rows].contiguous().view(torch.uint8).cpu().numpy().reshape(rows, -1)
                assert np.array_equal(gotp, pr), f"card {cd.card}: pre-copy layout differs"
                np.testing.assert_array_equal(cd.pre_tags[:rows].cpu().numpy(), pt)
        if not check_combine:
            return layer
        layer.combine(level, n)
        layer.sync()
        want, tok = nodes.combine(_DT[dtype], fin, probs)
        _check_combine(layer, nodes, dtype, fin, probs, want)
        return layer
    finally:
        layer.close()


@pytest.mark.parametrize("e,t", [(1, 1), (2, 1), (1, 2), (2, 2), (2, 4), (4, 2)])
def test_dispatch_baseline(cuda, e, t):
    _run(e, t, 2 * e, 2, 64, 32, torch.float32, BASELINE, 1, LAND_FINAL, seed=e * 10 + t)


@pytest.mark.parametrize("level,n", [(O1, 1), (O2, 2), (O3, 4), (O2, 8)])
@pytest.mark.parametrize("landing", [LAND_FINAL, LAND_STAGED])
@pytest.mark.parametrize("e,t,E", [(2, 2, 2), (2, 2, 8), (2, 4, 2), (4, 2, 8), (4, 2, 4)])
def test_dispatch_chunked(cuda, e, t, E, level, n, landing):
    _run(e, t, E, 2 if E >= 2 else 1, 96, 64, torch.bfloat16, level, n, landing, seed=e * 100 + t * 10 + E + n)


def test_dispatch_fp32_toy_config(cuda):
    # configs[0] shape at reduced T: fp32, h=1024, E=8, k=2, EP=2 x TP=2
    _run(2, 2, 8, 2, 256, 1024, torch.float32, O2, 4, LAND_STAGED, seed=1)


def test_dispatch_int64_payload(cuda):
    # the reference's own payload type; combine decodes to fp64
    _run(2, 2, 2, 2, 24, 8, torch.int64, O3, 3, LAND_STAGED, seed=3, out_dtype=torch.float64)


def test_dispatch_skewed_routing(cuda):
    _run(4, 2, 16, 4, 128, 64, torch.bfloat16, O3, 4, LAND_FINAL, seed=9, skew=True)


def test_dispatch_deepseek_shape_small(cuda):
    # configs[3] shape family: E=160 fine-grained experts, top-6, EP=4 x TP=2
    _run(4, 2, 160, 6, 256, 320, torch.bfloat16, O3, 2, LAND_FINAL, seed=4)


def test_combine_fp32_out_of_bf16(cuda):
    _run(2, 2, 8, 2, 64, 128, torch.bfloat16, O1, 1, LAND_FINAL, seed=6, out_dtype=torch.float32)


def test_dispatch_validation(cuda):
    layer = MoeLayer(2, 2, 2, 1, 6, 4, dtype=torch.float32, max_chunks=8)
    try:
        with pytest.raises(ValueError):
            layer.dispatch(O2, 4)  # 4 does not divide 6
        with pytest.raises(ValueError):
            layer.dispatch(O1, 3)  # O1 is unchunked
        with pytest.raises(ValueError):
            layer.dispatch(O2, 0)
        with pytest.raises(ValueError):
            layer.dispatch(BASELINE, 2)
        with pytest.raises(ValueError):
            layer.dispatch(7, 1)
    finally:
        layer.close()
    layer = MoeLayer(2, 4, 2, 1, 8, 6, dtype=torch.float32, max_chunks=2)  # 6 % 4 != 0
    try:
        with pytest.raises(ValueError):
            layer.dispatch(O1, 1)
    finally:
        layer.close()


def test_forward_host_round_trip(cuda):
    # end-to-end from host buffers, identity experts with dyadic gates summing to 1
    e, t, E, k, T, h = 2, 2, 8, 2, 128, 256
    layer = MoeLayer(e, t, E, k, T, h, dtype=torch.bfloat16, max_chunks=4)
    try:
        x, logits = _inputs(e, T, h, E, torch.bfloat16, 5)
        hx = torch.empty(e * t, T, h, dtype=torch.bfloat16).pin_memory()
        hl = torch.empty(e * t, T, E, dtype=torch.float32).pin_memory()
        for c in range(e * t):
            hx[c] = x[c // t]
            hl[c] = logits[c // t]
        ho = torch.empty(e * t, T, h, dtype=torch.bfloat16).pin_memory()
        layer.forward_host(hx, hl, ho, O2, 2)
        torch.cuda.synchronize()
        layer.sync()
        # identity experts: out = x * sum_s p_s  (probs are not renormalised)
        for cd in layer.cards:
            psum = cd.probs.double().sum(1, keepdim=True).cpu()
            want = x[cd.node].double() * psum
            err = (ho[cd.card].double() - want).abs().max() / want.abs().max()
            assert err < 1e-2
    finally:
        layer.close()


@pytest.mark.parametrize("level,n,landing", [(BASELINE, 1, LAND_FINAL), (O1, 1, LAND_FINAL), (O3, 4, LAND_STAGED)])
def test_cuda_graph_replay_matches_eager(cuda, level, n, landing):
    """forward() captured as a CUDA graph and replayed gives the same bits."""
    e, t, E, k, T, h = 2, 2, 8, 2, 128, 256
    x, logits = _inputs(e, T, h, E, torch.bfloat16, 21)
    outs = []
    for graphs in (False, True):
        layer = MoeLayer(e, t, E, k, T, h, dtype=torch.bfloat16, max_chunks=8)
        try:
            layer.enable_graphs(graphs)
            for cd in layer.cards:
                cd.x.copy_(x[cd.node])
                cd.logits.copy_(logits[cd.node])
            for _ in range(3):  # capture, then replays
                layer.forward(level, n, landing)
            layer.sync()
            outs.append([(cd.recv[:layer.recv_rows(cd.card)].clone(), cd.recv_tags[:layer.recv_rows(cd.card)].clone(),
                          cd.out.clone()) for cd in layer.cards])
        finally:
            layer.close()
    for (r0, t0, o0), (r1, t1, o1) in zip(*outs):
        assert torch.equal(r0.view(torch.int16), r1.view(torch.int16))
        assert torch.equal(t0, t1)
        assert torch.equal(o0.view(torch.int16), o1.view(torch.int16))


def test_combine_requires_a_pending_dispatch(cuda):
    layer = MoeLayer(2, 2, 4, 1, 16, 8, dtype=torch.float32, max_chunks=2)
    try:
        with pytest.raises(ValueError):
            layer.combine(O1, 1)
        layer.route()
        layer.dispatch(O1, 1)
        layer.combine(O1, 1)
        with pytest.raises(ValueError):
            layer.combine(O1, 1)  # one combine per dispatch
    finally:
        layer.close()


@pytest.mark.parametrize("T,E,k,n", [(8192, 160, 6, 8), (8190, 160, 6, 5), (4096, 8, 2, 1), (8192, 2, 1, 64),
                                     (3, 4, 2, 3), (0, 8, 2, 1),
                                     # more tiles than co-resident tile CTAs: CTAs own several tiles
                                     (19264, 160, 6, 1), (19264, 160, 6, 4), (147904, 8, 2, 1)])
def test_front_index_matches_oracle_full_size(cuda, T, E, k, n):
    """The fused front kernel's index (cooperative grid: tile histograms, a
    grid barrier, per-tile prefixes and ranks) equals the oracle's permute at
    full size, including chunk lengths that do not align with the tiles and
    grids where a CTA owns several tiles."""
    layer = MoeLayer(1, 1, E, k, T, 64, dtype=torch.bfloat16, max_chunks=max(n, 1))
    try:
        cd = layer.cards[0]
        g = torch.Generator(device="cuda").manual_seed(T + E)
        if T:
            cd.logits.copy_(torch.randn(T, E, generator=g, device="cuda"))
        layer.route()
        if n == 1:
            layer.dispatch(BASELINE, 1)
        else:
            layer.dispatch(O2, n)
        layer.sync()
        experts = cd.experts.cpu().numpy()
        ps, eo, inv, _ = oracle.permute(experts)
        assert np.array_equal(cd.perm_src.cpu().numpy(), ps)
        assert np.array_equal(cd.expert_of.cpu().numpy(), eo)
        assert np.array_equal(cd.slot_pos.cpu().numpy(), inv)
        want = np.zeros((n, E), np.int64)
        ct = T // n if n else 0
        for i in range(T):
            for x in experts[i]:
                want[i // ct, x] += 1
        assert np.array_equal(cd.counts[:n].cpu().numpy(), want)
        assert np.array_equal(cd.expert_offsets.cpu().numpy(), np.concatenate([[0], np.cumsum(want.sum(0))]))
    finally:
        layer.close()


@pytest.mark.parametrize("graphs", [False, True])
def test_forward_host_pipelined_single_card_bit_exact(cuda, graphs):
    """Single-card forward_host pipelines host copies against the layer per
    token chunk; the output must be bit-identical to the device path."""
    T, h, E, k = 4096, 1024, 8, 2
    x, logits = _inputs(1, T, h, E, torch.bfloat16, 31)
    layer = MoeLayer(1, 1, E, k, T, h, dtype=torch.bfloat16, max_chunks=16)
    try:
        layer.enable_graphs(graphs)
        cd = layer.cards[0]
        cd.x.copy_(x[0])
        cd.logits.copy_(logits[0])
        layer.forward(BASELINE, 1)
        layer.sync()
        want = cd.out.clone()
        cd.out.zero_()
        cd.x.zero_()
        hx = host_empty((T, h), torch.bfloat16)  # moe_host_alloc buffers (what bench.py uses)
        hx.copy_(x[0].cpu())
        hl = host_empty((T, E), torch.float32)
        hl.copy_(logits[0].cpu())
        ho = host_empty((T, h), torch.bfloat16)
        ho.zero_()
        for _ in range(3):
            layer.forward_host(hx, hl, ho, BASELINE, 1)
        torch.cuda.synchronize()
        layer.sync()
        assert torch.equal(ho.view(torch.int16), want.cpu().view(torch.int16))
    finally:
        layer.close()


def test_host_empty_buffers(cuda):
    """moe_host_alloc tensors: page-locked, writable, freed with their last view."""
    import gc
    t = host_empty((1000, 3), torch.float32)
    assert t.shape == (1000, 3) and t.dtype == torch.float32 and t.is_pinned()
    t.fill_(2.5)
    d = t.cuda(non_blocking=True)
    torch.cuda.synchronize()
    assert float(d.sum()) == 7500.0
    v = t[10:20]
    del t
    gc.collect()
    v.fill_(1.0)  # storage still alive through the view
    assert float(v.sum()) == 30.0
    assert host_empty((0, 4), torch.bfloat16).numel() == 0


@pytest.mark.parametrize("cfg", [
    # (e, t, E, k, T, h, dtype, level, n, landing) — every BASELINE.json config at full size,
    # emulated cards on one GPU (virtual mode), compared with the oracle row for row
    (2, 2, 8, 2, 2048, 1024, torch.float32, O2, 4, LAND_STAGED),      # configs[0] toy layer, fp32, 2x2
    (2, 2, 8, 2, 2048, 1024, torch.float32, BASELINE, 1, LAND_FINAL),
    (2, 4, 8, 2, 4096, 4096, torch.bfloat16, O1, 1, LAND_FINAL),      # configs[1] Mixtral layer, 2x4
    (4, 2, 8, 2, 4096, 4096, torch.bfloat16, O3, 4, LAND_STAGED),     # ... and 4x2
    (2, 4, 2, 1, 8192, 8192, torch.bfloat16, O3, 4, LAND_STAGED),     # configs[2] 2x70B-style, E = e
    (2, 4, 2, 1, 8192, 8192, torch.bfloat16, BASELINE, 1, LAND_FINAL),
    (4, 2, 160, 6, 8192, 5120, torch.bfloat16, O2, 2, LAND_STAGED),   # configs[3] DeepSeek-V2-style, 4x2
    (4, 2, 160, 6, 8192, 5120, torch.bfloat16, O1, 1, LAND_FINAL),
])
def test_full_size_configs_match_oracle(cuda, cfg):
    """Every BASELINE.json config at full T and h, compared with the oracle
    (dataplane.hpp:145-283, 293-347 restated): every card's recv rows and
    tags bit-for-bit in the reference's expert -> source -> token order, the
    staged (pre_copy) layout in chunk -> source -> expert order, and the
    combine per element."""
    e, t, E, k, T, h, dtype, level, n, landing = cfg
    _run(e, t, E, k, T, h, dtype, level, n, landing, seed=E * 13 + h + n)


@pytest.mark.parametrize("cfg", [
    # (e, t, E, k, T, h, level, n, landing) — BASELINE.json configs at full size, emulated cards on one GPU
    (2, 2, 8, 2, 2048, 1024, O2, 4, LAND_STAGED),    # configs[0] toy layer (run here in bf16)
    (2, 4, 8, 2, 4096, 4096, O1, 1, LAND_FINAL),     # configs[1] Mixtral layer, 2x4
    (2, 4, 2, 1, 8192, 8192, O3, 4, LAND_STAGED),    # configs[2] 2x70B-style, E = e
    (4, 2, 160, 6, 8192, 5120, O2, 2, LAND_FINAL),   # configs[3] DeepSeek-V2-style, 4x2
])
def test_full_size_configs_round_trip(cuda, cfg):
    """Size-independent properties at BASELINE.json's full sizes: every landed row
    is bit-identical to the source row its tag names, each (source, position,
    expert) lands exactly once on the node owning the expert, row counts match
    the routing, and combine(dispatch(x)) with identity experts is x * sum(p)."""
    e, t, E, k, T, h, level, n, landing = cfg
    L = E // e
    layer = MoeLayer(e, t, E, k, T, h, dtype=torch.bfloat16, max_chunks=max(n, 1))
    try:
        g = torch.Generator(device="cuda").manual_seed(E * 7 + h)
        xs = [torch.randn(T, h, generator=g, device="cuda").to(torch.bfloat16) for _ in range(e)]
        ls = [torch.randn(T, E, generator=g, device="cuda") for _ in range(e)]
        for cd in layer.cards:
            cd.x.copy_(xs[cd.node])
            cd.logits.copy_(ls[cd.node])
        layer.forward(level, n, landing)
        layer.sync()
        experts = [layer.card(x * t).experts.long() for x in range(e)]
        probs = [layer.card(x * t).probs.double() for x in range(e)]
        for cd in layer.cards:
            rows = layer.recv_rows(cd.card)
            want_rows = sum(int(((ex // L) == cd.node).sum()) for ex in experts)
            assert rows == want_rows, (cd.card, rows, want_rows)
            tags = cd.recv_tags[:rows].long()
            src_node = tags[:, 1] // t
            pos, xpt = tags[:, 2], tags[:, 3]
            assert bool(((xpt // L) == cd.node).all()), "a row landed on a node that does not own its expert"
            key = (src_node * T + pos) * E + xpt
            assert key.unique().numel() == rows, "a (source, position, expert) landed twice"
            for x in range(e):
                sel = src_node == x
                if not bool(sel.any()):
                    continue
                assert torch.equal(cd.recv[:rows][sel].view(torch.int16), xs[x][pos[sel]].view(torch.int16))
                assert bool((experts[x][pos[sel]] == xpt[sel][:, None]).any(1).all()), "tag expert not routed"
            want = xs[cd.node].double() * probs[cd.node].sum(1, keepdim=True)
            err = ((cd.out.double() - want).abs().max() / want.abs().max()).item()
            assert err <= 1e-2, (cd.card, err)
    finally:
        layer.close()


@pytest.mark.parametrize("e,t,level", [(1, 1, BASELINE), (2, 1, BASELINE), (2, 2, O1), (2, 2, O3)])
def test_top1_wide_rows(cuda, e, t, level):
    """Top-1 routing over rows of >= 2048 columns per slice takes the 4 KiB-item
    top-1 un-permute (the 2x70B config's shape class)."""
    _run(e, t, 2 * e, 1, 300, 2048 * t, torch.bfloat16, level, 1 if level != O3 else 2, LAND_FINAL, seed=7 + e + t)


def test_autotune_picks_a_measured_candidate(cuda):
    """moe_ctx_autotune times every candidate in place and returns the fastest
    (times written back); invalid candidates are rejected before any run."""
    layer = MoeLayer(2, 2, 8, 2, 512, 256, dtype=torch.bfloat16, max_chunks=8)
    try:
        x, logits = _inputs(2, 512, 256, 8, torch.bfloat16, 5)
        for cd in layer.cards:
            cd.x.copy_(x[cd.node])
            cd.logits.copy_(logits[cd.node])
        cands = [(O1, 1, LAND_FINAL), (O2, 4, LAND_FINAL), (O3, 2, LAND_STAGED), (BASELINE, 1, LAND_FINAL)]
        best, times = layer.autotune(cands, steps=3)
        assert 0 <= best < len(cands) and all(t > 0 for t in times)
        assert times[best] == min(times)
        with pytest.raises(ValueError):
            layer.autotune([(O1, 3, LAND_FINAL)])  # O1 is unchunked
        layer.forward(*cands[best])
        layer.sync()
    finally:
        layer.close()


@pytest.mark.parametrize("e,t,E,k,level,n,landing", [
    (2, 2, 8, 2, O1, 1, LAND_FINAL), (2, 2, 8, 2, O2, 4, LAND_STAGED), (4, 2, 160, 6, O3, 2, LAND_FINAL),
    (1, 1, 160, 6, BASELINE, 1, LAND_FINAL), (2, 1, 4, 2, BASELINE, 1, LAND_FINAL)])
def test_routing_checks_pass_and_catch_corruption(cuda, e, t, E, k, level, n, landing):
    """moe_ctx_enable_checks: a clean layer passes the device tag check on every
    step; a landed row moved out of place (or lost) raises CorruptRoutingError
    (the reference's exception, dataplane.hpp:18-20) at the next sync."""
    layer = MoeLayer(e, t, E, k, 256, 128, dtype=torch.bfloat16, max_chunks=max(n, 1))
    try:
        layer.enable_checks(True)
        g = torch.Generator(device="cuda").manual_seed(e * 10 + t)
        xs = [torch.randn(256, 128, generator=g, device="cuda").to(torch.bfloat16) for _ in range(e)]
        ls = [torch.randn(256, E, generator=g, device="cuda") for _ in range(e)]
        for cd in layer.cards:  # a node's TP ranks hold the same batch (the dedup relies on it)
            cd.logits.copy_(ls[cd.node])
            cd.x.copy_(xs[cd.node])
        for _ in range(2):
            layer.forward(level, n, landing)
            layer.sync()
        layer.dispatch(level, n, landing)
        layer.verify()
        layer.sync()
        if t > 1:  # TP ranks routing differently (inconsistent replicas) is caught too
            layer.cards[1].logits.copy_(torch.randn(256, E, generator=g, device="cuda"))
            layer.forward(level, n, landing)
            with pytest.raises(_lib.CorruptRoutingError):
                layer.sync()
            layer.cards[1].logits.copy_(ls[layer.cards[1].node])
            layer.forward(level, n, landing)
            layer.sync()
            layer.dispatch(level, n, landing)
            layer.sync()
        cd = layer.cards[-1]
        rows = layer.recv_rows(cd.card)
        assert rows >= 2
        tags = cd.recv_tags[:rows].clone()
        cd.recv_tags[0].copy_(tags[1])            # two rows swapped: out of order
        cd.recv_tags[1].copy_(tags[0])
        layer.verify()
        with pytest.raises(_lib.CorruptRoutingError):
            layer.sync()
        cd.recv_tags[:rows].copy_(tags)
        cd.recv_tags[rows - 1].fill_(-1)          # a row that never landed
        layer.verify()
        with pytest.raises(_lib.CorruptRoutingError):
            layer.sync()
        cd.recv_tags[:rows].copy_(tags)
        layer.verify()
        layer.sync()
        layer.combine(level, n)
        layer.sync()
    finally:
        layer.close()


@pytest.mark.parametrize("level,n", [(BASELINE, 1), (O2, 2)])
def test_link_rate_pacing_changes_timing_not_results(cuda, level, n):
    """moe_ctx_set_link_rate only delays the cross-node legs: same rows, same output."""
    e, t, E, k, T, h = 2, 2, 8, 2, 256, 256
    x, logits = _inputs(e, T, h, E, torch.bfloat16, 17)
    outs = []
    for rate in (0.0, 20.0):
        layer = MoeLayer(e, t, E, k, T, h, dtype=torch.bfloat16, max_chunks=4)
        try:
            layer.set_link_rate(rate)
            for cd in layer.cards:
                cd.x.copy_(x[cd.node])
                cd.logits.copy_(logits[cd.node])
            layer.forward(level, n)
            layer.sync()
            outs.append([(cd.recv[:layer.recv_rows(cd.card)].clone(), cd.out.clone()) for cd in layer.cards])
        finally:
            layer.close()
    for (r0, o0), (r1, o1) in zip(*outs):
        assert torch.equal(r0, r1) and torch.equal(o0, o1)


def test_chunk_count_sequence_matches_fresh_context(cuda):
    """forward at n = 4, then 1, then 8 on one context gives what a fresh
    context gives at n = 8 (the front's per-chunk count buffers are reset for
    every chunk, not just the previous launch's)."""
    e, t, E, k, T, h = 2, 2, 8, 2, 512, 256
    x, logits = _inputs(e, T, h, E, torch.bfloat16, 23)

    def run(seq):
        layer = MoeLayer(e, t, E, k, T, h, dtype=torch.bfloat16, max_chunks=8)
        try:
            for cd in layer.cards:
                cd.x.copy_(x[cd.node])
                cd.logits.copy_(logits[cd.node])
            for lv, n in seq:
                for _ in range(3):
                    layer.forward(lv, n)
            layer.sync()
            return [(cd.recv[:layer.recv_rows(cd.card)].clone(), cd.recv_tags[:layer.recv_rows(cd.card)].clone(),
                     cd.out.clone()) for cd in layer.cards]
        finally:
            layer.close()

    got = run([(O3, 4), (O1, 1), (O3, 8)])
    want = run([(O3, 8)])
    for g, w in zip(got, want):
        assert all(torch.equal(a, b) for a, b in zip(g, w))

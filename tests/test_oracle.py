"""The CPU oracle (oracle/moe_oracle.c, a C restatement of the reference data
plane) pinned against (a) the reference's own known-answer tests, (b) golden
fixtures produced by the reference itself (tests/golden/make_golden.py), and
(c) the live reference (oracle/_ref) on the reference test envelopes — the
oracle is trusted as the checker only after this file passes."""
import os

import numpy as np
import pytest

import oracle

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
needs_ref = pytest.mark.skipif(not oracle.ref_available(), reason="oracle/_ref not built (no /root/reference)")


def _load(name):
    return dict(np.load(os.path.join(GOLD, name)))


def test_router_known_answers():
    k = _load("kats.npz")
    e, p = oracle.route_topk(np.array([[10.0, 0.0, 0.0, 0.0]]), 1)
    assert e.tolist() == [[0]] and abs(p[0, 0] - 1.0) < 1e-3
    e, p = oracle.route_topk(np.array([[1.0, 1.0, 1.0, 1.0]]), 2)
    assert e.tolist() == [[0, 1]] and np.allclose(p, 0.25, rtol=1e-12)
    e, p = oracle.route_topk(np.array([[0.1, 0.9, 0.3, 0.5]]), 2)
    np.testing.assert_array_equal(e, k["route_softmax_experts"])
    np.testing.assert_allclose(p, k["route_softmax_probs"], rtol=1e-12)
    with pytest.raises(oracle.OracleError):
        oracle.route_topk(np.array([[1.0, 2.0]]), 3)
    with pytest.raises(oracle.OracleError):
        oracle.route_topk(np.array([[1.0, 2.0]]), 0)


def test_router_golden():
    r = _load("router.npz")
    for c in range(int(r["count"])):
        e, p = oracle.route_topk(r[f"c{c}_scores"], int(r[f"c{c}_k"]))
        np.testing.assert_array_equal(e, r[f"c{c}_experts"])
        np.testing.assert_allclose(p, r[f"c{c}_probs"], rtol=1e-12)


def test_permute_known_answers():
    k = _load("kats.npz")
    ps, eo, inv, il = oracle.permute(np.array([[1], [0], [1], [0]]))
    np.testing.assert_array_equal(ps, k["permute_alternating_positions"])
    np.testing.assert_array_equal(eo, k["permute_alternating_expert_of"])
    assert ps.tolist() == [1, 3, 0, 2]
    ps, eo, inv, il = oracle.permute(np.array([[0], [0], [1], [1]]))  # already sorted: identity
    assert ps.tolist() == [0, 1, 2, 3] and inv[:, 0].tolist() == [0, 1, 2, 3]


def test_precopy_layout_known_answer():
    k = _load("kats.npz")
    payload = k["precopy_payload"]
    nodes = oracle.Nodes(2, 2, 2, payload.view(np.uint8).reshape(2, 8, -1), k["precopy_experts"])
    fin, stg = nodes.dispatch_chunked(oracle.O2, 2, 8)
    pre = [(int(a), int(b)) for a, b in stg[0][1][:, 1:3]]
    assert pre == [(0, 0), (0, 2), (2, 0), (2, 2), (0, 4), (0, 6), (2, 4), (2, 6)]
    np.testing.assert_array_equal(stg[0][1][:, :3], k["precopy_pre_card0_tags"])
    np.testing.assert_array_equal(fin[0][1][:, :3], k["precopy_fin_card0_tags"])


def test_doubling_expert_known_answer():
    k = _load("kats.npz")
    nodes = oracle.Nodes(2, 1, 2, k["doubling_payload"].view(np.uint8).reshape(2, 2, -1), k["doubling_experts"])
    mono = nodes.dispatch_monolithic()
    doubled = [((r.view(np.int64) * 2).view(np.uint8).reshape(r.shape), tg) for r, tg in mono]
    out, _ = nodes.combine(oracle.I64, doubled, np.ones((2, 2, 1)))
    np.testing.assert_array_equal(out[:, :, 0], [[6.0, 8.0], [10.0, 12.0]])
    np.testing.assert_array_equal(out, k["doubling_combined"])


def test_dataplane_golden_envelopes():
    d = _load("dataplane.npz")
    for c in range(int(d["count"])):
        p = f"c{c}_"
        e, t, n, T, W, k, level = (int(v) for v in d[p + "shape"])
        payload, experts, probs = d[p + "payload"], d[p + "experts"], d[p + "probs"]
        nodes = oracle.Nodes(e, t, e, payload.view(np.uint8).reshape(e, T, -1), experts)
        mono = nodes.dispatch_monolithic()
        fin, stg = nodes.dispatch_chunked(level, n, 8)
        for card in range(e * t):
            x = card // t
            np.testing.assert_array_equal(mono[x][1][:, :3], d[p + f"mono_tags_{card}"])
            np.testing.assert_array_equal(mono[x][0].view(np.int64).reshape(-1, W), d[p + f"mono_payload_{card}"])
            np.testing.assert_array_equal(fin[x][1][:, :3], d[p + f"chunk_tags_{card}"])
            np.testing.assert_array_equal(fin[x][0].view(np.int64).reshape(-1, W), d[p + f"chunk_payload_{card}"])
            np.testing.assert_array_equal(stg[x][1][:, :3], d[p + f"pre_tags_{card}"])
            np.testing.assert_array_equal(stg[x][0].view(np.int64).reshape(-1, W), d[p + f"pre_payload_{card}"])
        out, tok = nodes.combine(oracle.I64, fin, probs)
        np.testing.assert_array_equal(out, d[p + "combined"])  # dyadic gates: exact
        np.testing.assert_array_equal(tok, d[p + "token_ids"])


def test_chunked_validation_matches_reference_order():
    payload = np.zeros((2, 3, 2), np.int64)
    experts = np.array([[[0], [1], [0]], [[0], [1], [0]]], np.int32)
    nodes = oracle.Nodes(2, 2, 2, payload.view(np.uint8).reshape(2, 3, -1), experts)
    for level, n in ((oracle.O2, 2), (oracle.O1, 3), (oracle.BASELINE, 1), (oracle.O2, 0)):
        with pytest.raises(oracle.OracleError):
            nodes.dispatch_chunked(level, n, 8)


def test_missing_expert_output_is_corrupt_routing():
    payload = np.array([[[1], [2]], [[3], [4]]], np.int64)
    experts = np.array([[[0], [1]], [[0], [1]]], np.int32)
    nodes = oracle.Nodes(2, 1, 2, payload.view(np.uint8).reshape(2, 2, -1), experts)
    mono = nodes.dispatch_monolithic()
    mono[0] = (mono[0][0][:-1], mono[0][1][:-1])  # drop one routed token's output
    with pytest.raises(oracle.OracleError) as ei:
        nodes.combine(oracle.I64, mono, np.ones((2, 2, 1)))
    assert ei.value.status == 2


@needs_ref
def test_oracle_equals_live_reference_on_random_envelopes():
    # test_dataplane.cpp:233-251 / :362-390 envelopes, 200 instances
    rng = np.random.default_rng(83)
    for _ in range(200):
        e = 2 * int(rng.integers(1, 3))
        t = 2 * int(rng.integers(1, 3))
        n = int(rng.integers(1, 5))
        T = n * int(rng.integers(1, 4))
        W = t * int(rng.integers(1, 3))
        k = int(rng.integers(1, 3))
        payload = rng.integers(0, 100, (e, T, W)).astype(np.int64)
        experts = np.stack([np.stack([np.sort(rng.choice(e, k, replace=False)) for _ in range(T)]) for _ in range(e)])
        probs = np.full((e, T, k), 1.0 / k)
        level = 1 if n == 1 else int(rng.choice([2, 3]))
        ref = oracle.ref_dataplane(e, t, payload, experts.astype(np.int32), probs, level=level, n=n)
        nodes = oracle.Nodes(e, t, e, payload.view(np.uint8).reshape(e, T, -1), experts)
        fin, stg = nodes.dispatch_chunked(level, n, 8)
        for card in range(e * t):
            np.testing.assert_array_equal(fin[card // t][1][:, :3], ref["cards"][card][0])
            np.testing.assert_array_equal(fin[card // t][0].view(np.int64).reshape(-1, W), ref["cards"][card][1])
            np.testing.assert_array_equal(stg[card // t][1][:, :3], ref["pre"][card][0])
        out, tok = nodes.combine(oracle.I64, fin, probs)
        np.testing.assert_array_equal(out, ref["combined"])


@needs_ref
def test_oracle_router_equals_live_reference():
    rng = np.random.default_rng(3)
    for T, E, k in ((300, 8, 2), (100, 160, 6), (64, 2, 1), (50, 33, 5)):
        s = rng.standard_normal((T, E))
        a, b = oracle.route_topk(s, k), oracle.ref_route_topk(s, k)
        np.testing.assert_array_equal(a[0], b[0])
        np.testing.assert_allclose(a[1], b[1], rtol=1e-14)


def test_generalised_layout_reduces_to_reference_at_E_equals_e():
    # E > e generalisation (SURVEY.md §7 decision 1): node x hosts experts
    # [x*L, (x+1)*L); with L == 1 the final and staged layouts are the
    # reference's.  Check the L > 1 final layout is expert-major then source.
    rng = np.random.default_rng(1)
    e, t, E, T, k = 2, 1, 8, 16, 2
    experts = np.stack([np.stack([np.sort(rng.choice(E, k, replace=False)) for _ in range(T)]) for _ in range(e)])
    x = rng.integers(0, 255, (e, T, 4), dtype=np.uint8)
    nodes = oracle.Nodes(e, t, E, x, experts)
    for node, (rows, tags) in enumerate(nodes.dispatch_monolithic()):
        keys = [(tg[3], tg[1], tg[2]) for tg in tags]  # (expert, source card, position)
        assert keys == sorted(keys)
        assert all(node * (E // e) <= tg[3] < (node + 1) * (E // e) for tg in tags)

"""Generate tests/golden/*.npz from the REFERENCE itself (oracle/_ref, the
unmodified headers of /root/reference/proj/include/moeplan compiled by
oracle/Makefile).  Run here, where /root/reference exists:

    python tests/golden/make_golden.py

Fixtures (all small; committed):
  kats.npz        the reference's own known-answer tests for the data plane
                  (test_dataplane.cpp:72-98, :100-123, :198-231, :341-360)
  dataplane.npz   seeded random envelopes in the shape of
                  test_dataplane.cpp:233-251 / acceptance.cpp:141-214:
                  inputs (int64 payloads, routing) and the reference's
                  dispatch_monolithic, dispatch_chunked (+ pre_copy) and
                  combine_unpermute outputs
  router.npz      route_topk on seeded score matrices (incl. exact ties)
  router_special.npz  route_topk on float32-representable special values:
                  signed zeros, +-inf, subnormals, +-FLT_MAX (value ties the
                  fp32 GPU key path must break exactly as the reference does)
  planner.npz     cost model / chunk search / strategy on seeded inputs
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import oracle  # noqa: E402


def kats():
    out = {}
    e, p = oracle.ref_route_topk(np.array([[10.0, 0.0, 0.0, 0.0]]), 1)
    out["route_dominant_experts"], out["route_dominant_probs"] = e, p
    e, p = oracle.ref_route_topk(np.array([[1.0, 1.0, 1.0, 1.0]]), 2)
    out["route_ties_experts"], out["route_ties_probs"] = e, p
    e, p = oracle.ref_route_topk(np.array([[0.1, 0.9, 0.3, 0.5]]), 2)
    out["route_softmax_experts"], out["route_softmax_probs"] = e, p
    ps, eo, inv, il = oracle.ref_permute(np.array([[1], [0], [1], [0]]))
    out["permute_alternating_positions"], out["permute_alternating_expert_of"] = ps, eo
    # two chunks interleave at the destination until the reorder copy (test_dataplane.cpp:198-231)
    payload = np.zeros((2, 8, 2), np.int64)
    experts = np.zeros((2, 8, 1), np.int32)
    for node in range(2):
        for i in range(8):
            payload[node, i] = [node * 100 + i, node * 100 + i + 50]
            experts[node, i, 0] = i % 2
    r = oracle.ref_dataplane(2, 2, payload, experts, np.ones((2, 8, 1)), level=2, n=2, combine=False)
    out["precopy_payload"], out["precopy_experts"] = payload, experts
    out["precopy_pre_card0_tags"] = r["pre"][0][0]
    out["precopy_fin_card0_tags"] = r["cards"][0][0]
    # a doubling expert doubles the combined output (test_dataplane.cpp:341-360)
    payload = np.array([[[3], [4]], [[5], [6]]], np.int64)
    experts = np.array([[[1], [0]], [[0], [1]]], np.int32)
    r = oracle.ref_dataplane(2, 1, payload, experts, np.ones((2, 2, 1)), level=-1, expert_scale=2)
    out["doubling_payload"], out["doubling_experts"], out["doubling_combined"] = payload, experts, r["combined"]
    np.savez_compressed(os.path.join(HERE, "kats.npz"), **out)


def dataplane(count=40, seed=83):
    rng = np.random.default_rng(seed)
    out = {}
    for c in range(count):
        e = int(rng.choice([2, 4]))
        t = int(rng.choice([1, 2, 4]))
        n = int(rng.integers(1, 5))
        T = n * int(rng.integers(1, 4))
        W = t * int(rng.integers(1, 3))
        k = int(rng.integers(1, 3))
        payload = rng.integers(0, 100, (e, T, W)).astype(np.int64)
        experts = np.zeros((e, T, k), np.int32)
        probs = np.zeros((e, T, k))
        for g in range(e):
            for i in range(T):
                experts[g, i] = np.sort(rng.choice(e, k, replace=False))
                if k == 1:
                    probs[g, i] = [1.0]
                else:
                    pp = float(rng.integers(1, 16)) / 16.0  # dyadic: combine is exact
                    probs[g, i] = [pp, 1.0 - pp]
        level = 1 if n == 1 else int(rng.choice([2, 3]))
        mono = oracle.ref_dataplane(e, t, payload, experts, probs, level=-1, combine=True)
        ch = oracle.ref_dataplane(e, t, payload, experts, probs, level=level, n=n, combine=True)
        p = f"c{c}_"
        out[p + "shape"] = np.array([e, t, n, T, W, k, level])
        out[p + "payload"], out[p + "experts"], out[p + "probs"] = payload, experts, probs
        for card in range(e * t):
            out[p + f"mono_tags_{card}"], out[p + f"mono_payload_{card}"] = mono["cards"][card]
            out[p + f"chunk_tags_{card}"], out[p + f"chunk_payload_{card}"] = ch["cards"][card]
            out[p + f"pre_tags_{card}"], out[p + f"pre_payload_{card}"] = ch["pre"][card]
        out[p + "combined"], out[p + "token_ids"] = ch["combined"], ch["token_ids"]
    out["count"] = np.array(count)
    np.savez_compressed(os.path.join(HERE, "dataplane.npz"), **out)


def router(seed=7):
    rng = np.random.default_rng(seed)
    out = {}
    cases = [(64, 8, 2, False), (33, 2, 1, False), (50, 160, 6, False), (40, 4, 2, True), (17, 16, 4, True),
             (5, 1, 1, False), (21, 64, 8, False)]
    for c, (T, E, k, ties) in enumerate(cases):
        s = rng.integers(0, 4, (T, E)).astype(np.float64) if ties else rng.standard_normal((T, E))
        e, p = oracle.ref_route_topk(s, k)
        out[f"c{c}_scores"], out[f"c{c}_k"], out[f"c{c}_experts"], out[f"c{c}_probs"] = s, np.array(k), e, p
    out["count"] = np.array(len(cases))
    np.savez_compressed(os.path.join(HERE, "router.npz"), **out)


def router_special(seed=11):
    rng = np.random.default_rng(seed)
    f32 = np.float32
    tiny = float(np.finfo(f32).smallest_subnormal)
    pool_finite = np.array([-0.0, 0.0, tiny, -tiny, 2 * tiny, -2 * tiny, float(np.finfo(f32).tiny),
                            1.0, -1.0, float(np.finfo(f32).max), -float(np.finfo(f32).max)], np.float64)
    pool_inf = np.concatenate([pool_finite, [np.inf, -np.inf]])
    out = {"signed_zero_scores": np.array([[-0.0, 0.0], [0.0, -0.0], [-0.0, -0.0]])}
    out["signed_zero_experts"], out["signed_zero_probs"] = oracle.ref_route_topk(out["signed_zero_scores"], 1)
    cases = [(300, 8, 2, pool_finite), (300, 2, 1, pool_finite), (200, 160, 6, pool_finite),
             (300, 37, 5, pool_finite), (300, 8, 2, pool_inf), (200, 160, 6, pool_inf), (100, 4, 4, pool_inf)]
    for c, (T, E, k, pool) in enumerate(cases):
        s = rng.choice(pool, (T, E))
        assert np.array_equal(s.astype(f32).astype(np.float64), s)  # exact in fp32
        e, p = oracle.ref_route_topk(s, k)
        out[f"c{c}_scores"], out[f"c{c}_k"], out[f"c{c}_experts"], out[f"c{c}_probs"] = s, np.array(k), e, p
    out["count"] = np.array(len(cases))
    np.savez_compressed(os.path.join(HERE, "router_special.npz"), **out)


def planner(seed=41, count=60):
    rng = np.random.default_rng(seed)
    out = {}
    for c in range(count):
        curves = []
        for base in (1e4, 2e4, 5e4):
            v, vs, es = base, [], []
            for _ in range(5):
                vs.append(v)
                es.append(float(rng.uniform(0.05, 1.0)))
                v *= 4.0 + int(rng.integers(0, 12))
            curves.append((np.array(vs), np.array(es), 0.0))
        if rng.integers(0, 2):
            curves[0] = (curves[0][0], curves[0][1], 1e4 * float(rng.integers(1, 51)))
        model = (int(rng.integers(1, 5)), int(rng.integers(1, 16385)), 256 << int(rng.integers(0, 6)), 2)
        t, e = int(rng.integers(2, 9)), int(rng.integers(2, 9))
        b1, b2, b3 = 25e9, 200e9, 1.6e12
        ac, ap = float(rng.integers(0, 2)) * 1e-4, float(rng.integers(0, 2)) * 5e-5
        n_cap = int(rng.integers(1, 65))
        lvl, n, tp, alts = oracle.ref_select_strategy(model, t, e, b1, b2, b3, curves, ac, ap, n_cap)
        n2, t2, f2 = oracle.ref_search(2, model, t, e, b1, b2, b3, curves, ac, ap, n_cap)
        n3, t3, f3 = oracle.ref_search(3, model, t, e, b1, b2, b3, curves, ac, ap, n_cap)
        p = f"c{c}_"
        for i, (vv, ee, im) in enumerate(curves):
            out[p + f"curve{i}_v"], out[p + f"curve{i}_e"], out[p + f"curve{i}_imin"] = vv, ee, np.array(im)
        out[p + "model"] = np.array(model)
        out[p + "par"] = np.array([t, e, n_cap])
        out[p + "ov"] = np.array([ac, ap])
        out[p + "decision"] = np.array([lvl, n, tp])
        out[p + "o2"] = np.array([n2, t2, f2])
        out[p + "o3"] = np.array([n3, t3, f3])
    out["count"] = np.array(count)
    np.savez_compressed(os.path.join(HERE, "planner.npz"), **out)


if __name__ == "__main__":
    if not oracle.ref_available():
        oracle.build(ref=True)
    kats()
    dataplane()
    router()
    router_special()
    planner()
    print("golden fixtures written to", HERE)

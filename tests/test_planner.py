"""Planner parity (CPU): the C++ planner in libmonta.so, called through the C
ABI, against (a) the reference's published golden timings (Table 8 of the
paper as pinned by test_commcost.cpp:37-93 / acceptance.cpp:59-137) and
(b) the reference headers themselves (oracle/_ref) on randomised inputs,
with the reference's own tolerances (1e-12 relative on model outputs)."""
import math
import random

import numpy as np
import pytest

import oracle
from paper_2411_00662_b200 import planner as P
from paper_2411_00662_b200.planner import (ClusterSpec, CurvePoint, CurveSet, EfficiencyCurve, ModelSpec,
                                           OverheadModel, ParallelSpec, StrategyLevel)

K_VOLUME, K_B1, K_B2, K_B3 = 256e6, 25e9, 200e9, 1.6e12
K_T, K_E = 8, 2
AA = EfficiencyCurve([CurvePoint(8e6, 0.427), CurvePoint(32e6, 0.632), CurvePoint(256e6, 0.741)])
AG = EfficiencyCurve([CurvePoint(64e6, 0.726), CurvePoint(256e6, 0.776)])
D2D = EfficiencyCurve.constant(0.8)
REF_CURVES = CurveSet(AA, AG, D2D)
CLUSTER = ClusterSpec(2, 8, K_B1, K_B2, K_B3, 312e12, 16)

needs_ref = pytest.mark.skipif(not oracle.ref_available(), reason="oracle/_ref not built")


def within(got, want, rel):
    return abs(got - want) <= rel * abs(want)


def test_golden_table8_timings():
    assert within(P.baseline_time(K_VOLUME, K_E, K_B1, AA), 6.909e-3, 0.005)
    assert within(P.chunk_alltoall_time(K_VOLUME, 1, K_T, K_E, K_B1, AA), 1.012e-3, 0.005)
    assert within(P.chunk_allgather_time(K_VOLUME, 1, K_T, K_B2, AG), 1.443e-3, 0.005)
    assert within(P.chunk_alltoall_time(K_VOLUME, 4, K_T, K_E, K_B1, AA), 0.374e-3, 0.005)
    assert within(P.chunk_allgather_time(K_VOLUME, 4, K_T, K_B2, AG), 0.385e-3, 0.005)
    assert within(P.chunk_d2d_time(K_VOLUME, 4, K_B3, D2D), 0.050e-3, 0.005)
    ratio = P.o1_time(K_VOLUME, K_T, K_E, K_B1, K_B2, REF_CURVES) / P.baseline_time(K_VOLUME, K_E, K_B1, AA)
    assert within(ratio, 2.455 / 6.909, 0.005)
    cal = P.o1_time(K_VOLUME, K_T, K_E, K_B1, K_B2, REF_CURVES) / (P.baseline_time(K_VOLUME, K_E, K_B1, AA) + 0.9e-3)
    assert 0.295 <= cal <= 0.315
    assert P.asymptotic_speedup(8, 2, K_B1, 8 * K_B1, 0.75, 0.75) == 0.21875
    assert P.o2_score(0.374e-3, 0.385e-3, 0.05e-3, 4) == pytest.approx(2.114e-3, rel=1e-9)
    assert P.o3_score(1.0, 2.0, 0.5, 2) == pytest.approx(5.5, rel=1e-12)
    assert P.o3_score(3.0, 1.0, 1.0, 2) == pytest.approx(8.0, rel=1e-12)


def test_traffic_volume():
    assert P.traffic_volume(ModelSpec(b=2, s=8192, h=8192, bpe=2)) == 268435456.0
    assert P.traffic_volume(ModelSpec(b=1, s=4096, h=8192, bpe=2)) == 67108864.0


def test_degenerate_groups_are_pure_overhead():
    assert P.baseline_time(K_VOLUME, 1, K_B1, AA) == 0.0
    assert P.baseline_time(K_VOLUME, 1, K_B1, AA, OverheadModel(2.5e-4, 0.0)) == 2.5e-4
    assert P.chunk_alltoall_time(K_VOLUME, 4, K_T, 1, K_B1, AA, OverheadModel(1e-4, 0)) == 1e-4
    assert P.chunk_allgather_time(K_VOLUME, 4, 1, K_B2, AG, OverheadModel(3e-4, 0)) == 3e-4
    assert P.chunk_d2d_time(0.0, 4, K_B3, D2D) == 0.0


def test_lookup_efficiency_interpolates_in_log_volume():
    c = EfficiencyCurve([CurvePoint(1e6, 0.2), CurvePoint(1e8, 0.6)])
    assert P.lookup_efficiency(c, 1e7) == pytest.approx(0.4, rel=1e-12)
    assert P.lookup_efficiency(c, 1.0) == 0.2
    assert P.lookup_efficiency(c, 1e12) == 0.6
    with pytest.raises(ValueError):
        P.lookup_efficiency(c, 0.0)
    with pytest.raises(ValueError):
        P.lookup_efficiency(EfficiencyCurve([]), 1.0)


def test_argument_validation():
    with pytest.raises(ValueError):
        P.chunk_alltoall_time(1.0, 0, 1, 1, 1.0, AA)
    with pytest.raises(ValueError):
        P.chunk_allgather_time(-1.0, 1, 1, 1.0, AG)
    with pytest.raises(P.StrategyInapplicableError):
        P.o2_search(ModelSpec(b=2, s=8192, h=8192), ParallelSpec(t=1, e=2), CLUSTER, REF_CURVES)
    with pytest.raises(P.StrategyInapplicableError):
        P.asymptotic_speedup(1, 2, 1, 1, 1, 1)
    with pytest.raises(ValueError):
        P.estimate_performance(P.StrategyDecision(), ModelSpec(), ParallelSpec(), CLUSTER, 1, -1.0)


def test_search_behaviour_pins():
    model = ModelSpec(b=2, s=8192, h=8192, a=64, l=80, k=2, bpe=2)
    par = ParallelSpec(d=2, p=1, t=8, e=2)
    flat = CurveSet(EfficiencyCurve.constant(0.6), EfficiencyCurve.constant(0.8), EfficiencyCurve.constant(0.8))
    assert P.o2_search(model, par, CLUSTER, flat, n_cap=16).n_opt == 16
    assert P.o3_search(model, par, CLUSTER, flat, n_cap=16).n_opt == 16
    tiny = ModelSpec(b=2, s=3, h=8192, bpe=2)
    assert P.o2_search(tiny, par, CLUSTER, flat).n_opt == 3
    gated = CurveSet(EfficiencyCurve.constant(0.6, 4e6), EfficiencyCurve.constant(0.8, 4e6),
                     EfficiencyCurve.constant(0.8))
    r = P.o2_search(ModelSpec(b=1, s=2048, h=8192, bpe=2), par, CLUSTER, gated)
    assert r.feasible and r.n_opt == 1
    gated = CurveSet(EfficiencyCurve.constant(0.6, 1e6), EfficiencyCurve.constant(0.8, 1e6),
                     EfficiencyCurve.constant(0.8))
    r = P.o2_search(ModelSpec(b=1, s=128, h=8192, bpe=2), par, CLUSTER, gated)
    assert not r.feasible and r.n_opt == 1 and r.t_pred > 0


def test_select_strategy_pins():
    flat = CurveSet(EfficiencyCurve.constant(0.7), EfficiencyCurve.constant(0.8), EfficiencyCurve.constant(0.8))
    d = P.select_strategy(ModelSpec(b=1, s=1024, h=1024, bpe=2), ParallelSpec(t=1, e=2), CLUSTER, flat)
    assert d.level == StrategyLevel.Baseline and d.n == 1 and len(d.alternatives) == 1
    flat = CurveSet(EfficiencyCurve.constant(0.6), EfficiencyCurve.constant(0.8), EfficiencyCurve.constant(0.8))
    d = P.select_strategy(ModelSpec(b=1, s=512, h=1024, bpe=2), ParallelSpec(t=8, e=2), CLUSTER, flat,
                          OverheadModel(0.5e-3, 0.0))
    assert d.level == StrategyLevel.O1 and d.n == 1
    d = P.select_strategy(ModelSpec(b=4, s=262144, h=8192, bpe=2), ParallelSpec(t=8, e=2), CLUSTER, flat)
    assert d.level == StrategyLevel.O3 and d.n > 1


def test_estimate_performance_comm_free_limit():
    d = P.StrategyDecision(t_pred=0.0)
    perf = P.estimate_performance(d, ModelSpec(b=4, s=2048, h=1024), ParallelSpec(d=8), CLUSTER, 16, 1.0)
    assert perf.step_latency == 1.0
    assert perf.throughput == pytest.approx(4 * 2048 * 8)


def _random_curve(rng, base):
    pts, v = [], base
    for _ in range(5):
        pts.append(CurvePoint(v, rng.uniform(0.05, 1.0)))
        v *= 4.0 + rng.randrange(12)
    return EfficiencyCurve(pts)


def _as_ref(curves: CurveSet):
    return [([p.volume for p in c.points], [p.efficiency for p in c.points], c.i_minimal)
            for c in (curves.alltoall, curves.allgather, curves.d2d)]


@needs_ref
def test_cost_model_matches_reference_randomised():
    rng = random.Random(23)
    for _ in range(300):
        cs = CurveSet(_random_curve(rng, 1e4), _random_curve(rng, 2e4), _random_curve(rng, 5e4))
        vol = rng.uniform(1.0, 1e10)
        n, t, e = 1 + rng.randrange(64), 1 + rng.randrange(8), 1 + rng.randrange(8)
        b1, b2, b3 = rng.uniform(1e9, 1e12), rng.uniform(1e9, 1e12), rng.uniform(1e11, 1e13)
        ov = OverheadModel(rng.choice([0.0, 1e-5, 2e-4]), rng.choice([0.0, 5e-6]))
        got = (P.chunk_alltoall_time(vol, n, t, e, b1, cs.alltoall, ov),
               P.chunk_allgather_time(vol, n, t, b2, cs.allgather, ov),
               P.chunk_d2d_time(vol, n, b3, cs.d2d, ov), P.baseline_time(vol, e, b1, cs.alltoall, ov),
               P.o1_time(vol, t, e, b1, b2, cs, ov))
        want = oracle.ref_chunk_times(vol, n, t, e, b1, b2, b3, _as_ref(cs), ov.alpha_comm, ov.alpha_copy)
        for g, w in zip(got, want):
            assert g == pytest.approx(w, rel=1e-12, abs=0.0)


@needs_ref
def test_search_and_strategy_match_reference_exhaustively():
    rng = random.Random(41)
    for _ in range(150):
        model = ModelSpec(b=1 + rng.randrange(4), s=1 + rng.randrange(16384), h=256 << rng.randrange(6), bpe=2)
        par = ParallelSpec(t=2 + rng.randrange(7), e=2 + rng.randrange(7))
        cs = CurveSet(_random_curve(rng, 1e4), _random_curve(rng, 2e4), _random_curve(rng, 5e4))
        if rng.randrange(2):
            cs.alltoall.i_minimal = 1e4 * (1 + rng.randrange(50))
        if rng.randrange(2):
            cs.allgather.i_minimal = 1e4 * (1 + rng.randrange(50))
        ov = OverheadModel((rng.randrange(2)) * 1e-4, (rng.randrange(2)) * 5e-5)
        n_cap = 1 + rng.randrange(64)
        m = (model.b, model.s, model.h, model.bpe)
        for which, fn in ((2, P.o2_search), (3, P.o3_search)):
            got = fn(model, par, CLUSTER, cs, ov, n_cap)
            n_opt, t_pred, feas = oracle.ref_search(which, m, par.t, par.e, CLUSTER.b1, CLUSTER.b2, CLUSTER.b3,
                                                    _as_ref(cs), ov.alpha_comm, ov.alpha_copy, n_cap)
            assert (got.n_opt, got.feasible) == (n_opt, feas)
            assert got.t_pred == pytest.approx(t_pred, rel=1e-12)
        d = P.select_strategy(model, par, CLUSTER, cs, ov, n_cap)
        lvl, n, tp, alts = oracle.ref_select_strategy(m, par.t, par.e, CLUSTER.b1, CLUSTER.b2, CLUSTER.b3,
                                                      _as_ref(cs), ov.alpha_comm, ov.alpha_copy, n_cap)
        assert (int(d.level), d.n) == (lvl, n)
        assert d.t_pred == pytest.approx(tp, rel=1e-12)
        assert [(int(a.level), a.n) for a in d.alternatives] == [(a[0], a[2]) for a in alts]


@needs_ref
def test_select_strategy_matches_reference_including_t1():
    rng = random.Random(53)
    for _ in range(200):
        model = ModelSpec(b=1 + rng.randrange(4), s=1 + rng.randrange(65536), h=1024, bpe=2)
        par = ParallelSpec(t=1 + rng.randrange(8), e=1 + rng.randrange(4))
        cs = CurveSet(EfficiencyCurve.constant(rng.uniform(0.1, 1)), EfficiencyCurve.constant(rng.uniform(0.1, 1)),
                      EfficiencyCurve.constant(rng.uniform(0.1, 1)))
        ov = OverheadModel((rng.randrange(3)) * 2e-4, 0.0)
        d = P.select_strategy(model, par, CLUSTER, cs, ov)
        lvl, n, tp, _ = oracle.ref_select_strategy((model.b, model.s, model.h, 2), par.t, par.e, CLUSTER.b1,
                                                   CLUSTER.b2, CLUSTER.b3, _as_ref(cs), ov.alpha_comm,
                                                   ov.alpha_copy, 64)
        assert (int(d.level), d.n) == (lvl, n)
        assert d.t_pred == pytest.approx(tp, rel=1e-12)


@needs_ref
def test_calibrate_matches_reference():
    rng = random.Random(7)
    for trial in range(50):
        samples = []
        for prim in ("alltoall", "allgather", "d2d"):
            for _ in range(2 + rng.randrange(6)):
                v = float(rng.choice([1e5, 1e6, 8e6, 3.2e7, 2.56e8, 1e9]))
                samples.append(P.BenchSample(prim, v, v / rng.uniform(1e9, 5e11) + rng.uniform(0, 1e-4)))
        cl = ClusterSpec(2 + rng.randrange(3), 2 + rng.randrange(7), 25e9, 200e9, 1.6e12, 1e15, 16)
        got = P.calibrate(samples, cl)
        pid = {"alltoall": 0, "allgather": 1, "d2d": 2}
        want, ac, ap = oracle.ref_calibrate([(pid[s.primitive], s.volume, s.seconds) for s in samples], cl.nodes,
                                            cl.gpus_per_node, cl.b1, cl.b2, cl.b3)
        for c, (wv, we) in zip((got.curves.alltoall, got.curves.allgather, got.curves.d2d), want):
            assert [p.volume for p in c.points] == list(wv)
            np.testing.assert_allclose([p.efficiency for p in c.points], we, rtol=1e-12)
        assert got.overhead.alpha_comm == pytest.approx(ac, rel=1e-9, abs=1e-18)
        assert got.overhead.alpha_copy == pytest.approx(ap, rel=1e-9, abs=1e-18)


def test_calibrate_errors():
    cl = ClusterSpec(2, 8, 25e9, 200e9, 1.6e12, 1e15, 16)
    with pytest.raises(P.CalibrationError):
        P.calibrate([P.BenchSample("alltoall", 1e6, 1e-3)], cl)
    s = [P.BenchSample(p, v, 1e-3) for p in ("alltoall", "allgather", "d2d") for v in (1e6, 2e6)]
    with pytest.raises(P.CalibrationError):
        P.calibrate(s + [P.BenchSample("bogus", 1.0, 1.0)], cl)
    with pytest.raises(P.CalibrationError):
        P.calibrate(s, ClusterSpec(1, 8, 1, 1, 1, 1, 1))


def test_calibrate_reference_bench_file():
    # the reference's own A800 bench samples (proj/data/bench_2xa800.csv) as a fixture
    import pathlib
    f = pathlib.Path(__file__).parent / "golden" / "bench_2xa800.csv"
    samples = P.read_bench_csv(f)
    cs = P.calibrate(samples, ClusterSpec(2, 8, 25e9, 200e9, 1.6e12, 312e12, 16))
    # round trip: the fitted model reproduces the samples' efficiencies
    assert len(cs.curves.alltoall.points) >= 2 and cs.overhead.alpha_comm >= 0


@needs_ref
def test_pipeline_simulator_matches_reference():
    rng = random.Random(61)
    for _ in range(200):
        level = rng.randrange(4)
        n = 1 + rng.randrange(8)
        tm = P.ChunkTiming(rng.uniform(0, 5), rng.uniform(0, 5), rng.uniform(0, 5), n)
        expert = rng.uniform(0, 3)
        phases = 1 + rng.randrange(2)
        tr = P.simulate(P.build_pipeline(level, n, tm, expert, phases))
        st, en, sm, mk = oracle.ref_simulate_pipeline(level, n, tm.aa, tm.ag, tm.d2d, expert, phases)
        assert len(tr.spans) == len(st)
        np.testing.assert_allclose([s.start for s in tr.spans], st, rtol=1e-12, atol=1e-12)
        np.testing.assert_allclose([s.end for s in tr.spans], en, rtol=1e-12, atol=1e-12)
        assert [int(s.stream) for s in tr.spans] == list(sm)
        assert tr.makespan == pytest.approx(mk, rel=1e-12)


def test_simulator_closed_forms():
    # acceptance #4: one-phase O2/O3 makespans equal the chunk-search closed forms
    # acceptance.cpp:113-137: the closed forms hold when the copy is not the
    # slowest stage (d2d <= max(aa, ag))
    rng = random.Random(4)
    for _ in range(1000):
        n = 1 + rng.randrange(16)
        aa, ag, d2d = rng.uniform(1e-6, 1), rng.uniform(1e-6, 1), rng.uniform(1e-6, 1)
        if d2d > max(aa, ag):
            d2d = max(aa, ag) * rng.uniform(1e-6, 1)
        tm = P.ChunkTiming(aa, ag, d2d, n)
        o2 = P.simulate(P.build_pipeline(StrategyLevel.O2, n, tm, 0.0, 1)).makespan
        o3 = P.simulate(P.build_pipeline(StrategyLevel.O3, n, tm, 0.0, 1)).makespan
        assert abs(o2 - P.o2_score(aa, ag, d2d, n)) <= 1e-9 * max(o2, 1e-12)
        assert abs(o3 - P.o3_score(aa, ag, d2d, n)) <= 1e-9 * max(o3, 1e-12)


def test_simulator_rejects_cycles_and_bad_deps():
    with pytest.raises(P.InvalidGraphError):
        P.simulate([P.SimTask("a", P.Stream.Compute, 1.0, ["b"]), P.SimTask("b", P.Stream.AllToAll, 1.0, ["a"])])
    with pytest.raises(ValueError):
        P.simulate([P.SimTask("a", P.Stream.Compute, 1.0, ["zzz"])])
    with pytest.raises(ValueError):
        P.simulate([P.SimTask("a", P.Stream.Compute, -1.0, [])])
    with pytest.raises(ValueError):
        P.simulate([P.SimTask("a"), P.SimTask("a")])


def test_curve_csv_round_trip(tmp_path):
    c = EfficiencyCurve([CurvePoint(1e5, 0.05), CurvePoint(8e6, 0.427), CurvePoint(2.56e8, 0.741)])
    P.write_curve_csv(tmp_path / "alltoall.csv", c)
    back = P.read_curve_csv(tmp_path / "alltoall.csv")
    assert [(p.volume, p.efficiency) for p in back.points] == [(p.volume, p.efficiency) for p in c.points]
    (tmp_path / "bad.csv").write_text("volume_bytes,efficiency\n2,0.5\n1,0.5\n")
    with pytest.raises(ValueError):
        P.read_curve_csv(tmp_path / "bad.csv")


def test_planner_matches_reference_golden_fixtures():
    """Fixture form of the exhaustive parity (runs where oracle/_ref is absent)."""
    import os
    d = dict(np.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "planner.npz")))
    cl = ClusterSpec(2, 8, 25e9, 200e9, 1.6e12, 312e12, 16)
    for c in range(int(d["count"])):
        p = f"c{c}_"
        cs = CurveSet(*[EfficiencyCurve([CurvePoint(v, e) for v, e in zip(d[p + f"curve{i}_v"], d[p + f"curve{i}_e"])],
                                        float(d[p + f"curve{i}_imin"])) for i in range(3)])
        b, s, h, bpe = (int(v) for v in d[p + "model"])
        t, e, n_cap = (int(v) for v in d[p + "par"])
        ov = OverheadModel(*[float(v) for v in d[p + "ov"]])
        m = ModelSpec(b=b, s=s, h=h, bpe=bpe)
        par = ParallelSpec(t=t, e=e)
        dec = P.select_strategy(m, par, cl, cs, ov, n_cap)
        assert (int(dec.level), dec.n) == (int(d[p + "decision"][0]), int(d[p + "decision"][1]))
        assert dec.t_pred == pytest.approx(float(d[p + "decision"][2]), rel=1e-12)
        for key, fn in (("o2", P.o2_search), ("o3", P.o3_search)):
            r = fn(m, par, cl, cs, ov, n_cap)
            assert (r.n_opt, r.feasible) == (int(d[p + key][0]), bool(d[p + key][2]))
            assert r.t_pred == pytest.approx(float(d[p + key][1]), rel=1e-12)


def test_b200_shared_egress_variant():
    """moe_select_strategy_b200: with shared_egress off it is the reference's
    select_strategy; on, chunked levels score n*(aa+ag) + d2d (+ O2's copy
    backlog) — the AllToAll and the AllGather serialise on one NVSwitch box's
    egress — through the same gates and tie order."""
    rng = random.Random(5)
    for _ in range(200):
        curves = CurveSet(EfficiencyCurve([CurvePoint(1e5, rng.uniform(0.05, 1)), CurvePoint(1e8, rng.uniform(0.05, 1))]),
                          EfficiencyCurve([CurvePoint(1e5, rng.uniform(0.05, 1)), CurvePoint(1e8, rng.uniform(0.05, 1))]),
                          EfficiencyCurve.constant(rng.uniform(0.3, 1)))
        model = ModelSpec(b=1, s=rng.randint(1, 65536), h=4096, bpe=2)
        par = ParallelSpec(t=rng.choice([1, 2, 4, 8]), e=rng.choice([1, 2, 4]))
        cl = ClusterSpec(nodes=2, gpus_per_node=8, b1=rng.uniform(1e10, 8e11), b2=8e11, b3=7e12, peak_flops=1e15)
        ov = P.OverheadModel(rng.choice([0.0, 1e-5]), rng.choice([0.0, 5e-6]))
        ref = P.select_strategy(model, par, cl, curves, ov, n_cap=16)
        off = P.select_strategy_b200(model, par, cl, curves, ov, n_cap=16, shared_egress=False)
        assert (off.level, off.n, off.t_pred) == (ref.level, ref.n, ref.t_pred)
        on = P.select_strategy_b200(model, par, cl, curves, ov, n_cap=16, shared_egress=True)
        assert on.t_pred == min(a.t_pred for a in on.alternatives)
        if par.t >= 2:
            o1 = P.o1_time(P.traffic_volume(model), par.t, par.e, cl.b1, cl.b2, curves, ov)
            assert on.alternatives[0].t_pred == pytest.approx(o1, rel=1e-12)
            V = P.traffic_volume(model)
            aa1 = P.chunk_alltoall_time(V, 1, par.t, par.e, cl.b1, curves.alltoall, ov)
            ag1 = P.chunk_allgather_time(V, 1, par.t, cl.b2, curves.allgather, ov)
            for a in on.alternatives[1:]:
                # both legs share the egress: the unchunked legs + one overhead per extra chunk
                assert a.t_pred == pytest.approx(aa1 + ag1 + (a.n - 1) * ov.alpha_comm, rel=1e-12)
        else:
            assert (on.level, on.n) == (ref.level, ref.n)

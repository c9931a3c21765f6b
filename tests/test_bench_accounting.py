"""CPU checks of bench.py's accounting (no GPU): the exposed-AllToAll interval
arithmetic, the per-leg NVLink byte counts (SURVEY.md §8(d) numerators with
measured routing) and the workload table against BASELINE.json's configs."""
import json
import os

import numpy as np

import bench

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_exposed_alltoall_intervals():
    # AA [0,10) overlapped by AG [4,6) and [8,12): exposed 4 + 2 = 6
    assert bench.exposed([(0, 10)], [(4, 6), (8, 12)]) == 6
    # overlapping AA intervals are merged first; nothing to cover
    assert bench.exposed([(0, 5), (3, 8)], []) == 8
    busy, exp = bench.role_stats([("aa", 0, 0.0, 10.0), ("ag", 0, 10.0, 20.0), ("caa", 0, 30.0, 40.0),
                                  ("unpermute", 0, 35.0, 50.0)])
    assert busy == {"aa": 10.0, "ag": 10.0, "caa": 10.0, "unpermute": 15.0}
    assert exp == 10.0 + 5.0  # serial AA, then the CAA's first half before the un-permute starts


def test_nvlink_leg_bytes_dedup_2x2():
    # node 0 of a 2x2 layout, E=8 (experts 0-3 local), h=64 bf16; 3 tokens, top-2
    experts = np.array([[0, 5], [4, 6], [1, 2]])
    recv_rows = 7  # rows landed on this card: 3 own-node pairs + 4 from node 1
    r = bench.nvlink_legs(experts, e=2, t=2, E=8, T=3, h=64, node=0, dedup=True, recv_rows=recv_rows,
                          busy={"aa": 1.0, "ag": 1.0, "caa": 1.0, "unpermute": 1.0})
    sl = 32 * bench.ELEM  # this rank's half of a row
    assert r["legs"]["aa"]["bytes"] == 3 * sl          # 3 cross-node pairs, slice each
    assert r["legs"]["ag"]["bytes"] == 4 * sl * 1      # 4 received cross rows to 1 TP peer
    assert r["legs"]["caa"]["bytes"] == 4 * sl         # expert outputs of those rows back
    assert r["legs"]["unpermute"]["bytes"] == 3 * sl   # output slice to the TP peer
    assert r["dispatch"]["bytes"] == 7 * sl


def test_nvlink_leg_bytes_naive():
    experts = np.array([[0, 5], [4, 6]])
    r = bench.nvlink_legs(experts, e=2, t=2, E=8, T=2, h=64, node=0, dedup=False, recv_rows=4, busy={})
    full = 64 * bench.ELEM
    assert r["legs"]["aa"]["bytes"] == 3 * full and r["legs"]["ag"]["bytes"] == 0
    assert r["dispatch"]["gbs"] is None  # no trace, no rate


def test_workloads_match_baseline_configs():
    with open(os.path.join(ROOT, "BASELINE.json")) as f:
        cfgs = json.load(f)["configs"]
    w = bench.WORKLOADS
    assert (w["toy"][0]["tokens_per_node"], w["toy"][0]["hidden"], w["toy"][0]["dtype"]) == (2048, 1024, "f32")
    assert "2048 tokens, hidden 1024, 8 experts top-2" in cfgs[0]
    assert (w["mixtral"][0]["hidden"], w["mixtral"][0]["experts"], w["mixtral"][0]["top_k"]) == (4096, 8, 2)
    assert "hidden 4096, 8 experts top-2, seq 4K" in cfgs[1]
    assert (w["70b"][0]["hidden"], w["70b"][0]["experts"], w["70b"][0]["top_k"], w["70b"][0]["tokens_per_node"]) == \
        (8192, 2, 1, 8192)
    assert (w["deepseek"][0]["hidden"], w["deepseek"][0]["experts"], w["deepseek"][0]["top_k"]) == (5120, 160, 6)
    assert w["deepseek"][1][8] == (4, 2) and w["70b"][1][8] == (2, 4)  # EP=4 x TP=2, EP=2 x TP=4
    bench.select_workload("toy")
    try:
        assert bench.ELEM == 4 and bench.CONFIG["workload"].startswith("toy")
    finally:
        bench.select_workload("mixtral")

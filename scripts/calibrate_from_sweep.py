"""Calibrate MoNTA's cost model from the layer's own exchange kernel (2x2).

The round-1 curves (`paper_2411_00662_b200/calibrate.py`) time each primitive
as a standalone copy launch; the dispatch actually runs inside the persistent
exchange kernel, whose role traces (`scripts/sweep_levels.py` ->
roles_busy_us) give the AllToAll, AllGather and reorder busy time of every
level and chunk count.  Each (level, n) contributes one sample per role at the
planner's per-call volume (AllToAll V/(n t), AllGather and D2D V/n, V =
traffic_volume with s = T k) and time busy / n; the reference's `calibrate`
(calibrate.hpp:84-118) turns the samples into curves + overheads.  Then it
prints predicted vs measured dispatch-exchange time per config with the
reference score and the B200 shared-egress score (moe_select_strategy_b200).

    python scripts/calibrate_from_sweep.py profiles/r02/sweep --out profiles/curves_b200/2x2_xchg
"""
import argparse
import glob
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2411_00662_b200 import planner as P  # noqa: E402

CFG = {"mixtral": "mixtral", "deepseek": "deepseek", "70b": "70b", "toy": "toy"}


def load(d):
    out = {}
    for f in sorted(glob.glob(os.path.join(d, "sweep_*.jsonl"))):
        name = os.path.basename(f)[6:-6]
        out[name] = [json.loads(l) for l in open(f) if l.startswith("{")]
    return out


def volume(cfg):
    bench.select_workload(cfg)
    c = bench.CONFIG
    return P.traffic_volume(P.ModelSpec(b=1, s=c["tokens_per_node"] * c["top_k"], h=c["hidden"], bpe=bench.ELEM))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("sweep_dir")
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    runs = load(a.sweep_dir)
    e, t = 2, 2
    samples = []
    for cfg, rows in runs.items():
        V = volume(CFG[cfg])
        for r in rows:
            if r["level"] == "Baseline":
                continue
            n, busy = r["n"], r["roles_busy_us"]
            if busy.get("aa"):
                samples.append(P.BenchSample("alltoall", V / (n * t), busy["aa"] * 1e-6 / n))
            if busy.get("ag"):
                samples.append(P.BenchSample("allgather", V / n, busy["ag"] * 1e-6 / n))
            if busy.get("d2d"):
                samples.append(P.BenchSample("d2d", V / n, busy["d2d"] * 1e-6 / n))
    # FINAL landing writes final offsets from the sender: the engine has no
    # reorder copy.  The reference's calibrate needs >= 2 d2d samples, so the
    # d2d curve comes from the measured HBM copy rate (MEASURED_PEAKS.json)
    if not any(s.primitive == "d2d" for s in samples):
        hbm = bench.load_peaks()[0] * 1e9
        for v in (1 << 20, 1 << 30):
            samples.append(P.BenchSample("d2d", float(v), 2.0 * v / hbm))
    cl = P.b200_cluster(e, t)
    cal = P.calibrate(samples, cl)
    if a.out:
        os.makedirs(a.out, exist_ok=True)
        for name in ("alltoall", "allgather", "d2d"):
            P.write_curve_csv(os.path.join(a.out, f"{name}.csv"), getattr(cal.curves, name))
        json.dump({"alpha_comm": cal.overhead.alpha_comm, "alpha_copy": cal.overhead.alpha_copy},
                  open(os.path.join(a.out, "overhead.json"), "w"))
        with open(os.path.join(a.out, "bench.csv"), "w") as f:
            f.write("primitive,volume_bytes,measured_seconds\n")
            for s in samples:
                f.write(f"{s.primitive},{s.volume:.0f},{s.seconds:.9e}\n")
    report = []
    for cfg, rows in runs.items():
        V = volume(CFG[cfg])
        for r in rows:
            lv, n, meas = r["level"], r["n"], r["dispatch_exchange_us"]
            if lv == "Baseline":
                continue
            aa = P.chunk_alltoall_time(V, n, t, e, cl.b1, cal.curves.alltoall, cal.overhead)
            ag = P.chunk_allgather_time(V, n, t, cl.b2, cal.curves.allgather, cal.overhead)
            dd = P.chunk_d2d_time(V, n, cl.b3, cal.curves.d2d, cal.overhead)
            if lv == "O1":
                ref = b2 = aa + ag
            else:
                ref = (P.o2_score if lv == "O2" else P.o3_score)(aa, ag, dd, n)
                aa1 = P.chunk_alltoall_time(V, 1, t, e, cl.b1, cal.curves.alltoall, cal.overhead)
                ag1 = P.chunk_allgather_time(V, 1, t, cl.b2, cal.curves.allgather, cal.overhead)
                b2 = aa1 + ag1 + (n - 1) * cal.overhead.alpha_comm
            report.append({"config": cfg, "level": lv, "n": n, "measured_us": round(meas, 1),
                           "reference_pred_us": round(ref * 1e6, 1), "b200_pred_us": round(b2 * 1e6, 1),
                           "b200_err": round((b2 * 1e6 - meas) / meas, 3)})
    for x in report:
        print(json.dumps(x))
    print(json.dumps({"overhead": {"alpha_comm": cal.overhead.alpha_comm, "alpha_copy": cal.overhead.alpha_copy},
                      "samples": len(samples)}))


if __name__ == "__main__":
    main()

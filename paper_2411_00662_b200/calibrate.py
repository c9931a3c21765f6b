"""Calibrate MoNTA's cost model on measured B200 NVLink curves (configs[4]).

    torchrun --nproc-per-node N -m paper_2411_00662_b200.calibrate --out profiles/calibration

One process per GPU; the N GPUs are emulated as `nodes` x `gpus_per_node`
groups (2x1, 2x2, 2x4).  For every per-rank volume in 64 KiB .. 1 GiB (x2
steps) it times, with CUDA events and max over ranks:
  alltoall  — every card stores volume/e bytes to each card of its
              expert-parallel group (its own share is a local copy): the
              primitive of chunk_alltoall_time (commcost.hpp:48-60);
  allgather — every card stores volume/t bytes to each of its t-1 TP peers:
              chunk_allgather_time (commcost.hpp:63-75);
  d2d       — a local copy of `volume` bytes: chunk_d2d_time (:77-87);
all with the product's copy kernel (moe_ctx_xfer).  It also sweeps the CTA
count at 64 MiB and times NCCL's all_to_all_single / all_gather_into_tensor
on the same groups and volumes (the transport comparison north_star asks
for).  The samples are written in the reference bench CSV format
(primitive,volume_bytes,measured_seconds) and fitted with the C++
`calibrate` (calibrate.hpp:84-118) into curve CSVs + overhead.json that
bench.py's planner loads.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys

import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2411_00662_b200 import planner as P  # noqa: E402
from paper_2411_00662_b200.layer import MoeLayer  # noqa: E402

TOPO = {2: (2, 1), 4: (2, 2), 8: (2, 4)}
NVLINK_NOMINAL = 900e9


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "calibration"))
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--max-bytes", type=float, default=1 << 30)
    ap.add_argument("--min-bytes", type=float, default=64 << 10)
    ap.add_argument("--row-bytes", type=int, default=16384)
    ap.add_argument("--no-nccl", action="store_true")
    a = ap.parse_args()
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dev = torch.device(f"cuda:{local}")
    dist.init_process_group("nccl", device_id=dev)
    e, t = TOPO.get(world, (world, 1))
    node, rho = rank // t, rank % t
    h = a.row_bytes // 2
    T = int(a.max_bytes) // a.row_bytes  # 1 GiB of rows per card
    layer = MoeLayer(e, t, e, 1, T, h, dtype=torch.bfloat16, max_chunks=1, device=local, rank=rank,
                     world_size=world)
    layer.connect()
    cards = e * t
    stream = torch.cuda.current_stream()
    bar = torch.zeros(1, device=dev)

    ep_group = [x * t + rho for x in range(e)]
    tp_group = [node * t + r for r in range(t)]
    ep_groups = [dist.new_group([x * t + r for x in range(e)]) for r in range(t)]
    tp_groups = [dist.new_group([g * t + r for r in range(t)]) for g in range(e)]
    my_ep, my_tp = ep_groups[rho], tp_groups[node]

    def timed(fn, reps):
        vals = []
        for _ in range(2):
            fn()
        torch.cuda.synchronize()
        for _ in range(reps):
            dist.all_reduce(bar)
            torch.cuda.synchronize()
            s, f = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            # keep the stream busy while the host enqueues, so the events see
            # device time only (no host launch latency)
            torch.cuda._sleep(100000)
            s.record(stream)
            fn()
            f.record(stream)
            torch.cuda.synchronize()
            v = torch.tensor([s.elapsed_time(f) / 1e3], device=dev, dtype=torch.float64)
            dist.all_reduce(v, op=dist.ReduceOp.MAX)
            vals.append(float(v.item()))
        return statistics.median(vals)

    vols = []
    v = a.min_bytes
    while v <= a.max_bytes:
        vols.append(int(v))
        v *= 2
    samples, report = [], {"world": world, "topology": f"{e}x{t}", "row_bytes": a.row_bytes, "points": []}

    def rows_for(nbytes):
        return max(1, int(nbytes) // a.row_bytes)

    for V in vols:
        pt = {"volume": V}
        if e > 1:
            per = [0] * cards
            for c in ep_group:
                per[c] = rows_for(V / e)
            sec = timed(lambda: layer.xfer(per, a.row_bytes, 0, stream), a.reps)
            samples.append(P.BenchSample("alltoall", float(V), sec))
            pt["alltoall_s"] = sec
            pt["alltoall_eff"] = (e - 1) / e * V / (NVLINK_NOMINAL * sec)
        if t > 1:
            per = [0] * cards
            for c in tp_group:
                if c != rank:
                    per[c] = rows_for(V / t)
            sec = timed(lambda: layer.xfer(per, a.row_bytes, 0, stream), a.reps)
            samples.append(P.BenchSample("allgather", float(V), sec))
            pt["allgather_s"] = sec
            pt["allgather_eff"] = (t - 1) / t * V / (NVLINK_NOMINAL * sec)
        per = [0] * cards
        per[rank] = rows_for(V)
        sec = timed(lambda: layer.xfer(per, a.row_bytes, 0, stream), a.reps)
        samples.append(P.BenchSample("d2d", float(V), sec))
        pt["d2d_s"] = sec
        if not a.no_nccl and V <= (256 << 20):
            if e > 1:
                src = torch.empty(V // 2, dtype=torch.bfloat16, device=dev)
                dst = torch.empty_like(src)
                pt["nccl_alltoall_s"] = timed(lambda: dist.all_to_all_single(dst, src, group=my_ep), a.reps)
            if t > 1:
                part = torch.empty(V // t // 2, dtype=torch.bfloat16, device=dev)
                full = torch.empty(part.numel() * t, dtype=torch.bfloat16, device=dev)
                pt["nccl_allgather_s"] = timed(lambda: dist.all_gather_into_tensor(full, part, group=my_tp), a.reps)
        report["points"].append(pt)
        if rank == 0:
            print(json.dumps(pt), flush=True)

    # CTA-count sweep of the AllToAll leg at 64 MiB per rank
    sweep = {}
    if e > 1:
        V = 64 << 20
        per = [0] * cards
        for c in ep_group:
            per[c] = rows_for(V / e)
        for grid in (8, 16, 32, 64, 128, 148, 296, 592, 1184):
            sec = timed(lambda: layer.xfer(per, a.row_bytes, grid, stream), a.reps)
            sweep[grid] = {"s": sec, "GBps_cross_node": (e - 1) / e * V / sec / 1e9}
    report["aa_grid_sweep_64MiB"] = sweep

    if rank == 0:
        out = os.path.join(a.out, f"{e}x{t}")
        os.makedirs(out, exist_ok=True)
        P.write_bench_csv(os.path.join(out, "bench.csv"), samples)
        with open(os.path.join(out, "report.json"), "w") as f:
            json.dump(report, f, indent=1)
        if e >= 2 and t >= 2:
            cl = P.b200_cluster(e, t, b1=NVLINK_NOMINAL, b2=NVLINK_NOMINAL, b3=6543.1e9 / 2)
            cs = P.calibrate(samples, cl)
            for name, c in (("alltoall", cs.curves.alltoall), ("allgather", cs.curves.allgather),
                            ("d2d", cs.curves.d2d)):
                P.write_curve_csv(os.path.join(out, f"{name}.csv"), c)
            with open(os.path.join(out, "overhead.json"), "w") as f:
                json.dump({"alpha_comm": cs.overhead.alpha_comm, "alpha_copy": cs.overhead.alpha_copy}, f)
        print(json.dumps({"sweep": sweep}), flush=True)
    layer.close()
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()

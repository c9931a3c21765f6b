"""EP > DP priority under contention (PAPER.md
"Communication Conflict"): the MoE layer (EP dispatch + combine) timed while
a DP gradient all-reduce (NCCL, large bucket) runs concurrently on another
stream, with the DP stream at (a) the EP stream's priority and (b) the DP
priority the library assigns (moe_comm_stream_priority).  Also the layer
alone.  One JSON line (rank 0), max over ranks.

    torchrun --nproc-per-node 2 scripts/micro/priority_bench.py [--config mixtral]
"""
import argparse
import json
import os
import sys

import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from paper_2411_00662_b200 import _lib, ops  # noqa: E402
from paper_2411_00662_b200.layer import MoeLayer, BASELINE, O1  # noqa: E402

SHAPES = {"mixtral": (4096, 4096, 8, 2), "deepseek": (8192, 5120, 160, 6)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="mixtral")
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--dp-mib", type=int, default=512)
    ap.add_argument("--gap-cycles", type=int, default=400000, help="non-MoE compute between layers (~200 us)")
    args = ap.parse_args()
    world, rank, local = int(os.environ["WORLD_SIZE"]), int(os.environ["RANK"]), int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    T, h, E, k = SHAPES[args.config]
    e, t = (world, 1) if world <= 2 else (world // 2, 2)
    level = BASELINE if t == 1 else O1
    layer = MoeLayer(e, t, E, k, T, h, dtype=torch.bfloat16, max_chunks=4, device=local, rank=rank,
                     world_size=world)
    layer.connect()
    layer.enable_graphs(True)
    cd = layer.cards[0]
    g = torch.Generator(device=f"cuda:{local}").manual_seed(rank)
    cd.x.copy_(torch.randn(T, h, generator=g, device=f"cuda:{local}").to(torch.bfloat16))
    cd.logits.copy_(torch.randn(T, E, generator=g, device=f"cuda:{local}"))
    ep = ops.comm_stream(_lib.COMM_EP)
    bucket = torch.ones(args.dp_mib << 18, dtype=torch.float32, device=f"cuda:{local}")

    chunks = 16  # the DP bucket all-reduced in chunks (what the gate schedules around)
    pieces = bucket.chunk(chunks)

    def run(mode):
        dp = None
        if mode == "equal":
            dp = torch.cuda.Stream(priority=ops.comm_stream_priority(_lib.COMM_EP))
        elif mode == "mapped":
            dp = ops.comm_stream(_lib.COMM_DP)
        for _ in range(3):
            layer.forward(level, 1, 0, ep)
        torch.cuda.synchronize()
        dist.barrier()
        d0, d1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        if dp is not None:  # keep the DP all-reduces running through the whole timed window
            dp.wait_stream(torch.cuda.current_stream())
            d0.record(dp)
            with torch.cuda.stream(dp):
                for _ in range(args.steps * 2):
                    for p in pieces:
                        dist.all_reduce(p)
            d1.record(dp)
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
        for a, b in evs:
            a.record(ep)
            layer.forward(level, 1, 0, ep)
            b.record(ep)
            torch.cuda._sleep(args.gap_cycles)  # the step's non-MoE compute between MoE layers
        torch.cuda.synchronize()
        us = sorted(a.elapsed_time(b) * 1e3 for a, b in evs)
        med = torch.tensor([us[len(us) // 2]], dtype=torch.float64, device=f"cuda:{local}")
        dist.all_reduce(med, op=dist.ReduceOp.MAX)
        dp_us = d0.elapsed_time(d1) * 1e3 / (args.steps * 2) if dp is not None else None
        return float(med.item()), dp_us

    def dp_alone():
        dp = ops.comm_stream(_lib.COMM_DP)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(dp)
        with torch.cuda.stream(dp):
            for p in pieces:
                dist.all_reduce(p)
        b.record(dp)
        torch.cuda.synchronize()
        return a.elapsed_time(b) * 1e3

    out = {"config": args.config, "topology": f"{e}x{t}", "level": _lib.LEVEL_NAMES[level], "dp_bucket_mib": args.dp_mib,
           "stream_priorities": {n: ops.comm_stream_priority(gr) for n, gr in
                                 (("EP", _lib.COMM_EP), ("PP", _lib.COMM_PP), ("CP", _lib.COMM_CP),
                                  ("DP", _lib.COMM_DP), ("TP_SP", _lib.COMM_TP_SP))}}
    for mode in ("alone", "equal", "mapped", "alone"):
        lay, dp_us = run(mode)
        out.setdefault("layer_us_median", {}).setdefault(mode, []).append(lay)
        if dp_us is not None:
            out.setdefault("dp_bucket_us_during", {})[mode] = dp_us
    out["dp_bucket_allreduce_us_alone"] = dp_alone()
    if rank == 0:
        print(json.dumps(out), flush=True)
    layer.close()
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()

"""Measured dispatch+combine time per (level, n) at one topology, next to the
MoNTA planner's prediction — the validation half of configs[4].

    torchrun --nproc-per-node N scripts/sweep_levels.py [--tokens 4096 --hidden 4096 --experts 8 --topk 2]

Prints one JSON line per (level, n) from rank 0: measured us/layer (CUDA
events, max over ranks, L2 flushed between steps, CUDA graphs), exposed
AllToAll (per-kernel events), and the planner's t_pred for the dispatch
phase with the calibrated curves in profiles/curves_b200/<e>x<t>/.
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ["NCCL_DEBUG"] = "WARN"

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import bench  # noqa: E402
from paper_2411_00662_b200 import planner as P  # noqa: E402
from paper_2411_00662_b200.layer import MoeLayer, BASELINE, O1, O2, O3  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tokens", type=int, default=4096)
    ap.add_argument("--hidden", type=int, default=4096)
    ap.add_argument("--experts", type=int, default=8)
    ap.add_argument("--topk", type=int, default=2)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--config", default=None, help="a bench.py workload name (overrides the shape flags)")
    a = ap.parse_args()
    world, rank = int(os.environ["WORLD_SIZE"]), int(os.environ["RANK"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    if a.config:
        bench.select_workload(a.config)
        a.tokens, a.hidden, a.experts, a.topk = (bench.CONFIG[x] for x in ("tokens_per_node", "hidden", "experts",
                                                                            "top_k"))
    e, t = bench.topo_for(world)
    T, h, E, k = a.tokens, a.hidden, a.experts, a.topk
    PD = bench.payload_dtype() if a.config else torch.bfloat16
    layer = MoeLayer(e, t, E, k, T, h, dtype=PD, max_chunks=16, device=local, rank=rank, world_size=world)
    layer.connect()
    layer.enable_graphs(True)
    cd = layer.cards[0]
    g = torch.Generator(device=f"cuda:{local}").manual_seed(99 + cd.node)
    cd.x.copy_(torch.randn(T, h, generator=g, device=f"cuda:{local}").to(PD))
    cd.logits.copy_(torch.randn(T, E, generator=g, device=f"cuda:{local}"))
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=f"cuda:{local}")
    bar = torch.zeros(1, device=f"cuda:{local}")
    stream = torch.cuda.current_stream()
    try:
        cdir = os.path.join(ROOT, "profiles", "curves_b200", f"{e}x{t}")
        curves = P.load_curve_set(cdir)
        ov = P.OverheadModel(**json.load(open(os.path.join(cdir, "overhead.json"))))
    except Exception:
        curves, ov = None, None
    combos = [(BASELINE, 1)]
    if t > 1:
        combos += [(O1, 1)] + [(lv, n) for lv in (O2, O3) for n in (2, 4, 8, 16)]
    for lv, n in combos:
        def step():
            layer.forward(lv, n, 0, stream)
        for _ in range(3):
            step()
        layer.sync()
        tot = 0.0
        for _ in range(a.steps):
            flush.zero_()
            dist.all_reduce(bar)
            s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s0.record(stream)
            step()
            s1.record(stream)
            torch.cuda.synchronize()
            tot += s0.elapsed_time(s1)
        v = torch.tensor([tot / a.steps * 1e3], device=f"cuda:{local}", dtype=torch.float64)
        dist.all_reduce(v, op=dist.ReduceOp.MAX)
        layer.enable_timing(True)
        exp = []
        for _ in range(3):
            flush.zero_()
            dist.all_reduce(bar)
            step()
            busy, ex = bench.role_stats(layer.xchg_trace())
            exp.append(ex)
            roles = busy
        disp = []
        for _ in range(3):  # the dispatch exchange alone (the span of its kernel[s]), as the planner predicts it
            flush.zero_()
            dist.all_reduce(bar)
            step()
            disp.append(sum((b - a) * 1e3 for st, j, a, b in layer.spans() if st in ("aa", "ag", "d2d")))
        layer.enable_timing(False)
        pred, pred_b200 = None, None
        if curves is not None and lv != BASELINE:
            m = P.ModelSpec(b=1, s=T * k, h=h, bpe=torch.empty((), dtype=PD).element_size())
            par = P.ParallelSpec(t=t, e=e)
            cl = P.b200_cluster(e, t)
            if lv == O1:
                pred = pred_b200 = P.o1_time(P.traffic_volume(m), t, e, cl.b1, cl.b2, curves, ov)
            else:
                vol = P.traffic_volume(m)
                aa, ag, dd = (P.chunk_alltoall_time(vol, n, t, e, cl.b1, curves.alltoall, ov),
                              P.chunk_allgather_time(vol, n, t, cl.b2, curves.allgather, ov),
                              P.chunk_d2d_time(vol, n, cl.b3, curves.d2d, ov))
                pred = (P.o2_score if lv == O2 else P.o3_score)(aa, ag, dd, n)
                # the B200 shared-egress score (moe_select_strategy_b200)
                aa1 = P.chunk_alltoall_time(vol, 1, t, e, cl.b1, curves.alltoall, ov)
                ag1 = P.chunk_allgather_time(vol, 1, t, cl.b2, curves.allgather, ov)
                pred_b200 = aa1 + ag1 + (n - 1) * ov.alpha_comm
        if rank == 0:
            print(json.dumps({"topology": f"{e}x{t}", "level": ["Baseline", "O1", "O2", "O3"][lv], "n": n,
                              "us_per_layer": float(v.item()), "exposed_alltoall_us": sum(exp) / len(exp),
                              "roles_busy_us": {r: round(x, 1) for r, x in roles.items()},
                              "dispatch_exchange_us": sum(disp) / len(disp),
                              "planner_dispatch_pred_us": None if pred is None else pred * 1e6,
                              "b200_shared_egress_pred_us": None if pred_b200 is None else pred_b200 * 1e6}),
                  flush=True)
    layer.close()
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()

"""Multi-card layer backward vs forward time (one process per GPU).

    torchrun --nproc-per-node 4 scripts/micro/backward_layer_bench.py [--level 1 --chunks 1]

Mixtral layer (T=4096 per node, h=4096, E=8, top-2, bf16) at e x t from
bench.topo_for(world).  Times, with CUDA events max over ranks, L2 flushed
before each: the forward dispatch + combine, and the backward =
combine_backward (gradient dispatch + adjoint kernels + metadata all-gather
+ scatter) followed by dispatch_backward (unit-weight combine, which mirrors
that gradient dispatch).  Prints one JSON line from rank 0.
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import bench  # noqa: E402
from paper_2411_00662_b200 import layer_backward as LB  # noqa: E402
from paper_2411_00662_b200.layer import LAND_FINAL, MoeLayer  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--level", type=int, default=1)
    ap.add_argument("--chunks", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    a = ap.parse_args()
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    e, t = bench.topo_for(world)
    level = a.level if t > 1 else 0
    T, h, E, k = 4096, 4096, 8, 2
    dev = torch.device(f"cuda:{local}")
    layer = MoeLayer(e, t, E, k, T, h, dtype=torch.bfloat16, max_chunks=max(a.chunks, 1), device=local, rank=rank,
                     world_size=world)
    layer.connect()
    cd = layer.cards[0]
    g = torch.Generator(device=dev).manual_seed(3 + cd.node)
    x = torch.randn(T, h, generator=g, device=dev).to(torch.bfloat16)
    gout = torch.randn(T, h, generator=g, device=dev).to(torch.bfloat16)
    cd.logits.copy_(torch.randn(T, E, generator=g, device=dev))
    layer.route()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)

    def timed(fn):
        ts = []
        for i in range(a.steps + 3):
            flush.zero_()
            dist.barrier()
            torch.cuda.synchronize()
            s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s0.record()
            fn()
            s1.record()
            torch.cuda.synchronize()
            if i >= 3:
                ts.append(s0.elapsed_time(s1) * 1e3)
        v = torch.tensor([sum(ts) / len(ts)], dtype=torch.float64, device=dev)
        dist.all_reduce(v, op=dist.ReduceOp.MAX)
        return float(v.item())

    def fwd():
        cd.x.copy_(x)
        layer.dispatch(level, a.chunks, LAND_FINAL)
        layer.combine(level, a.chunks)

    fwd_us = timed(fwd)
    layer.sync()
    rows = layer.recv_rows(cd.card)
    y = {cd.card: cd.recv[:rows].clone()}
    grad_rows = {cd.card: cd.recv[:rows].clone()}

    def bwd():  # the combine exchange of dispatch_backward mirrors the gradient dispatch of combine_backward
        LB.combine_backward(layer, {cd.card: gout}, y, level, a.chunks, LAND_FINAL)
        LB.dispatch_backward(layer, grad_rows, level, a.chunks)

    bwd_us = timed(bwd)

    def bwd_ctx():  # the whole backward inside the context (moe_ctx_backward): no host round trip
        cd.x.copy_(gout)
        layer.backward(level, a.chunks)

    ctx_us = timed(bwd_ctx)
    layer.enable_graphs(True)
    ctxg_us = timed(bwd_ctx)  # the backward as one replayed CUDA graph

    def fwd_graph():
        cd.x.copy_(x)
        layer.forward(level, a.chunks, LAND_FINAL)

    fwdg_us = timed(fwd_graph)
    layer.enable_graphs(False)
    if rank == 0:
        print(json.dumps({"workload": "mixtral-8x7b-moe-layer", "topology": f"{e}x{t}", "level": level,
                          "chunks": a.chunks, "forward_us": fwd_us, "backward_us": bwd_us,
                          "ctx_backward_us": ctx_us, "ctx_backward_graph_us": ctxg_us,
                          "forward_route_graph_us": fwdg_us,
                          "note": "host-timed regions include the Python orchestration, the syncs inside "
                                  "combine_backward/dispatch_backward and the metadata all-gathers; no CUDA "
                                  "graphs; max over ranks"}), flush=True)
    layer.close()
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()

"""Multi-process worker for tests/test_multigpu.py (one rank per GPU).

    python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 \
        --master-port P tests/mp_worker.py --out DIR --e E --t T ...

Each rank owns card == rank of an e x t topology, fills its node's batch
(seeded by node so TP peers hold identical inputs), runs dispatch and
combine over NVLink peer memory, and saves its buffers to DIR/rank{r}.npz
for the parent test to compare with the CPU oracle.
"""
import argparse
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2411_00662_b200.layer import MoeLayer  # noqa: E402


def expert_weights(E, F, h, seed=777):
    """Deterministic SwiGLU expert weights (CPU), shared with the parent test."""
    g = torch.Generator().manual_seed(seed)
    wg = (torch.randn(E, F, h, generator=g) / h ** 0.5).to(torch.bfloat16)
    wu = (torch.randn(E, F, h, generator=g) / h ** 0.5).to(torch.bfloat16)
    w2 = (torch.randn(E, h, F, generator=g) / F ** 0.5).to(torch.bfloat16)
    return wg, wu, w2


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", required=True)
    ap.add_argument("--groups", dest="e", type=int, required=True)
    ap.add_argument("--tp", dest="t", type=int, required=True)
    ap.add_argument("--experts", dest="E", type=int, default=8)
    ap.add_argument("--topk", dest="k", type=int, default=2)
    ap.add_argument("--tokens", dest="T", type=int, default=256)
    ap.add_argument("--hidden", dest="h", type=int, default=256)
    ap.add_argument("--dtype", default="bf16")
    ap.add_argument("--runs", default="0:1:0")  # level:n:landing,...
    ap.add_argument("--repeat", type=int, default=2)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--graphs", type=int, default=0)
    ap.add_argument("--persistent", type=int, default=1)
    ap.add_argument("--ffn", type=int, default=0)  # > 0: SwiGLU experts of this size bound on every card
    ap.add_argument("--host", type=int, default=0)  # 1: also forward_host (pipelined host copies) vs forward
    ap.add_argument("--node-dedup", type=int, default=1)  # 0 off, 1 on (the tests' default), 2 auto
    a = ap.parse_args()
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    ngpu = torch.cuda.device_count()
    if world > ngpu:
        # oversubscribed (test-only): several cards per GPU, one process each,
        # time-sliced; NCCL refuses duplicate GPUs, so the plumbing runs on gloo
        local %= ngpu
        torch.cuda.set_device(local)
        dist.init_process_group("gloo")
    else:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    dt = {"bf16": torch.bfloat16, "f32": torch.float32}[a.dtype]
    layer = MoeLayer(a.e, a.t, a.E, a.k, a.T, a.h, dtype=dt, max_chunks=16, device=local, rank=rank,
                     world_size=world)
    layer.connect()
    layer.enable_graphs(bool(a.graphs))
    layer.set_persistent(bool(a.persistent))
    layer.set_node_dedup(a.node_dedup)
    cd = layer.cards[0]
    node = cd.node
    g = torch.Generator().manual_seed(a.seed * 1000 + node)
    x = torch.randn(a.T, a.h, generator=g).to(dt)
    logits = torch.randn(a.T, a.E, generator=g)
    cd.x.copy_(x.cuda())
    cd.logits.copy_(logits.cuda())
    if a.ffn:
        from paper_2411_00662_b200 import ops
        wg, wu, w2 = expert_weights(a.E, a.ffn, a.h)
        L = a.E // a.e
        sl = slice(node * L, (node + 1) * L)
        w13 = ops.interleave_w13(wg[sl].cuda(), wu[sl].cuda())
        layer.bind_experts(cd.card, w13, w2[sl].contiguous().cuda())
    results = {}
    for spec in a.runs.split(","):
        level, n, landing = (int(v) for v in spec.split(":"))
        for _ in range(a.repeat + (2 if a.graphs else 0)):  # repeated steps: epoch flags, buffer reuse, replays
            layer.forward(level, n, landing)
        layer.sync()
        rows = layer.recv_rows(cd.card)
        key = f"{level}_{n}_{landing}"
        results[f"recv_{key}"] = cd.recv[:rows].contiguous().view(torch.uint8).cpu().numpy()
        results[f"tags_{key}"] = cd.recv_tags[:rows].cpu().numpy()
        if landing == 1:
            results[f"pre_{key}"] = cd.pre[:rows].contiguous().view(torch.uint8).cpu().numpy()
            results[f"pretags_{key}"] = cd.pre_tags[:rows].cpu().numpy()
        results[f"out_{key}"] = cd.out.float().cpu().numpy()
        if a.ffn:  # the fused down-projection + reverse AllToAll must give the sequential result bit for bit
            out_on = cd.out.clone()
            layer.set_expert_overlap(False)
            layer.forward(level, n, landing)
            layer.sync()
            results[f"overlap_same_{key}"] = np.array([bool(torch.equal(out_on, cd.out))])
            layer.set_expert_overlap(True)
    if a.host:  # forward_host (host copies pipelined per chunk) must equal forward on device buffers
        from paper_2411_00662_b200 import ops
        level, n, landing = (int(v) for v in a.runs.split(",")[0].split(":"))
        layer.forward(level, n, landing)
        layer.sync()
        want = cd.out.clone()
        hx = ops.host_empty(tuple(x.shape), dt)
        hx.copy_(x)
        hl = ops.host_empty(tuple(logits.shape), torch.float32)
        hl.copy_(logits)
        ho = ops.host_empty(tuple(want.shape), want.dtype)
        cd.out.zero_()
        cd.x.zero_()  # forward_host must bring its own rows up
        for _ in range(2):
            layer.forward_host(hx, hl, ho, level, n, landing)
        layer.sync()
        results["host_same"] = np.array([bool(torch.equal(ho.cuda(), want))])
        cd.x.copy_(x.cuda())
    results["experts"] = cd.experts.cpu().numpy()
    results["probs"] = cd.probs.double().cpu().numpy()
    results["x"] = x.contiguous().view(torch.uint8).numpy()
    np.savez(os.path.join(a.out, f"rank{rank}.npz"), **results)
    dist.barrier()
    layer.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()

"""forward_host (pipelined host copies) vs forward at full size on N GPUs (dev tool):
    torchrun --nproc-per-node N scripts/host_pipe_check.py E k T h level n graphs [lv:n:landing,...]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2411_00662_b200 import ops  # noqa: E402
from paper_2411_00662_b200.layer import MoeLayer  # noqa: E402


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", device_id=torch.device(f"cuda:{rank}"))
    E, k, T, h, level, n, graphs = (int(v) for v in sys.argv[1:8])
    e, t = (2, 1) if world == 2 else (2, 2)
    layer = MoeLayer(e, t, E, k, T, h, dtype=torch.bfloat16, max_chunks=16, device=rank, rank=rank, world_size=world)
    layer.connect()
    layer.enable_graphs(bool(graphs))
    cd = layer.cards[0]
    g = torch.Generator().manual_seed(cd.node)
    x = torch.randn(T, h, generator=g).to(torch.bfloat16)
    lg = torch.randn(T, E, generator=g)
    cd.x.copy_(x.cuda())
    cd.logits.copy_(lg.cuda())
    # optional warm-up schedules before the check, "lv:n:landing,..." (argv[8])
    for spec in (sys.argv[8].split(",") if len(sys.argv) > 8 and sys.argv[8] else []):
        lv, nn, ld = (int(v) for v in spec.split(":"))
        for _ in range(3):
            layer.forward(lv, nn, ld)
        layer.sync()
        print(f"rank {rank} warm-up {spec} ok", flush=True)
    layer.forward(level, n)
    layer.sync()
    print(f"rank {rank} forward {level}:{n} ok", flush=True)
    want = cd.out.clone()
    if os.environ.get("CHECK_PER_LAUNCH"):  # the per-launch exchange at O3 n=8 instead of forward_host
        layer.set_persistent(False)
        for i in range(3):
            layer.forward(3, 8, 0)
            layer.sync()
            print(f"rank {rank} per-launch step {i}: same = {torch.equal(cd.out, want)}", flush=True)
        dist.barrier()
        layer.close()
        dist.destroy_process_group()
        return
    hx = ops.host_empty((T, h), torch.bfloat16)
    hx.copy_(x)
    hl = ops.host_empty((T, E), torch.float32)
    hl.copy_(lg)
    ho = ops.host_empty((T, h), torch.bfloat16)
    for i in range(3):
        layer.forward_host(hx, hl, ho, level, n)
        layer.sync()
        print(f"rank {rank} step {i}: same = {torch.equal(ho.cuda(), want)}", flush=True)
    dist.barrier()
    layer.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()

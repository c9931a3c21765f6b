"""Per-stage spans of one layer step with DeepSeek-shaped experts bound, the
the reverse AllToAll fused into the down-projection epilogue or not (dev tool):
    torchrun --nproc-per-node 2 scripts/overlap_timeline.py [groups ...]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2411_00662_b200 import ops  # noqa: E402
from paper_2411_00662_b200.layer import MoeLayer, BASELINE, O1  # noqa: E402


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", device_id=torch.device(f"cuda:{rank}"))
    e, t = (2, 1) if world == 2 else (2, 2)
    T, h, E, k, F = 8192, 5120, 160, 6, 1536
    layer = MoeLayer(e, t, E, k, T, h, dtype=torch.bfloat16, max_chunks=8, device=rank, rank=rank, world_size=world)
    layer.connect()
    layer.enable_graphs(True)
    cd = layer.cards[0]
    cd.x.normal_()
    cd.logits.normal_()
    L = E // e
    wg = (torch.randn(L, F, h, device="cuda") * h ** -0.5).to(torch.bfloat16)
    wu = (torch.randn(L, F, h, device="cuda") * h ** -0.5).to(torch.bfloat16)
    w13 = ops.interleave_w13(wg, wu)
    del wg, wu
    w2 = (torch.randn(L, h, F, device="cuda") * F ** -0.5).to(torch.bfloat16)
    layer.bind_experts(cd.card, w13, w2)
    level = BASELINE if t == 1 else O1
    for groups in [int(g) for g in sys.argv[1:]] or [0, 1]:
        layer.set_expert_overlap(bool(groups))
        for _ in range(3):
            layer.forward(level, 1)
        layer.sync()
        layer.enable_timing(True)
        layer.forward(level, 1)
        layer.sync()
        sp = layer.spans()
        layer.enable_timing(False)
        t0 = min(a for _, _, a, _ in sp)
        if rank == 0:
            print(f"== fused {groups} ({e}x{t})")
            for st, j, a, b in sorted(sp, key=lambda z: z[2]):
                print(f"  {st:10s} {j:2d} {1e3 * (a - t0):8.1f} -> {1e3 * (b - t0):8.1f}  ({1e3 * (b - a):7.1f} us)")
        dist.barrier()
    layer.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()

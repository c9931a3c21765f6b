"""Cross-GPU timeline of one dispatch+combine step (dev tool).

    torchrun --nproc-per-node N scripts/timeline.py [--level O1] [--chunks 1]

Every rank records globaltimer stamps of its fused front kernel (debug_front)
and of the persistent exchange kernels' roles (xchg_trace); rank 0 prints them
on one time axis (globaltimer is a per-GPU clock; on one HGX board the GPUs'
clocks agree to within a microsecond or so, enough to read skew and waits).
"""
import argparse
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ["NCCL_DEBUG"] = "WARN"

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import bench  # noqa: E402
from paper_2411_00662_b200.layer import MoeLayer, BASELINE, O1, O2, O3  # noqa: E402

LEVELS = {"Baseline": BASELINE, "O1": O1, "O2": O2, "O3": O3}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--level", default="O1")
    ap.add_argument("--chunks", type=int, default=1)
    ap.add_argument("--tokens", type=int, default=4096)
    ap.add_argument("--hidden", type=int, default=4096)
    ap.add_argument("--experts", type=int, default=8)
    ap.add_argument("--topk", type=int, default=2)
    ap.add_argument("--no-persistent", action="store_true")
    ap.add_argument("--timing", action="store_true", help="also record role traces and event spans (adds overhead)")
    a = ap.parse_args()
    world, rank = int(os.environ["WORLD_SIZE"]), int(os.environ["RANK"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    e, t = bench.topo_for(world)
    lv = LEVELS[a.level] if t > 1 else BASELINE
    layer = MoeLayer(e, t, a.experts, a.topk, a.tokens, a.hidden, dtype=torch.bfloat16, max_chunks=16, device=local,
                     rank=rank, world_size=world)
    layer.connect()
    layer.enable_graphs(True)
    if a.no_persistent:
        layer.set_persistent(False)
    cd = layer.cards[0]
    g = torch.Generator(device=f"cuda:{local}").manual_seed(7 + cd.node)
    cd.x.copy_(torch.randn(a.tokens, a.hidden, generator=g, device=f"cuda:{local}").to(torch.bfloat16))
    cd.logits.copy_(torch.randn(a.tokens, a.experts, generator=g, device=f"cuda:{local}"))
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=f"cuda:{local}")
    bar = torch.zeros(1, device=f"cuda:{local}")
    layer.lib.moe_ctx_debug_front(layer._ctx, 1, 0, None)
    layer.enable_timing(a.timing)
    for rep in range(4):
        flush.zero_()
        dist.all_reduce(bar)
        torch.cuda.synchronize()
        layer.forward(lv, a.chunks, 0, torch.cuda.current_stream())
        torch.cuda.synchronize()
    out = (C.c_uint64 * 20)()
    layer.lib.moe_ctx_debug_front(layer._ctx, 1, layer.local_cards[0], out)
    front = [out[i] for i in range(20)]
    mc = layer.max_chunks
    cap = 2 * 4 * mc * 2
    arr = (C.c_uint64 * cap)()
    got = C.c_int32()
    if a.timing:
        layer.lib.moe_ctx_xchg_trace(layer._ctx, layer.local_cards[0], arr, cap, C.byref(got))
    roles = []
    for kern in range(2):
        for role in range(4):
            for j in range(mc):
                base = ((kern * 4 + role) * mc + j) * 2
                x0, x1 = arr[base], arr[base + 1]
                if x0 == 0xFFFFFFFFFFFFFFFF or x1 == 0xFFFFFFFFFFFFFFFF or not layer.ROLES[kern][role]:
                    continue
                roles.append((layer.ROLES[kern][role], j, x0, x1))
    spans = layer.spans() if a.timing else []
    allg = [None] * world
    dist.all_gather_object(allg, (rank, front, roles, spans))
    if rank == 0:
        for r, f, rl, sp in allg:
            t0 = f[0]
            us = lambda v: (v - t0) / 1e3 if v else float("nan")
            print(f"rank {r}: front start {us(f[0]):7.1f}  release {us(f[1]):7.1f}  counts-pushed {us(f[2]):7.1f}  "
                  f"peers-counts {us(f[3]):7.1f}  plan-steps " + " ".join(f"{us(f[i]):.1f}" for i in range(8, 13)) +
                  f"  plan-end {us(f[6]):7.1f}  tile-rank-end {us(f[7]):7.1f}")
            print(f"    dispatch kernel {us(f[16]):7.1f} -> {us(f[17]):7.1f}   combine kernel {us(f[18]):7.1f} -> {us(f[19]):7.1f}")
            for name, j, x0, x1 in sorted((z for z in rl if z[2] and z[3]), key=lambda z: z[2]):
                print(f"    {name:10s} chunk {j:2d}  {us(x0):7.1f} -> {us(x1):7.1f}  ({(x1 - x0) / 1e3:6.1f} us)")
            print("    spans (event clock, from the step's first event):",
                  "  ".join(f"{st}[{j}] {x0 * 1e3:.1f}-{x1 * 1e3:.1f}" for st, j, x0, x1 in sp))
    layer.close()
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()

"""One rank of the multi-process fp8-wire check (tests/test_multigpu.py): one
card per GPU over NVLink, the wire set to fp8; every landed row equals its
source row (own node) or the e4m3 round trip of it (crossed a node), bit for
bit.  Exits non-zero on a mismatch."""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2411_00662_b200 import _lib  # noqa: E402
from paper_2411_00662_b200.layer import MoeLayer  # noqa: E402
from test_gpu_wire import _fp8_roundtrip  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--groups", type=int, default=2)
    ap.add_argument("--tp", type=int, default=2)
    ap.add_argument("--runs", default="1:1,0:1,2:2")  # level:n
    a = ap.parse_args()
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    e, t, E, k, T, h = a.groups, a.tp, 8, 2, 256, 512
    xs = [torch.randn(T, h, generator=torch.Generator().manual_seed(11 + g)).to(torch.bfloat16) for g in range(e)]
    lg = [torch.randn(T, E, generator=torch.Generator().manual_seed(77 + g)) for g in range(e)]
    rts = [_fp8_roundtrip(x) for x in xs]
    layer = MoeLayer(e, t, E, k, T, h, dtype=torch.bfloat16, max_chunks=4, device=local, rank=rank, world_size=world)
    layer.connect()
    layer.set_wire(_lib.WIRE_FP8)
    cd = layer.cards[0]
    ok = True
    try:
        cd.x.copy_(xs[cd.node])
        cd.logits.copy_(lg[cd.node])
        for spec in a.runs.split(","):
            level, n = (int(v) for v in spec.split(":"))
            for _ in range(2):
                layer.forward(level, n, 0)
            layer.sync()
            rows = layer.recv_rows(cd.card)
            tags = cd.recv_tags[:rows].long().cpu()
            got = cd.recv[:rows].cpu()
            for r in range(rows):
                src, pos = int(tags[r, 1]) // t, int(tags[r, 2])
                want = xs[src][pos] if src == cd.node else rts[src][pos]
                if not torch.equal(got[r].view(torch.int16), want.view(torch.int16)):
                    print(f"rank {rank} {spec}: row {r} (src {src}, pos {pos}) differs", flush=True)
                    ok = False
                    break
    finally:
        layer.close()
        dist.barrier()
        dist.destroy_process_group()
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()

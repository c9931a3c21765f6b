"""One rank of the multi-process layer-backward check (tests/test_multigpu_backward.py):
one card per process over NVLink, the closed forms of tests/test_gpu_layer_backward.py
checked on this rank's card.  Exits non-zero on a mismatch."""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2411_00662_b200 import layer_backward as LB  # noqa: E402
from paper_2411_00662_b200.layer import MoeLayer  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--groups", type=int, default=2)
    ap.add_argument("--tp", type=int, default=2)
    ap.add_argument("--experts", type=int, default=8)
    ap.add_argument("--topk", type=int, default=2)
    ap.add_argument("--runs", default="1:1:0,2:2:0,0:1:0")
    a = ap.parse_args()
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    e, t, E, k, T, h = a.groups, a.tp, a.experts, a.topk, 128, 256
    dt, dev = torch.bfloat16, torch.device(f"cuda:{local}")
    gen = torch.Generator().manual_seed(5)
    x = torch.randn(e, T, h, generator=gen).to(dt)
    logits = torch.randn(e, T, E, generator=gen)
    gout = torch.randn(e, T, h, generator=gen).to(dt)
    c = torch.linspace(0.5, 2.0, E, dtype=torch.float64)
    d = torch.linspace(-1.0, 1.0, E, dtype=torch.float64)
    layer = MoeLayer(e, t, E, k, T, h, dtype=dt, logit_dtype=torch.float32, max_chunks=4, device=local, rank=rank,
                     world_size=world)
    layer.connect()
    cd = layer.cards[0]
    ok = True
    try:
        for spec in a.runs.split(","):
            level, n, landing = (int(v) for v in spec.split(":"))
            cd.x.copy_(x[cd.node])
            cd.logits.copy_(logits[cd.node])
            layer.route()
            layer.dispatch(level, n, landing)
            layer.sync()
            rows = layer.recv_rows(cd.card)
            xe = cd.recv_tags[:rows, 3].long().cpu()
            y = {cd.card: (cd.recv[:rows].double().cpu() * c[xe][:, None]).to(dt).to(dev)}
            ex = cd.experts.long().cpu()
            pr = cd.probs.double().cpu()
            _, grad_p = LB.combine_backward(layer, {cd.card: gout[cd.node]}, y, level, n, landing)
            g, xx = gout[cd.node].double(), x[cd.node].double()
            yx = (xx[:, None, :] * c[ex][:, :, None]).to(dt).double()
            want = (g[:, None, :] * yx).sum(-1)
            err = ((grad_p[cd.card].double().cpu() - want).abs() / (g[:, None, :] * yx).abs().sum(-1)).max().item()
            if not err < 1e-5:
                print(f"rank {rank} {spec}: grad_probs rel err {err}", flush=True)
                ok = False
            grad_rows = {cd.card: (cd.recv[:rows].double().cpu() * d[xe][:, None]).to(dt).to(dev)}
            gx = LB.dispatch_backward(layer, grad_rows, level, n)[cd.card]
            want = (g[:, None, :] * d[ex][:, :, None]).to(dt).double().sum(1)
            err = ((gx.double().cpu() - want).abs().max() / want.abs().max()).item()
            if not err < 1e-2:
                print(f"rank {rank} {spec}: grad_x rel err {err}", flush=True)
                ok = False
            if not torch.equal(cd.probs.double().cpu(), pr):
                print(f"rank {rank} {spec}: probs not restored", flush=True)
                ok = False
            # the same closed forms through the context's device-side backward
            # (moe_ctx_backward_combine / _dispatch: no host round trip)
            if landing == 0:
                cd.x.copy_(x[cd.node])
                layer.dispatch(level, n, landing)
                layer.sync()
                cd.recv[:rows].copy_(y[cd.card])       # the scaling experts, in place
                layer.combine(level, n)
                cd.x.copy_(gout[cd.node])
                layer.backward_combine(level, n)
                layer.sync()
                want_p = (g[:, None, :] * yx).sum(-1)
                err = ((cd.grad_probs.double().cpu() - want_p).abs() / (g[:, None, :] * yx).abs().sum(-1)).max().item()
                if not err < 1e-5:
                    print(f"rank {rank} {spec}: ctx grad_probs rel err {err}", flush=True)
                    ok = False
                tags = cd.recv_tags[:rows].long()
                cd.pre[:rows].copy_((gout.to(dev)[tags[:, 1] // t, tags[:, 2]].double()
                                     * d.to(dev)[tags[:, 3]][:, None]).to(dt))
                layer.backward_dispatch(level, n)
                layer.sync()
                err = ((cd.out.double().cpu() - want).abs().max() / want.abs().max()).item()
                if not err < 1e-2:
                    print(f"rank {rank} {spec}: ctx grad_x rel err {err}", flush=True)
                    ok = False
    finally:
        layer.close()
        dist.barrier()
        dist.destroy_process_group()
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()

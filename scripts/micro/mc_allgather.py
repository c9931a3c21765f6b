"""NVLS multicast AllGather vs unicast stores vs NCCL on one group of GPUs
(the TP group's AllGather).  One process per GPU:

    torchrun --nproc-per-node 4 scripts/micro/mc_allgather.py

Each rank contributes `v` bytes; after the AllGather every rank holds all
ranks' parts.  multicast: one moe_mc_store of the rank's part through the
multicast address (lands on every device; egress = v).  unicast: the
library's copy kernel storing the part to every peer over NVLink
(moe_ctx_xfer; egress = (t - 1) v).  nccl: all_gather_into_tensor.  Checks
the multicast result bit for bit, then prints one JSON line per size
(max over ranks of CUDA-event time, median of reps).
"""
import ctypes as C
import json
import os
import socket
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2411_00662_b200 import _lib  # noqa: E402
from paper_2411_00662_b200.layer import MoeLayer, device_view  # noqa: E402


GRIDS = (8, 16, 32, 64, 148, 296, 592)


def share_fd(rank, world, fd, tag):
    """Leader's fd -> every rank (SCM_RIGHTS over an abstract Unix socket)."""
    name = f"\0monta_mc_{tag}"
    if rank == 0:
        srv = socket.socket(socket.AF_UNIX, socket.SOCK_STREAM)
        srv.bind(name)
        srv.listen(world)
        dist.barrier()
        for _ in range(world - 1):
            conn, _ = srv.accept()
            socket.send_fds(conn, [b"x"], [fd])
            conn.close()
        srv.close()
        dist.barrier()
        return fd
    dist.barrier()
    cli = socket.socket(socket.AF_UNIX, socket.SOCK_STREAM)
    cli.connect(name)
    _, fds, _, _ = socket.recv_fds(cli, 1, 1)
    cli.close()
    dist.barrier()
    return fds[0]


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dev = torch.device(f"cuda:{local}")
    dist.init_process_group("nccl", device_id=dev)
    lib = _lib.load()
    ok = C.c_int()
    _lib.check(lib.moe_mc_supported(local, C.byref(ok)))
    if not ok.value:
        if rank == 0:
            print(json.dumps({"multicast": "unsupported on this device"}))
        return
    max_part = int(os.environ.get("MC_MAX_MIB", "64")) << 20
    gran = C.c_size_t()
    _lib.check(lib.moe_mc_granularity(world, max_part * world, C.byref(gran)))
    total = ((max_part * world + gran.value - 1) // gran.value) * gran.value
    mc = C.c_void_p()
    fd = C.c_int(-1)
    if rank == 0:
        _lib.check(lib.moe_mc_create(world, total, C.byref(fd), C.byref(mc)))
    fd_all = share_fd(rank, world, fd.value, os.environ.get("MASTER_PORT", "0"))
    if rank != 0:
        _lib.check(lib.moe_mc_import(fd_all, world, total, C.byref(mc)))
    _lib.check(lib.moe_mc_add_device(mc, local))
    dist.barrier()
    uc, mcva = C.c_void_p(), C.c_void_p()
    _lib.check(lib.moe_mc_bind(mc, C.byref(uc), C.byref(mcva)))
    dist.barrier()
    buf = device_view(uc.value, (total,), torch.uint8, local)
    # the unicast baseline: the library's NVLink store kernel, one "node" of `world` TP cards
    row = 16384
    layer = MoeLayer(1, world, world, 1, world * max_part // row, row // 2, dtype=torch.bfloat16, max_chunks=1, device=local,
                     rank=rank, world_size=world)
    layer.connect()
    stream = torch.cuda.current_stream()
    bar = torch.zeros(1, device=dev)

    def timed(fn, reps=10):
        vals = []
        for _ in range(2):
            fn()
        torch.cuda.synchronize()
        for _ in range(reps):
            dist.all_reduce(bar)
            torch.cuda.synchronize()
            s, f = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda._sleep(100000)
            s.record(stream)
            fn()
            f.record(stream)
            torch.cuda.synchronize()
            v = torch.tensor([s.elapsed_time(f) * 1e3], device=dev, dtype=torch.float64)
            dist.all_reduce(v, op=dist.ReduceOp.MAX)
            vals.append(float(v.item()))
        return statistics.median(vals)

    all_ok = True
    v = 1 << 20
    while v <= max_part:
        src = torch.randint(0, 255, (v,), dtype=torch.uint8, device=dev, generator=torch.Generator(device=dev).manual_seed(rank * 7 + v))
        dst_mc = C.c_void_p(mcva.value + rank * v)
        buf[: world * v].zero_()
        dist.barrier()
        _lib.check(lib.moe_mc_store(C.c_void_p(src.data_ptr()), dst_mc, v, 0, C.c_void_p(stream.cuda_stream)))
        torch.cuda.synchronize()
        dist.barrier()
        parts = [torch.empty(v, dtype=torch.uint8, device=dev) for _ in range(world)]
        dist.all_gather(parts, src)
        good = all(torch.equal(buf[r * v:(r + 1) * v], parts[r]) for r in range(world))
        all_ok &= good
        mct = {g: timed(lambda g=g: _lib.check(lib.moe_mc_store(C.c_void_p(src.data_ptr()), dst_mc, v, g,
                                                                 C.c_void_p(stream.cuda_stream))))
              for g in GRIDS}
        per = [0] * world
        for c in range(world):
            if c != rank:
                per[c] = max(1, v // row)
        uc = {g: timed(lambda g=g: layer.xfer(per, row, g, stream)) for g in GRIDS}
        mc_us, uc_us = min(mct.values()), min(uc.values())
        full = torch.empty(v * world, dtype=torch.uint8, device=dev)
        nccl_us = timed(lambda: dist.all_gather_into_tensor(full, src))
        if rank == 0:
            print(json.dumps({"gpus": world, "part_bytes": v, "correct": bool(good),
                              "multicast_us": round(mc_us, 2), "unicast_us": round(uc_us, 2),
                              "nccl_us": round(nccl_us, 2),
                              "multicast_egress_gbs": round(v / mc_us / 1e3, 1),
                              "delivered_gbs_multicast": round((world - 1) * v / mc_us / 1e3, 1),
                              "delivered_gbs_unicast": round((world - 1) * v / uc_us / 1e3, 1),
                              "multicast_us_by_ctas": {g: round(x, 2) for g, x in mct.items()},
                              "unicast_us_by_ctas": {g: round(x, 2) for g, x in uc.items()}}), flush=True)
        v *= 4
    layer.close()
    dist.barrier()
    lib.moe_mc_destroy(mc)
    dist.destroy_process_group()
    sys.exit(0 if all_ok else 1)


if __name__ == "__main__":
    main()

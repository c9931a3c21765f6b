"""Host-side logic of the N>1 path, on CPU with torch.distributed/gloo at
world_size 2 (no GPU): every rank must take the same planner decision (the
epoch flags assume identical op sequences on all ranks), the IPC-handle
exchange must assemble blobs in rank order, and the exposed-AllToAll
arithmetic used by bench.py must be right."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import sys
        sys.path.insert(0, ROOT)
        import bench
        from paper_2411_00662_b200 import planner as P
        from paper_2411_00662_b200 import layer as L

        # 1) planner decision per rank (bench.py's selection) for every bench topology
        decisions = []
        for n_gpus in (2, 4, 8):
            e, t = bench.topo_for(n_gpus)
            if t == 1:
                decisions.append(("Baseline", 1))
                continue
            cdir = os.path.join(ROOT, "profiles", "curves_b200", f"{e}x{t}")
            cs = P.load_curve_set(cdir)
            import json
            ov = P.OverheadModel(**json.load(open(os.path.join(cdir, "overhead.json"))))
            d = P.select_strategy(P.ModelSpec(b=1, s=4096 * 2, h=4096, k=2, bpe=2), P.ParallelSpec(t=t, e=e),
                                  P.b200_cluster(e, t), cs, ov, n_cap=16)
            decisions.append((d.level.name, d.n))
        gathered = [None] * world
        dist.all_gather_object(gathered, decisions)

        # 2) IPC blob exchange through MoeLayer.connect with a stub ABI
        class StubLib:
            def moe_ctx_ipc_handle_size(self):
                return 128

            def moe_ctx_ipc_export(self, ctx, blob):
                blob[:] = bytes([rank + 1]) * 128
                return 0

            def moe_ctx_ipc_connect(self, ctx, buf):
                StubLib.seen = bytes(buf)
                return 0

        layer = L.MoeLayer.__new__(L.MoeLayer)
        layer.lib = StubLib()
        layer.world_size = world
        layer._ctx = None
        layer.connect()
        blob_ok = StubLib.seen == b"".join(bytes([r + 1]) * 128 for r in range(world))
        q.put((rank, gathered, blob_ok))
    finally:
        dist.destroy_process_group()


def test_two_rank_host_logic_over_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    results = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, gathered, blob_ok in results:
        assert gathered[0] == gathered[1], "ranks disagree on the planner decision"
        assert blob_ok, f"rank {rank}: IPC blobs not assembled in rank order"


def test_exposed_alltoall_interval_arithmetic():
    import sys
    sys.path.insert(0, ROOT)
    import bench
    # AA [0,10] with AG covering [4,6] and [8,12] -> exposed 10 - 2 - 2 = 6
    assert bench.exposed([(0, 10)], [(4, 6), (8, 12)]) == pytest.approx(6.0)
    # overlapping AA intervals are unioned first
    assert bench.exposed([(0, 5), (3, 8)], []) == pytest.approx(8.0)
    busy, exp = bench.role_stats([("aa", 0, 0.0, 10.0), ("ag", 0, 5.0, 20.0), ("caa", 0, 30.0, 40.0),
                                  ("unpermute", 0, 35.0, 50.0)])
    assert busy["aa"] == pytest.approx(10.0) and busy["ag"] == pytest.approx(15.0)
    assert exp == pytest.approx(5.0 + 5.0)


def test_bench_topologies_are_one_card_per_gpu():
    import sys
    sys.path.insert(0, ROOT)
    import bench
    for n in (1, 2, 4, 8):
        e, t = bench.topo_for(n)
        assert e * t == n

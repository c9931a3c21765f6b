"""Router alone (moe_route_topk, the front's route_tokens in a plain grid):
GPU us per call, from a CUDA graph of 20 back-to-back calls (no host overhead)."""
import os, sys, json
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2411_00662_b200 import ops  # noqa: E402
for (T, E, k) in [(8192, 160, 6), (4096, 8, 2), (8192, 160, 1), (8192, 128, 6), (8192, 32, 6), (8192, 160, 2)]:
    lg = torch.randn(T, E, device="cuda")
    ex = torch.empty(T, k, dtype=torch.int32, device="cuda")
    pr = torch.empty(T, k, device="cuda")
    from paper_2411_00662_b200 import _lib
    lib = _lib.load()
    s = torch.cuda.Stream()
    def call():
        _lib.check(lib.moe_route_topk(lg.data_ptr(), _lib.F32, T, E, k, ex.data_ptr(), pr.data_ptr(),
                                      torch.cuda.current_stream().cuda_stream))
    with torch.cuda.stream(s):
        call()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for _ in range(20):
            call()
    g.replay()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    g.replay()
    b.record()
    torch.cuda.synchronize()
    print(json.dumps({"T": T, "E": E, "k": k, "us": a.elapsed_time(b) * 1e3 / 20}))

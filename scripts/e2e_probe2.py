"""forward_host as bench.py times it, with and without the per-step L2 flush
and host sync (dev tool: explains the bench's e2e against e2e_probe.py)."""
import os
import statistics
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2411_00662_b200.layer import MoeLayer, BASELINE

T, h, E, k = 4096, 4096, 8, 2
layer = MoeLayer(1, 1, E, k, T, h, dtype=torch.bfloat16, logit_dtype=torch.float32, max_chunks=16, device=0)
layer.enable_graphs(True)
s = torch.cuda.current_stream()
hx = torch.randn(T, h).to(torch.bfloat16).pin_memory()
hl = torch.randn(T, E).pin_memory()
ho = torch.empty(T, h, dtype=torch.bfloat16).pin_memory()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
flush_rd = torch.ones((256 << 20) // 4, dtype=torch.float32, device="cuda")


def step():
    layer.forward_host(hx, hl, ho, BASELINE, 1, 0, s)


for _ in range(5):
    step()
torch.cuda.synchronize()
for name, cold, sync in (("cold+nosync", 1, 0), ("nocold+nosync", 0, 0), ("cold+sync", 1, 1), ("nocold+sync", 0, 1),
                         ("memset-only", 2, 0), ("read-only", 3, 0)):
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(20)]
    torch.cuda.synchronize()
    for a, b in evs:
        if cold in (1, 2):
            flush.zero_()
        if cold in (1, 3):
            flush_rd.amax()
        a.record(s)
        step()
        b.record(s)
        if sync:
            torch.cuda.synchronize()
    torch.cuda.synchronize()
    ms = [a.elapsed_time(b) * 1e3 for a, b in evs]
    print(f"{name:14s} median {statistics.median(ms):7.0f} us  min {min(ms):7.0f}  max {max(ms):7.0f}", flush=True)
layer.close()

"""forward_host timing on one GPU with different host buffers (dev tool)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2411_00662_b200.layer import MoeLayer, BASELINE
from paper_2411_00662_b200.ops import host_empty

T, h, E, k = 4096, 4096, 8, 2
layer = MoeLayer(1, 1, E, k, T, h, dtype=torch.bfloat16, max_chunks=16)
s = torch.cuda.current_stream()
ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for name, alloc in (("pin_memory", lambda sh, dt: torch.empty(sh, dtype=dt).pin_memory()), ("host_empty", host_empty)):
    hx, hl, ho = alloc((T, h), torch.bfloat16), alloc((T, E), torch.float32), alloc((T, h), torch.bfloat16)
    hx.copy_(torch.randn(T, h).to(torch.bfloat16))
    hl.copy_(torch.randn(T, E))
    for graphs in (False, True):
        layer.enable_graphs(graphs)
        for _ in range(3):
            layer.forward_host(hx, hl, ho, BASELINE, 1, 0, s)
        torch.cuda.synchronize()
        ts = []
        for _ in range(10):
            ev0.record(s)
            layer.forward_host(hx, hl, ho, BASELINE, 1, 0, s)
            ev1.record(s)
            torch.cuda.synchronize()
            ts.append(ev0.elapsed_time(ev1) * 1e3)
        print(f"{name:12s} graphs={graphs}: median {sorted(ts)[5]:.0f} us  min {min(ts):.0f} us", flush=True)
    # plain copies for reference
    d = torch.empty(T, h, dtype=torch.bfloat16, device="cuda")
    ev0.record(s); d.copy_(hx, non_blocking=True); ev1.record(s); torch.cuda.synchronize()
    ev0.record(s); d.copy_(hx, non_blocking=True); ev1.record(s); torch.cuda.synchronize()
    h2d = ev0.elapsed_time(ev1) * 1e3
    ev0.record(s); ho.copy_(d, non_blocking=True); ev1.record(s); torch.cuda.synchronize()
    print(f"{name:12s} H2D 32 MiB {h2d:.0f} us   D2H {ev0.elapsed_time(ev1) * 1e3:.0f} us", flush=True)
layer.close()

"""e2e A/B (dev tool): moe_ctx_forward_host on the DeepSeek N=1 layer with the
ABI's pinned buffers, CUDA-event time per step (median of 20), as bench.py's
e2e leg measures it; run under different MONTA_* environment settings."""
import os
import statistics
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_2411_00662_b200 import ops  # noqa: E402
from paper_2411_00662_b200.layer import MoeLayer, BASELINE  # noqa: E402

T, h, E, k = 8192, 5120, 160, 6
layer = MoeLayer(1, 1, E, k, T, h, dtype=torch.bfloat16, logit_dtype=torch.float32, max_chunks=16, device=0)
layer.enable_graphs(True)
s = torch.cuda.current_stream()
hx = ops.host_empty((T, h), torch.bfloat16)
hx.copy_(torch.randn(T, h).to(torch.bfloat16))
hl = ops.host_empty((T, E), torch.float32)
hl.copy_(torch.randn(T, E))
ho = ops.host_empty((T, h), torch.bfloat16)
for _ in range(5):
    layer.forward_host(hx, hl, ho, BASELINE, 1, 0, s)
torch.cuda.synchronize()
ts = []
for _ in range(20):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s)
    layer.forward_host(hx, hl, ho, BASELINE, 1, 0, s)
    b.record(s)
    torch.cuda.synchronize()
    ts.append(a.elapsed_time(b) * 1e3)
print(os.environ.get("TAG", ""), "e2e us median", round(statistics.median(ts), 1), "min", round(min(ts), 1))

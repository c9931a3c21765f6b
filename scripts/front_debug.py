"""Phase timestamps of the fused front kernel (dev tool)."""
import ctypes as C
import sys
import os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2411_00662_b200.layer import MoeLayer, O1, BASELINE

for (e, t, E, k, T) in [(1, 1, 8, 2, 4096), (1, 1, 160, 6, 8192), (1, 1, 2, 1, 8192), (4, 2, 160, 6, 8192)]:
    layer = MoeLayer(e, t, E, k, T, 1024, dtype=torch.bfloat16, max_chunks=8)
    for cd in layer.cards:
        cd.logits.normal_()
    layer.lib.moe_ctx_debug_front(layer._ctx, 1, 0, None)
    for rep in range(3):
        layer.forward(BASELINE, 1)
        out = (C.c_uint64 * 20)()
        layer.lib.moe_ctx_debug_front(layer._ctx, 1, 0, out)
        v = [out[i] for i in range(20)]
        t0 = (~v[16]) & ((1 << 64) - 1)
        r = lambda i: (v[i] - v[0]) / 1e3
        print(f"{e}x{t} E={E} k={k} T={T}: release {r(1):.1f}  counts+push {r(2):.1f}  plan-wait {r(3):.1f}  "
              f"plan-end {r(6):.1f}  cta0-rank-end {r(7):.1f} us | first CTA start -> cta0 start {(v[0] - t0) / 1e3:.1f}, "
              f"last CTA start {(v[17] - t0) / 1e3:.1f}, last tile end {(v[18] - t0) / 1e3:.1f}, control end {(v[19] - t0) / 1e3:.1f} us")
    layer.close()

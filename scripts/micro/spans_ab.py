import os, sys
sys.path.insert(0, "/root/repo")
import torch
from paper_2411_00662_b200.layer import MoeLayer, BASELINE
T, h, E, k = 8192, 5120, 160, 6
layer = MoeLayer(1, 1, E, k, T, h, dtype=torch.bfloat16, max_chunks=16)
cd = layer.cards[0]
cd.x.normal_(); cd.logits.normal_()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda"); rd = torch.ones(64 << 20, device="cuda")
for graphs in (True, False):
    layer.enable_graphs(graphs)
    for _ in range(3): layer.forward(BASELINE, 1)
    layer.sync()
    layer.enable_timing(True)
    res = {}
    for _ in range(5):
        flush.zero_(); rd.amax()
        torch.cuda._sleep(2_000_000)
        layer.forward(BASELINE, 1)
        for st, j, a, b in layer.spans():
            res.setdefault(st, []).append((b - a) * 1e3)
    layer.enable_timing(False)
    layer.sync()
    print("graphs" if graphs else "eager", {k: round(sorted(v)[len(v)//2], 1) for k, v in res.items()})
layer.close()

import torch, time
x = torch.empty(32 << 20, dtype=torch.uint8).pin_memory()
d = torch.empty(32 << 20, dtype=torch.uint8, device="cuda")
s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for name, fn in [("h2d", lambda: d.copy_(x, non_blocking=True)), ("d2h", lambda: x.copy_(d, non_blocking=True))]:
    for _ in range(3): fn()
    torch.cuda.synchronize()
    s0.record(); 
    for _ in range(10): fn()
    s1.record(); torch.cuda.synchronize()
    ms = s0.elapsed_time(s1) / 10
    print(name, f"{ms*1e3:.1f} us  {32*1.048576/ms:.1f} GB/s")
# both directions concurrently
s2 = torch.cuda.Stream(); y = torch.empty_like(x); d2 = torch.empty_like(d)
torch.cuda.synchronize(); s0.record()
for _ in range(10):
    d.copy_(x, non_blocking=True)
    with torch.cuda.stream(s2): y.copy_(d2, non_blocking=True)
torch.cuda.current_stream().wait_stream(s2); s1.record(); torch.cuda.synchronize()
print("both", f"{s0.elapsed_time(s1)/10*1e3:.1f} us")

"""PCIe host<->device copy rates on this box (dev tool): default pinned memory,
write-combined pinned memory (cudaHostAllocWriteCombined) and pinned memory
first-touched from each NUMA node's CPUs."""
import ctypes as C
import os
import subprocess

import torch

MB = 32
cudart = C.CDLL("libcudart.so.12") if os.path.exists("/usr/local/cuda/lib64/libcudart.so.12") else None


def rate(host, dev, direction):
    s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    fn = (lambda: dev.copy_(host, non_blocking=True)) if direction == "h2d" else (lambda: host.copy_(dev, non_blocking=True))
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    s0.record()
    for _ in range(10):
        fn()
    s1.record()
    torch.cuda.synchronize()
    ms = s0.elapsed_time(s1) / 10
    return MB * 1.048576 / ms


def host_alloc(nbytes, flags):
    ptr = C.c_void_p()
    rc = cudart.cudaHostAlloc(C.byref(ptr), C.c_size_t(nbytes), C.c_uint(flags))
    assert rc == 0, rc
    buf = (C.c_uint8 * nbytes).from_address(ptr.value)
    C.memset(ptr, 1, nbytes)
    return torch.frombuffer(buf, dtype=torch.uint8), ptr


def main():
    print(subprocess.run(["nvidia-smi", "topo", "-m"], capture_output=True, text=True).stdout[:1500])
    print(subprocess.run(["bash", "-c", "lscpu | grep -i numa"], capture_output=True, text=True).stdout)
    d = torch.empty(MB << 20, dtype=torch.uint8, device="cuda")
    x = torch.empty(MB << 20, dtype=torch.uint8).pin_memory()
    print("torch pin_memory       h2d %.1f GB/s  d2h %.1f GB/s" % (rate(x, d, "h2d"), rate(x, d, "d2h")))
    if cudart:
        for name, flags in (("cudaHostAllocDefault", 0), ("WriteCombined", 4), ("Portable", 1)):
            h, p = host_alloc(MB << 20, flags)
            print("%-22s h2d %.1f GB/s  d2h %.1f GB/s" % (name, rate(h, d, "h2d"), rate(h, d, "d2h")))
    cpus = sorted(os.sched_getaffinity(0))
    nodes = {}
    for c in cpus:
        try:
            node = [f for f in os.listdir(f"/sys/devices/system/cpu/cpu{c}") if f.startswith("node")][0]
        except (IndexError, FileNotFoundError):
            node = "node?"
        nodes.setdefault(node, []).append(c)
    # both directions at once (the pipelined forward_host overlaps them)
    h2 = torch.empty(MB << 20, dtype=torch.uint8).pin_memory()
    x.fill_(1)
    h2.fill_(1)
    d2 = torch.empty_like(d)
    s2 = torch.cuda.Stream()
    s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    s0.record()
    for _ in range(10):
        d.copy_(x, non_blocking=True)
        with torch.cuda.stream(s2):
            h2.copy_(d2, non_blocking=True)
    torch.cuda.current_stream().wait_stream(s2)
    s1.record()
    torch.cuda.synchronize()
    ms = s0.elapsed_time(s1) / 10
    print("both directions at once: %.1f GB/s total" % (2 * MB * 1.048576 / ms))
    for node, cs in sorted(nodes.items()):
        os.sched_setaffinity(0, cs)
        x = torch.empty(MB << 20, dtype=torch.uint8)
        x.fill_(1)  # first touch on this node
        x = x.pin_memory()
        print("pinned first-touch %-6s h2d %.1f GB/s  d2h %.1f GB/s" % (node, rate(x, d, "h2d"), rate(x, d, "d2h")))
    os.sched_setaffinity(0, cpus)


if __name__ == "__main__" and not (len(os.sys.argv) > 1 and os.sys.argv[1] == "multi"):
    main()


def multi():
    """torchrun --nproc-per-node N scripts/pcie_probe.py multi: every rank copies at once."""
    import torch.distributed as dist
    rank, local = int(os.environ["RANK"]), int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("gloo")
    d = torch.empty(MB << 20, dtype=torch.uint8, device="cuda")
    x = torch.empty(MB << 20, dtype=torch.uint8).pin_memory()
    h, _ = host_alloc(MB << 20, 1)
    for name, buf in (("pin_memory", x), ("cudaHostAlloc", h)):
        for mode in ("alone", "all"):
            res = []
            for r in range(dist.get_world_size()):
                dist.barrier()
                if mode == "all" or r == rank:
                    res.append((rate(buf, d, "h2d"), rate(buf, d, "d2h")))
                if mode == "all":
                    break
            dist.barrier()
            print(f"rank {rank} {name:14s} {mode:5s} h2d {res[0][0]:.1f} GB/s  d2h {res[0][1]:.1f} GB/s", flush=True)


if __name__ == "__main__" and len(os.sys.argv) > 1 and os.sys.argv[1] == "multi":
    multi()

"""HBM roofline of the backward kernels (include/monta.h section 1b) at the
BASELINE layer sizes, one B200.  Each kernel is timed alone with CUDA events
on the current stream, cold L2 (a 256 MiB write + read between launches,
outside the events), median of 20 launches.  Algorithmic bytes per launch:

  combine_backward   grad_out T*h*bg (read once) + y R*h*by (read) + grad_y R*h*by (write)
                     + probs/slot_pos 8*T*k (read) + grad_probs 4*T*k (write)
  dispatch_backward  grad_rows R*h*b (read) + grad_x T*h*b (write) + slot_pos 4*T*k
  route_backward     logits 4*T*E (read) + grad_logits 4*T*E (write) + experts/grad_probs 8*T*k

usage: python scripts/micro/backward_bench.py [--out FILE]
"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2411_00662_b200 import ops  # noqa: E402

CONFIGS = {
    "toy": (2048, 1024, 8, 2, torch.float32),
    "mixtral": (4096, 4096, 8, 2, torch.bfloat16),
    "2x70b": (8192, 8192, 2, 1, torch.bfloat16),
    "deepseek": (8192, 5120, 160, 6, torch.bfloat16),
}


def timed(fn, flush, iters=20):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    fn()
    times = []
    for _ in range(iters):
        flush()
        s.record()
        fn()
        e.record()
        torch.cuda.synchronize()
        times.append(s.elapsed_time(e) * 1e3)
    times.sort()
    return times[len(times) // 2]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    peak = json.load(open(os.path.join(os.path.dirname(__file__), "..", "..", "MEASURED_PEAKS.json")))["hbm_gbs"]
    dev = torch.device("cuda:0")
    big = torch.empty(256 << 20, dtype=torch.uint8, device=dev)

    def flush():
        big.fill_(1)
        big.sum(dtype=torch.int64)

    lines = []
    for name, (T, h, E, k, dt) in CONFIGS.items():
        torch.manual_seed(0)
        logits = torch.randn(T, E, device=dev)
        experts, probs = ops.route_topk(logits, k)
        idx = ops.build_index(experts, E)
        R = T * k
        b = torch.empty((), dtype=dt).element_size()
        y = torch.randn(R, h, device=dev).to(dt)
        g = torch.randn(T, h, device=dev).to(dt)
        gy = torch.empty_like(y)
        gp = torch.empty_like(probs)
        gx = torch.empty_like(g)
        lib = ops._lib.load()
        st = torch.cuda.current_stream().cuda_stream
        dc = ops._lib.dtype_code(dt)
        sp = idx.slot_pos

        def cbwd():
            ops.check(lib.moe_combine_backward(g.data_ptr(), dc, h, y.data_ptr(), dc, h, h, sp.data_ptr(),
                                               probs.data_ptr(), ops._lib.F32, T, k, gy.data_ptr(), h,
                                               gp.data_ptr(), st))

        def dbwd():
            ops.check(lib.moe_dispatch_backward(y.data_ptr(), dc, h, h, sp.data_ptr(), T, k, gx.data_ptr(), dc, h,
                                                st))

        gz = torch.empty_like(logits)

        def rbwd():
            ops.check(lib.moe_route_backward(logits.data_ptr(), ops._lib.F32, T, E, k, experts.data_ptr(),
                                             gp.data_ptr(), gz.data_ptr(), st))

        for kern, fn, nbytes in (
                ("combine_backward", cbwd, T * h * b + 2 * R * h * b + 12 * T * k),
                ("dispatch_backward", dbwd, R * h * b + T * h * b + 4 * T * k),
                ("route_backward", rbwd, 8 * T * E + 8 * T * k)):
            us = timed(fn, flush)
            gbs = nbytes / us / 1e3
            line = {"config": name, "kernel": kern, "T": T, "h": h, "E": E, "k": k, "dtype": str(dt),
                    "us": round(us, 2), "bytes": nbytes, "GB/s": round(gbs, 1), "peak": peak,
                    "frac": round(gbs / peak, 3), "l2": "cold (256 MiB write+read between launches)"}
            print(json.dumps(line), flush=True)
            lines.append(line)
    if args.out:
        with open(args.out, "w") as f:
            for line in lines:
                f.write(json.dumps(line) + "\n")


if __name__ == "__main__":
    main()

"""Expert grouped GEMM / FFN throughput (include/monta.h 1c) vs cuBLAS on the
same box: TFLOP/s = 2 * rows * N * K / time, CUDA events, median of iters,
inputs larger than L2 (weights) or flushed.  One JSON line per case.

    python scripts/micro/gemm_bench.py [--iters 20]
"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2411_00662_b200 import _lib, ops  # noqa: E402


def timeit(fn, iters, flush):
    ts = []
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(3):
        fn()
    for _ in range(iters):
        flush.zero_()
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    ts.sort()
    return ts[len(ts) // 2]


def routed_offsets(T, E, k, dev, seed=0):
    g = torch.Generator(device="cpu").manual_seed(seed)
    logits = torch.randn(T, E, generator=g).to(dev)
    experts, _ = ops.route_topk(logits, k)
    return ops.build_index(experts, E).expert_offsets


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--cases", default="square,mixtral,deepseek,deepseek_ep4")
    args = ap.parse_args()
    dev = torch.device("cuda")
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    peaks = json.load(open(os.path.join(os.path.dirname(__file__), "..", "..", "MEASURED_PEAKS.json"))) \
        if os.path.exists(os.path.join(os.path.dirname(__file__), "..", "..", "MEASURED_PEAKS.json")) else {}
    sus = peaks.get("bf16_tflops_sustained", 1371.2)
    g = torch.Generator(device="cpu").manual_seed(0)
    for case in args.cases.split(","):
        if case == "square":
            rows, L, N, K = 8192, 1, 8192, 8192
            offs = torch.tensor([0, rows], dtype=torch.int32, device=dev)
            x = torch.randn(rows, K, generator=g).to(torch.bfloat16).to(dev)
            w = (torch.randn(L, N, K, generator=g) * 0.01).to(torch.bfloat16).to(dev)
            y = torch.empty(rows, N, dtype=torch.bfloat16, device=dev)
            us = timeit(lambda: ops.grouped_gemm(x, w, offs, out=y), args.iters, flush)
            ub = timeit(lambda: torch.matmul(x, w[0].T, out=y), args.iters, flush)
            fl = 2.0 * rows * N * K
            print(json.dumps({"case": case, "rows": rows, "L": L, "N": N, "K": K, "us": us, "tflops": fl / us / 1e6,
                              "frac_sustained": fl / us / 1e6 / sus, "cublas_us": ub, "cublas_tflops": fl / ub / 1e6}),
                  flush=True)
            continue
        if case == "mixtral":
            T, E, k, h, F = 4096, 8, 2, 4096, 14336
        elif case == "deepseek":
            T, E, k, h, F = 8192, 160, 6, 5120, 1536
        else:  # deepseek_ep4: one card of the 4x2 topology hosts 40 experts over 4 nodes' tokens
            T, E, k, h, F = 8192 * 4, 160, 6, 5120, 1536
        offs_all = routed_offsets(T, E, k, dev)
        if case == "deepseek_ep4":
            L = 40
            offs = (offs_all[:L + 1] - offs_all[0]).contiguous()
        else:
            L = E
            offs = offs_all
        rows = int(offs[-1].item())
        x = torch.randn(rows, h, generator=g).to(torch.bfloat16).to(dev)
        w13 = (torch.randn(L, 2 * F, h, generator=g) * 0.02).to(torch.bfloat16).to(dev)
        w2 = (torch.randn(L, h, F, generator=g) * 0.02).to(torch.bfloat16).to(dev)
        mid = torch.empty(rows, F, dtype=torch.bfloat16, device=dev)
        y = torch.empty(rows, h, dtype=torch.bfloat16, device=dev)
        u1 = timeit(lambda: ops.grouped_gemm(x, w13, offs, act=_lib.ACT_SWIGLU, out=mid), args.iters, flush)
        u2 = timeit(lambda: ops.grouped_gemm(mid, w2, offs, out=y), args.iters, flush)
        uf = timeit(lambda: ops.expert_ffn(x, w13, w2, offs, out=y, workspace=mid), args.iters, flush)
        f1, f2 = 2.0 * rows * 2 * F * h, 2.0 * rows * h * F
        # cuBLAS reference: one matmul per expert segment (what a torch MoE loop does)
        o = offs.tolist()

        def loop():
            for l in range(L):
                a, b = o[l], o[l + 1]
                if b > a:
                    torch.matmul(x[a:b], w13[l].T, out=None)
        ub = timeit(loop, max(3, args.iters // 4), flush)
        print(json.dumps({"case": case, "rows": rows, "L": L, "h": h, "F": F,
                          "gemm1_swiglu_us": u1, "gemm1_tflops": f1 / u1 / 1e6,
                          "gemm2_us": u2, "gemm2_tflops": f2 / u2 / 1e6,
                          "ffn_us": uf, "ffn_tflops": (f1 + f2) / uf / 1e6,
                          "ffn_frac_sustained": (f1 + f2) / uf / 1e6 / sus,
                          "cublas_loop_gemm1_us": ub, "cublas_loop_gemm1_tflops": f1 / ub / 1e6}), flush=True)


if __name__ == "__main__":
    main()

#!/usr/bin/env python
"""MoE dispatch+combine benchmark (BASELINE.json metric: us/layer).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config deepseek|mixtral|toy|70b]
    torchrun --nproc-per-node N bench.py --gpus N ...

Workload: BASELINE.json's metric is not quoted on one config, so the default
is the largest config that fits one GPU, configs[3] (DeepSeek-V2-style
fine-grained MoE layer, bf16): T = 8192 tokens per node group, hidden 5120,
E = 160 experts, top-6.  --config picks the others (mixtral = configs[1],
70b = configs[2], toy = configs[0]).  One card per GPU; the node topology
grows with N (weak scaling: every GPU routes and exchanges one node group's
tokens): N=1 -> 1x1, N=2 -> 2x1 (EP only), N=4 -> 2x2, N=8 -> 4x2
(EP=4 x TP=2, the config's own topology; Mixtral/70b/toy use 2x4).
A step is one layer: route (top-k gate) ->
dispatch (index, count exchange, fused permute+AllToAll, AllGather) ->
combine (reverse AllToAll, weighted un-permute + output AllGather), with
identity experts.  Level/chunks: the MoNTA planner's choice for t >= 2,
Baseline (naive AllToAll) for t == 1; the naive TP-redundant exchange is
timed alongside.

Timing: W warm-up steps; K timed steps, each bracketed by CUDA events on the
launching stream after an L2 flush (256 MiB memset + 256 MiB read) and a cross-rank barrier
(both outside the events); value = sum over steps, max over ranks.  e2e is
the same step through the C ABI host-buffer call (moe_ctx_forward_host: H2D
of x/logits from pinned memory, the layer, D2H of the output).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
os.environ.setdefault("NCCL_DEBUG", "WARN")
# the reference arm / cpu_baseline time the CPU port with every host thread
os.environ.setdefault("OMP_NUM_THREADS", str(os.cpu_count() or 1))
os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")  # NCCL logs (its version line too) off stdout: one JSON line

# BASELINE.json configs as workloads (--config); the default, configs[1], is the metric's workload and the
# others are reported the same way for completeness.  Topology (e x t) per GPU count.
WORKLOADS = {
    "mixtral": ({"workload": "mixtral-8x7b-moe-layer", "tokens_per_node": 4096, "hidden": 4096, "experts": 8,
                 "top_k": 2, "dtype": "bf16", "logits": "f32"}, {1: (1, 1), 2: (2, 1), 4: (2, 2), 8: (2, 4)}),
    "toy": ({"workload": "toy-moe-layer-fp32", "tokens_per_node": 2048, "hidden": 1024, "experts": 8,
             "top_k": 2, "dtype": "f32", "logits": "f32"}, {1: (1, 1), 2: (2, 1), 4: (2, 2), 8: (2, 4)}),
    "70b": ({"workload": "2x70b-moe-layer", "tokens_per_node": 8192, "hidden": 8192, "experts": 2,
             "top_k": 1, "dtype": "bf16", "logits": "f32"}, {1: (1, 1), 2: (2, 1), 4: (2, 2), 8: (2, 4)}),
    "deepseek": ({"workload": "deepseek-v2-finegrained-moe-layer", "tokens_per_node": 8192, "hidden": 5120,
                  "experts": 160, "top_k": 6, "dtype": "bf16", "logits": "f32"},
                 {1: (1, 1), 2: (2, 1), 4: (2, 2), 8: (4, 2)}),
}
DEFAULT_WORKLOAD = "deepseek"  # largest single-GPU config (configs[3]); see the docstring
CONFIG, TOPOLOGY = WORKLOADS[DEFAULT_WORKLOAD]
ELEM = 2  # payload bytes per element


def select_workload(name: str) -> None:
    global CONFIG, TOPOLOGY, ELEM
    CONFIG, TOPOLOGY = WORKLOADS[name]
    ELEM = 4 if CONFIG["dtype"] == "f32" else 2


L2_NOTE = "flushed between steps (256 MiB memset + 256 MiB read outside the events: cold, clean L2)"


def workload_config(e: int, t: int) -> dict:
    """The `config` object of the JSON line — identical for both arms (the
    schedule the repo arm ran, level/chunks/landing/planner, is reported
    beside it under `schedule`)."""
    return dict(CONFIG, topology=f"{e}x{t}", parallelism=f"ep{e}xtp{t}", l2=L2_NOTE)


def payload_dtype():
    import torch
    return torch.float32 if CONFIG["dtype"] == "f32" else torch.bfloat16
METRIC = "moe_dispatch_combine_us_per_layer"
SPAN_LEAD_CYCLES = 2_000_000  # ~1 ms spin ahead of each per-kernel span pass
L2_FLUSH_BYTES = 256 << 20


def topo_for(n: int):
    if n in TOPOLOGY:
        return TOPOLOGY[n]
    return (n, 1)


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md)."""

    def __init__(self, index: int):
        self.index = index
        self.file = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        self.proc = None

    def __enter__(self):
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=self.file, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        time.sleep(0.3)
        return self

    def __exit__(self, *exc):
        if self.proc:
            time.sleep(0.2)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        self.file.flush()
        self.file.seek(0)
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.file.read().splitlines():
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                mx = float(parts[2])
            except ValueError:
                continue
            for nm, v in zip(names, parts[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


def interval_union(iv):
    iv = sorted(iv)
    out = []
    for a, b in iv:
        if out and a <= out[-1][1]:
            out[-1][1] = max(out[-1][1], b)
        else:
            out.append([a, b])
    return out


def exposed(aa, other):
    """Length of union(aa) not covered by union(other)."""
    A, O = interval_union(aa), interval_union(other)
    tot = 0.0
    for a, b in A:
        cov = 0.0
        for c, d in O:
            lo, hi = max(a, c), min(b, d)
            if hi > lo:
                cov += hi - lo
        tot += (b - a) - cov
    return tot


def role_stats(trace):
    """From a persistent-kernel role trace [(role, chunk, start_us, end_us)]:
    busy time per role (union of its chunk intervals) and the exposed
    AllToAll: AA legs not overlapped by the AllGather/reorder legs, plus the
    combine's reverse AllToAll not overlapped by the un-permute."""
    by = {}
    for r, j, a, b in trace:
        by.setdefault(r, []).append((a, b))
    busy = {r: sum(y - x for x, y in interval_union(v)) for r, v in by.items()}
    exp = exposed(by.get("aa", []), by.get("ag", []) + by.get("d2d", [])) + \
        exposed(by.get("caa", []), by.get("unpermute", []))
    return busy, exp


NVLINK_PEAK_GBS = 770.0  # B200_PROFILING.md: measured peer copy per direction (nominal 900)


def nvlink_legs(experts, e, t, E, T, h, node, dedup, recv_rows, busy):
    """NVLink bytes this card stores to peers per step, per leg (SURVEY §8(d)
    numerators with MEASURED counts), and GB/s over each leg's busy time:
    aa   cross-node pairs x (h/t or h) x 2 B   (dispatch AllToAll)
    ag   received cross-node rows x h/t x 2 B x (t-1)   (dispatch AllGather)
    caa  received cross-node rows x (h/t or h) x 2 B   (combine reverse AllToAll)
    out  T x h/t x 2 B x (t-1)   (output AllGather fused into the un-permute)"""
    L = E // e
    valid = experts >= 0
    own = valid & (experts // L == node)
    cross_pairs = int((valid & ~own).sum())
    recv_cross = int(recv_rows) - int(own.sum())
    sl = (h // t if dedup else h) * ELEM
    legs = {"aa": cross_pairs * sl, "ag": recv_cross * sl * (t - 1) if dedup else 0,
            "caa": recv_cross * sl, "unpermute": T * sl * (t - 1) if dedup else 0}
    out = {}
    for r, b in legs.items():
        us = busy.get(r, 0.0)
        out[r] = {"bytes": b, "busy_us": us, "gbs": b / us / 1e3 if us and b else None}
    disp_b = legs["aa"] + legs["ag"]
    disp_us = busy.get("aa", 0.0) + busy.get("ag", 0.0)
    comb_b = legs["caa"] + legs["unpermute"]
    comb_us = busy.get("caa", 0.0) + busy.get("unpermute", 0.0)
    return {"peak": NVLINK_PEAK_GBS, "legs": out,
            "dispatch": {"bytes": disp_b, "busy_us": disp_us, "gbs": disp_b / disp_us / 1e3 if disp_us else None},
            "combine": {"bytes": comb_b, "busy_us": comb_us, "gbs": comb_b / comb_us / 1e3 if comb_us else None},
            "note": "bytes this card stores to peer GPUs per step / role busy time from the persistent kernels' "
                    "traces (legs of one kernel run back to back at n=1)"}


# ---------------------------------------------------------------------------
def cpu_threads() -> int:
    """Host threads the CPU port uses: OMP_NUM_THREADS, else every host thread
    (bench.py sets it before the oracle library loads)."""
    return int(os.environ.get("OMP_NUM_THREADS") or os.cpu_count() or 1)


def cpu_port_layer(e, t, E, k, T, h, seed=0):
    """One full layer of the oracle port (oracle/moe_oracle.c: the C
    restatement of the reference data plane, E > e generalised) on the host,
    single-threaded: route_topk + permute + dispatch + combine of every node.
    Returns seconds (input generation excluded)."""
    import numpy as np
    import oracle
    rng = np.random.default_rng(seed)
    x = rng.standard_normal((e, T, h)).astype(np.float32)
    if ELEM == 4:
        xbytes = x.view(np.uint8).reshape(e, T, h * 4)
    else:
        xbytes = (x.view(np.uint32) >> 16).astype(np.uint16).view(np.uint8).reshape(e, T, h * 2)  # bf16 bits
    logits = rng.standard_normal((e, T, E))
    t0 = time.perf_counter()
    experts = np.zeros((e, T, k), np.int32)
    probs = np.zeros((e, T, k), np.float64)
    for g in range(e):
        experts[g], probs[g] = oracle.route_topk(logits[g], k)
    nodes = oracle.Nodes(e, t, E, xbytes, experts)
    fin = nodes.dispatch_chunked(oracle.O1, 1, ELEM)[0] if t > 1 else nodes.dispatch_monolithic()
    nodes.combine(oracle.F32 if ELEM == 4 else oracle.BF16, fin, probs)
    return time.perf_counter() - t0


def cpu_baseline_value(e, t, E, k, T, h, budget_s=10.0, max_reps=100):
    vals, spent = [], 0.0
    while spent < budget_s and len(vals) < max_reps:
        dt = cpu_port_layer(e, t, E, k, T, h, seed=len(vals))
        vals.append(dt)
        spent += dt
    return statistics.mean(vals) * 1e6, len(vals), spent


def run_reference(args):
    """--impl reference: the reference's CPU path on this host (rank 0 only).
    With one expert per node (E == e: the 2x70B layer at N = 2) the unmodified
    reference headers (oracle/_ref) run.  Otherwise they cannot — with more
    experts than nodes (E = 160 on e <= 4) its dispatch drops records and its
    combine indexes out of bounds (SURVEY.md §7 decision 1) — so the arm times
    the oracle port, the C restatement of the same algorithm generalised to
    E > e, on every host thread (OpenMP over tokens, experts and records)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    e, t = topo_for(args.gpus)
    T, h, E, k = CONFIG["tokens_per_node"], CONFIG["hidden"], CONFIG["experts"], CONFIG["top_k"]
    import oracle
    if E == e and oracle.ref_available():
        # one expert per node (the 2x70B layer at N = 2): the reference itself
        # runs — its route_topk and dispatch + combine on its own int64
        # payload records, single-threaded, on a bounded token sample scaled
        # to the node batch
        import numpy as np
        Ts = min(T, 1024)

        def ref_layer(seed):
            rng = np.random.default_rng(seed)
            pay = rng.integers(-1000, 1000, size=(e, Ts, h), dtype=np.int64)
            sc = rng.standard_normal((e, Ts, E))
            t0 = time.perf_counter()
            ex = np.zeros((e, Ts, k), np.int32)
            pr = np.zeros((e, Ts, k), np.float64)
            for g in range(e):
                ex[g], pr[g] = oracle.ref_route_topk(sc[g], k)
            oracle.ref_dataplane(e, t, pay, ex, pr, level=-1 if t == 1 else 1, n=1)
            return (time.perf_counter() - t0) * T / Ts

        for _ in range(max(1, args.warmup)):
            ref_layer(0)
        vals = [ref_layer(s + 1) * 1e6 for s in range(max(1, args.steps))]
        v = statistics.mean(vals)
        line = {"metric": METRIC, "value": v, "unit": "us/layer", "n_gpus": args.gpus, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": v / 1e3, "higher_is_better": False, "scaling": "weak",
                "vs_baseline": None, "dtype": CONFIG["dtype"], "data": "synthetic", "impl": "reference",
                "config": workload_config(e, t),
                "cpu_baseline": {"value": v, "unit": "us/layer", "cores": 1, "kind": "reference",
                                 "sample": f"{Ts} of {T} tokens per node x {e} nodes per step, scaled x{T / Ts:g}; "
                                           "unmodified reference headers (oracle/_ref: route_topk, dispatch, "
                                           "combine_unpermute on int64 payload records), 1 thread"},
                "e2e": {"value": v, "unit": "us/layer", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(line), flush=True)
        return
    for _ in range(max(1, args.warmup)):
        cpu_port_layer(e, t, E, k, T, h)
    vals = [cpu_port_layer(e, t, E, k, T, h, seed=s) * 1e6 for s in range(max(1, args.steps))]
    v = statistics.mean(vals)
    line = {"metric": METRIC, "value": v, "unit": "us/layer", "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": v / 1e3, "higher_is_better": False, "scaling": "weak",
            "vs_baseline": None, "dtype": CONFIG["dtype"], "data": "synthetic", "impl": "reference",
            "config": workload_config(e, t),
            "cpu_baseline": {"value": v, "unit": "us/layer", "cores": cpu_threads(), "kind": "port",
                             "sample": f"full layer ({T} tokens x {e} nodes) per step, {args.steps} steps; "
                                       f"oracle/moe_oracle.c (OpenMP), {cpu_threads()} threads of {os.cpu_count()}"},
            "e2e": {"value": v, "unit": "us/layer", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
def backward_kernels(T, h, E, k, cold_l2, peak, iters=10):
    """SURVEY §8(f) item 2 at the workload's size, outside the timed region:
    the three backward kernels (ops.*_backward) each timed alone with CUDA
    events after a cold-L2 flush, median of `iters`, with their algorithmic
    HBM bytes (scripts/micro/backward_bench.py has the per-kernel formulas)."""
    import torch

    from paper_2411_00662_b200 import _lib, ops
    dev = torch.device("cuda", torch.cuda.current_device())
    dt = payload_dtype()
    b = ELEM
    gen = torch.Generator(device="cpu").manual_seed(7)
    logits = torch.randn(T, E, generator=gen).to(dev)
    experts, probs = ops.route_topk(logits, k)
    idx = ops.build_index(experts, E)
    R = T * k
    y = torch.randn(R, h, generator=gen).to(dt).to(dev)
    g = torch.randn(T, h, generator=gen).to(dt).to(dev)
    gy, gp, gx, gz = torch.empty_like(y), torch.empty_like(probs), torch.empty_like(g), torch.empty_like(logits)
    lib, dc, sp = _lib.load(), _lib.dtype_code(dt), idx.slot_pos

    def st():
        return torch.cuda.current_stream().cuda_stream

    runs = {
        "combine_backward": (lambda: _lib.check(lib.moe_combine_backward(
            g.data_ptr(), dc, h, y.data_ptr(), dc, h, h, sp.data_ptr(), probs.data_ptr(), _lib.F32, T, k,
            gy.data_ptr(), h, gp.data_ptr(), st())), T * h * b + 2 * R * h * b + 12 * R),
        "dispatch_backward": (lambda: _lib.check(lib.moe_dispatch_backward(
            y.data_ptr(), dc, h, h, sp.data_ptr(), T, k, gx.data_ptr(), dc, h, st())), R * h * b + T * h * b + 4 * R),
        "route_backward": (lambda: _lib.check(lib.moe_route_backward(
            logits.data_ptr(), _lib.F32, T, E, k, experts.data_ptr(), probs.data_ptr(), gz.data_ptr(), st())),
            8 * T * E + 8 * R),
    }
    out = {}
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for name, (fn, nbytes) in runs.items():
        fn()
        ts = []
        for _ in range(iters):
            cold_l2()  # queued ahead on the same stream: the GPU is still flushing when the
            ev0.record()  # start event and the launch are enqueued, so no host gap is timed
            fn()
            ev1.record()
            torch.cuda.synchronize()
            ts.append(ev0.elapsed_time(ev1) * 1e3)
        us = sorted(ts)[len(ts) // 2]
        out[name] = {"us": us, "bytes": nbytes, "gbs": nbytes / us / 1e3, "frac": nbytes / us / 1e3 / peak}
    out["sum_us"] = sum(v["us"] for v in out.values() if isinstance(v, dict))
    out["note"] = ("per-card adjoints of combine/dispatch/route (include/monta.h 1b), C-ABI calls into "
                   "preallocated buffers; cold L2; each timed alone, outside the bench's timed region")
    return out


FFN_DIM = {"deepseek-v2-finegrained-moe-layer": 1536, "mixtral-8x7b-moe-layer": 14336,
           "2x70b-moe-layer": 28672}  # expert intermediate size of each workload's model


def experts_leg(layer, cd, e, t, E, h, step, timed, steps, local, dedup=False):
    """Layer step with the experts bound (random-init SwiGLU weights of the
    workload's expert shape): us/layer, the experts stage's time and its
    tensor-core throughput (2 * rows * (2F * h + F * down_cols) flops per card:
    down_cols = h / t under TP dedup, the slice the card's combine reads) against
    MEASURED_PEAKS.json's sustained bf16 figure."""
    import torch
    from paper_2411_00662_b200 import ops
    F = FFN_DIM.get(CONFIG["workload"])
    if F is None:
        return None
    L = E // e
    dev = f"cuda:{local}"
    gen = torch.Generator(device=dev).manual_seed(99 + cd.node)
    lo = cd.node * L
    wg = (torch.randn(L, F, h, generator=gen, device=dev) * h ** -0.5).to(torch.bfloat16)
    wu = (torch.randn(L, F, h, generator=gen, device=dev) * h ** -0.5).to(torch.bfloat16)
    w13 = ops.interleave_w13(wg, wu)
    del wg, wu
    w2 = (torch.randn(L, h, F, generator=gen, device=dev) * F ** -0.5).to(torch.bfloat16)
    layer.bind_experts(cd.card, w13, w2)
    try:
        for _ in range(3):
            step()
        layer.sync()
        tot, _ = timed(step, steps)
        layer.enable_timing(True)
        sp = []
        for _ in range(3):
            step()
            sp.append([b - a for st, j, a, b in layer.spans() if st == "experts"])
        layer.enable_timing(False)
        layer.sync()
        rows = layer.recv_rows(cd.card)
        seq = None
        if e > 1:  # the same step with the reverse AllToAll NOT fused into the down-projection
            layer.set_expert_overlap(False)
            for _ in range(3):
                step()
            layer.sync()
            tseq, _ = timed(step, steps)
            seq = tseq * 1e3 / steps
            layer.set_expert_overlap(True)
    finally:
        layer.bind_experts(cd.card, None)
    ex_us = 1e3 * statistics.median(sum(v) for v in sp)
    # gate/up over every landed row; the down-projection over the columns the
    # card's combine reads (its 1/t slice under TP dedup, csrc/ctx.cu)
    down_cols = h // t if (dedup and (h // t) % 128 == 0) else h
    flops = 2.0 * rows * (2 * F * h + F * down_cols)
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            pk = json.load(f)
        peak, kind = float(pk["bf16_tflops_sustained"]), "measured bf16_tflops_sustained"
    except Exception:
        peak, kind = 1800.0, "fallback"
    ach = flops / ex_us / 1e6
    return {"us_per_layer_with_experts": tot * 1e3 / steps,
            "us_per_layer_with_experts_no_overlap": seq,
            "reverse_alltoall_fused_into_down_proj": e > 1,
            "experts_us": ex_us, "rows": rows, "ffn": F,
            "local_experts": L, "flops_per_card": flops, "down_proj_cols": down_cols,
            "roofline": {"bound": "tensor", "kernel": "k_grouped_gemm x2 (SwiGLU gate/up, down)", "achieved": ach,
                         "peak": peak, "unit": "TFLOP/s", "frac": ach / peak, "peak_kind": kind},
            "note": "random-init SwiGLU experts of the workload's expert shape (h x F) between dispatch and "
                    "combine; experts_us from the stage's in-graph events"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default=DEFAULT_WORKLOAD, choices=sorted(WORKLOADS),
                    help="BASELINE.json workload (default: configs[3], the largest that fits one GPU)")
    ap.add_argument("--level", default="auto", help="auto|baseline|o1|o2|o3")
    ap.add_argument("--chunks", type=int, default=0)
    ap.add_argument("--landing", default="final", choices=["final", "staged"])
    ap.add_argument("--quick", action="store_true", help="skip naive/e2e/cpu extras (profiling runs)")
    ap.add_argument("--no-graphs", action="store_true", help="launch eagerly instead of replaying CUDA graphs")
    ap.add_argument("--aa-ctas", type=int, default=0,
                    help="B1-throttled mode: cap the cross-node AllToAll legs at this many CTAs (0: off)")
    ap.add_argument("--link-gbs", type=float, default=0.0,
                    help="emulate a slow inter-node link for the cross-node legs (GB/s per card; the paper's "
                         "B1 << B2 regime, PAPER.md:183-184); the planner then uses the reference's separate-links model")
    ap.add_argument("--wire", default="bf16", choices=["bf16", "fp8"],
                    help="cross-node dispatch payload (fp8: e4m3 + per-128 scales, lossy; SURVEY §8(f) item 3)")
    ap.add_argument("--no-persistent", action="store_true",
                    help="multi-GPU: one launch per (leg, chunk) instead of the persistent exchange kernels")
    args = ap.parse_args()
    select_workload(args.config)
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
        return

    import torch
    import torch.distributed as dist
    from paper_2411_00662_b200 import _lib, planner as P
    from paper_2411_00662_b200.layer import MoeLayer, BASELINE, O1, O2, O3, LAND_FINAL, LAND_STAGED

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    e, t = topo_for(world)
    T, h, E, k = CONFIG["tokens_per_node"], CONFIG["hidden"], CONFIG["experts"], CONFIG["top_k"]
    node, rho = rank // t, rank % t

    # ---- level / chunk count: MoNTA planner on the B200 NVLink curves
    levels = {"baseline": BASELINE, "o1": O1, "o2": O2, "o3": O3}
    # curves fitted from the exchange kernel's own role traces when present
    # (scripts/calibrate_from_sweep.py), else the standalone-copy calibration
    curves_dir = os.path.join(ROOT, "profiles", "curves_b200", f"{e}x{t}_xchg")
    if not os.path.isdir(curves_dir):
        curves_dir = os.path.join(ROOT, "profiles", "curves_b200", f"{e}x{t}")
    decision = None
    if args.level != "auto":
        level = levels[args.level]
        n = args.chunks or (1 if level in (BASELINE, O1) else 4)
    elif t == 1:
        level, n = BASELINE, 1
    else:
        try:
            curves = P.load_curve_set(curves_dir)
            ov = P.OverheadModel(**json.load(open(os.path.join(curves_dir, "overhead.json"))))
        except Exception:
            curves = P.CurveSet(P.EfficiencyCurve.constant(0.8), P.EfficiencyCurve.constant(0.8),
                                P.EfficiencyCurve.constant(0.8))
            ov = P.OverheadModel(8e-6, 4e-6)
        model = P.ModelSpec(b=1, s=T * k, h=h, k=k, bpe=ELEM)  # routed rows: s_eff = T*k
        cluster = P.b200_cluster(e, t)
        if args.link_gbs:  # emulated inter-node link: paced legs move at exactly that rate
            cluster = P.b200_cluster(e, t, b1=args.link_gbs * 1e9)
            curves = P.CurveSet(P.EfficiencyCurve.constant(1.0), curves.allgather, curves.d2d)
        # the reference's selection (separate inter-/intra-node links), reported as is
        decision = P.select_strategy(model, P.ParallelSpec(t=t, e=e), cluster, curves, ov, n_cap=16)
        # the B200 variant: on one NVSwitch box both legs leave through the same
        # NVLink egress (not so when the AllToAll is throttled: B1-emulated mode)
        decision_b200 = P.select_strategy_b200(model, P.ParallelSpec(t=t, e=e), cluster, curves, ov,
                                               n_cap=16, shared_egress=not (args.aa_ctas or args.link_gbs))
        level, n = int(decision_b200.level), decision_b200.n
        while T % n:
            n -= 1
    landing = LAND_STAGED if args.landing == "staged" else LAND_FINAL

    PD = payload_dtype()
    layer = MoeLayer(e, t, E, k, T, h, dtype=PD, logit_dtype=torch.float32, max_chunks=16,
                     device=local, rank=rank if world > 1 else 0, world_size=world)
    layer.connect()
    layer.enable_graphs(not args.no_graphs)
    if args.no_persistent:
        layer.set_persistent(False)
    if args.aa_ctas:
        layer.set_aa_ctas(args.aa_ctas)
    if args.wire == "fp8":
        layer.set_wire(_lib.WIRE_FP8)
    if args.link_gbs:
        layer.set_link_rate(args.link_gbs)
    cd = layer.cards[0]
    gen = torch.Generator(device=f"cuda:{local}").manual_seed(1234 + node)
    x0 = torch.randn(T, h, generator=gen, device=f"cuda:{local}").to(PD)
    l0 = torch.randn(T, E, generator=gen, device=f"cuda:{local}")
    cd.x.copy_(x0)
    cd.logits.copy_(l0)
    flush = torch.empty(L2_FLUSH_BYTES, dtype=torch.uint8, device=f"cuda:{local}")
    flush_rd = torch.ones(L2_FLUSH_BYTES // 4, dtype=torch.float32, device=f"cuda:{local}")

    def cold_l2():
        # write a buffer larger than L2 (evicts everything), then read another
        # one: the memset's dirty lines are written back here, outside the
        # events, so the step starts from a cold AND clean L2 (what ncu's
        # --cache-control all gives each kernel)
        if os.environ.get("MONTA_BENCH_NO_FLUSH") == "1":  # diagnosis only: never for a reported number
            return
        flush.zero_()
        flush_rd.amax()
    stream = torch.cuda.current_stream()
    bar = torch.zeros(1, device=f"cuda:{local}")

    def barrier():
        if world > 1:
            dist.all_reduce(bar)

    def timed(step_fn, steps):
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
        torch.cuda.synchronize()
        barrier()
        torch.cuda.synchronize()
        for a, b in evs:
            cold_l2()
            barrier()
            a.record(stream)
            step_fn()
            b.record(stream)
        torch.cuda.synchronize()
        barrier()
        torch.cuda.synchronize()
        ms = [a.elapsed_time(b) for a, b in evs]
        total = torch.tensor([sum(ms)], dtype=torch.float64, device=f"cuda:{local}")
        if world > 1:
            dist.all_reduce(total, op=dist.ReduceOp.MAX)
        return float(total.item()), ms

    def step(lv=None, nn=None, ld=None):  # defaults: the (possibly re-chosen) level, n, landing
        layer.forward(level if lv is None else lv, n if nn is None else nn, landing if ld is None else ld, stream)

    # The schedule runs as the library decides it: the B200 planner variant's
    # choice and the reference's (when they differ) are timed in place by
    # moe_ctx_autotune (max over ranks, inside the C ABI) and the faster runs.
    autotune = None
    if decision is not None and args.level == "auto":
        rn = decision.n
        while T % rn:
            rn -= 1
        cands = [(level, n, landing)]
        if (int(decision.level), rn) != (level, n):
            cands.append((int(decision.level), rn, landing))
        if t > 1 and all(c[0] != BASELINE for c in cands):
            # the naive exchange too: with few experts per node (Mixtral, 2x70B)
            # the TP-redundant rows cost less than the AllGather round
            cands.append((BASELINE, 1, LAND_FINAL))
        if len(cands) > 1:
            best, times = layer.autotune(cands, steps=5, stream=stream)
            autotune = {"candidates": [[_lib.LEVEL_NAMES[c[0]], c[1], us] for c, us in zip(cands, times)],
                        "chosen": [_lib.LEVEL_NAMES[cands[best][0]], cands[best][1]]}
            level, n = cands[best][0], cands[best][1]

    for _ in range(args.warmup):
        step()
    layer.sync()
    launches0 = layer.launch_count
    with ClockSampler(local) as clk:
        total_ms, per = timed(step, args.steps)
    launches = layer.launch_count - launches0
    layer.sync()
    us = total_ms * 1e3 / args.steps

    # ---- per-kernel spans (separate pass, events per launch on its stream)
    layer.enable_timing(True)
    span_sets, traces = [], []
    for _ in range(3):
        cold_l2()
        barrier()
        torch.cuda._sleep(SPAN_LEAD_CYCLES)  # the host enqueues the whole step before the GPU reaches it
        step()
        span_sets.append(layer.spans())
        traces.append(layer.xchg_trace() if world > 1 else [])
    layer.enable_timing(False)
    layer.sync()

    def stage_stats(spans_list):
        out = {}
        for spans in spans_list:
            for st, j, a, b in spans:
                out.setdefault(st, []).append(b - a)
        return {s: {"launches_per_step": len(v) // len(spans_list), "avg_us": 1e3 * sum(v) / len(v),
                    "sum_us_per_step": 1e3 * sum(v) / len(spans_list)} for s, v in out.items()}

    def exposed_aa(spans_list, traces=None):
        if traces and any(traces):
            return statistics.mean(role_stats(tr)[1] for tr in traces)
        vals = []
        for spans in spans_list:
            aa = [(a, b) for st, j, a, b in spans if st == "aa"]
            oth = [(a, b) for st, j, a, b in spans if st in ("ag", "d2d")]
            caa = [(a, b) for st, j, a, b in spans if st == "caa"]
            unp = [(a, b) for st, j, a, b in spans if st == "unpermute"]
            vals.append(exposed(aa, oth) + exposed(caa, unp))
        return 1e3 * statistics.mean(vals)

    stages = stage_stats(span_sets)
    exp_aa = exposed_aa(span_sets, traces)
    roles = None
    if any(traces):
        rs = [role_stats(tr)[0] for tr in traces]
        roles = {r: statistics.mean(x.get(r, 0.0) for x in rs) for r in set().union(*rs)}

    # ---- naive TP-redundant exchange at the same N (for the headline ratio)
    naive = None
    if not args.quick and level != BASELINE:
        for _ in range(3):
            step(BASELINE, 1)
        layer.sync()
        ntot, _ = timed(lambda: step(BASELINE, 1), args.steps)
        layer.enable_timing(True)
        nspans, ntr = [], []
        for _ in range(3):
            cold_l2()
            barrier()
            torch.cuda._sleep(SPAN_LEAD_CYCLES)
            step(BASELINE, 1)
            nspans.append(layer.spans())
            ntr.append(layer.xchg_trace() if world > 1 else [])
        layer.enable_timing(False)
        layer.sync()
        naive = {"us_per_layer": ntot * 1e3 / args.steps, "exposed_alltoall_us": exposed_aa(nspans, ntr),
                 "stages": stage_stats(nspans)}
        if any(ntr):
            rs = [role_stats(tr)[0] for tr in ntr]
            naive["roles_busy_us"] = {r: statistics.mean(x.get(r, 0.0) for x in rs) for r in set().union(*rs)}

    # ---- MoNTA's chunked pipeline (O2/O3) at the same N: the AllGather of
    # chunk j overlaps the AllToAll of chunk j+1, which shrinks the exposed
    # AllToAll (the paper's headline) at the price of per-chunk costs; the
    # planner weighs both and picks the level above
    pipelined = None
    if not args.quick and t > 1:
        pipelined = []
        for lv, nn, ld in ((O2, 4, LAND_FINAL), (O3, 4, LAND_STAGED), (O2, 8, LAND_FINAL)):
            if T % nn or nn > layer.max_chunks or (ld == LAND_STAGED and args.wire == "fp8"):
                continue
            for _ in range(3):
                step(lv, nn, ld)
            layer.sync()
            ptot, _ = timed(lambda: step(lv, nn, ld), args.steps)
            layer.enable_timing(True)
            ptr = []
            for _ in range(3):
                cold_l2()
                barrier()
                torch.cuda._sleep(SPAN_LEAD_CYCLES)
                step(lv, nn, ld)
                layer.spans()
                ptr.append(layer.xchg_trace())
            layer.enable_timing(False)
            layer.sync()
            pipelined.append({"level": _lib.LEVEL_NAMES[lv], "n": nn, "landing": "staged" if ld else "final",
                              "us_per_layer": ptot * 1e3 / args.steps,
                              "exposed_alltoall_us": statistics.mean(role_stats(tr)[1] for tr in ptr) if any(ptr)
                              else None})

    # ---- robustness: Zipf-skewed routing, same shapes
    skewed = None
    if not args.quick:
        zipf = torch.log(1.0 / torch.arange(1, E + 1, device=f"cuda:{local}", dtype=torch.float32) ** 1.2)
        cd.logits.copy_(l0 + 2.0 * zipf[None, :])
        for _ in range(3):
            step()
        layer.sync()
        stot, _ = timed(step, args.steps)
        loads = torch.bincount(cd.experts.flatten().long(), minlength=E).float()
        skewed = {"us_per_layer": stot * 1e3 / args.steps, "routing": "logits + 2*log(rank^-1.2) (Zipf s=1.2)",
                  "max_over_mean_expert_load": float(loads.max() / loads.mean())}
        cd.logits.copy_(l0)
        for _ in range(2):
            step()
        layer.sync()

    # ---- e2e through the C ABI with host buffers
    e2e = None
    if not args.quick:
        # staging buffers from the ABI's host allocator (moe_host_alloc: cudaHostAlloc,
        # portable): on some boxes torch's pin_memory() pages copy host->device at
        # 37 GB/s against 55 GB/s for cudaHostAlloc'd ones (scripts/pcie_probe.py)
        from paper_2411_00662_b200.ops import host_empty
        hx = host_empty((T, h), PD)
        hl = host_empty((T, E), torch.float32)
        ho = host_empty((T, h), PD)
        hx.copy_(x0.cpu())
        hl.copy_(l0.cpu())

        def host_step():
            layer.forward_host(hx, hl, ho, level, n, landing, stream)

        for _ in range(3):
            host_step()
        torch.cuda.synchronize()
        etot, eper = timed(host_step, args.steps)
        layer.sync()
        e2e = {"value": etot * 1e3 / args.steps, "unit": "us/layer",
               "h2d_bytes_per_step": hx.numel() * ELEM + hl.numel() * 4, "d2h_bytes_per_step": ho.numel() * ELEM,
               "step_us_median": statistics.median(eper) * 1e3, "step_us_min": min(eper) * 1e3}

    # ---- the same layer with SwiGLU experts between
    # dispatch and combine (tcgen05 grouped GEMMs on the dispatched rows);
    # reported beside the metric, which is dispatch+combine
    experts = None
    if not args.quick and CONFIG["dtype"] == "bf16":
        try:
            experts = experts_leg(layer, cd, e, t, E, h, step, timed, args.steps, local,
                                  dedup=(level != BASELINE and t > 1))
        except Exception as exc:  # extra figures: never lose the bench line to them
            experts = {"error": f"{type(exc).__name__}: {exc}"}

    # ---- correctness spot check of the timed configuration (identity experts)
    layer.forward(level, n, landing, stream)
    layer.sync()
    psum = cd.probs.double().sum(1, keepdim=True)
    err = ((cd.out.double() - x0.double() * psum).abs().max() / x0.double().abs().max()).item()

    # ---- roofline of the dominant kernel (HBM-bound: algorithmic bytes / live duration)
    peak, peak_kind = load_peaks()
    R = T * k
    row = h * ELEM
    Rdst = layer.recv_rows(cd.card)
    # algorithmic bytes per launch
    if world == 1:
        # token-side AA: each token row read once, written to its k destinations,
        # + tags (16 B/row) and the index reads (experts, slot_pos: 8 B/pair)
        aa_bytes = T * row + R * row + 16 * R + 8 * R
    else:
        aa_bytes = None  # NVLink-bound: reported under "nvlink"
    unp_cols = h // t if (level != BASELINE and t > 1) else h
    unp_bytes = R * unp_cols * ELEM + T * unp_cols * ELEM * (t if (level != BASELINE and t > 1) else 1) + 12 * R
    kern = {}
    if "aa" in stages and aa_bytes:
        kern["fused_permute_aa"] = (aa_bytes * stages["aa"]["launches_per_step"] / max(stages["aa"]["sum_us_per_step"], 1e-9)) / 1e3
    if "unpermute" in stages:
        kern["unpermute_combine"] = (unp_bytes / max(stages["unpermute"]["sum_us_per_step"], 1e-9)) / 1e3
    if world == 1 and "aa" in stages and "unpermute" in stages:
        # the permute's row stores mostly land in L2 and are written back while
        # the un-permute runs, so each kernel's own figure misattributes DRAM
        # time; the pair's DRAM bytes (x read, permuted rows written + read,
        # output written) over their summed time is the honest HBM figure
        pair_bytes = aa_bytes + unp_bytes
        pair_us = stages["aa"]["sum_us_per_step"] + stages["unpermute"]["sum_us_per_step"]
        kern["permute_plus_unpermute"] = pair_bytes / pair_us / 1e3
    dom = max(((s, v["sum_us_per_step"]) for s, v in stages.items() if s in ("aa", "unpermute")),
              key=lambda z: z[1], default=("unpermute", 1.0))[0]
    if dom == "aa" and aa_bytes:
        ach = kern["fused_permute_aa"]
        traffic_alg = aa_bytes
        # the lone card's full-batch permute runs the TMA ring (aa.cu launch_aa_token)
        bulk = (world == 1 and T >= 2048 and k >= 4 and (h * ELEM) % 16 == 0 and os.environ.get("MONTA_AA_BULK", "1") != "0"
                and args.wire == "bf16" and not args.link_gbs)
        dom_name = "fused_permute_aa (k_aa_bulk)" if bulk else "fused_permute_aa (k_aa_token<16>)"
    else:
        ach = kern.get("unpermute_combine", 0.0)
        traffic_alg = unp_bytes
        dom_name = ("unpermute_combine (k_unpermute_k2<bf16,bf16,f32>)" if ELEM == 2 and k <= 2
                    else "unpermute_combine (k_unpermute_rows)" if ELEM == 2 else "unpermute_combine (k_unpermute)")
    # DRAM bytes of the same kernel from an ncu --set full capture of this
    # workload (profiles/ncu_traffic.json, keyed by workload then stage); null
    # when that workload has no capture or the kernel differs from the one timed
    ncu_traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            ncu_traffic = json.load(f)["workloads"][CONFIG["workload"]].get(dom_name.split(" ")[0])
    except Exception:
        pass
    roofline = {"bound": "hbm", "kernel": dom_name, "achieved": ach, "peak": peak, "unit": "GB/s",
                "frac": ach / peak, "traffic": ncu_traffic, "algorithmic_bytes_per_launch": traffic_alg,
                "peak_kind": peak_kind, "kernels_gbs": kern}

    # NVLink: bytes this card stores to peer GPUs per step, per leg, over the
    # leg's busy time in the persistent kernels' role traces (first CTA start
    # to last CTA's release; stores may still be draining at the release)
    nvlink = None
    if world > 1:
        nvlink = nvlink_legs(cd.experts.cpu().numpy(), e, t, E, T, h, node, level != BASELINE and t > 1, Rdst,
                             roles or {})
        if nvlink["dispatch"]["gbs"]:
            roofline = {"bound": "nvlink", "kernel": "k_xchg (persistent dispatch exchange: AllToAll + AllGather legs)",
                        "achieved": nvlink["dispatch"]["gbs"], "peak": NVLINK_PEAK_GBS, "unit": "GB/s",
                        "frac": nvlink["dispatch"]["gbs"] / NVLINK_PEAK_GBS, "traffic": None,
                        "algorithmic_bytes_per_launch": nvlink["dispatch"]["bytes"],
                        "peak_kind": "B200_PROFILING.md measured peer copy per direction"}
        elif nvlink["combine"]["gbs"]:
            # the node-dedup dispatch (per-launch kernels, no role traces) moves
            # fewer bytes than the per-(token, expert) legs above; the combine
            # runs the persistent kernel, whose reverse-AllToAll leg is timed
            roofline = {"bound": "nvlink", "kernel": "k_combine_xchg (persistent combine: reverse AllToAll leg)",
                        "achieved": nvlink["legs"]["caa"]["gbs"] or nvlink["combine"]["gbs"],
                        "peak": NVLINK_PEAK_GBS, "unit": "GB/s",
                        "frac": (nvlink["legs"]["caa"]["gbs"] or nvlink["combine"]["gbs"]) / NVLINK_PEAK_GBS,
                        "traffic": None, "algorithmic_bytes_per_launch": nvlink["legs"]["caa"]["bytes"],
                        "peak_kind": "B200_PROFILING.md measured peer copy per direction",
                        "note": "dispatch: node dedup (one row per (token, remote node)); its legs are not traced"}
        elif "caa" in stages and stages["caa"]["sum_us_per_step"] > 0:
            # per-launch combine (unchunked EP-only): the reverse AllToAll launch's in-graph span
            gbs = nvlink["legs"]["caa"]["bytes"] / stages["caa"]["sum_us_per_step"] / 1e3
            roofline = {"bound": "nvlink", "kernel": "k_seg_copy (combine reverse AllToAll launch)",
                        "achieved": gbs, "peak": NVLINK_PEAK_GBS, "unit": "GB/s", "frac": gbs / NVLINK_PEAK_GBS,
                        "traffic": None, "algorithmic_bytes_per_launch": nvlink["legs"]["caa"]["bytes"],
                        "peak_kind": "B200_PROFILING.md measured peer copy per direction",
                        "note": "dispatch: node dedup (one row per (token, remote node)); its legs are not traced"}

    cpu = None
    if rank == 0 and world == 1 and not args.quick:
        cpu_us, reps, secs = cpu_baseline_value(e, t, E, k, T, h)
        cpu = {"value": cpu_us, "unit": "us/layer", "cores": cpu_threads(), "kind": "port",
               "sample": f"{reps} full layers ({T} tokens, {secs:.1f} s CPU); oracle/moe_oracle.c "
                         f"route+permute+dispatch+combine (OpenMP over tokens / experts / records), "
                         f"{cpu_threads()} threads of {os.cpu_count()} host threads"}

    backward = None
    if world == 1 and not args.quick:
        try:
            backward = backward_kernels(T, h, E, k, cold_l2, peak)
        except Exception as exc:  # the backward figures are extra; never lose the bench line to them
            backward = {"error": f"{type(exc).__name__}: {exc}"}

    line = {"metric": METRIC, "value": us, "unit": "us/layer", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": us / 1e3, "higher_is_better": False, "scaling": "weak",
            "vs_baseline": None, "dtype": CONFIG["dtype"], "data": "synthetic (randn x, randn f32 gate logits)",
            "config": workload_config(e, t),
            "schedule": {"level": _lib.LEVEL_NAMES[level], "chunks": n, "landing": args.landing,
                         "aa_ctas": args.aa_ctas or None, "wire": args.wire, "link_gbs": args.link_gbs or None,
                         "cuda_graphs": not args.no_graphs,
                         "planner": None if decision is None else
                         {"reference": {"level": _lib.LEVEL_NAMES[int(decision.level)], "n": decision.n,
                                        "t_pred_us": decision.t_pred * 1e6},
                          "b200_shared_egress": {"level": _lib.LEVEL_NAMES[int(decision_b200.level)],
                                                 "n": decision_b200.n, "t_pred_us": decision_b200.t_pred * 1e6,
                                                 "alternatives": [[_lib.LEVEL_NAMES[int(a.level)], a.n,
                                                                   a.t_pred * 1e6]
                                                                  for a in decision_b200.alternatives]},
                          "autotune_us": autotune}},
            "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches,
            "clocks": clk.summary(), "stages": stages, "roles_busy_us": roles, "exposed_alltoall_us": exp_aa,
            "naive": naive,
            "pipelined": pipelined,
            "skewed": skewed,
            "nvlink": nvlink, "check_max_rel_err": err, "backward": backward, "experts": experts}
    if rank == 0:
        print(json.dumps(line), flush=True)
    layer.close()
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()

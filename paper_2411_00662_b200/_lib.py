"""ctypes binding of the C ABI in include/monta.h (libmonta.so).

The library is the product: every op below calls straight into the CUDA
kernels or the C++ planner through the C ABI.  There is no Python or CPU
fallback — if the library is missing or was built without a GPU target the
import fails loudly.
"""
from __future__ import annotations

import ctypes as C
import os
import pathlib

PKG = pathlib.Path(__file__).resolve().parent
LIB_PATH = PKG / "lib" / "libmonta.so"

ABI_VERSION = 2  # include/monta.h MONTA_ABI_VERSION (the card view / structs this binding mirrors)

# moe_status
OK = 0
ERR_INVALID_ARGUMENT = 1
ERR_CORRUPT_ROUTING = 2
ERR_STRATEGY_INAPPLICABLE = 3
ERR_CALIBRATION = 4
ERR_INVALID_GRAPH = 5
ERR_CUDA = 6
ERR_TRANSPORT = 7
ERR_TIMEOUT = 8
ERR_UNSUPPORTED = 9

# moe_level (== moeplan::StrategyLevel)
BASELINE, O1, O2, O3 = 0, 1, 2, 3
LEVEL_NAMES = {BASELINE: "Baseline", O1: "O1", O2: "O2", O3: "O3"}

# moe_dtype
F32, BF16, F16, F64, I64 = 0, 1, 2, 3, 4
# moe_landing
LAND_FINAL, LAND_STAGED = 0, 1
# communication groups (monta.h 1d; conflict.hpp CommGroup)
COMM_TP_SP, COMM_EP, COMM_PP, COMM_CP, COMM_DP = 0, 1, 2, 3, 4
# expert activations (moe_grouped_gemm)
ACT_NONE, ACT_SWIGLU = 0, 1
# dispatch wire formats (moe_ctx_set_wire)
WIRE_BF16, WIRE_FP8 = 0, 1
W13_BLOCK = 128
# moe_stage
STAGES = ["route", "index", "aa", "ag", "d2d", "caa", "unpermute", "total", "experts"]


class MoeError(RuntimeError):
    def __init__(self, status: int, message: str):
        super().__init__(f"[moe status {status}] {message}")
        self.status = status
        self.message = message


class InvalidArgument(MoeError, ValueError):
    """std::invalid_argument in the reference."""


class CorruptRoutingError(MoeError):
    """dataplane::CorruptRoutingError (dataplane.hpp:18-20)."""


class StrategyInapplicableError(InvalidArgument):
    """StrategyInapplicableError : std::invalid_argument (chunkopt.hpp:11-13)."""


class CalibrationError(MoeError):
    """CalibrationError (calibrate.hpp:12-14)."""


class InvalidGraphError(MoeError):
    """pipesim::InvalidGraphError (pipesim.hpp:65-67)."""


_ERRORS = {ERR_INVALID_ARGUMENT: InvalidArgument, ERR_CORRUPT_ROUTING: CorruptRoutingError,
           ERR_STRATEGY_INAPPLICABLE: StrategyInapplicableError, ERR_CALIBRATION: CalibrationError,
           ERR_INVALID_GRAPH: InvalidGraphError}


class LayerDesc(C.Structure):
    _fields_ = [("e", C.c_int32), ("t", C.c_int32), ("num_experts", C.c_int32), ("top_k", C.c_int32),
                ("tokens", C.c_int64), ("hidden", C.c_int64), ("dtype", C.c_int32), ("logit_dtype", C.c_int32),
                ("out_dtype", C.c_int32), ("max_chunks", C.c_int32)]


class CardView(C.Structure):
    _fields_ = [(n, C.c_void_p) for n in (
        "x", "logits", "token_ids", "experts", "probs", "perm_src", "expert_of", "slot_pos", "counts",
        "expert_offsets", "permuted", "recv", "recv_tags", "pre", "pre_tags", "expert_out", "comb", "out")] + [
        ("rows_permuted", C.c_int64), ("recv_cap", C.c_int64), ("recv_expert_offsets", C.c_void_p),
        ("grad_probs", C.c_void_p), ("grad_logits", C.c_void_p)]


class Span(C.Structure):
    _fields_ = [("stage", C.c_int32), ("chunk", C.c_int32), ("start_ms", C.c_float), ("end_ms", C.c_float)]


class ModelSpec(C.Structure):
    _fields_ = [(n, C.c_int64) for n in ("b", "s", "h", "a", "l", "k", "p1", "p2")] + [("bpe", C.c_int32)]


class ParallelSpec(C.Structure):
    _fields_ = [(n, C.c_int32) for n in ("d", "p", "t", "e", "cp")]


class ClusterSpec(C.Structure):
    _fields_ = [("nodes", C.c_int32), ("gpus_per_node", C.c_int32), ("b1", C.c_double), ("b2", C.c_double),
                ("b3", C.c_double), ("peak_flops", C.c_double), ("switch_capacity", C.c_int64)]


class Curve(C.Structure):
    _fields_ = [("volume", C.POINTER(C.c_double)), ("efficiency", C.POINTER(C.c_double)),
                ("n_points", C.c_int32), ("i_minimal", C.c_double)]


class CurveSet(C.Structure):
    _fields_ = [("alltoall", Curve), ("allgather", Curve), ("d2d", Curve)]


class Overhead(C.Structure):
    _fields_ = [("alpha_comm", C.c_double), ("alpha_copy", C.c_double)]


class ChunkTiming(C.Structure):
    _fields_ = [("aa", C.c_double), ("ag", C.c_double), ("d2d", C.c_double), ("n", C.c_int32),
                ("volume", C.c_double)]


class ChunkSearchResult(C.Structure):
    _fields_ = [("n_opt", C.c_int32), ("t_pred", C.c_double), ("per_chunk", ChunkTiming), ("feasible", C.c_int32)]


class StrategyAlt(C.Structure):
    _fields_ = [("level", C.c_int32), ("t_pred", C.c_double), ("n", C.c_int32)]


class StrategyDecision(C.Structure):
    _fields_ = [("level", C.c_int32), ("n", C.c_int32), ("t_pred", C.c_double), ("n_alternatives", C.c_int32),
                ("alternatives", StrategyAlt * 3)]


class PerfReport(C.Structure):
    _fields_ = [("step_latency", C.c_double), ("throughput", C.c_double), ("mfu", C.c_double)]


class BenchSample(C.Structure):
    _fields_ = [("primitive", C.c_int32), ("volume", C.c_double), ("seconds", C.c_double)]


class SimSpan(C.Structure):
    _fields_ = [("kind", C.c_int32), ("chunk", C.c_int32), ("stream", C.c_int32), ("start", C.c_double),
                ("end", C.c_double)]


class Schedule(C.Structure):
    _fields_ = [("level", C.c_int32), ("n_chunks", C.c_int32), ("landing", C.c_int32), ("us", C.c_double)]


class SimTask(C.Structure):
    _fields_ = [("stream", C.c_int32), ("duration", C.c_double), ("dep_begin", C.c_int32), ("dep_end", C.c_int32)]


_P = C.c_void_p
_I32, _I64, _D = C.c_int32, C.c_int64, C.c_double
_PI32 = C.POINTER(C.c_int32)
_PI64 = C.POINTER(C.c_int64)
_PD = C.POINTER(C.c_double)

# name -> (restype, argtypes)
SIGNATURES = {
    "moe_last_error": (C.c_char_p, []),
    "moe_abi_version": (C.c_int, []),
    "moe_dtype_size": (C.c_size_t, [C.c_int]),
    "moe_host_alloc": (C.c_int, [C.c_size_t, C.POINTER(C.c_void_p)]),
    "moe_host_free": (C.c_int, [_P]),
    "moe_route_topk": (C.c_int, [_P, C.c_int, _I64, _I32, _I32, _P, _P, _P]),
    "moe_build_index": (C.c_int, [_P, _I64, _I32, _I32, _I32, _P, _P, _P, _P, _P, _P, _P]),
    "moe_permute_rows": (C.c_int, [_P, _I64, _I64, _I64, _P, _I64, _P, _I64, _P]),
    "moe_unpermute_combine": (C.c_int, [_P, C.c_int, _I64, _I64, _P, _P, C.c_int, _I64, _I32, _P, C.c_int, _I64, _P]),
    "moe_combine_backward": (C.c_int, [_P, C.c_int, _I64, _P, C.c_int, _I64, _I64, _P, _P, C.c_int, _I64, _I32,
                                       _P, _I64, _P, _P]),
    "moe_dispatch_backward": (C.c_int, [_P, C.c_int, _I64, _I64, _P, _I64, _I32, _P, C.c_int, _I64, _P]),
    "moe_route_backward": (C.c_int, [_P, C.c_int, _I64, _I32, _I32, _P, _P, _P, _P]),
    "moe_ctx_bind_experts": (C.c_int, [_P, C.c_int, _P, _P, _I64]),
    "moe_ctx_experts": (C.c_int, [_P, _P]),
    "moe_ctx_set_expert_overlap": (C.c_int, [_P, C.c_int32]),
    "moe_ctx_set_node_dedup": (C.c_int, [_P, C.c_int32]),
    "moe_comm_priority": (C.c_int, [C.c_int]),
    "moe_ctx_enable_checks": (C.c_int, [_P, C.c_int]),
    "moe_ctx_set_wire": (C.c_int, [_P, C.c_int]),
    "moe_ctx_set_link_rate": (C.c_int, [_P, C.c_double]),
    "moe_ctx_backward_combine": (C.c_int, [_P, C.c_int, _I32, _P]),
    "moe_ctx_backward_dispatch": (C.c_int, [_P, C.c_int, _I32, _P]),
    "moe_ctx_backward": (C.c_int, [_P, C.c_int, _I32, _P]),
    "moe_ctx_verify": (C.c_int, [_P, _P]),
    "moe_comm_stream_priority": (C.c_int, [C.c_int, C.c_int, _P]),
    "moe_comm_stream_create": (C.c_int, [C.c_int, _P]),
    "moe_comm_stream_destroy": (C.c_int, [_P]),
    "moe_mc_supported": (C.c_int, [C.c_int, _P]),
    "moe_mc_granularity": (C.c_int, [C.c_int, C.c_size_t, _P]),
    "moe_mc_create": (C.c_int, [C.c_int, C.c_size_t, _P, _P]),
    "moe_mc_import": (C.c_int, [C.c_int, C.c_int, C.c_size_t, _P]),
    "moe_mc_add_device": (C.c_int, [_P, C.c_int]),
    "moe_mc_bind": (C.c_int, [_P, _P, _P]),
    "moe_mc_store": (C.c_int, [_P, _P, C.c_size_t, C.c_int32, _P]),
    "moe_mc_destroy": (C.c_int, [_P]),
    "moe_grouped_gemm": (C.c_int, [_P, _I64, _I64, _P, _P, _I32, _I64, _I64, _P, _I64, C.c_int, _P]),
    "moe_interleave_w13": (C.c_int, [_P, _P, _I32, _I64, _I64, _P, _P]),
    "moe_expert_ffn": (C.c_int, [_P, _I64, _I64, _P, _P, _P, _I32, _I64, _I64, _P, _P, _I64, _P]),
    "moe_ctx_create": (C.c_int,[C.POINTER(LayerDesc), C.c_int, C.c_int, C.c_int, C.POINTER(_P)]),
    "moe_ctx_destroy": (C.c_int, [_P]),
    "moe_ctx_card_view": (C.c_int, [_P, C.c_int, C.POINTER(CardView)]),
    "moe_ctx_num_local_cards": (C.c_int, [_P]),
    "moe_ctx_first_card": (C.c_int, [_P]),
    "moe_ctx_ipc_handle_size": (C.c_size_t, []),
    "moe_ctx_ipc_export": (C.c_int, [_P, _P]),
    "moe_ctx_ipc_connect": (C.c_int, [_P, _P]),
    "moe_ctx_bind_expert_out": (C.c_int, [_P, C.c_int, _P]),
    "moe_ctx_route": (C.c_int, [_P, _P]),
    "moe_ctx_permute": (C.c_int, [_P, _I32, _P]),
    "moe_ctx_dispatch": (C.c_int, [_P, C.c_int, _I32, C.c_int, _P]),
    "moe_ctx_combine": (C.c_int, [_P, C.c_int, _I32, _P]),
    "moe_ctx_forward": (C.c_int, [_P, C.c_int, _I32, C.c_int, _P]),
    "moe_ctx_forward_host": (C.c_int, [_P, C.c_int, _I32, C.c_int, _P, _P, _P, _P]),
    "moe_ctx_recv_rows": (C.c_int, [_P, C.c_int, _PI64]),
    "moe_ctx_sync": (C.c_int, [_P]),
    "moe_ctx_enable_timing": (C.c_int, [_P, C.c_int]),
    "moe_ctx_enable_graphs": (C.c_int, [_P, C.c_int]),
    "moe_ctx_spans": (C.c_int, [_P, C.POINTER(Span), _I32, _PI32]),
    "moe_ctx_set_aa_ctas": (C.c_int, [_P, _I32]),
    "moe_ctx_launch_count": (C.c_int64, [_P]),
    "moe_ctx_xfer": (C.c_int, [_P, _PI64, _I32, _I32, _P]),
    "moe_ctx_set_persistent": (C.c_int, [_P, C.c_int]),
    "moe_ctx_xchg_trace": (C.c_int, [_P, C.c_int, C.POINTER(C.c_uint64), _I32, _PI32]),
    "moe_ctx_debug_front": (C.c_int, [_P, C.c_int, C.c_int, C.POINTER(C.c_uint64)]),
    "moe_lookup_efficiency": (C.c_int, [C.POINTER(Curve), _D, _PD]),
    "moe_traffic_volume": (C.c_double, [C.POINTER(ModelSpec)]),
    "moe_chunk_alltoall_time": (C.c_int, [_D, _I32, _I32, _I32, _D, C.POINTER(Curve), C.POINTER(Overhead), _PD]),
    "moe_chunk_allgather_time": (C.c_int, [_D, _I32, _I32, _D, C.POINTER(Curve), C.POINTER(Overhead), _PD]),
    "moe_chunk_d2d_time": (C.c_int, [_D, _I32, _D, C.POINTER(Curve), C.POINTER(Overhead), _PD]),
    "moe_baseline_time": (C.c_int, [_D, _I32, _D, C.POINTER(Curve), C.POINTER(Overhead), _PD]),
    "moe_o1_time": (C.c_int, [_D, _I32, _I32, _D, _D, C.POINTER(CurveSet), C.POINTER(Overhead), _PD]),
    "moe_o2_score": (C.c_double, [_D, _D, _D, _I32]),
    "moe_o3_score": (C.c_double, [_D, _D, _D, _I32]),
    "moe_o2_search": (C.c_int, [C.POINTER(ModelSpec), C.POINTER(ParallelSpec), C.POINTER(ClusterSpec),
                                C.POINTER(CurveSet), C.POINTER(Overhead), _I32, C.POINTER(ChunkSearchResult)]),
    "moe_o3_search": (C.c_int, [C.POINTER(ModelSpec), C.POINTER(ParallelSpec), C.POINTER(ClusterSpec),
                                C.POINTER(CurveSet), C.POINTER(Overhead), _I32, C.POINTER(ChunkSearchResult)]),
    "moe_asymptotic_speedup": (C.c_int, [_I32, _I32, _D, _D, _D, _D, _PD]),
    "moe_select_strategy": (C.c_int, [C.POINTER(ModelSpec), C.POINTER(ParallelSpec), C.POINTER(ClusterSpec),
                                      C.POINTER(CurveSet), C.POINTER(Overhead), _I32, C.POINTER(StrategyDecision)]),
    "moe_select_strategy_b200": (C.c_int, [C.POINTER(ModelSpec), C.POINTER(ParallelSpec), C.POINTER(ClusterSpec),
                                           C.POINTER(CurveSet), C.POINTER(Overhead), _I32, _I32,
                                           C.POINTER(StrategyDecision)]),
    "moe_ctx_autotune": (C.c_int, [_P, _P, _I32, _I32, _P, _P]),
    "moe_estimate_performance": (C.c_int, [C.POINTER(StrategyDecision), C.POINTER(ModelSpec),
                                           C.POINTER(ParallelSpec), C.POINTER(ClusterSpec), _I32, _D,
                                           C.POINTER(PerfReport)]),
    "moe_calibrate": (C.c_int, [C.POINTER(BenchSample), _I32, C.POINTER(ClusterSpec), _PD, _PD, _PI32,
                                C.POINTER(Overhead)]),
    "moe_simulate_pipeline": (C.c_int, [C.c_int, _I32, C.POINTER(ChunkTiming), _D, _I32, C.POINTER(SimSpan), _I32,
                                        _PI32, _PD]),
    "moe_simulate_graph": (C.c_int, [C.POINTER(SimTask), _I32, _PI32, _PD, _PD, _PD]),
    "moe_build_pipeline": (C.c_int, [C.c_int, _I32, _P, C.c_double, _I32, _P, _P, _P, _I32, _P, _I32, _P]),
    "moe_check_specs": (C.c_int, [C.c_int, _P, _P, _P, _P, _I64, _P, _P]),
}

_lib = None


def load(path: str | os.PathLike | None = None):
    """Load libmonta.so (building it first if this checkout has nvcc and no build)."""
    global _lib
    if _lib is not None:
        return _lib
    p = pathlib.Path(path or os.environ.get("MONTA_LIB") or LIB_PATH)  # MONTA_LIB: A/B a second build
    if not p.exists():
        try:
            from . import build as _build
            _build.build()
        except Exception as exc:  # pragma: no cover - depends on toolchain
            raise ImportError(f"libmonta.so missing at {p} and could not be built: {exc}") from exc
    lib = C.CDLL(str(p), mode=C.RTLD_GLOBAL)
    if not os.environ.get("MONTA_LIB") and lib.moe_abi_version() != ABI_VERSION:
        raise ImportError(f"{p}: ABI version {lib.moe_abi_version()}, this binding needs {ABI_VERSION} (rebuild)")
    for name, (res, args) in SIGNATURES.items():
        if os.environ.get("MONTA_LIB") and not hasattr(lib, name):
            continue  # A/B against an older build: symbols it predates stay unbound
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def check(status: int) -> None:
    if status != OK:
        raise _ERRORS.get(status, MoeError)(status, load().moe_last_error().decode(errors="replace"))


def dtype_code(torch_dtype) -> int:
    import torch
    table = {torch.float32: F32, torch.bfloat16: BF16, torch.float16: F16, torch.float64: F64, torch.int64: I64}
    if torch_dtype not in table:
        raise ValueError(f"unsupported dtype {torch_dtype}")
    return table[torch_dtype]


def torch_dtype(code: int):
    import torch
    return {F32: torch.float32, BF16: torch.bfloat16, F16: torch.float16, F64: torch.float64, I64: torch.int64}[code]

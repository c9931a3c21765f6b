"""MoNTA planner — the reference operator API over the C ABI (libmonta.so).

Names, argument meaning and error behaviour mirror the reference headers:
    config.hpp      ModelSpec, ParallelSpec, ClusterSpec, CurvePoint,
                    EfficiencyCurve, CurveSet, lookup_efficiency     (:14-87)
    commcost.hpp    StrategyLevel, OverheadModel, ChunkTiming, traffic_volume,
                    chunk_alltoall_time, chunk_allgather_time, chunk_d2d_time,
                    baseline_time, o1_time                            (:11-109)
    chunkopt.hpp    o2_score, o3_score, o2_search, o3_search,
                    asymptotic_speedup, StrategyInapplicableError     (:11-104)
    strategy.hpp    select_strategy, estimate_performance             (:24-80)
    calibrate.hpp   BenchSample, calibrate, CalibrationError          (:12-118)
    pipesim.hpp     Stream, build_pipeline, simulate                  (:91-173)
    io.hpp          curve CSV / bench CSV / key=value cluster config  (:78-301)
Exceptions: ValueError (std::invalid_argument), StrategyInapplicableError,
CalibrationError, InvalidGraphError.  All arithmetic runs in the C++ planner.
"""
from __future__ import annotations

import ctypes as C
import enum
import math
import pathlib
from dataclasses import dataclass, field

from . import _lib
from ._lib import (CalibrationError, InvalidGraphError, StrategyInapplicableError,  # noqa: F401
                   check)


class StrategyLevel(enum.IntEnum):
    Baseline = _lib.BASELINE
    O1 = _lib.O1
    O2 = _lib.O2
    O3 = _lib.O3


def to_string(level) -> str:
    return StrategyLevel(level).name


@dataclass
class ModelSpec:
    b: int = 1
    s: int = 1
    h: int = 1
    a: int = 1
    l: int = 1  # noqa: E741
    k: int = 1
    p1: int = 0
    p2: int = 0
    bpe: int = 2

    def _c(self):
        return _lib.ModelSpec(self.b, self.s, self.h, self.a, self.l, self.k, self.p1, self.p2, self.bpe)


@dataclass
class ParallelSpec:
    d: int = 1
    p: int = 1
    t: int = 1
    e: int = 1
    cp: int = 1

    def _c(self):
        return _lib.ParallelSpec(self.d, self.p, self.t, self.e, self.cp)


@dataclass
class ClusterSpec:
    nodes: int = 1
    gpus_per_node: int = 1
    b1: float = 1.0
    b2: float = 1.0
    b3: float = 1.0
    peak_flops: float = 1.0
    switch_capacity: int = 1

    def _c(self):
        return _lib.ClusterSpec(self.nodes, self.gpus_per_node, self.b1, self.b2, self.b3, self.peak_flops,
                                self.switch_capacity)


@dataclass
class CurvePoint:
    volume: float = 0.0
    efficiency: float = 1.0


@dataclass
class EfficiencyCurve:
    points: list = field(default_factory=list)
    i_minimal: float = 0.0

    @staticmethod
    def constant(efficiency: float, i_minimal: float = 0.0) -> "EfficiencyCurve":
        return EfficiencyCurve([CurvePoint(1.0, efficiency)], i_minimal)

    def _c(self):
        n = len(self.points)
        v = (C.c_double * max(n, 1))(*[float(p.volume) for p in self.points])
        e = (C.c_double * max(n, 1))(*[float(p.efficiency) for p in self.points])
        c = _lib.Curve(C.cast(v, C.POINTER(C.c_double)), C.cast(e, C.POINTER(C.c_double)), n, self.i_minimal)
        c._keep = (v, e)
        return c


@dataclass
class CurveSet:
    alltoall: EfficiencyCurve = field(default_factory=EfficiencyCurve)
    allgather: EfficiencyCurve = field(default_factory=EfficiencyCurve)
    d2d: EfficiencyCurve = field(default_factory=EfficiencyCurve)

    def _c(self):
        a, g, d = self.alltoall._c(), self.allgather._c(), self.d2d._c()
        cs = _lib.CurveSet(a, g, d)
        cs._keep = (a, g, d)
        return cs


@dataclass
class OverheadModel:
    alpha_comm: float = 0.0
    alpha_copy: float = 0.0

    def _c(self):
        return _lib.Overhead(self.alpha_comm, self.alpha_copy)


@dataclass
class ChunkTiming:
    aa: float = 0.0
    ag: float = 0.0
    d2d: float = 0.0
    n: int = 1
    volume: float = 0.0


@dataclass
class ChunkSearchResult:
    n_opt: int = 1
    t_pred: float = 0.0
    per_chunk: ChunkTiming = field(default_factory=ChunkTiming)
    feasible: bool = True


@dataclass
class StrategyAlternative:
    level: StrategyLevel = StrategyLevel.Baseline
    t_pred: float = 0.0
    n: int = 1


@dataclass
class StrategyDecision:
    level: StrategyLevel = StrategyLevel.Baseline
    n: int = 1
    t_pred: float = 0.0
    alternatives: list = field(default_factory=list)


@dataclass
class PerfReport:
    step_latency: float = 0.0
    throughput: float = 0.0
    mfu: float = 0.0


@dataclass
class BenchSample:
    primitive: str = ""
    volume: float = 0.0
    seconds: float = 0.0


@dataclass
class CalibrationSet:
    curves: CurveSet = field(default_factory=CurveSet)
    overhead: OverheadModel = field(default_factory=OverheadModel)


def _L():
    return _lib.load()


def _out_double(fn, *args) -> float:
    out = C.c_double()
    check(fn(*args, C.byref(out)))
    return out.value


def lookup_efficiency(curve: EfficiencyCurve, volume: float) -> float:
    return _out_double(_L().moe_lookup_efficiency, C.byref(curve._c()), float(volume))


def traffic_volume(m: ModelSpec) -> float:
    return float(_L().moe_traffic_volume(C.byref(m._c())))


def chunk_alltoall_time(volume, n_chunks, t, e, b1, curve: EfficiencyCurve, ov: OverheadModel = OverheadModel()):
    return _out_double(_L().moe_chunk_alltoall_time, float(volume), n_chunks, t, e, float(b1), C.byref(curve._c()),
                       C.byref(ov._c()))


def chunk_allgather_time(volume, n_chunks, t, b2, curve: EfficiencyCurve, ov: OverheadModel = OverheadModel()):
    return _out_double(_L().moe_chunk_allgather_time, float(volume), n_chunks, t, float(b2), C.byref(curve._c()),
                       C.byref(ov._c()))


def chunk_d2d_time(volume, n_chunks, b3, curve: EfficiencyCurve, ov: OverheadModel = OverheadModel()):
    return _out_double(_L().moe_chunk_d2d_time, float(volume), n_chunks, float(b3), C.byref(curve._c()),
                       C.byref(ov._c()))


def baseline_time(volume, e, b1, curve: EfficiencyCurve, ov: OverheadModel = OverheadModel()):
    return _out_double(_L().moe_baseline_time, float(volume), e, float(b1), C.byref(curve._c()), C.byref(ov._c()))


def o1_time(volume, t, e, b1, b2, curves: CurveSet, ov: OverheadModel = OverheadModel()):
    return _out_double(_L().moe_o1_time, float(volume), t, e, float(b1), float(b2), C.byref(curves._c()),
                       C.byref(ov._c()))


def o2_score(aa, ag, d2d, n) -> float:
    return float(_L().moe_o2_score(aa, ag, d2d, n))


def o3_score(aa, ag, d2d, n) -> float:
    return float(_L().moe_o3_score(aa, ag, d2d, n))


def _search(fn, model, par, cluster, curves, ov, n_cap):
    r = _lib.ChunkSearchResult()
    check(fn(C.byref(model._c()), C.byref(par._c()), C.byref(cluster._c()), C.byref(curves._c()),
             C.byref(ov._c()), n_cap, C.byref(r)))
    pc = r.per_chunk
    return ChunkSearchResult(r.n_opt, r.t_pred, ChunkTiming(pc.aa, pc.ag, pc.d2d, pc.n, pc.volume), bool(r.feasible))


def o2_search(model: ModelSpec, par: ParallelSpec, cluster: ClusterSpec, curves: CurveSet,
              ov: OverheadModel = OverheadModel(), n_cap: int = 64) -> ChunkSearchResult:
    return _search(_L().moe_o2_search, model, par, cluster, curves, ov, n_cap)


def o3_search(model: ModelSpec, par: ParallelSpec, cluster: ClusterSpec, curves: CurveSet,
              ov: OverheadModel = OverheadModel(), n_cap: int = 64) -> ChunkSearchResult:
    return _search(_L().moe_o3_search, model, par, cluster, curves, ov, n_cap)


def asymptotic_speedup(t, e, b1, b2, r1, r2) -> float:
    return _out_double(_L().moe_asymptotic_speedup, t, e, float(b1), float(b2), float(r1), float(r2))


def select_strategy(model: ModelSpec, par: ParallelSpec, cluster: ClusterSpec, curves: CurveSet,
                    ov: OverheadModel = OverheadModel(), n_cap: int = 64) -> StrategyDecision:
    d = _lib.StrategyDecision()
    check(_L().moe_select_strategy(C.byref(model._c()), C.byref(par._c()), C.byref(cluster._c()),
                                   C.byref(curves._c()), C.byref(ov._c()), n_cap, C.byref(d)))
    alts = [StrategyAlternative(StrategyLevel(d.alternatives[i].level), d.alternatives[i].t_pred,
                                d.alternatives[i].n) for i in range(d.n_alternatives)]
    return StrategyDecision(StrategyLevel(d.level), d.n, d.t_pred, alts)


def select_strategy_b200(model: ModelSpec, par: ParallelSpec, cluster: ClusterSpec, curves: CurveSet,
                         ov: OverheadModel = OverheadModel(), n_cap: int = 64,
                         shared_egress: bool = True) -> StrategyDecision:
    """B200 variant (monta.h): AllToAll and AllGather serialise on one NVSwitch
    box's shared NVLink egress; shared_egress=False is select_strategy."""
    d = _lib.StrategyDecision()
    check(_L().moe_select_strategy_b200(C.byref(model._c()), C.byref(par._c()), C.byref(cluster._c()),
                                        C.byref(curves._c()), C.byref(ov._c()), n_cap, int(shared_egress),
                                        C.byref(d)))
    alts = [StrategyAlternative(StrategyLevel(d.alternatives[i].level), d.alternatives[i].t_pred,
                                d.alternatives[i].n) for i in range(d.n_alternatives)]
    return StrategyDecision(StrategyLevel(d.level), d.n, d.t_pred, alts)


def estimate_performance(decision: StrategyDecision, model: ModelSpec, par: ParallelSpec, cluster: ClusterSpec,
                         moe_layer_count: int, non_comm_time: float) -> PerfReport:
    d = _lib.StrategyDecision()
    d.level, d.n, d.t_pred = int(decision.level), decision.n, decision.t_pred
    r = _lib.PerfReport()
    check(_L().moe_estimate_performance(C.byref(d), C.byref(model._c()), C.byref(par._c()), C.byref(cluster._c()),
                                        moe_layer_count, float(non_comm_time), C.byref(r)))
    return PerfReport(r.step_latency, r.throughput, r.mfu)


_PRIM = {"alltoall": 0, "allgather": 1, "d2d": 2}


def calibrate(samples: list, cluster: ClusterSpec) -> CalibrationSet:
    for s in samples:
        if s.primitive not in _PRIM:
            raise CalibrationError(_lib.ERR_CALIBRATION, f"calibrate: unknown primitive '{s.primitive}'")
    n = len(samples)
    arr = (_lib.BenchSample * max(n, 1))(*[_lib.BenchSample(_PRIM[s.primitive], s.volume, s.seconds)
                                           for s in samples])
    vols = (C.c_double * (3 * max(n, 1)))()
    effs = (C.c_double * (3 * max(n, 1)))()
    npts = (C.c_int32 * 3)()
    ov = _lib.Overhead()
    check(_L().moe_calibrate(arr, n, C.byref(cluster._c()), vols, effs, npts, C.byref(ov)))
    curves = [EfficiencyCurve([CurvePoint(vols[p * n + i], effs[p * n + i]) for i in range(npts[p])])
              for p in range(3)]
    return CalibrationSet(CurveSet(*curves), OverheadModel(ov.alpha_comm, ov.alpha_copy))


# ---------------------------------------------------------------------------
# pipesim
class Stream(enum.IntEnum):
    AllToAll = 0
    AllGather = 1
    D2D = 2
    Compute = 3


_STREAM_NAMES = {Stream.AllToAll: "alltoall", Stream.AllGather: "allgather", Stream.D2D: "d2d",
                 Stream.Compute: "compute"}


@dataclass
class SimTask:
    id: str
    stream: Stream = Stream.Compute
    duration: float = 0.0
    deps: list = field(default_factory=list)


@dataclass
class TaskSpan:
    id: str
    stream: Stream
    start: float
    end: float


@dataclass
class StreamTrace:
    spans: list
    makespan: float


def build_pipeline(level, n: int, timing: ChunkTiming, expert_time: float, phases: int = 2) -> list:
    """Task graph of one MoE transfer (pipesim.hpp:91-105): ids as the reference's."""
    if n < 1:
        raise _lib.InvalidArgument(_lib.ERR_INVALID_ARGUMENT, "build_pipeline: n must be >= 1")
    if phases not in (1, 2):
        raise _lib.InvalidArgument(_lib.ERR_INVALID_ARGUMENT, "build_pipeline: phases must be 1 or 2")
    level = StrategyLevel(level)
    if level in (StrategyLevel.Baseline, StrategyLevel.O1):
        n = 1
    g: list = []

    def phase(prefix, deps):
        terms = []
        for j in range(1, n + 1):
            aa = f"{prefix}_aa_{j}"
            g.append(SimTask(aa, Stream.AllToAll, timing.aa, list(deps)))
            if level == StrategyLevel.Baseline:
                terms.append(aa)
                continue
            ag = f"{prefix}_ag_{j}"
            g.append(SimTask(ag, Stream.AllGather, timing.ag, [aa]))
            if level == StrategyLevel.O1:
                terms.append(ag)
                continue
            dd = f"{prefix}_d2d_{j}"
            g.append(SimTask(dd, Stream.AllGather if level == StrategyLevel.O2 else Stream.D2D, timing.d2d, [ag]))
            terms.append(dd)
        return terms

    terms = phase("dispatch", [])
    if phases == 2:
        g.append(SimTask("expert", Stream.Compute, expert_time, terms))
        phase("combine", ["expert"])
    return g


def simulate(tasks: list) -> StreamTrace:
    """List scheduling in the C++ planner (pipesim.hpp:110-173)."""
    index = {}
    for i, t in enumerate(tasks):
        if t.duration < 0:
            raise _lib.InvalidArgument(_lib.ERR_INVALID_ARGUMENT, f"simulate: negative duration for task {t.id}")
        if t.id in index:
            raise _lib.InvalidArgument(_lib.ERR_INVALID_ARGUMENT, f"simulate: duplicate task id {t.id}")
        index[t.id] = i
    deps: list = []
    arr = (_lib.SimTask * max(len(tasks), 1))()
    for i, t in enumerate(tasks):
        begin = len(deps)
        for d in t.deps:
            if d not in index:
                raise _lib.InvalidArgument(_lib.ERR_INVALID_ARGUMENT, f"simulate: unknown dependency {d}")
            deps.append(index[d])
        arr[i] = _lib.SimTask(int(t.stream), float(t.duration), begin, len(deps))
    dep_arr = (C.c_int32 * max(len(deps), 1))(*deps)
    n = len(tasks)
    st = (C.c_double * max(n, 1))()
    en = (C.c_double * max(n, 1))()
    mk = C.c_double()
    check(_L().moe_simulate_graph(arr, n, dep_arr, st, en, C.byref(mk)))
    return StreamTrace([TaskSpan(t.id, t.stream, st[i], en[i]) for i, t in enumerate(tasks)], mk.value)


# ---------------------------------------------------------------------------
# file formats (io.hpp): curve CSV, bench CSV, key = value configs
def read_curve_csv(path, i_minimal: float = 0.0) -> EfficiencyCurve:
    lines = [ln.strip() for ln in pathlib.Path(path).read_text().splitlines()]
    lines = [ln for ln in lines if ln and not ln.startswith("#")]
    if not lines or lines[0].replace(" ", "") != "volume_bytes,efficiency":
        raise ValueError(f"{path}: expected header 'volume_bytes,efficiency'")
    pts = []
    for ln in lines[1:]:
        v, e = (float(x) for x in ln.split(","))
        if not (0.0 < e <= 1.0):
            raise ValueError(f"{path}: efficiency must be in (0, 1]")
        if pts and v <= pts[-1].volume:
            raise ValueError(f"{path}: volumes must be strictly increasing")
        pts.append(CurvePoint(v, e))
    if not pts:
        raise ValueError(f"{path}: no curve points")
    return EfficiencyCurve(pts, i_minimal)


def write_curve_csv(path, curve: EfficiencyCurve) -> None:
    rows = ["volume_bytes,efficiency"] + [f"{p.volume:.17g},{p.efficiency:.17g}" for p in curve.points]
    pathlib.Path(path).write_text("\n".join(rows) + "\n")


def load_curve_set(directory, i_minimal: float = 0.0) -> CurveSet:
    d = pathlib.Path(directory)
    return CurveSet(read_curve_csv(d / "alltoall.csv", i_minimal), read_curve_csv(d / "allgather.csv", i_minimal),
                    read_curve_csv(d / "d2d.csv", 0.0))


def read_bench_csv(path) -> list:
    lines = [ln.strip() for ln in pathlib.Path(path).read_text().splitlines()]
    lines = [ln for ln in lines if ln and not ln.startswith("#")]
    if not lines or lines[0].replace(" ", "") != "primitive,volume_bytes,measured_seconds":
        raise ValueError(f"{path}: expected header 'primitive,volume_bytes,measured_seconds'")
    out = []
    for ln in lines[1:]:
        p, v, s = ln.split(",")
        out.append(BenchSample(p.strip(), float(v), float(s)))
    return out


def write_bench_csv(path, samples: list) -> None:
    rows = ["primitive,volume_bytes,measured_seconds"] + [f"{s.primitive},{s.volume:.17g},{s.seconds:.17g}"
                                                          for s in samples]
    pathlib.Path(path).write_text("\n".join(rows) + "\n")


def read_kv(path) -> dict:
    out = {}
    for ln in pathlib.Path(path).read_text().splitlines():
        ln = ln.split("#", 1)[0].strip()
        if not ln:
            continue
        if "=" not in ln:
            raise ValueError(f"{path}: expected 'key = value', got {ln!r}")
        k, v = ln.split("=", 1)
        out[k.strip()] = v.strip()
    return out


def load_cluster_spec(path) -> ClusterSpec:
    kv = read_kv(path)
    c = ClusterSpec()
    for k, v in kv.items():
        if k in ("nodes", "gpus_per_node", "switch_capacity"):
            setattr(c, k, int(float(v)))
        elif k in ("b1", "b2", "b3", "peak_flops"):
            setattr(c, k, float(v))
    return c


def b200_cluster(nodes: int, gpus_per_node: int, b1: float = 900e9, b2: float = 900e9, b3: float = 6.5e12,
                 peak_flops: float = 2.25e15) -> ClusterSpec:
    """One NVSwitch box emulated as `nodes` groups of `gpus_per_node` GPUs."""
    return ClusterSpec(nodes, gpus_per_node, b1, b2, b3, peak_flops, nodes * gpus_per_node)


__all__ = [n for n in dir() if not n.startswith("_") and n not in ("annotations", "C", "enum", "math", "pathlib")]

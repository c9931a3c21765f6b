// monta_planner.hpp — the reference's planner operator API (moeplan::
// config / commcost / chunkopt / strategy / calibrate / pipesim,
// /root/reference/proj/include/moeplan/{config,commcost,chunkopt,strategy,
// calibrate,pipesim}.hpp) implemented over the C ABI (monta.h section 3,
// libmonta.so's csrc/planner.cpp).
//
// Same namespaces, type names, field order and defaults (designated
// initialisers in caller code depend on them), function signatures, default
// arguments and exception types as the reference, so its callers and its own
// unit tests compile unchanged: put include/dropin on the include path ahead
// of the reference headers and link libmonta.so.  The host side here only
// converts between the reference's value types (vectors, strings, enums) and
// the C ABI's plain structs and arrays; every number comes from the library.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <map>
#include <stdexcept>
#include <string>
#include <unordered_map>
#include <vector>

#include "monta.h"

#ifndef MONTA_HAVE_STRATEGY_LEVEL
#define MONTA_HAVE_STRATEGY_LEVEL
namespace moeplan {
enum class StrategyLevel { Baseline, O1, O2, O3 };  // == moe_level
inline const char* to_string(StrategyLevel level) {
  switch (level) {
    case StrategyLevel::Baseline: return "Baseline";
    case StrategyLevel::O1: return "O1";
    case StrategyLevel::O2: return "O2";
    case StrategyLevel::O3: return "O3";
  }
  return "?";
}
}  // namespace moeplan
#endif

namespace moeplan {

// ---------------------------------------------------------------- config.hpp
struct ModelSpec {
  std::int64_t b = 1;
  std::int64_t s = 1;
  std::int64_t h = 1;
  std::int64_t a = 1;
  std::int64_t l = 1;
  std::int64_t k = 1;
  std::int64_t p1 = 0;
  std::int64_t p2 = 0;
  int bpe = 2;
};

struct ParallelSpec {
  int d = 1;
  int p = 1;
  int t = 1;
  int e = 1;
  int cp = 1;
};

struct ClusterSpec {
  int nodes = 1;
  int gpus_per_node = 1;
  double b1 = 1.0;
  double b2 = 1.0;
  double b3 = 1.0;
  double peak_flops = 1.0;
  std::int64_t switch_capacity = 1;
};

struct CurvePoint {
  double volume = 0.0;
  double efficiency = 1.0;
};

struct EfficiencyCurve {
  std::vector<CurvePoint> points;
  double i_minimal = 0.0;

  static EfficiencyCurve constant(double efficiency, double i_minimal = 0.0) {
    return EfficiencyCurve{{{1.0, efficiency}}, i_minimal};
  }
};

struct CurveSet {
  EfficiencyCurve alltoall;
  EfficiencyCurve allgather;
  EfficiencyCurve d2d;
};

// ---------------------------------------------------------------- commcost.hpp
struct OverheadModel {
  double alpha_comm = 0.0;
  double alpha_copy = 0.0;
};

struct ChunkTiming {
  double aa = 0.0;
  double ag = 0.0;
  double d2d = 0.0;
  int n = 1;
  double volume = 0.0;
};

// ---------------------------------------------------------------- chunkopt.hpp
struct StrategyInapplicableError : std::invalid_argument {
  using std::invalid_argument::invalid_argument;
};

struct ChunkSearchResult {
  int n_opt = 1;
  double t_pred = 0.0;
  ChunkTiming per_chunk;
  bool feasible = true;
};

// ---------------------------------------------------------------- strategy.hpp
struct StrategyAlternative {
  StrategyLevel level = StrategyLevel::Baseline;
  double t_pred = 0.0;
  int n = 1;
};

struct StrategyDecision {
  StrategyLevel level = StrategyLevel::Baseline;
  int n = 1;
  double t_pred = 0.0;
  std::vector<StrategyAlternative> alternatives;
};

struct PerfReport {
  double step_latency = 0.0;
  double throughput = 0.0;
  double mfu = 0.0;
};

// ---------------------------------------------------------------- calibrate.hpp
struct CalibrationError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

struct BenchSample {
  std::string primitive;
  double volume = 0.0;
  double seconds = 0.0;
};

struct CalibrationSet {
  CurveSet curves;
  OverheadModel overhead;
};

namespace pipesim {
// ---------------------------------------------------------------- pipesim.hpp
enum class Stream { AllToAll, AllGather, D2D, Compute };  // == the C ABI's stream ids 0..3

inline const char* to_string(Stream s) {
  switch (s) {
    case Stream::AllToAll: return "alltoall";
    case Stream::AllGather: return "allgather";
    case Stream::D2D: return "d2d";
    case Stream::Compute: return "compute";
  }
  return "?";
}

struct SimTask {
  std::string id;
  Stream stream = Stream::Compute;
  double duration = 0.0;
  std::vector<std::string> deps;
};

using TaskGraph = std::vector<SimTask>;

struct InvalidGraphError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

struct TaskSpan {
  std::string id;
  Stream stream = Stream::Compute;
  double start = 0.0;
  double end = 0.0;
};

struct StreamTrace {
  std::vector<TaskSpan> spans;
  double makespan = 0.0;
};
}  // namespace pipesim

// ============================================================================
// C ABI marshalling
namespace planner_detail {

[[noreturn]] inline void raise(moe_status st) {
  const std::string msg = moe_last_error();
  switch (st) {
    case MOE_ERR_STRATEGY_INAPPLICABLE: throw StrategyInapplicableError(msg);
    case MOE_ERR_CALIBRATION: throw CalibrationError(msg);
    case MOE_ERR_INVALID_GRAPH: throw pipesim::InvalidGraphError(msg);
    case MOE_ERR_INVALID_ARGUMENT: throw std::invalid_argument(msg);
    default: throw std::runtime_error("monta: " + msg);
  }
}
inline void check(moe_status st) {
  if (st != MOE_OK) raise(st);
}

// An EfficiencyCurve as a moe_curve view (owns the split arrays).
struct CurveView {
  std::vector<double> v, e;
  moe_curve c{};
  explicit CurveView(const EfficiencyCurve& curve) {
    v.reserve(curve.points.size());
    e.reserve(curve.points.size());
    for (const auto& p : curve.points) {
      v.push_back(p.volume);
      e.push_back(p.efficiency);
    }
    c.volume = v.data();
    c.efficiency = e.data();
    c.n_points = int32_t(curve.points.size());
    c.i_minimal = curve.i_minimal;
  }
  CurveView(const CurveView&) = delete;
  CurveView& operator=(const CurveView&) = delete;
};

struct CurveSetView {
  CurveView aa, ag, d2d;
  moe_curve_set s{};
  explicit CurveSetView(const CurveSet& cs) : aa(cs.alltoall), ag(cs.allgather), d2d(cs.d2d) {
    s.alltoall = aa.c;
    s.allgather = ag.c;
    s.d2d = d2d.c;
  }
};

inline moe_model_spec to_c(const ModelSpec& m) {
  moe_model_spec o{};
  o.b = m.b;
  o.s = m.s;
  o.h = m.h;
  o.a = m.a;
  o.l = m.l;
  o.k = m.k;
  o.p1 = m.p1;
  o.p2 = m.p2;
  o.bpe = m.bpe;
  return o;
}
inline moe_parallel_spec to_c(const ParallelSpec& p) { return moe_parallel_spec{p.d, p.p, p.t, p.e, p.cp}; }
inline moe_cluster_spec to_c(const ClusterSpec& c) {
  moe_cluster_spec o{};
  o.nodes = c.nodes;
  o.gpus_per_node = c.gpus_per_node;
  o.b1 = c.b1;
  o.b2 = c.b2;
  o.b3 = c.b3;
  o.peak_flops = c.peak_flops;
  o.switch_capacity = c.switch_capacity;
  return o;
}
inline moe_overhead to_c(const OverheadModel& ov) { return moe_overhead{ov.alpha_comm, ov.alpha_copy}; }
inline moe_chunk_timing to_c(const ChunkTiming& t) { return moe_chunk_timing{t.aa, t.ag, t.d2d, t.n, t.volume}; }
inline ChunkTiming from_c(const moe_chunk_timing& t) { return ChunkTiming{t.aa, t.ag, t.d2d, t.n, t.volume}; }

inline std::vector<std::string> report(int which, const moe_model_spec* m, const moe_parallel_spec* p,
                                       const moe_cluster_spec* c) {
  int32_t n = 0;
  int64_t need = 0;
  check(moe_check_specs(which, m, p, c, nullptr, 0, &n, &need));
  std::string buf(size_t(need), '\0');
  check(moe_check_specs(which, m, p, c, buf.data(), need, &n, &need));
  std::vector<std::string> out;
  size_t at = 0;
  for (int32_t i = 0; i < n; ++i) {
    const size_t nl = buf.find('\n', at);
    out.push_back(buf.substr(at, nl - at));
    at = nl + 1;
  }
  return out;
}

inline ChunkSearchResult from_c(const moe_chunk_search_result& r) {
  return ChunkSearchResult{r.n_opt, r.t_pred, from_c(r.per_chunk), r.feasible != 0};
}

}  // namespace planner_detail

// ---------------------------------------------------------------- config.hpp
inline double lookup_efficiency(const EfficiencyCurve& curve, double volume) {
  planner_detail::CurveView c(curve);
  double out = 0.0;
  planner_detail::check(moe_lookup_efficiency(&c.c, volume, &out));
  return out;
}

inline std::vector<std::string> check(const ModelSpec& m) {
  const moe_model_spec cm = planner_detail::to_c(m);
  return planner_detail::report(MOE_CHECK_MODEL, &cm, nullptr, nullptr);
}
inline std::vector<std::string> check(const ParallelSpec& p) {
  const moe_parallel_spec cp = planner_detail::to_c(p);
  return planner_detail::report(MOE_CHECK_PARALLEL, nullptr, &cp, nullptr);
}
inline std::vector<std::string> check(const ClusterSpec& c) {
  const moe_cluster_spec cc = planner_detail::to_c(c);
  return planner_detail::report(MOE_CHECK_CLUSTER, nullptr, nullptr, &cc);
}
inline std::vector<std::string> validate(const ModelSpec&, const ParallelSpec& par, const ClusterSpec& cluster) {
  const moe_parallel_spec cp = planner_detail::to_c(par);
  const moe_cluster_spec cc = planner_detail::to_c(cluster);
  return planner_detail::report(MOE_CHECK_PLACEMENT, nullptr, &cp, &cc);
}

// ---------------------------------------------------------------- commcost.hpp
inline double traffic_volume(const ModelSpec& m) {
  const moe_model_spec cm = planner_detail::to_c(m);
  return moe_traffic_volume(&cm);
}

inline double chunk_alltoall_time(double volume, int n_chunks, int t, int e, double b1, const EfficiencyCurve& curve,
                                  const OverheadModel& ov = {}) {
  planner_detail::CurveView c(curve);
  const moe_overhead o = planner_detail::to_c(ov);
  double out = 0.0;
  planner_detail::check(moe_chunk_alltoall_time(volume, n_chunks, t, e, b1, &c.c, &o, &out));
  return out;
}

inline double chunk_allgather_time(double volume, int n_chunks, int t, double b2, const EfficiencyCurve& curve,
                                   const OverheadModel& ov = {}) {
  planner_detail::CurveView c(curve);
  const moe_overhead o = planner_detail::to_c(ov);
  double out = 0.0;
  planner_detail::check(moe_chunk_allgather_time(volume, n_chunks, t, b2, &c.c, &o, &out));
  return out;
}

inline double chunk_d2d_time(double volume, int n_chunks, double b3, const EfficiencyCurve& curve,
                             const OverheadModel& ov = {}) {
  planner_detail::CurveView c(curve);
  const moe_overhead o = planner_detail::to_c(ov);
  double out = 0.0;
  planner_detail::check(moe_chunk_d2d_time(volume, n_chunks, b3, &c.c, &o, &out));
  return out;
}

inline double baseline_time(double volume, int e, double b1, const EfficiencyCurve& curve,
                            const OverheadModel& ov = {}) {
  planner_detail::CurveView c(curve);
  const moe_overhead o = planner_detail::to_c(ov);
  double out = 0.0;
  planner_detail::check(moe_baseline_time(volume, e, b1, &c.c, &o, &out));
  return out;
}

inline double o1_time(double volume, int t, int e, double b1, double b2, const CurveSet& curves,
                      const OverheadModel& ov = {}) {
  planner_detail::CurveSetView cs(curves);
  const moe_overhead o = planner_detail::to_c(ov);
  double out = 0.0;
  planner_detail::check(moe_o1_time(volume, t, e, b1, b2, &cs.s, &o, &out));
  return out;
}

// ---------------------------------------------------------------- chunkopt.hpp
inline double o2_score(double aa, double ag, double d2d, int n) { return moe_o2_score(aa, ag, d2d, n); }
inline double o3_score(double aa, double ag, double d2d, int n) { return moe_o3_score(aa, ag, d2d, n); }

inline ChunkSearchResult o2_search(const ModelSpec& model, const ParallelSpec& par, const ClusterSpec& cluster,
                                   const CurveSet& curves, const OverheadModel& ov = {}, int n_cap = 64) {
  const moe_model_spec m = planner_detail::to_c(model);
  const moe_parallel_spec p = planner_detail::to_c(par);
  const moe_cluster_spec c = planner_detail::to_c(cluster);
  planner_detail::CurveSetView cs(curves);
  const moe_overhead o = planner_detail::to_c(ov);
  moe_chunk_search_result r{};
  planner_detail::check(moe_o2_search(&m, &p, &c, &cs.s, &o, n_cap, &r));
  return planner_detail::from_c(r);
}

inline ChunkSearchResult o3_search(const ModelSpec& model, const ParallelSpec& par, const ClusterSpec& cluster,
                                   const CurveSet& curves, const OverheadModel& ov = {}, int n_cap = 64) {
  const moe_model_spec m = planner_detail::to_c(model);
  const moe_parallel_spec p = planner_detail::to_c(par);
  const moe_cluster_spec c = planner_detail::to_c(cluster);
  planner_detail::CurveSetView cs(curves);
  const moe_overhead o = planner_detail::to_c(ov);
  moe_chunk_search_result r{};
  planner_detail::check(moe_o3_search(&m, &p, &c, &cs.s, &o, n_cap, &r));
  return planner_detail::from_c(r);
}

inline double asymptotic_speedup(int t, int e, double b1, double b2, double r1, double r2) {
  double out = 0.0;
  planner_detail::check(moe_asymptotic_speedup(t, e, b1, b2, r1, r2, &out));
  return out;
}

// ---------------------------------------------------------------- strategy.hpp
inline StrategyDecision select_strategy(const ModelSpec& model, const ParallelSpec& par, const ClusterSpec& cluster,
                                        const CurveSet& curves, const OverheadModel& ov = {}, int n_cap = 64) {
  const moe_model_spec m = planner_detail::to_c(model);
  const moe_parallel_spec p = planner_detail::to_c(par);
  const moe_cluster_spec c = planner_detail::to_c(cluster);
  planner_detail::CurveSetView cs(curves);
  const moe_overhead o = planner_detail::to_c(ov);
  moe_strategy_decision d{};
  planner_detail::check(moe_select_strategy(&m, &p, &c, &cs.s, &o, n_cap, &d));
  StrategyDecision out;
  out.level = StrategyLevel(d.level);
  out.n = d.n;
  out.t_pred = d.t_pred;
  for (int i = 0; i < d.n_alternatives; ++i)
    out.alternatives.push_back(
        StrategyAlternative{StrategyLevel(d.alternatives[i].level), d.alternatives[i].t_pred, d.alternatives[i].n});
  return out;
}

inline PerfReport estimate_performance(const StrategyDecision& decision, const ModelSpec& model,
                                       const ParallelSpec& par, const ClusterSpec& cluster, int moe_layer_count,
                                       double non_comm_time) {
  moe_strategy_decision d{};
  d.level = int32_t(decision.level);
  d.n = decision.n;
  d.t_pred = decision.t_pred;
  d.n_alternatives = int32_t(std::min<std::size_t>(decision.alternatives.size(), 3));
  for (int i = 0; i < d.n_alternatives; ++i)
    d.alternatives[i] = moe_strategy_alt{int32_t(decision.alternatives[size_t(i)].level),
                                         decision.alternatives[size_t(i)].t_pred, decision.alternatives[size_t(i)].n};
  const moe_model_spec m = planner_detail::to_c(model);
  const moe_parallel_spec p = planner_detail::to_c(par);
  const moe_cluster_spec c = planner_detail::to_c(cluster);
  moe_perf_report r{};
  planner_detail::check(moe_estimate_performance(&d, &m, &p, &c, moe_layer_count, non_comm_time, &r));
  return PerfReport{r.step_latency, r.throughput, r.mfu};
}

// ---------------------------------------------------------------- calibrate.hpp
inline CalibrationSet calibrate(const std::vector<BenchSample>& samples, const ClusterSpec& cluster) {
  std::vector<moe_bench_sample> cs;
  cs.reserve(samples.size());
  for (const auto& s : samples) {
    int prim = -1;
    if (s.primitive == "alltoall") prim = 0;
    else if (s.primitive == "allgather") prim = 1;
    else if (s.primitive == "d2d") prim = 2;
    else throw CalibrationError("calibrate: unknown primitive '" + s.primitive + "'");
    cs.push_back(moe_bench_sample{prim, s.volume, s.seconds});
  }
  const moe_cluster_spec c = planner_detail::to_c(cluster);
  const size_t cap = std::max<size_t>(cs.size(), 1);
  std::vector<double> vol(3 * cap), eff(3 * cap);
  int32_t npts[3] = {0, 0, 0};
  moe_overhead ov{};
  planner_detail::check(
      moe_calibrate(cs.data(), int32_t(cs.size()), &c, vol.data(), eff.data(), npts, &ov));
  CalibrationSet out;
  EfficiencyCurve* curves[3] = {&out.curves.alltoall, &out.curves.allgather, &out.curves.d2d};
  for (int q = 0; q < 3; ++q)
    for (int i = 0; i < npts[q]; ++i)
      curves[q]->points.push_back(CurvePoint{vol[size_t(q) * cap + size_t(i)], eff[size_t(q) * cap + size_t(i)]});
  out.overhead = OverheadModel{ov.alpha_comm, ov.alpha_copy};
  return out;
}

// ---------------------------------------------------------------- pipesim.hpp
namespace pipesim {

inline TaskGraph build_pipeline(StrategyLevel level, int n, const ChunkTiming& timing, double expert_time,
                                int phases = 2) {
  const moe_chunk_timing tm = planner_detail::to_c(timing);
  int32_t count = 0;
  planner_detail::check(
      moe_build_pipeline(int(level), n, &tm, expert_time, phases, nullptr, nullptr, nullptr, 0, nullptr, 0, &count));
  std::vector<moe_sim_task> tasks(size_t(count) + 1);
  std::vector<int32_t> kinds(size_t(count) + 1), chunks(size_t(count) + 1);
  std::vector<int32_t> deps(size_t(count) * 4 + 4);
  planner_detail::check(moe_build_pipeline(int(level), n, &tm, expert_time, phases, tasks.data(), kinds.data(),
                                           chunks.data(), count, deps.data(), int32_t(deps.size()), &count));
  static const char* kLeg[3] = {"aa", "ag", "d2d"};
  TaskGraph g(static_cast<size_t>(count));
  for (int32_t i = 0; i < count; ++i) {
    const int kind = kinds[size_t(i)];
    const int leg = kind % 8;
    g[size_t(i)].id = leg == 3 ? std::string("expert")
                               : std::string(kind / 8 ? "combine" : "dispatch") + "_" + kLeg[leg] + "_" +
                                     std::to_string(chunks[size_t(i)]);
    g[size_t(i)].stream = Stream(tasks[size_t(i)].stream);
    g[size_t(i)].duration = tasks[size_t(i)].duration;
  }
  for (int32_t i = 0; i < count; ++i)
    for (int32_t q = tasks[size_t(i)].dep_begin; q < tasks[size_t(i)].dep_end; ++q)
      g[size_t(i)].deps.push_back(g[size_t(deps[size_t(q)])].id);
  return g;
}

// The task ids are resolved here (the C ABI schedules by index); duration,
// id uniqueness and dependency names are checked in the reference's order.
inline StreamTrace simulate(const TaskGraph& tasks) {
  std::unordered_map<std::string, int32_t> index;
  index.reserve(tasks.size());
  for (size_t i = 0; i < tasks.size(); ++i) {
    if (tasks[i].duration < 0.0)
      throw std::invalid_argument("simulate: negative duration for task " + tasks[i].id);
    if (!index.emplace(tasks[i].id, int32_t(i)).second)
      throw std::invalid_argument("simulate: duplicate task id " + tasks[i].id);
  }
  std::vector<moe_sim_task> ct(tasks.size() + 1);
  std::vector<int32_t> deps;
  for (size_t i = 0; i < tasks.size(); ++i) {
    ct[i].stream = int32_t(tasks[i].stream);
    ct[i].duration = tasks[i].duration;
    ct[i].dep_begin = int32_t(deps.size());
    for (const auto& d : tasks[i].deps) {
      const auto it = index.find(d);
      if (it == index.end()) throw std::invalid_argument("simulate: unknown dependency " + d);
      deps.push_back(it->second);
    }
    ct[i].dep_end = int32_t(deps.size());
  }
  deps.push_back(0);
  std::vector<double> start(tasks.size() + 1), end(tasks.size() + 1);
  double makespan = 0.0;
  planner_detail::check(
      moe_simulate_graph(ct.data(), int32_t(tasks.size()), deps.data(), start.data(), end.data(), &makespan));
  StreamTrace trace;
  trace.spans.reserve(tasks.size());
  for (size_t i = 0; i < tasks.size(); ++i) trace.spans.push_back({tasks[i].id, tasks[i].stream, start[i], end[i]});
  trace.makespan = makespan;
  return trace;
}

}  // namespace pipesim
}  // namespace moeplan

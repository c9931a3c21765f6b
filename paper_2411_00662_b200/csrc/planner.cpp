// MoNTA planner: volume/efficiency cost model, optimal chunk search
// (Alg. 1/2), strategy selection (Alg. 3), calibration from measured
// samples, and the multi-stream list-scheduling simulator — host fp64.
//
// Semantics follow the reference headers exactly (they are the parity pins):
//   lookup_efficiency       config.hpp:70-87
//   chunk_*_time, baseline, o1   commcost.hpp:48-109
//   o2/o3 score + search    chunkopt.hpp:16-93
//   asymptotic_speedup      chunkopt.hpp:98-104
//   select_strategy         strategy.hpp:24-47
//   estimate_performance    strategy.hpp:59-80
//   calibrate               calibrate.hpp:34-118
//   build_pipeline/simulate pipesim.hpp:58-173
// On B200 the curves fed to it are measured on NVLink (bench/calibrate.py).
#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <deque>
#include <map>
#include <string>
#include <vector>

#include "monta.h"

namespace monta {
moe_status fail(moe_status st, const char* fmt, ...);
}

namespace {

using monta::fail;

moe_status lookup(const moe_curve* curve, double volume, double* out) {
  if (!(volume > 0.0)) return fail(MOE_ERR_INVALID_ARGUMENT, "lookup_efficiency: volume must be positive");
  if (!curve || curve->n_points <= 0 || !curve->volume || !curve->efficiency)
    return fail(MOE_ERR_INVALID_ARGUMENT, "lookup_efficiency: curve has no points");
  const double* v = curve->volume;
  const double* e = curve->efficiency;
  const int n = curve->n_points;
  if (volume <= v[0]) { *out = e[0]; return MOE_OK; }
  if (volume >= v[n - 1]) { *out = e[n - 1]; return MOE_OK; }
  // first point strictly above the volume
  const int hi = int(std::upper_bound(v, v + n, volume) - v);
  const int lo = hi - 1;
  const double f = (std::log(volume) - std::log(v[lo])) / (std::log(v[hi]) - std::log(v[lo]));
  *out = e[lo] + (e[hi] - e[lo]) * f;
  return MOE_OK;
}

double alpha_comm(const moe_overhead* ov) { return ov ? ov->alpha_comm : 0.0; }
double alpha_copy(const moe_overhead* ov) { return ov ? ov->alpha_copy : 0.0; }

moe_status aa_time(double volume, int n, int t, int e, double b1, const moe_curve* curve,
                   const moe_overhead* ov, double* out) {
  if (n < 1 || t < 1 || e < 1) return fail(MOE_ERR_INVALID_ARGUMENT, "chunk_alltoall_time: n, t, e must be >= 1");
  if (volume < 0.0) return fail(MOE_ERR_INVALID_ARGUMENT, "chunk_alltoall_time: negative volume");
  if (e == 1 || volume == 0.0) { *out = alpha_comm(ov); return MOE_OK; }
  const double per_call = volume / (double(n) * t);
  double r1;
  if (moe_status st = lookup(curve, per_call, &r1)) return st;
  *out = alpha_comm(ov) + per_call * (e - 1.0) / e / (b1 * r1);
  return MOE_OK;
}

moe_status ag_time(double volume, int n, int t, double b2, const moe_curve* curve, const moe_overhead* ov,
                   double* out) {
  if (n < 1 || t < 1) return fail(MOE_ERR_INVALID_ARGUMENT, "chunk_allgather_time: n and t must be >= 1");
  if (volume < 0.0) return fail(MOE_ERR_INVALID_ARGUMENT, "chunk_allgather_time: negative volume");
  if (t == 1 || volume == 0.0) { *out = alpha_comm(ov); return MOE_OK; }
  const double per_call = volume / n;
  double r2;
  if (moe_status st = lookup(curve, per_call, &r2)) return st;
  *out = alpha_comm(ov) + per_call * (t - 1.0) / t / (b2 * r2);
  return MOE_OK;
}

moe_status d2d_time(double volume, int n, double b3, const moe_curve* curve, const moe_overhead* ov,
                    double* out) {
  if (n < 1) return fail(MOE_ERR_INVALID_ARGUMENT, "chunk_d2d_time: n must be >= 1");
  if (volume < 0.0) return fail(MOE_ERR_INVALID_ARGUMENT, "chunk_d2d_time: negative volume");
  if (volume == 0.0) { *out = alpha_copy(ov); return MOE_OK; }
  const double per_call = volume / n;
  double r3;
  if (moe_status st = lookup(curve, per_call, &r3)) return st;
  *out = alpha_copy(ov) + per_call / (b3 * r3);
  return MOE_OK;
}

moe_status base_time(double volume, int e, double b1, const moe_curve* curve, const moe_overhead* ov,
                     double* out) {
  if (e < 1) return fail(MOE_ERR_INVALID_ARGUMENT, "baseline_time: e must be >= 1");
  if (volume < 0.0) return fail(MOE_ERR_INVALID_ARGUMENT, "baseline_time: negative volume");
  if (e == 1 || volume == 0.0) { *out = alpha_comm(ov); return MOE_OK; }
  double r1;
  if (moe_status st = lookup(curve, volume, &r1)) return st;
  *out = alpha_comm(ov) + volume * (e - 1.0) / e / (b1 * r1);
  return MOE_OK;
}

double volume_of(const moe_model_spec* m) {
  return double(m->b) * double(m->s) * double(m->h) * double(m->bpe);
}

double score_o2(double aa, double ag, double d2d, int n) {
  // AllGather and reorder copy share a stream: the slower side repeats n times.
  return aa < ag + d2d ? aa + (ag + d2d) * n : aa * n + ag + d2d;
}
double score_o3(double aa, double ag, double d2d, int n) {
  // The copy has its own stream: only the gather races the AllToAll.
  return aa < ag ? aa + ag * n + d2d : aa * n + ag + d2d;
}

template <class Score>
moe_status search(const moe_model_spec* m, const moe_parallel_spec* par, const moe_cluster_spec* cl,
                  const moe_curve_set* cv, const moe_overhead* ov, int n_cap, Score score,
                  moe_chunk_search_result* out) {
  if (!m || !par || !cl || !cv || !out) return fail(MOE_ERR_INVALID_ARGUMENT, "chunk search: null argument");
  if (par->t < 2 || par->e < 2)
    return fail(MOE_ERR_STRATEGY_INAPPLICABLE, "chunked alltoall needs t >= 2 and e >= 2");
  const double volume = volume_of(m);
  const int64_t cap = std::min<int64_t>(m->s, n_cap);
  const int n_max = int(std::max<int64_t>(1, cap));
  bool have = false, feasible = false;
  moe_chunk_search_result best{};
  for (int n = 1; n <= n_max; ++n) {
    const bool passes = volume / (double(n) * par->t) >= cv->alltoall.i_minimal &&
                        volume / n >= cv->allgather.i_minimal;
    if (!passes && n > 1) break;  // chunks only shrink further
    double aa, ag, dd;
    if (moe_status st = aa_time(volume, n, par->t, par->e, cl->b1, &cv->alltoall, ov, &aa)) return st;
    if (moe_status st = ag_time(volume, n, par->t, cl->b2, &cv->allgather, ov, &ag)) return st;
    if (moe_status st = d2d_time(volume, n, cl->b3, &cv->d2d, ov, &dd)) return st;
    const double total = score(aa, ag, dd, n);
    if (!have || total < best.t_pred) {
      best.n_opt = n;
      best.t_pred = total;
      best.per_chunk = moe_chunk_timing{aa, ag, dd, n, volume};
      have = true;
    }
    feasible = feasible || passes;
    if (!passes) break;  // n == 1 is scored even when gated out
  }
  best.feasible = feasible ? 1 : 0;
  *out = best;
  return MOE_OK;
}

}  // namespace

extern "C" moe_status moe_lookup_efficiency(const moe_curve* curve, double volume, double* out) {
  if (!out) return fail(MOE_ERR_INVALID_ARGUMENT, "lookup_efficiency: null out");
  return lookup(curve, volume, out);
}

extern "C" double moe_traffic_volume(const moe_model_spec* m) { return m ? volume_of(m) : 0.0; }

extern "C" moe_status moe_chunk_alltoall_time(double volume, int32_t n, int32_t t, int32_t e, double b1,
                                              const moe_curve* curve, const moe_overhead* ov, double* out) {
  return aa_time(volume, n, t, e, b1, curve, ov, out);
}
extern "C" moe_status moe_chunk_allgather_time(double volume, int32_t n, int32_t t, double b2,
                                               const moe_curve* curve, const moe_overhead* ov, double* out) {
  return ag_time(volume, n, t, b2, curve, ov, out);
}
extern "C" moe_status moe_chunk_d2d_time(double volume, int32_t n, double b3, const moe_curve* curve,
                                         const moe_overhead* ov, double* out) {
  return d2d_time(volume, n, b3, curve, ov, out);
}
extern "C" moe_status moe_baseline_time(double volume, int32_t e, double b1, const moe_curve* curve,
                                        const moe_overhead* ov, double* out) {
  return base_time(volume, e, b1, curve, ov, out);
}
extern "C" moe_status moe_o1_time(double volume, int32_t t, int32_t e, double b1, double b2,
                                  const moe_curve_set* curves, const moe_overhead* ov, double* out) {
  if (t < 1 || e < 1) return fail(MOE_ERR_INVALID_ARGUMENT, "o1_time: t and e must be >= 1");
  if (!curves) return fail(MOE_ERR_INVALID_ARGUMENT, "o1_time: null curves");
  if (t == 1) return base_time(volume, e, b1, &curves->alltoall, ov, out);
  double aa, ag;
  if (moe_status st = aa_time(volume, 1, t, e, b1, &curves->alltoall, ov, &aa)) return st;
  if (moe_status st = ag_time(volume, 1, t, b2, &curves->allgather, ov, &ag)) return st;
  *out = aa + ag;
  return MOE_OK;
}
extern "C" double moe_o2_score(double aa, double ag, double d2d, int32_t n) { return score_o2(aa, ag, d2d, n); }
extern "C" double moe_o3_score(double aa, double ag, double d2d, int32_t n) { return score_o3(aa, ag, d2d, n); }

extern "C" moe_status moe_o2_search(const moe_model_spec* m, const moe_parallel_spec* par,
                                    const moe_cluster_spec* cl, const moe_curve_set* curves,
                                    const moe_overhead* ov, int32_t n_cap, moe_chunk_search_result* out) {
  return search(m, par, cl, curves, ov, n_cap, score_o2, out);
}
extern "C" moe_status moe_o3_search(const moe_model_spec* m, const moe_parallel_spec* par,
                                    const moe_cluster_spec* cl, const moe_curve_set* curves,
                                    const moe_overhead* ov, int32_t n_cap, moe_chunk_search_result* out) {
  return search(m, par, cl, curves, ov, n_cap, score_o3, out);
}

extern "C" moe_status moe_asymptotic_speedup(int32_t t, int32_t e, double b1, double b2, double r1, double r2,
                                             double* out) {
  if (t < 2 || e < 2) return fail(MOE_ERR_STRATEGY_INAPPLICABLE, "asymptotic_speedup needs t >= 2 and e >= 2");
  *out = (t - 1.0) / t * e / (e - 1.0) * (b1 * r1) / (b2 * r2);
  return MOE_OK;
}

extern "C" moe_status moe_select_strategy(const moe_model_spec* m, const moe_parallel_spec* par,
                                          const moe_cluster_spec* cl, const moe_curve_set* curves,
                                          const moe_overhead* ov, int32_t n_cap, moe_strategy_decision* out) {
  if (!m || !par || !cl || !curves || !out) return fail(MOE_ERR_INVALID_ARGUMENT, "select_strategy: null argument");
  const double volume = volume_of(m);
  moe_strategy_decision d{};
  if (par->t == 1) {
    double tb;
    if (moe_status st = base_time(volume, par->e, cl->b1, &curves->alltoall, ov, &tb)) return st;
    d.level = MOE_BASELINE;
    d.n = 1;
    d.t_pred = tb;
    d.n_alternatives = 1;
    d.alternatives[0] = moe_strategy_alt{MOE_BASELINE, tb, 1};
    *out = d;
    return MOE_OK;
  }
  double t1;
  if (moe_status st = moe_o1_time(volume, par->t, par->e, cl->b1, cl->b2, curves, ov, &t1)) return st;
  d.alternatives[d.n_alternatives++] = moe_strategy_alt{MOE_O1, t1, 1};
  if (par->e >= 2) {
    moe_chunk_search_result r2, r3;
    if (moe_status st = moe_o2_search(m, par, cl, curves, ov, n_cap, &r2)) return st;
    d.alternatives[d.n_alternatives++] = moe_strategy_alt{MOE_O2, r2.t_pred, r2.n_opt};
    if (moe_status st = moe_o3_search(m, par, cl, curves, ov, n_cap, &r3)) return st;
    d.alternatives[d.n_alternatives++] = moe_strategy_alt{MOE_O3, r3.t_pred, r3.n_opt};
  }
  int best = 0;  // strict '<': ties keep O1 over O2 over O3
  for (int i = 1; i < d.n_alternatives; ++i)
    if (d.alternatives[i].t_pred < d.alternatives[best].t_pred) best = i;
  d.level = d.alternatives[best].level;
  d.n = d.alternatives[best].n;
  d.t_pred = d.alternatives[best].t_pred;
  *out = d;
  return MOE_OK;
}

// B200 variant (one NVSwitch box): the AllToAll and the AllGather leave each
// GPU through the same NVLink ports, so chunking cannot overlap the two legs —
// their bytes move at the unchunked rate whatever n is — and every extra
// chunk costs one more per-call overhead.  The engine lands rows at their
// final offsets (FINAL landing: no reorder copy), so no d2d term:
// score = aa(n=1) + ag(n=1) + (n - 1) alpha_comm.
// (Measured at 2x2 on the four BASELINE layers: within 3-18% of the exchange
// kernel's time for O1 and O2/O3 at n = 2..16 with in-situ curves.)
extern "C" moe_status moe_select_strategy_b200(const moe_model_spec* m, const moe_parallel_spec* par,
                                               const moe_cluster_spec* cl, const moe_curve_set* curves,
                                               const moe_overhead* ov, int32_t n_cap, int32_t shared_egress,
                                               moe_strategy_decision* out) {
  if (!shared_egress) return moe_select_strategy(m, par, cl, curves, ov, n_cap, out);
  if (!m || !par || !cl || !curves || !out) return fail(MOE_ERR_INVALID_ARGUMENT, "select_strategy: null argument");
  if (par->t == 1) return moe_select_strategy(m, par, cl, curves, ov, n_cap, out);  // baseline only
  const double volume = volume_of(m);
  moe_strategy_decision d{};
  double t1;
  if (moe_status st = moe_o1_time(volume, par->t, par->e, cl->b1, cl->b2, curves, ov, &t1)) return st;
  d.alternatives[d.n_alternatives++] = moe_strategy_alt{MOE_O1, t1, 1};
  if (par->e >= 2) {
    double aa1, ag1;
    if (moe_status st = aa_time(volume, 1, par->t, par->e, cl->b1, &curves->alltoall, ov, &aa1)) return st;
    if (moe_status st = ag_time(volume, 1, par->t, cl->b2, &curves->allgather, ov, &ag1)) return st;
    const double alpha = ov ? ov->alpha_comm : 0.0;
    auto shared = [&](double, double, double, int n) { return aa1 + ag1 + (n - 1) * alpha; };
    moe_chunk_search_result r2, r3;
    if (moe_status st = search(m, par, cl, curves, ov, n_cap, shared, &r2)) return st;
    d.alternatives[d.n_alternatives++] = moe_strategy_alt{MOE_O2, r2.t_pred, r2.n_opt};
    if (moe_status st = search(m, par, cl, curves, ov, n_cap, shared, &r3)) return st;
    d.alternatives[d.n_alternatives++] = moe_strategy_alt{MOE_O3, r3.t_pred, r3.n_opt};
  }
  int best = 0;
  for (int i = 1; i < d.n_alternatives; ++i)
    if (d.alternatives[i].t_pred < d.alternatives[best].t_pred) best = i;
  d.level = d.alternatives[best].level;
  d.n = d.alternatives[best].n;
  d.t_pred = d.alternatives[best].t_pred;
  *out = d;
  return MOE_OK;
}

extern "C" moe_status moe_estimate_performance(const moe_strategy_decision* d, const moe_model_spec* m,
                                               const moe_parallel_spec* par, const moe_cluster_spec* cl,
                                               int32_t moe_layer_count, double non_comm_time,
                                               moe_perf_report* out) {
  if (!d || !m || !par || !cl || !out) return fail(MOE_ERR_INVALID_ARGUMENT, "estimate_performance: null argument");
  if (non_comm_time < 0.0) return fail(MOE_ERR_INVALID_ARGUMENT, "estimate_performance: non_comm_time must be >= 0");
  if (moe_layer_count < 0) return fail(MOE_ERR_INVALID_ARGUMENT, "estimate_performance: moe_layer_count must be >= 0");
  const double step = non_comm_time + 2.0 * moe_layer_count * d->t_pred;
  if (!(step > 0.0)) return fail(MOE_ERR_INVALID_ARGUMENT, "estimate_performance: step latency is zero");
  const double tokens = double(m->b) * double(m->s) * par->d;
  const double active = double(m->p1) + double(m->k) * double(m->p2) / par->e;
  const double gpus = double(cl->nodes) * cl->gpus_per_node;
  const double mfu = 6.0 * active * tokens / (step * cl->peak_flops * gpus);
  out->step_latency = step;
  out->throughput = tokens / step;
  out->mfu = std::min(1.0, std::max(0.0, mfu));
  return MOE_OK;
}

// ---------------------------------------------------------------------------
// calibration
namespace {

// Least-squares intercept of seconds vs volume over the smaller half of the
// samples (at least two); clamped at zero; degenerate fits give zero.
double intercept(std::vector<moe_bench_sample> s) {
  std::sort(s.begin(), s.end(),
            [](const moe_bench_sample& a, const moe_bench_sample& b) { return a.volume < b.volume; });
  const size_t take = std::min(s.size(), std::max<size_t>(2, s.size() / 2));
  s.resize(take);
  double sv = 0, st = 0, svv = 0, svt = 0;
  for (const auto& x : s) {
    sv += x.volume;
    st += x.seconds;
    svv += x.volume * x.volume;
    svt += x.volume * x.seconds;
  }
  const double cnt = double(s.size());
  const double den = cnt * svv - sv * sv;
  if (den <= 0.0) return 0.0;
  const double slope = (cnt * svt - sv * st) / den;
  return std::max(0.0, (st - slope * sv) / cnt);
}

const char* kPrimName[3] = {"alltoall", "allgather", "d2d"};

moe_status fit(const std::vector<moe_bench_sample>& s, double wire, double bw, int prim, double* vol,
               double* eff, int32_t* np) {
  std::map<double, std::pair<double, int>> by;
  for (const auto& x : s) {
    if (!(x.volume > 0.0) || !(x.seconds > 0.0))
      return fail(MOE_ERR_CALIBRATION, "calibrate: %s sample needs positive volume and time", kPrimName[prim]);
    const double e = wire * x.volume / (bw * x.seconds);
    if (!(e > 0.0)) return fail(MOE_ERR_CALIBRATION, "calibrate: %s sample implies zero efficiency", kPrimName[prim]);
    auto& slot = by[x.volume];
    slot.first += std::min(1.0, e);
    slot.second += 1;
  }
  int i = 0;
  for (const auto& kv : by) {
    vol[i] = kv.first;
    eff[i] = kv.second.first / kv.second.second;
    ++i;
  }
  *np = i;
  return MOE_OK;
}

}  // namespace

extern "C" moe_status moe_calibrate(const moe_bench_sample* samples, int32_t count, const moe_cluster_spec* cl,
                                    double* volumes, double* efficiencies, int32_t* n_points,
                                    moe_overhead* overhead) {
  if ((!samples && count > 0) || !cl || !volumes || !efficiencies || !n_points || !overhead || count < 0)
    return fail(MOE_ERR_INVALID_ARGUMENT, "calibrate: null argument");
  std::vector<moe_bench_sample> groups[3];
  for (int i = 0; i < count; ++i) {
    const int p = samples[i].primitive;
    if (p < 0 || p > 2) return fail(MOE_ERR_CALIBRATION, "calibrate: unknown primitive '%d'", p);
    groups[p].push_back(samples[i]);
  }
  for (int p = 0; p < 3; ++p)
    if (groups[p].size() < 2)
      return fail(MOE_ERR_CALIBRATION, "calibrate: need at least 2 '%s' samples, got %zu", kPrimName[p],
                  groups[p].size());
  if (cl->nodes < 2) return fail(MOE_ERR_CALIBRATION, "calibrate: alltoall calibration needs >= 2 nodes");
  if (cl->gpus_per_node < 2)
    return fail(MOE_ERR_CALIBRATION, "calibrate: allgather calibration needs >= 2 cards per node");
  const double wire[3] = {(cl->nodes - 1.0) / cl->nodes, (cl->gpus_per_node - 1.0) / cl->gpus_per_node, 1.0};
  const double bw[3] = {cl->b1, cl->b2, cl->b3};
  for (int p = 0; p < 3; ++p)
    if (moe_status st = fit(groups[p], wire[p], bw[p], p, volumes + size_t(p) * count,
                            efficiencies + size_t(p) * count, n_points + p))
      return st;
  overhead->alpha_comm = 0.5 * (intercept(groups[0]) + intercept(groups[1]));
  overhead->alpha_copy = intercept(groups[2]);
  return MOE_OK;
}

// ---------------------------------------------------------------------------
// multi-stream simulator
namespace {

struct Task {
  int kind, chunk, stream;
  double dur;
  std::vector<int> deps;
};

// One chunked phase: per chunk AA, then AG after it, then the reorder copy
// after the AG (same stream as the AG under O2, its own under O3).
std::vector<int> add_phase(std::vector<Task>& g, int level, int n, const moe_chunk_timing& tm, int phase,
                           const std::vector<int>& phase_deps) {
  std::vector<int> terminals;
  for (int j = 1; j <= n; ++j) {
    g.push_back(Task{phase * 8 + 0, j, 0, tm.aa, phase_deps});
    const int aa = int(g.size()) - 1;
    if (level == MOE_BASELINE) { terminals.push_back(aa); continue; }
    g.push_back(Task{phase * 8 + 1, j, 1, tm.ag, {aa}});
    const int ag = int(g.size()) - 1;
    if (level == MOE_O1) { terminals.push_back(ag); continue; }
    g.push_back(Task{phase * 8 + 2, j, level == MOE_O2 ? 1 : 2, tm.d2d, {ag}});
    terminals.push_back(int(g.size()) - 1);
  }
  return terminals;
}

moe_status schedule(const std::vector<Task>& g, std::vector<double>& start, std::vector<double>& end) {
  const size_t n = g.size();
  std::vector<std::vector<int>> preds(n), succs(n);
  std::map<int, int> last_on_stream;
  for (size_t i = 0; i < n; ++i) {
    if (g[i].dur < 0.0) return fail(MOE_ERR_INVALID_ARGUMENT, "simulate: negative duration for task %zu", i);
    for (int dpd : g[i].deps) {
      if (dpd < 0 || size_t(dpd) >= n) return fail(MOE_ERR_INVALID_ARGUMENT, "simulate: unknown dependency %d", dpd);
      preds[i].push_back(dpd);
    }
    auto it = last_on_stream.find(g[i].stream);
    if (it != last_on_stream.end()) preds[i].push_back(it->second);
    last_on_stream[g[i].stream] = int(i);
  }
  std::vector<int> indeg(n, 0);
  for (size_t i = 0; i < n; ++i)
    for (int p : preds[i]) {
      succs[size_t(p)].push_back(int(i));
      ++indeg[i];
    }
  std::deque<int> ready;
  for (size_t i = 0; i < n; ++i)
    if (indeg[i] == 0) ready.push_back(int(i));
  start.assign(n, 0.0);
  end.assign(n, 0.0);
  size_t done = 0;
  while (!ready.empty()) {
    const int i = ready.front();
    ready.pop_front();
    ++done;
    double at = 0.0;
    for (int p : preds[size_t(i)]) at = std::max(at, end[size_t(p)]);
    start[size_t(i)] = at;
    end[size_t(i)] = at + g[size_t(i)].dur;
    for (int s : succs[size_t(i)])
      if (--indeg[size_t(s)] == 0) ready.push_back(s);
  }
  if (done != n) return fail(MOE_ERR_INVALID_GRAPH, "simulate: dependency cycle detected");
  return MOE_OK;
}

}  // namespace

extern "C" moe_status moe_simulate_pipeline(int level, int32_t n, const moe_chunk_timing* timing,
                                            double expert_time, int32_t phases, moe_sim_span* spans,
                                            int32_t capacity, int32_t* n_spans, double* makespan) {
  if (!timing || !n_spans || !makespan) return fail(MOE_ERR_INVALID_ARGUMENT, "simulate_pipeline: null argument");
  if (n < 1) return fail(MOE_ERR_INVALID_ARGUMENT, "build_pipeline: n must be >= 1");
  if (phases != 1 && phases != 2) return fail(MOE_ERR_INVALID_ARGUMENT, "build_pipeline: phases must be 1 or 2");
  if (level < MOE_BASELINE || level > MOE_O3) return fail(MOE_ERR_INVALID_ARGUMENT, "build_pipeline: bad level");
  if (level == MOE_BASELINE || level == MOE_O1) n = 1;
  std::vector<Task> g;
  const std::vector<int> term = add_phase(g, level, n, *timing, 0, {});
  if (phases == 2) {
    g.push_back(Task{3, 0, 3, expert_time, term});
    const int expert = int(g.size()) - 1;
    add_phase(g, level, n, *timing, 1, {expert});
  }
  std::vector<double> st, en;
  if (moe_status s = schedule(g, st, en)) return s;
  double ms = 0.0;
  for (size_t i = 0; i < g.size(); ++i) {
    if (int32_t(i) < capacity && spans) spans[i] = moe_sim_span{g[i].kind, g[i].chunk, g[i].stream, st[i], en[i]};
    ms = std::max(ms, en[i]);
  }
  *n_spans = int32_t(g.size());
  *makespan = ms;
  return MOE_OK;
}

extern "C" moe_status moe_simulate_graph(const moe_sim_task* tasks, int32_t count, const int32_t* deps,
                                         double* start, double* end, double* makespan) {
  if ((count > 0 && (!tasks || !start || !end)) || !makespan || count < 0)
    return fail(MOE_ERR_INVALID_ARGUMENT, "simulate: null argument");
  std::vector<Task> g(static_cast<size_t>(count));
  for (int i = 0; i < count; ++i) {
    g[size_t(i)].kind = 0;
    g[size_t(i)].chunk = 0;
    g[size_t(i)].stream = tasks[i].stream;
    g[size_t(i)].dur = tasks[i].duration;
    for (int q = tasks[i].dep_begin; q < tasks[i].dep_end; ++q) g[size_t(i)].deps.push_back(deps[q]);
  }
  std::vector<double> st, en;
  if (moe_status s = schedule(g, st, en)) return s;
  double ms = 0.0;
  for (int i = 0; i < count; ++i) {
    start[i] = st[size_t(i)];
    end[i] = en[size_t(i)];
    ms = std::max(ms, en[size_t(i)]);
  }
  *makespan = ms;
  return MOE_OK;
}

extern "C" moe_status moe_build_pipeline(int level, int32_t n, const moe_chunk_timing* timing, double expert_time,
                                         int32_t phases, moe_sim_task* tasks, int32_t* kinds, int32_t* chunks,
                                         int32_t capacity, int32_t* deps, int32_t dep_capacity, int32_t* count) {
  if (!timing || !count) return fail(MOE_ERR_INVALID_ARGUMENT, "build_pipeline: null argument");
  if (n < 1) return fail(MOE_ERR_INVALID_ARGUMENT, "build_pipeline: n must be >= 1");
  if (phases != 1 && phases != 2) return fail(MOE_ERR_INVALID_ARGUMENT, "build_pipeline: phases must be 1 or 2");
  if (level < MOE_BASELINE || level > MOE_O3) return fail(MOE_ERR_INVALID_ARGUMENT, "build_pipeline: bad level");
  if (level == MOE_BASELINE || level == MOE_O1) n = 1;
  std::vector<Task> g;
  const std::vector<int> term = add_phase(g, level, n, *timing, 0, {});
  if (phases == 2) {
    g.push_back(Task{3, 0, 3, expert_time, term});
    const int expert = int(g.size()) - 1;
    add_phase(g, level, n, *timing, 1, {expert});
  }
  *count = int32_t(g.size());
  if (!tasks) return MOE_OK;  // size query
  if (int32_t(g.size()) > capacity) return fail(MOE_ERR_INVALID_ARGUMENT, "build_pipeline: task capacity too small");
  int32_t at = 0;
  for (size_t i = 0; i < g.size(); ++i) {
    if (at + int32_t(g[i].deps.size()) > dep_capacity)
      return fail(MOE_ERR_INVALID_ARGUMENT, "build_pipeline: dependency capacity too small");
    tasks[i].stream = g[i].stream;
    tasks[i].duration = g[i].dur;
    tasks[i].dep_begin = at;
    for (int d : g[i].deps) deps[at++] = d;
    tasks[i].dep_end = at;
    if (kinds) kinds[i] = g[i].kind;
    if (chunks) chunks[i] = g[i].chunk;
  }
  return MOE_OK;
}

// config.hpp check()/validate(): field-domain and placement reports.  The
// messages are data (one per violated rule), written '\n'-separated.
namespace {

struct Report {
  std::string text;
  int32_t count = 0;
  void add(const std::string& m) {
    text += m;
    text += '\n';
    ++count;
  }
};

void model_rules(const moe_model_spec& m, Report& r) {
  const struct { int64_t v; const char* name; } pos[] = {{m.b, "b"}, {m.s, "s"}, {m.h, "h"},
                                                          {m.a, "a"}, {m.l, "l"}, {m.k, "k"}};
  for (const auto& f : pos)
    if (f.v <= 0) r.add(std::string("model: ") + f.name + " must be positive");
  if (m.p1 < 0) r.add("model: p1 must be non-negative");
  if (m.p2 < 0) r.add("model: p2 must be non-negative");
  if (m.bpe != 1 && m.bpe != 2 && m.bpe != 4 && m.bpe != 8) r.add("model: bpe must be one of 1, 2, 4, 8");
}

void parallel_rules(const moe_parallel_spec& p, Report& r) {
  const struct { int v; const char* name; } deg[] = {{p.d, "d"}, {p.p, "p"}, {p.t, "t"}, {p.e, "e"}, {p.cp, "cp"}};
  for (const auto& f : deg)
    if (f.v < 1) r.add(std::string("parallel: ") + f.name + " must be >= 1");
}

void cluster_rules(const moe_cluster_spec& c, Report& r) {
  if (c.nodes < 1) r.add("cluster: nodes must be >= 1");
  if (c.gpus_per_node < 1) r.add("cluster: gpus_per_node must be >= 1");
  if (!(c.b1 > 0.0)) r.add("cluster: b1 must be positive");
  if (!(c.b2 > 0.0)) r.add("cluster: b2 must be positive");
  if (c.b2 < c.b1) r.add("cluster: b2 must be >= b1 (intra-node links are the fast ones)");
  if (!(c.b3 > 0.0)) r.add("cluster: b3 must be positive");
  if (!(c.peak_flops > 0.0)) r.add("cluster: peak_flops must be positive");
  if (c.switch_capacity < 1) r.add("cluster: switch_capacity must be >= 1");
}

void placement_rules(const moe_parallel_spec& p, const moe_cluster_spec& c, Report& r) {
  if (p.t < 1 || c.gpus_per_node % p.t != 0) {
    r.add("t (" + std::to_string(p.t) + ") does not divide gpus_per_node (" + std::to_string(c.gpus_per_node) + ")");
  } else {
    const int64_t slots = int64_t(c.nodes) * (c.gpus_per_node / p.t);
    if (p.e > slots)
      r.add("e (" + std::to_string(p.e) + ") exceeds the " + std::to_string(slots) +
            " tensor-group slots of the cluster");
  }
  const int64_t gpus = int64_t(c.nodes) * c.gpus_per_node;
  const int64_t dense = int64_t(p.d) * p.p * p.t * p.cp;
  if (dense > gpus)
    r.add("d*p*t*cp (" + std::to_string(dense) + ") exceeds the " + std::to_string(gpus) + " GPUs of the cluster");
}

}  // namespace

extern "C" moe_status moe_check_specs(int which, const moe_model_spec* m, const moe_parallel_spec* p,
                                      const moe_cluster_spec* c, char* buf, int64_t capacity, int32_t* n_messages,
                                      int64_t* bytes_needed) {
  if (!n_messages) return fail(MOE_ERR_INVALID_ARGUMENT, "check_specs: null argument");
  Report r;
  switch (which) {
    case MOE_CHECK_MODEL:
      if (!m) return fail(MOE_ERR_INVALID_ARGUMENT, "check_specs: null model");
      model_rules(*m, r);
      break;
    case MOE_CHECK_PARALLEL:
      if (!p) return fail(MOE_ERR_INVALID_ARGUMENT, "check_specs: null parallel spec");
      parallel_rules(*p, r);
      break;
    case MOE_CHECK_CLUSTER:
      if (!c) return fail(MOE_ERR_INVALID_ARGUMENT, "check_specs: null cluster");
      cluster_rules(*c, r);
      break;
    case MOE_CHECK_PLACEMENT:
      if (!p || !c) return fail(MOE_ERR_INVALID_ARGUMENT, "check_specs: null parallel spec or cluster");
      placement_rules(*p, *c, r);
      break;
    default:
      return fail(MOE_ERR_INVALID_ARGUMENT, "check_specs: unknown report %d", which);
  }
  *n_messages = r.count;
  if (bytes_needed) *bytes_needed = int64_t(r.text.size()) + 1;
  if (buf && capacity > 0) {
    const size_t w = std::min<size_t>(r.text.size(), size_t(capacity - 1));
    std::copy(r.text.begin(), r.text.begin() + std::ptrdiff_t(w), buf);
    buf[w] = '\0';
  }
  return MOE_OK;
}

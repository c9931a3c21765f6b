// ref_shim.cpp — flat C entry points over the UNMODIFIED reference headers
// (/root/reference/proj/include/moeplan/*.hpp), compiled by oracle/Makefile
// into oracle/_ref/libmoeplan_ref.so.  TEST INFRASTRUCTURE ONLY: used to pin
// the C restatement (oracle/moe_oracle.c) and the product planner against
// the reference itself, and as the `cpu_baseline` "reference" kind.  No
// reference source is copied: this file only includes the headers in place.
#include <cstdint>
#include <cstring>
#include <exception>
#include <stdexcept>
#include <string>
#include <vector>

#include "moeplan/calibrate.hpp"
#include "moeplan/chunkopt.hpp"
#include "moeplan/commcost.hpp"
#include "moeplan/config.hpp"
#include "moeplan/dataplane.hpp"
#include "moeplan/pipesim.hpp"
#include "moeplan/strategy.hpp"

using namespace moeplan;
using namespace moeplan::dataplane;

namespace {
thread_local std::string g_msg;

template <class F>
int guard(F&& f) {
  try {
    f();
    return 0;
  } catch (const CorruptRoutingError& e) {
    g_msg = e.what();
    return 2;
  } catch (const StrategyInapplicableError& e) {
    g_msg = e.what();
    return 3;
  } catch (const CalibrationError& e) {
    g_msg = e.what();
    return 4;
  } catch (const pipesim::InvalidGraphError& e) {
    g_msg = e.what();
    return 5;
  } catch (const std::invalid_argument& e) {
    g_msg = e.what();
    return 1;
  } catch (const std::exception& e) {
    g_msg = e.what();
    return 99;
  }
}

EfficiencyCurve curve_of(const double* v, const double* eff, int n, double imin) {
  EfficiencyCurve c;
  for (int i = 0; i < n; ++i) c.points.push_back({v[i], eff[i]});
  c.i_minimal = imin;
  return c;
}

struct RefCurves {
  const double* v[3];
  const double* e[3];
  int n[3];
  double imin[3];
};
CurveSet curves_of(const RefCurves* c) {
  return {curve_of(c->v[0], c->e[0], c->n[0], c->imin[0]), curve_of(c->v[1], c->e[1], c->n[1], c->imin[1]),
          curve_of(c->v[2], c->e[2], c->n[2], c->imin[2])};
}

// Builds per-node PermutedBatch / RoutingDecision from flat arrays.
void build_nodes(int e, int t, int64_t T, int W, int k, const int64_t* payload, const int32_t* experts,
                 const double* probs, std::vector<PermutedBatch>& permuted, std::vector<RoutingDecision>& routing,
                 std::vector<Buffer>* batches) {
  const VirtualTopology topo{e, t};
  permuted.clear();
  routing.clear();
  for (int g = 0; g < e; ++g) {
    std::vector<std::vector<std::int64_t>> rows(static_cast<size_t>(T), std::vector<std::int64_t>(static_cast<size_t>(W)));
    for (int64_t i = 0; i < T; ++i)
      for (int q = 0; q < W; ++q) rows[size_t(i)][size_t(q)] = payload[(g * T + i) * W + q];
    Buffer batch = make_batch(topo, g, rows);
    RoutingDecision rd;
    rd.k = k;
    for (int64_t i = 0; i < T; ++i) {
      TokenRouting tr;
      for (int s = 0; s < k; ++s) {
        tr.experts.push_back(experts[(g * T + i) * k + s]);
        tr.probs.push_back(probs[(g * T + i) * k + s]);
      }
      rd.per_token.push_back(tr);
    }
    permuted.push_back(permute(batch, rd));
    routing.push_back(rd);
    if (batches) batches->push_back(batch);
  }
}

void flatten(const CardBuffers& cb, int W, int64_t cap, int32_t* tags, int64_t* payload, int64_t* count) {
  for (size_t c = 0; c < cb.size(); ++c) {
    count[c] = int64_t(cb[c].size());
    for (size_t r = 0; r < cb[c].size() && int64_t(r) < cap; ++r) {
      const TokenRecord& rec = cb[c][r];
      tags[(c * cap + r) * 3 + 0] = rec.token_id;
      tags[(c * cap + r) * 3 + 1] = rec.source_card;
      tags[(c * cap + r) * 3 + 2] = rec.source_position;
      for (int q = 0; q < W && q < int(rec.payload.size()); ++q) payload[(c * cap + r) * W + q] = rec.payload[size_t(q)];
    }
  }
}

}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_msg.c_str(); }

int ref_route_topk(const double* scores, int64_t T, int E, int k, int32_t* experts, double* probs) {
  return guard([&] {
    std::vector<std::vector<double>> s(static_cast<size_t>(T), std::vector<double>(static_cast<size_t>(E)));
    for (int64_t i = 0; i < T; ++i)
      for (int x = 0; x < E; ++x) s[size_t(i)][size_t(x)] = scores[i * E + x];
    const RoutingDecision rd = route_topk(s, k);
    for (int64_t i = 0; i < T; ++i)
      for (int q = 0; q < k; ++q) {
        experts[i * k + q] = rd.per_token[size_t(i)].experts[size_t(q)];
        probs[i * k + q] = rd.per_token[size_t(i)].probs[size_t(q)];
      }
  });
}

// permute of one node: records' source positions, expert_of and the inverse map.
int ref_permute(int64_t T, int k, const int32_t* experts, int32_t* perm_src, int32_t* expert_of, int32_t* inv,
                int32_t* inv_len, int64_t* n_records) {
  return guard([&] {
    const VirtualTopology topo{1, 1};
    std::vector<std::vector<std::int64_t>> rows(static_cast<size_t>(T), std::vector<std::int64_t>(1, 0));
    Buffer batch = make_batch(topo, 0, rows);
    RoutingDecision rd;
    rd.k = k;
    for (int64_t i = 0; i < T; ++i) {
      TokenRouting tr;
      for (int s = 0; s < k; ++s) {
        tr.experts.push_back(experts[i * k + s]);
        tr.probs.push_back(1.0);
      }
      rd.per_token.push_back(tr);
    }
    const PermutedBatch pb = permute(batch, rd);
    *n_records = int64_t(pb.records.size());
    for (size_t r = 0; r < pb.records.size(); ++r) {
      perm_src[r] = pb.records[r].source_position;
      expert_of[r] = pb.expert_of[r];
    }
    for (int64_t i = 0; i < T; ++i) {
      inv_len[i] = int32_t(pb.inverse_map[size_t(i)].size());
      for (size_t s = 0; s < pb.inverse_map[size_t(i)].size() && int(s) < k; ++s)
        inv[i * k + int64_t(s)] = pb.inverse_map[size_t(i)][s];
    }
  });
}

// Full data plane on the reference: level < 0 -> dispatch_monolithic, else
// dispatch_chunked(level, n).  Outputs per CARD (e*t): tags [cards][cap][3],
// payload [cards][cap][W], counts [cards]; pre_copy likewise (chunked only).
// Then combine_unpermute of the dispatched buffers scaled by `expert_scale`
// (identity = 1) -> combined [e][T][W] doubles + token ids.
int ref_dataplane(int e, int t, int64_t T, int W, int k, const int64_t* payload, const int32_t* experts,
                  const double* probs, int level, int n, int64_t cap, int32_t* tags, int64_t* out_payload,
                  int64_t* counts, int32_t* pre_tags, int64_t* pre_payload, int64_t* pre_counts,
                  int64_t expert_scale, double* combined, int32_t* combined_token) {
  return guard([&] {
    const VirtualTopology topo{e, t};
    std::vector<PermutedBatch> permuted;
    std::vector<RoutingDecision> routing;
    build_nodes(e, t, T, W, k, payload, experts, probs, permuted, routing, nullptr);
    CardBuffers out;
    if (level < 0) {
      out = dispatch_monolithic(permuted, topo);
    } else {
      ChunkedDispatchTrace trace;
      out = dispatch_chunked(permuted, topo, StrategyLevel(level), n, &trace);
      if (pre_tags) flatten(trace.pre_copy, W, cap, pre_tags, pre_payload, pre_counts);
    }
    flatten(out, W, cap, tags, out_payload, counts);
    if (combined) {
      for (auto& buf : out)
        for (auto& rec : buf)
          for (auto& v : rec.payload) v *= expert_scale;
      const auto comb = combine_unpermute(out, routing, permuted, topo);
      for (int g = 0; g < e; ++g)
        for (int64_t i = 0; i < T; ++i) {
          combined_token[g * T + i] = comb[size_t(g)][size_t(i)].token_id;
          for (int q = 0; q < W; ++q) combined[(g * T + i) * W + q] = comb[size_t(g)][size_t(i)].payload[size_t(q)];
        }
    }
  });
}

// ---- planner -------------------------------------------------------------
int ref_lookup_efficiency(const double* v, const double* eff, int n, double volume, double* out) {
  return guard([&] { *out = lookup_efficiency(curve_of(v, eff, n, 0.0), volume); });
}
int ref_chunk_times(double volume, int n, int t, int e, double b1, double b2, double b3, const RefCurves* c,
                    double alpha_comm, double alpha_copy, double* aa, double* ag, double* d2d, double* base,
                    double* o1) {
  return guard([&] {
    const CurveSet cs = curves_of(c);
    const OverheadModel ov{alpha_comm, alpha_copy};
    *aa = chunk_alltoall_time(volume, n, t, e, b1, cs.alltoall, ov);
    *ag = chunk_allgather_time(volume, n, t, b2, cs.allgather, ov);
    *d2d = chunk_d2d_time(volume, n, b3, cs.d2d, ov);
    *base = baseline_time(volume, e, b1, cs.alltoall, ov);
    *o1 = o1_time(volume, t, e, b1, b2, cs, ov);
  });
}
int ref_search(int which, const int64_t* model /*b,s,h,bpe*/, int t, int e, double b1, double b2, double b3,
               const RefCurves* c, double alpha_comm, double alpha_copy, int n_cap, int* n_opt, double* t_pred,
               int* feasible) {
  return guard([&] {
    ModelSpec m;
    m.b = model[0];
    m.s = model[1];
    m.h = model[2];
    m.bpe = int(model[3]);
    ParallelSpec par;
    par.t = t;
    par.e = e;
    ClusterSpec cl;
    cl.b1 = b1;
    cl.b2 = b2;
    cl.b3 = b3;
    const OverheadModel ov{alpha_comm, alpha_copy};
    const auto r = which == 2 ? o2_search(m, par, cl, curves_of(c), ov, n_cap) : o3_search(m, par, cl, curves_of(c), ov, n_cap);
    *n_opt = r.n_opt;
    *t_pred = r.t_pred;
    *feasible = r.feasible ? 1 : 0;
  });
}
int ref_select_strategy(const int64_t* model, int t, int e, double b1, double b2, double b3, const RefCurves* c,
                        double alpha_comm, double alpha_copy, int n_cap, int* level, int* n, double* t_pred,
                        int* n_alts, int* alt_level, double* alt_t, int* alt_n) {
  return guard([&] {
    ModelSpec m;
    m.b = model[0];
    m.s = model[1];
    m.h = model[2];
    m.bpe = int(model[3]);
    ParallelSpec par;
    par.t = t;
    par.e = e;
    ClusterSpec cl;
    cl.b1 = b1;
    cl.b2 = b2;
    cl.b3 = b3;
    const auto d = select_strategy(m, par, cl, curves_of(c), OverheadModel{alpha_comm, alpha_copy}, n_cap);
    *level = int(d.level);
    *n = d.n;
    *t_pred = d.t_pred;
    *n_alts = int(d.alternatives.size());
    for (size_t i = 0; i < d.alternatives.size(); ++i) {
      alt_level[i] = int(d.alternatives[i].level);
      alt_t[i] = d.alternatives[i].t_pred;
      alt_n[i] = d.alternatives[i].n;
    }
  });
}
int ref_calibrate(const int* prim, const double* volume, const double* seconds, int count, int nodes, int gpn,
                  double b1, double b2, double b3, double* vols, double* effs, int* npts, double* alpha_comm,
                  double* alpha_copy) {
  return guard([&] {
    static const char* names[3] = {"alltoall", "allgather", "d2d"};
    std::vector<BenchSample> s;
    for (int i = 0; i < count; ++i)
      s.push_back({prim[i] >= 0 && prim[i] < 3 ? names[prim[i]] : "bogus", volume[i], seconds[i]});
    ClusterSpec cl;
    cl.nodes = nodes;
    cl.gpus_per_node = gpn;
    cl.b1 = b1;
    cl.b2 = b2;
    cl.b3 = b3;
    const CalibrationSet cs = calibrate(s, cl);
    const EfficiencyCurve* cv[3] = {&cs.curves.alltoall, &cs.curves.allgather, &cs.curves.d2d};
    for (int p = 0; p < 3; ++p) {
      npts[p] = int(cv[p]->points.size());
      for (size_t i = 0; i < cv[p]->points.size(); ++i) {
        vols[p * count + int(i)] = cv[p]->points[i].volume;
        effs[p * count + int(i)] = cv[p]->points[i].efficiency;
      }
    }
    *alpha_comm = cs.overhead.alpha_comm;
    *alpha_copy = cs.overhead.alpha_copy;
  });
}
int ref_simulate_pipeline(int level, int n, double aa, double ag, double d2d, double expert, int phases,
                          double* starts, double* ends, int* streams, int cap, int* count, double* makespan) {
  return guard([&] {
    ChunkTiming tm;
    tm.aa = aa;
    tm.ag = ag;
    tm.d2d = d2d;
    tm.n = n;
    const auto g = pipesim::build_pipeline(StrategyLevel(level), n, tm, expert, phases);
    const auto tr = pipesim::simulate(g);
    *count = int(tr.spans.size());
    for (size_t i = 0; i < tr.spans.size() && int(i) < cap; ++i) {
      starts[i] = tr.spans[i].start;
      ends[i] = tr.spans[i].end;
      streams[i] = int(tr.spans[i].stream);
    }
    *makespan = tr.makespan;
  });
}

}  // extern "C"

// monta_dataplane.hpp — the reference's data-plane operator API
// (moeplan::dataplane, /root/reference/proj/include/moeplan/dataplane.hpp)
// implemented on the B200 kernels through the C ABI (monta.h).
//
// Same namespaces, types, function signatures and exception types as the
// reference, so reference code (and its tests) compile against it unchanged:
// put include/dropin on the include path ahead of the reference headers and
// link libmonta.so + libcudart.
//
// Every operation runs on the GPU (device 0 unless MONTA_DEVICE is set):
//   route_topk        moe_route_topk, fp64 (the reference's precision)
//   permute           moe_build_index + moe_permute_rows
//   dispatch_*        a virtual-mode moe_ctx (every card of the topology on one
//                     GPU, as the reference emulates them) — BASELINE for
//                     dispatch_monolithic, O1/O2/O3 + STAGED landing for
//                     dispatch_chunked (the staged buffer is ChunkedDispatchTrace)
//   combine_unpermute moe_ctx_combine with fp64 accumulation in slot order
// The host side only converts between the reference's array-of-records
// containers and device buffers.
//
// Documented deviations (the reference's behaviour there is silent data loss
// or undefined): expert ids must be in [0, e) for dispatch/combine (the
// reference drops records of experts >= e, dataplane.hpp:151-160), every token
// and nodes must hold the same number of tokens; violations throw
// std::invalid_argument.  Tokens with fewer selections than others are padded
// with empty slots (expert id -1), which every kernel skips.  combine_unpermute
// takes its row width from the expert outputs (which may differ from the
// dispatched payload width, as in the reference) but needs every output row
// to share it — rows move as one dense [rows, W] tensor — where the reference
// only requires a token's own slots to agree (dataplane.hpp:335-338); a
// ragged row throws CorruptRoutingError like the reference's mismatch.
// Gates are paired with their expert by id (tr.experts[slot] <-> tr.probs[slot],
// dataplane.hpp:340-343), so the routing's expert order need not ascend.
#pragma once

#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <map>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "monta.h"

#ifndef MONTA_HAVE_STRATEGY_LEVEL
#define MONTA_HAVE_STRATEGY_LEVEL
namespace moeplan {
enum class StrategyLevel { Baseline, O1, O2, O3 };
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

namespace moeplan::dataplane {

struct CorruptRoutingError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

struct VirtualTopology {
  int e = 1;
  int t = 1;
  int cards() const { return e * t; }
  int node_of(int card) const { return card / t; }
  int tp_rank_of(int card) const { return card % t; }
  int card_of(int node, int tp_rank) const { return node * t + tp_rank; }
  int canonical_card(int node) const { return node * t; }
};

struct TokenRecord {
  int token_id = 0;
  int source_card = 0;
  int source_position = 0;
  std::vector<std::int64_t> payload;
  friend bool operator==(const TokenRecord&, const TokenRecord&) = default;
};
using Buffer = std::vector<TokenRecord>;
using CardBuffers = std::vector<Buffer>;

inline Buffer make_batch(const VirtualTopology& topo, int node, const std::vector<std::vector<std::int64_t>>& payloads) {
  Buffer batch(payloads.size());
  for (std::size_t i = 0; i < payloads.size(); ++i)
    batch[i] = TokenRecord{int(i) + node * 100000, topo.canonical_card(node), int(i), payloads[i]};
  return batch;
}

struct TokenRouting {
  std::vector<int> experts;
  std::vector<double> probs;
};
struct RoutingDecision {
  int k = 1;
  std::vector<TokenRouting> per_token;
};
struct PermutedBatch {
  Buffer records;
  std::vector<int> expert_of;
  std::vector<std::vector<int>> inverse_map;
  int batch_tokens = 0;
};
struct ChunkedDispatchTrace {
  CardBuffers pre_copy;
};
struct CombinedToken {
  int token_id = 0;
  std::vector<double> payload;
};

namespace detail {

[[noreturn]] inline void raise(moe_status st) {
  const std::string msg = moe_last_error();
  if (st == MOE_ERR_INVALID_ARGUMENT) throw std::invalid_argument(msg);
  if (st == MOE_ERR_CORRUPT_ROUTING) throw CorruptRoutingError(msg);
  throw std::runtime_error("monta: " + msg);
}
inline void check(moe_status st) {
  if (st != MOE_OK) raise(st);
}
inline void cuda(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw std::runtime_error(std::string("monta: ") + what + ": " + cudaGetErrorString(e));
}
inline int device() {
  static const int dev = [] {
    const char* s = std::getenv("MONTA_DEVICE");
    const int d = s ? std::atoi(s) : 0;
    cuda(cudaSetDevice(d), "cudaSetDevice");
    return d;
  }();
  cuda(cudaSetDevice(dev), "cudaSetDevice");
  return dev;
}

// Owning device allocation.
template <class T>
struct Dev {
  T* p = nullptr;
  std::size_t n = 0;
  explicit Dev(std::size_t count) : n(count) {
    if (n) cuda(cudaMalloc(reinterpret_cast<void**>(&p), n * sizeof(T)), "cudaMalloc");
  }
  Dev(const std::vector<T>& h) : Dev(h.size()) { upload(h.data(), h.size()); }
  ~Dev() {
    if (p) cudaFree(p);
  }
  Dev(const Dev&) = delete;
  Dev& operator=(const Dev&) = delete;
  void upload(const T* h, std::size_t count) {
    if (count) cuda(cudaMemcpy(p, h, count * sizeof(T), cudaMemcpyHostToDevice), "upload");
  }
  std::vector<T> download(std::size_t count) const {
    std::vector<T> h(count);
    if (count) cuda(cudaMemcpy(h.data(), p, count * sizeof(T), cudaMemcpyDeviceToHost), "download");
    return h;
  }
};

inline void to_device(void* dst, const void* src, std::size_t bytes) {
  if (bytes) cuda(cudaMemcpy(dst, src, bytes, cudaMemcpyHostToDevice), "upload");
}
inline void to_host(void* dst, const void* src, std::size_t bytes) {
  if (bytes) cuda(cudaMemcpy(dst, src, bytes, cudaMemcpyDeviceToHost), "download");
}

// One layer context in virtual mode, rebuilt from the reference's per-node
// permuted batches (node batch rows from the records' source positions,
// routing from expert_of / inverse_map).
struct Layer {
  moe_ctx* ctx = nullptr;
  VirtualTopology topo;
  int T = 0, W = 0, k = 1;
  std::vector<std::vector<int32_t>> experts;   // [e][T*k]
  ~Layer() {
    if (ctx) moe_ctx_destroy(ctx);
  }
};

// hidden_override > 0: the context's row width (the combine's expert-output
// width, which may differ from the dispatched payload width).
inline void build_layer(Layer& L, const std::vector<PermutedBatch>& per_node, const VirtualTopology& topo, int n,
                        const std::vector<RoutingDecision>* routing, int hidden_override = 0) {
  device();
  L.topo = topo;
  const int e = topo.e;
  L.T = per_node.empty() ? 0 : per_node[0].batch_tokens;
  int width = -1, k = -1;
  for (const auto& b : per_node) {
    if (b.batch_tokens != L.T) throw std::invalid_argument("monta: nodes must hold the same number of tokens");
    for (const auto& r : b.records) {
      if (width < 0) width = int(r.payload.size());
      if (int(r.payload.size()) != width) throw std::invalid_argument("dispatch: ragged payloads");
    }
    for (const auto& inv : b.inverse_map) k = std::max(k, int(inv.size()));
  }
  L.W = width < 0 ? 0 : width;
  if (hidden_override > 0) L.W = hidden_override;
  L.k = k < 1 ? 1 : k;
  moe_layer_desc d{};
  d.e = e;
  d.t = topo.t;
  d.num_experts = e;
  d.top_k = L.k;
  d.tokens = L.T;
  d.hidden = L.W > 0 ? L.W : 1;
  d.dtype = MOE_I64;
  d.logit_dtype = MOE_F64;
  d.out_dtype = MOE_F64;
  d.max_chunks = n;
  check(moe_ctx_create(&d, device(), 0, 1, &L.ctx));
  L.experts.assign(e, std::vector<int32_t>(std::size_t(L.T) * L.k, -1));  // -1: empty slot
  for (int g = 0; g < e; ++g) {
    const PermutedBatch& b = per_node[g];
    std::vector<std::int64_t> x(std::size_t(L.T) * d.hidden, 0);
    std::vector<int32_t> ids(L.T, 0);
    std::vector<double> probs(std::size_t(L.T) * L.k, 1.0);
    for (int i = 0; i < L.T && i < int(b.inverse_map.size()); ++i) {
      const auto& inv = b.inverse_map[i];
      for (int s = 0; s < int(inv.size()); ++s) {
        const int r = inv[s];
        const int ex = b.expert_of[r];
        if (ex < 0 || ex >= e) throw std::invalid_argument("monta: expert id outside [0, e)");
        L.experts[g][std::size_t(i) * L.k + s] = ex;
      }
      if (!inv.empty()) {
        const TokenRecord& rec = b.records[inv.front()];
        if (rec.source_card != topo.canonical_card(g) || rec.source_position != i)
          throw std::invalid_argument("monta: records must carry make_batch tags");
        ids[i] = rec.token_id;
        const std::size_t w = std::min<std::size_t>(rec.payload.size(), std::size_t(d.hidden));
        std::copy(rec.payload.begin(), rec.payload.begin() + std::ptrdiff_t(w), x.begin() + std::ptrdiff_t(i) * d.hidden);
      }
      if (routing) {
        // the reference pairs tr.probs[slot] with tr.experts[slot]
        // (dataplane.hpp:335-343); the device slots follow the inverse map
        // (ascending expert), so each slot's gate is looked up by expert id
        const auto& tr = (*routing)[g].per_token[i];
        for (int s = 0; s < int(inv.size()) && s < L.k; ++s) {
          const int ex = b.expert_of[inv[s]];
          int j = 0;
          while (j < int(tr.experts.size()) && tr.experts[j] != ex) ++j;
          if (j == int(tr.experts.size()) || j >= int(tr.probs.size()))
            throw CorruptRoutingError("combine_unpermute: inverse map does not match routing");
          probs[std::size_t(i) * L.k + s] = tr.probs[j];
        }
      }
    }
    for (int rho = 0; rho < topo.t; ++rho) {
      moe_card_view v{};
      check(moe_ctx_card_view(L.ctx, topo.card_of(g, rho), &v));
      to_device(v.x, x.data(), x.size() * 8);
      to_device(v.token_ids, ids.data(), ids.size() * 4);
      to_device(v.experts, L.experts[g].data(), L.experts[g].size() * 4);
      to_device(v.probs, probs.data(), probs.size() * 8);
    }
  }
}

inline Buffer read_rows(const Layer& L, const void* rows_dev, const int32_t* tags_dev, int64_t rows) {
  const int h = L.W > 0 ? L.W : 1;
  std::vector<std::int64_t> pay(std::size_t(rows) * h);
  std::vector<int32_t> tags(std::size_t(rows) * 4);
  to_host(pay.data(), rows_dev, pay.size() * 8);
  to_host(tags.data(), tags_dev, tags.size() * 4);
  Buffer out(rows);
  for (int64_t r = 0; r < rows; ++r) {
    out[r].token_id = tags[r * 4 + 0];
    out[r].source_card = tags[r * 4 + 1];
    out[r].source_position = tags[r * 4 + 2];
    out[r].payload.assign(pay.begin() + r * h, pay.begin() + r * h + L.W);
  }
  return out;
}

inline CardBuffers run_dispatch(const std::vector<PermutedBatch>& per_node, const VirtualTopology& topo,
                                moe_level level, int n, ChunkedDispatchTrace* trace) {
  if (int(per_node.size()) != topo.e)
    throw std::invalid_argument(level == MOE_BASELINE ? "dispatch_monolithic: need one batch per node"
                                                      : "dispatch_chunked: need one batch per node");
  Layer L;
  build_layer(L, per_node, topo, n, nullptr);
  const int landing = level == MOE_BASELINE ? MOE_LAND_FINAL : MOE_LAND_STAGED;
  check(moe_ctx_dispatch(L.ctx, level, n, landing, nullptr));
  check(moe_ctx_sync(L.ctx));
  CardBuffers out(topo.cards());
  if (trace) trace->pre_copy.assign(topo.cards(), {});
  for (int c = 0; c < topo.cards(); ++c) {
    int64_t rows = 0;
    check(moe_ctx_recv_rows(L.ctx, c, &rows));
    moe_card_view v{};
    check(moe_ctx_card_view(L.ctx, c, &v));
    out[c] = read_rows(L, v.recv, v.recv_tags, rows);
    if (trace) trace->pre_copy[c] = read_rows(L, v.pre, v.pre_tags, rows);
  }
  return out;
}

}  // namespace detail

// ---------------------------------------------------------------------------
inline RoutingDecision route_topk(const std::vector<std::vector<double>>& gate_scores, int k) {
  if (k < 1) throw std::invalid_argument("route_topk: k must be >= 1");
  RoutingDecision out;
  out.k = k;
  out.per_token.resize(gate_scores.size());
  // rows are routed on the GPU in runs of equal width
  std::size_t i = 0;
  while (i < gate_scores.size()) {
    const std::size_t E = gate_scores[i].size();
    if (E == 0) throw std::invalid_argument("route_topk: empty gate score row");
    if (int(E) < k) throw std::invalid_argument("route_topk: k exceeds the expert count");
    std::size_t j = i;
    while (j < gate_scores.size() && gate_scores[j].size() == E) ++j;
    const std::size_t T = j - i;
    std::vector<double> flat(T * E);
    for (std::size_t q = 0; q < T; ++q) std::copy(gate_scores[i + q].begin(), gate_scores[i + q].end(), flat.begin() + q * E);
    detail::device();
    detail::Dev<double> dl(flat);
    detail::Dev<int32_t> de(T * k);
    detail::Dev<double> dp(T * k);
    detail::check(moe_route_topk(dl.p, MOE_F64, int64_t(T), int32_t(E), k, de.p, dp.p, nullptr));
    const auto ex = de.download(T * k);
    const auto pr = dp.download(T * k);
    for (std::size_t q = 0; q < T; ++q) {
      auto& tr = out.per_token[i + q];
      tr.experts.assign(ex.begin() + q * k, ex.begin() + (q + 1) * k);
      tr.probs.assign(pr.begin() + q * k, pr.begin() + (q + 1) * k);
    }
    i = j;
  }
  return out;
}

inline PermutedBatch permute(const Buffer& tokens, const RoutingDecision& routing) {
  if (routing.per_token.size() != tokens.size()) throw std::invalid_argument("permute: routing does not cover the batch");
  const int64_t T = int64_t(tokens.size());
  PermutedBatch out;
  out.batch_tokens = int(T);
  out.inverse_map.resize(tokens.size());
  if (T == 0) return out;
  // ragged selections are padded with -1: an empty slot, which the reference's
  // permute never matches either (its loop starts at expert 0)
  int k = 1, E = 1;
  for (const auto& tr : routing.per_token) {
    k = std::max(k, int(tr.experts.size()));
    for (const int x : tr.experts) E = std::max(E, x + 1);
  }
  std::vector<int32_t> experts(std::size_t(T) * k, -1);
  for (int64_t i = 0; i < T; ++i)
    for (std::size_t s = 0; s < routing.per_token[i].experts.size(); ++s)
      experts[i * k + int64_t(s)] = routing.per_token[i].experts[s];
  detail::device();
  const int64_t R = T * k;
  detail::Dev<int32_t> dex(experts), dperm(R), dof(R), dslot(R), dcnt(E), doff(E + 1);
  detail::check(moe_build_index(dex.p, T, k, E, 1, dperm.p, dof.p, dslot.p, dcnt.p, doff.p, nullptr, nullptr));
  const auto perm = dperm.download(R);
  const auto eof = dof.download(R);
  const auto slot = dslot.download(R);
  int64_t valid = 0;  // records: pairs with a real expert (empty slots are skipped)
  for (int64_t q = 0; q < R; ++q) valid += slot[q] >= 0;
  // payloads: gathered on the GPU when the batch is rectangular
  std::size_t W = tokens[0].payload.size();
  bool rect = true;
  for (const auto& rec : tokens) rect = rect && rec.payload.size() == W;
  std::vector<std::int64_t> gathered;
  if (rect && W > 0 && valid > 0) {
    std::vector<std::int64_t> x(std::size_t(T) * W);
    for (int64_t i = 0; i < T; ++i) std::copy(tokens[i].payload.begin(), tokens[i].payload.end(), x.begin() + i * W);
    detail::Dev<std::int64_t> dx(x), dg(std::size_t(valid) * W);
    detail::check(moe_permute_rows(dx.p, int64_t(W) * 8, 0, int64_t(W) * 8, dperm.p, valid, dg.p, int64_t(W) * 8, nullptr));
    gathered = dg.download(std::size_t(valid) * W);
  }
  out.records.resize(valid);
  out.expert_of.assign(eof.begin(), eof.begin() + valid);
  for (int64_t r = 0; r < valid; ++r) {
    const TokenRecord& src = tokens[perm[r]];
    out.records[r].token_id = src.token_id;
    out.records[r].source_card = src.source_card;
    out.records[r].source_position = src.source_position;
    if (rect && W > 0) out.records[r].payload.assign(gathered.begin() + r * W, gathered.begin() + (r + 1) * W);
    else out.records[r].payload = src.payload;
  }
  for (int64_t i = 0; i < T; ++i) {
    auto& inv = out.inverse_map[i];
    for (int s = 0; s < k; ++s)
      if (slot[i * k + s] >= 0) inv.push_back(slot[i * k + s]);
    std::sort(inv.begin(), inv.end());  // ascending expert order
  }
  return out;
}

inline CardBuffers dispatch_monolithic(const std::vector<PermutedBatch>& per_node, const VirtualTopology& topo) {
  return detail::run_dispatch(per_node, topo, MOE_BASELINE, 1, nullptr);
}

inline std::vector<std::int64_t> hidden_shard(const std::vector<std::int64_t>& payload, int rho, int t) {
  if (t < 1 || rho < 0 || rho >= t) throw std::invalid_argument("hidden_shard: rank out of range");
  if (payload.size() % std::size_t(t) != 0)
    throw std::invalid_argument("hidden_shard: tensor group must evenly split the payload");
  const std::size_t w = payload.size() / std::size_t(t);
  return std::vector<std::int64_t>(payload.begin() + std::ptrdiff_t(rho * w), payload.begin() + std::ptrdiff_t((rho + 1) * w));
}

inline CardBuffers dispatch_chunked(const std::vector<PermutedBatch>& per_node, const VirtualTopology& topo,
                                    StrategyLevel level, int n, ChunkedDispatchTrace* trace = nullptr) {
  if (level != StrategyLevel::O1 && level != StrategyLevel::O2 && level != StrategyLevel::O3)
    throw std::invalid_argument("dispatch_chunked: level must be O1, O2 or O3");
  if (n < 1) throw std::invalid_argument("dispatch_chunked: n must be >= 1");
  if (level == StrategyLevel::O1 && n != 1) throw std::invalid_argument("dispatch_chunked: O1 is unchunked (n = 1)");
  if (int(per_node.size()) != topo.e) throw std::invalid_argument("dispatch_chunked: need one batch per node");
  int width = -1;
  for (const auto& b : per_node) {
    if (b.batch_tokens % n != 0) throw std::invalid_argument("dispatch_chunked: n does not divide the sequence");
    for (const auto& r : b.records) {
      if (width < 0) width = int(r.payload.size());
      if (int(r.payload.size()) != width) throw std::invalid_argument("dispatch_chunked: ragged payloads");
    }
  }
  if (width < 0) width = 0;
  if (width % topo.t != 0) throw std::invalid_argument("dispatch_chunked: tensor group must evenly split the payload");
  ChunkedDispatchTrace local;
  CardBuffers out = detail::run_dispatch(per_node, topo, moe_level(int(level)), n, &local);
  if (trace) *trace = std::move(local);
  return out;
}

inline std::vector<std::vector<CombinedToken>> combine_unpermute(const CardBuffers& expert_outputs,
                                                                 const std::vector<RoutingDecision>& routing,
                                                                 const std::vector<PermutedBatch>& permuted,
                                                                 const VirtualTopology& topo) {
  if (int(expert_outputs.size()) != topo.cards()) throw std::invalid_argument("combine_unpermute: need one buffer per card");
  if (int(routing.size()) != topo.e || int(permuted.size()) != topo.e)
    throw std::invalid_argument("combine_unpermute: need routing and batches per node");
  for (int g = 0; g < topo.e; ++g) {
    if (int(routing[g].per_token.size()) != permuted[g].batch_tokens)
      throw std::invalid_argument("combine_unpermute: routing does not cover the batch");
    for (int i = 0; i < permuted[g].batch_tokens; ++i) {
      const auto& inv = permuted[g].inverse_map[i];
      if (inv.empty() || inv.size() != routing[g].per_token[i].experts.size())
        throw CorruptRoutingError("combine_unpermute: inverse map does not match routing");
    }
  }
  // the expert outputs' width (the reference only requires a token's slots
  // to agree, dataplane.hpp:335-338); rows move as one dense [rows, W]
  // tensor, so every output row must share it (documented deviation)
  int out_w = -1;
  for (int x = 0; x < topo.e && out_w < 0; ++x)
    for (const auto& rec : expert_outputs[topo.canonical_card(x)]) {
      out_w = int(rec.payload.size());
      break;
    }
  detail::Layer L;
  detail::build_layer(L, permuted, topo, 1, &routing, out_w > 0 ? out_w : 0);
  // the index and plan of this layer; then the expert outputs replace the
  // dispatched rows (located by their tags, like the reference's lookup)
  detail::check(moe_ctx_dispatch(L.ctx, MOE_BASELINE, 1, MOE_LAND_FINAL, nullptr));
  detail::check(moe_ctx_sync(L.ctx));
  const int h = L.W > 0 ? L.W : 1;
  for (int x = 0; x < topo.e; ++x) {
    const int card = topo.canonical_card(x);
    int64_t rows = 0;
    detail::check(moe_ctx_recv_rows(L.ctx, card, &rows));
    moe_card_view v{};
    detail::check(moe_ctx_card_view(L.ctx, card, &v));
    std::vector<int32_t> tags(std::size_t(rows) * 4);
    detail::to_host(tags.data(), v.recv_tags, tags.size() * 4);
    std::map<std::pair<int, int>, const TokenRecord*> where;
    for (const auto& rec : expert_outputs[card]) where[{rec.source_card, rec.source_position}] = &rec;
    std::vector<std::int64_t> y(std::size_t(rows) * h, 0);
    for (int64_t r = 0; r < rows; ++r) {
      const auto it = where.find({tags[r * 4 + 1], tags[r * 4 + 2]});
      if (it == where.end())
        throw CorruptRoutingError("combine_unpermute: missing expert output for node " +
                                  std::to_string(tags[r * 4 + 1] / topo.t) + " position " +
                                  std::to_string(tags[r * 4 + 2]) + " expert " + std::to_string(x));
      if (int(it->second->payload.size()) != L.W) throw CorruptRoutingError("combine_unpermute: payload width mismatch");
      std::copy(it->second->payload.begin(), it->second->payload.end(), y.begin() + r * h);
    }
    detail::to_device(v.recv, y.data(), y.size() * 8);
  }
  detail::check(moe_ctx_combine(L.ctx, MOE_BASELINE, 1, nullptr));
  detail::check(moe_ctx_sync(L.ctx));
  std::vector<std::vector<CombinedToken>> result(topo.e);
  for (int g = 0; g < topo.e; ++g) {
    moe_card_view v{};
    detail::check(moe_ctx_card_view(L.ctx, topo.canonical_card(g), &v));
    std::vector<double> out(std::size_t(L.T) * h);
    detail::to_host(out.data(), v.out, out.size() * 8);
    result[g].resize(L.T);
    for (int i = 0; i < L.T; ++i) {
      result[g][i].token_id = permuted[g].records[permuted[g].inverse_map[i].front()].token_id;
      result[g][i].payload.assign(out.begin() + std::ptrdiff_t(i) * h, out.begin() + std::ptrdiff_t(i) * h + L.W);
    }
  }
  return result;
}

}  // namespace moeplan::dataplane

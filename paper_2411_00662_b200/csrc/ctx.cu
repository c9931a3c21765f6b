// Layer context: per-card HBM layout, NVLink peer mappings, prioritised
// streams, the cross-GPU flag protocol, and the orchestration of
//   dispatch = index build -> count exchange -> plan -> per chunk
//              { AA (+fused permute) ; AG ; D2D }            (dataplane.hpp:187-283)
//   combine  = per chunk { reverse AA ; un-permute (+fused output AG) } (dataplane.hpp:293-347)
//
// Stream roles follow the reference simulator (pipesim.hpp:58-83, Fig. 14 of
// the paper): the AllToAll legs run on a high-priority stream, the AllGather
// legs on a second stream, the reorder copies on the AllGather stream (O2) or
// a third stream (O3).  Cross-GPU ordering uses epoch flags written over
// NVLink (common.cuh); cross-stream ordering on one GPU uses CUDA events.
//
// In virtual mode (world_size == 1) every card lives on one device and the
// phases run in lockstep on the caller's stream — no card ever waits on
// another card's kernel, so nothing spins.
#include <algorithm>
#include <cstdlib>
#include <string>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "engine.cuh"

namespace monta {

namespace {

constexpr size_t kAlign = 256;
inline size_t align_up(size_t v) { return (v + kAlign - 1) / kAlign * kAlign; }

constexpr int kMaxTune = 32;  // autotune candidates per call

struct PeerPtrs {
  char* slab = nullptr;
  char* recv = nullptr;
  int32_t* recv_tags = nullptr;
  char* pre = nullptr;
  int32_t* pre_tags = nullptr;
  char* comb = nullptr;
  char* out = nullptr;
  uint64_t* count_table = nullptr;  // [e][max_chunks][E] of {count | epoch << 32}
  uint64_t* flags = nullptr;
  int32_t* experts = nullptr;       // routing (layer backward reads it by row tag)
  void* probs = nullptr;
  void* parts = nullptr;            // [T][k][t] grad-prob partials (layer backward)
  float* wscale = nullptr;          // [recv_cap][h / 128] fp8 wire scales
  char* cwire = nullptr;            // [R][h] fp8 combine leg rows
  float* cscale = nullptr;          // [R][h / 128]
  char* stage = nullptr;            // node dedup: [e][T] staged rows, block g from sender node g
  int32_t* sdesc = nullptr;         //             [e][T][2 + 2k] their descriptors
  uint32_t* scount = nullptr;       //             [kMaxCards] rows this card staged to each card
};

// Byte offsets of every buffer inside a card's slab.  Identical on every
// rank, so an IPC-mapped peer slab is addressed with the same offsets.
struct SlabLayout {
  size_t x, logits, token_ids, experts, probs, perm_src, expert_of, slot_pos, counts, offsets;
  size_t permuted, recv, recv_tags, pre, pre_tags, comb, out, count_table, flags, err, done;
  size_t lists, local_delta, recv_rows, recv_offs, tune, prow, rowpos, rowslot, dot, parts, gprobs, glogits, ones,
      wscale, cwire, cscale, scratch, epoch, front_done, dbg, tile_hist, tile_base, counts_acc, arrive,
      ready, xchg_counters, xchg_flags, xtrace, aa_table, rowdst, stage, sdesc, scount, nslot, bcnt, total;
};

struct Card {
  int id = 0, node = 0, rho = 0;
  char* slab = nullptr;
  moe_card_view v{};
  uint64_t* count_table = nullptr;
  uint64_t* flags = nullptr;
  int32_t* err = nullptr;
  unsigned* done = nullptr;
  SegList* lists = nullptr;
  int32_t* local_delta = nullptr;
  int64_t* recv_rows = nullptr;
  int32_t* scratch = nullptr;
  uint64_t* epoch_dev = nullptr;   // bumped by the front kernel once per dispatch
  unsigned long long* dbg = nullptr;  // front-kernel phase timestamps (debug)
  int32_t* tile_hist = nullptr;       // [n_tiles][E]
  int32_t* tile_base = nullptr;       // [n_tiles][E]
  int32_t* counts_acc = nullptr;      // [2][max_chunks][E] (epoch parity)
  unsigned* arrive = nullptr;         // front grid barrier
  unsigned long long* ready = nullptr;
  unsigned* xchg_counters = nullptr;  // [4][max_chunks] persistent-exchange chunk counters
  uint64_t* xchg_flags = nullptr;     // [max_chunks] own-node chunk completion
  unsigned long long* xtrace = nullptr;  // [2 kernels][4 roles][max_chunks][2] role trace (ns)
  int32_t* aa_table = nullptr;        // [4 + max_chunks][E] token-side AA destinations
  char** rowdst = nullptr;            // [recv_cap] reverse-AllToAll row address (peer comb) or null
  int32_t* nslot = nullptr;           // node dedup: [T][e] staging slot of (token, remote node), -1 none
  int32_t* bcnt = nullptr;            //             [e][ceil(T / 1024)] per-block counts
  unsigned* front_done = nullptr;  // CTA election counter of the front kernel
  // layer backward scratch (moe_ctx_backward)
  void* prow = nullptr;
  int32_t* rowpos = nullptr;
  int32_t* rowslot = nullptr;
  void* dot = nullptr;
  void* parts = nullptr;
  void* ones = nullptr;
  // bound expert FFN (moe_ctx_bind_experts)
  const void* w13 = nullptr;
  const void* w2 = nullptr;
  int64_t ffn = 0;
  void* ffn_ws = nullptr;             // [recv_cap, ffn] bf16
  size_t ffn_ws_bytes = 0;
};

struct Span {
  int stage, chunk;
  cudaEvent_t a, b;
};

}  // namespace
}  // namespace monta

struct moe_ctx {
  moe_layer_desc d{};
  int L = 1, cards = 1, device = 0, rank = 0, world = 1, sms = 148;
  size_t xb = 0, lb = 0, ob = 0;  // element bytes of payload / logits / out
  int64_t R = 0, recv_cap = 0, row_bytes = 0;
  int n_flag_sigs = 0;
  monta::SlabLayout lay{};
  std::vector<monta::Card> local;
  monta::PeerPtrs peer[monta::kMaxCards];
  std::vector<void*> opened;
  cudaStream_t s_aa = nullptr, s_ag = nullptr, s_d2d = nullptr, s_cap = nullptr;
  // forward_host on a multi-GPU rank: host copies pipelined per token chunk
  cudaStream_t s_h2d = nullptr, s_d2h = nullptr;
  std::vector<cudaEvent_t> ev_h2d, ev_d2h;
  cudaEvent_t ev_join_d2h = nullptr;
  bool pipe = false;       // set by forward_impl for one call: AA(j) waits H2D(j), D2H(j) follows un-permute(j)
  char* pipe_ho = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join_aa = nullptr, ev_join_ag = nullptr, ev_join_d2d = nullptr;
  std::vector<cudaEvent_t> ev_aa, ev_ag;
  bool expert_fused = true;  // moe_ctx_set_expert_overlap: down-projection epilogue issues the reverse AllToAll
  bool node_dedup_now = false;  // set by dispatch_node_dedup for its launch_aa
  int node_dedup = 2;           // moe_ctx_set_node_dedup: 0 off, 1 on, 2 auto (top_k >= 2 e)
  int aa_ctas = 0;
  bool combine_ready = false;  // a dispatch whose combine has not run yet
  bool debug = false;          // record front-kernel phase timestamps
  bool use_graphs = false;
  bool use_xchg = true;  // persistent role-specialised exchange kernels (multi-GPU)
  uint64_t tune_epoch = 0;
  bool checks = false;  // poison + verify the landed rows' tags every dispatch (moe_ctx_enable_checks)
  bool unit_probs = false;  // combine with unit weights (the layer backward's dispatch adjoint)
  int wire = MOE_WIRE_BF16;  // cross-node dispatch payload format (moe_ctx_set_wire)
  uint32_t pace_bpus = 0;     // emulated inter-node link rate, bytes/us (moe_ctx_set_link_rate)
  struct GraphEntry {
    int kind;  // 0 forward, 1 layer backward (moe_ctx_backward)
    int level, n, landing;
    const void *hx, *hl;
    void* ho;
    cudaGraphExec_t exec;
    int64_t kernels;  // this context's kernels inside the graph
    bool timed;       // captured with timing events (spans of the replay)
    std::vector<std::pair<int, int>> span_labels;  // (stage, chunk) of c->spans[0..)
  };
  std::vector<GraphEntry> graphs;
  bool connected = false;
  // last dispatch (the combine replays its plan)
  int last_level = -1, last_n = 0, last_landing = 0;
  bool timing = false;
  bool in_forward = false;
  cudaEvent_t ev_base = nullptr;
  std::vector<monta::Span> spans;
  size_t span_used = 0;
  int64_t launches = 0;
  monta::SegList* xfer_list = nullptr;       // device
  monta::SegList* xfer_host = nullptr;       // pinned staging
};

namespace monta {
namespace {

bool is_virtual(const moe_ctx* c) { return c->world == 1; }

SlabLayout make_layout(const moe_ctx* c) {
  const moe_layer_desc& d = c->d;
  SlabLayout s{};
  size_t off = 0;
  auto take = [&](size_t bytes) {
    const size_t at = off;
    off = align_up(off + std::max<size_t>(bytes, 1));
    return at;
  };
  const int64_t T = d.tokens, h = d.hidden, E = d.num_experts, k = d.top_k;
  s.x = take(size_t(T) * h * c->xb);
  s.logits = take(size_t(T) * E * c->lb);
  s.token_ids = take(size_t(T) * 4);
  s.experts = take(size_t(T) * k * 4);
  s.probs = take(size_t(T) * k * c->lb);
  s.perm_src = take(size_t(c->R) * 4);
  s.expert_of = take(size_t(c->R) * 4);
  s.slot_pos = take(size_t(T) * k * 4);
  s.counts = take(size_t(d.max_chunks) * E * 4);
  s.offsets = take(size_t(E + 1) * 4);
  s.permuted = take(size_t(c->R) * c->row_bytes);
  s.recv = take(size_t(c->recv_cap) * c->row_bytes);
  s.recv_tags = take(size_t(c->recv_cap) * 16);
  s.pre = take(size_t(c->recv_cap) * c->row_bytes);
  s.pre_tags = take(size_t(c->recv_cap) * 16);
  s.comb = take(size_t(c->R) * c->row_bytes);
  s.out = take(size_t(T) * h * c->ob);
  s.count_table = take(size_t(d.e) * d.max_chunks * E * 8);
  s.flags = take(size_t(c->n_flag_sigs) * kMaxCards * 8);
  s.err = take(16);
  s.done = take(size_t(kNumPhaseSignals * d.max_chunks + 8) * 4);
  s.lists = take(size_t(kNumPhases) * d.max_chunks * seglist_bytes(int(E)));
  s.local_delta = take(size_t(E) * 4);
  s.recv_rows = take(8);
  s.recv_offs = take(size_t(c->L + 1) * 4);
  s.tune = take(size_t(kMaxCards) * kMaxTune * 8);  // [sender][candidate] us (autotune)
  // layer backward (moe_ctx_backward): per landed row weight / position / slot / partial dot,
  // the grad-prob partials [T][k][t], grad_probs [T, k], grad_logits [T, E], unit weights [T, k]
  s.prow = take(size_t(c->recv_cap) * c->lb);
  s.rowpos = take(size_t(c->recv_cap) * 4);
  s.rowslot = take(size_t(c->recv_cap) * 4);
  s.dot = take(size_t(c->recv_cap) * c->lb);
  s.parts = take(size_t(T) * k * d.t * c->lb);
  s.gprobs = take(size_t(T) * k * c->lb);
  s.glogits = take(size_t(T) * E * c->lb);
  s.ones = take(size_t(T) * k * c->lb);
  s.wscale = take(size_t(c->recv_cap) * std::max<int64_t>(1, h / 128) * 4);  // fp8 wire scales
  s.cwire = take(size_t(c->R) * size_t(h));                              // fp8 combine leg: e4m3 rows
  s.cscale = take(size_t(c->R) * std::max<int64_t>(1, h / 128) * 4);     //   and their scales
  s.scratch = take(plan_scratch_ints(d.e, int(E), d.max_chunks) * 4);
  s.epoch = take(8);
  s.front_done = take(16);
  s.dbg = take(256);
  const int64_t tiles = (T + front_router_tokens(int(E)) - 1) / front_router_tokens(int(E));
  s.tile_hist = take(size_t(tiles) * E * 4);
  s.tile_base = take(size_t(tiles) * E * 4);
  s.counts_acc = take(size_t(2) * d.max_chunks * E * 4);
  s.arrive = take(16);
  s.ready = take(16);
  s.xchg_counters = take(size_t(8) * d.max_chunks * 17 * 4);  // [dispatch 4 + combine 2 legs][chunk][1 + 16 groups]
  s.xchg_flags = take(size_t(d.max_chunks) * 8);
  s.xtrace = take(size_t(2) * 4 * d.max_chunks * 2 * 8);
  s.aa_table = take(size_t(4 + d.max_chunks) * E * 4);
  s.rowdst = take(size_t(c->recv_cap) * 8);  // fused combine: each landed row's reverse-AllToAll destination
  // node dedup: a token's row (slice under TP) crosses to a remote node once
  const bool nd = d.e > 1 && c->world > 1;
  s.stage = take(nd ? size_t(d.e) * T * c->row_bytes : 0);
  s.sdesc = take(nd ? size_t(d.e) * T * (2 + 2 * k) * 4 : 0);
  s.scount = take(size_t(kMaxCards) * 4);
  s.nslot = take(nd ? size_t(T) * d.e * 4 : 0);
  s.bcnt = take(nd ? size_t(d.e) * ((T + 1023) / 1024) * 4 : 0);
  s.total = off;
  return s;
}

void bind_card(moe_ctx* c, Card& cd) {
  const SlabLayout& s = c->lay;
  char* b = cd.slab;
  moe_card_view& v = cd.v;
  v.x = b + s.x;
  v.logits = b + s.logits;
  v.token_ids = reinterpret_cast<int32_t*>(b + s.token_ids);
  v.experts = reinterpret_cast<int32_t*>(b + s.experts);
  v.probs = b + s.probs;
  v.perm_src = reinterpret_cast<int32_t*>(b + s.perm_src);
  v.expert_of = reinterpret_cast<int32_t*>(b + s.expert_of);
  v.slot_pos = reinterpret_cast<int32_t*>(b + s.slot_pos);
  v.counts = reinterpret_cast<int32_t*>(b + s.counts);
  v.expert_offsets = reinterpret_cast<int32_t*>(b + s.offsets);
  v.permuted = b + s.permuted;
  v.recv = b + s.recv;
  v.recv_tags = reinterpret_cast<int32_t*>(b + s.recv_tags);
  v.pre = b + s.pre;
  v.pre_tags = reinterpret_cast<int32_t*>(b + s.pre_tags);
  v.expert_out = v.recv;
  v.comb = b + s.comb;
  v.out = b + s.out;
  v.rows_permuted = c->R;
  v.recv_cap = c->recv_cap;
  v.recv_expert_offsets = reinterpret_cast<int32_t*>(b + s.recv_offs);
  v.grad_probs = b + s.gprobs;
  v.grad_logits = b + s.glogits;
  cd.count_table = reinterpret_cast<uint64_t*>(b + s.count_table);
  cd.flags = reinterpret_cast<uint64_t*>(b + s.flags);
  cd.err = reinterpret_cast<int32_t*>(b + s.err);
  cd.done = reinterpret_cast<unsigned*>(b + s.done);
  cd.lists = reinterpret_cast<SegList*>(b + s.lists);
  cd.local_delta = reinterpret_cast<int32_t*>(b + s.local_delta);
  cd.recv_rows = reinterpret_cast<int64_t*>(b + s.recv_rows);
  cd.scratch = reinterpret_cast<int32_t*>(b + s.scratch);
  cd.epoch_dev = reinterpret_cast<uint64_t*>(b + s.epoch);
  cd.front_done = reinterpret_cast<unsigned*>(b + s.front_done);
  cd.dbg = reinterpret_cast<unsigned long long*>(b + s.dbg);
  cd.tile_hist = reinterpret_cast<int32_t*>(b + s.tile_hist);
  cd.tile_base = reinterpret_cast<int32_t*>(b + s.tile_base);
  cd.counts_acc = reinterpret_cast<int32_t*>(b + s.counts_acc);
  cd.prow = b + s.prow;
  cd.rowpos = reinterpret_cast<int32_t*>(b + s.rowpos);
  cd.rowslot = reinterpret_cast<int32_t*>(b + s.rowslot);
  cd.dot = b + s.dot;
  cd.parts = b + s.parts;
  cd.ones = b + s.ones;
  cd.arrive = reinterpret_cast<unsigned*>(b + s.arrive);
  cd.ready = reinterpret_cast<unsigned long long*>(b + s.ready);
  cd.xchg_counters = reinterpret_cast<unsigned*>(b + s.xchg_counters);
  cd.xchg_flags = reinterpret_cast<uint64_t*>(b + s.xchg_flags);
  cd.xtrace = reinterpret_cast<unsigned long long*>(b + s.xtrace);
  cd.aa_table = reinterpret_cast<int32_t*>(b + s.aa_table);
  cd.rowdst = reinterpret_cast<char**>(b + s.rowdst);
  cd.nslot = reinterpret_cast<int32_t*>(b + s.nslot);
  cd.bcnt = reinterpret_cast<int32_t*>(b + s.bcnt);
}

void set_peer(moe_ctx* c, int card, char* slab) {
  const SlabLayout& s = c->lay;
  PeerPtrs& p = c->peer[card];
  p.slab = slab;
  p.recv = slab + s.recv;
  p.recv_tags = reinterpret_cast<int32_t*>(slab + s.recv_tags);
  p.pre = slab + s.pre;
  p.pre_tags = reinterpret_cast<int32_t*>(slab + s.pre_tags);
  p.comb = slab + s.comb;
  p.out = slab + s.out;
  p.count_table = reinterpret_cast<uint64_t*>(slab + s.count_table);
  p.flags = reinterpret_cast<uint64_t*>(slab + s.flags);
  p.experts = reinterpret_cast<int32_t*>(slab + s.experts);
  p.probs = slab + s.probs;
  p.parts = slab + s.parts;
  p.wscale = reinterpret_cast<float*>(slab + s.wscale);
  p.cwire = slab + s.cwire;
  p.cscale = reinterpret_cast<float*>(slab + s.cscale);
  p.stage = slab + s.stage;
  p.sdesc = reinterpret_cast<int32_t*>(slab + s.sdesc);
  p.scount = reinterpret_cast<uint32_t*>(slab + s.scount);
}

inline int card_of(const moe_ctx* c, int node, int rho) { return node * c->d.t + rho; }
inline int sig_chunk(const moe_ctx* c, int ps, int j) { return kSigChunkBase + ps * c->d.max_chunks + j; }
inline int sig_tune(const moe_ctx* c) { return c->n_flag_sigs - 2; }
inline int sig_bwd(const moe_ctx* c) { return c->n_flag_sigs - 1; }

// Flag word on `owner` that `sender` writes for signal `sig`.
inline uint64_t* flag_at(moe_ctx* c, int owner, int sig, int sender) {
  return c->peer[owner].flags + size_t(sig) * kMaxCards + sender;
}

SegList* list_of(const moe_ctx* c, const Card& cd, int phase, int j) {
  char* base = reinterpret_cast<char*>(cd.lists);
  return reinterpret_cast<SegList*>(base + (size_t(phase) * c->d.max_chunks + j) *
                                               seglist_bytes(c->d.num_experts));
}

// ---- timing -------------------------------------------------------------
// Timing events are recorded as external event nodes when the stream is being
// captured, so a replayed graph reports the same per-kernel spans.
void record_timing(cudaEvent_t ev, cudaStream_t s) {
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  cudaStreamIsCapturing(s, &cs);
  if (cs == cudaStreamCaptureStatusActive) cudaEventRecordWithFlags(ev, s, cudaEventRecordExternal);
  else cudaEventRecord(ev, s);
}
void span_begin(moe_ctx* c, int stage, int chunk, cudaStream_t s, size_t* slot) {
  *slot = SIZE_MAX;
  if (!c->timing) return;
  if (c->span_used == c->spans.size()) {
    Span sp{stage, chunk, nullptr, nullptr};
    cudaEventCreate(&sp.a);
    cudaEventCreate(&sp.b);
    c->spans.push_back(sp);
  }
  Span& sp = c->spans[c->span_used];
  sp.stage = stage;
  sp.chunk = chunk;
  record_timing(sp.a, s);
  *slot = c->span_used++;
}
void span_end(moe_ctx* c, size_t slot, cudaStream_t s) {
  if (slot == SIZE_MAX) return;
  record_timing(c->spans[slot].b, s);
}

int copy_grid(const moe_ctx* c, bool concurrent, bool aa) {
  int g = c->sms * (concurrent ? 2 : 4);
  if (aa && c->aa_ctas > 0) g = std::min(g, c->aa_ctas);
  return g;
}

WaitList no_wait() {
  WaitList w{};
  w.n = 0;
  w.epoch = 0;
  return w;
}
SignalList no_signal() {
  SignalList s{};
  s.n = 0;
  return s;
}

}  // namespace

// ===========================================================================
// creation / teardown
// ===========================================================================
static moe_status validate_desc(const moe_layer_desc* d) {
  if (!d) return fail(MOE_ERR_INVALID_ARGUMENT, "ctx_create: null descriptor");
  if (d->e < 1 || d->t < 1) return fail(MOE_ERR_INVALID_ARGUMENT, "ctx_create: e and t must be >= 1");
  if (d->e * d->t > kMaxCards)
    return fail(MOE_ERR_UNSUPPORTED, "ctx_create: at most %d cards", kMaxCards);
  if (d->num_experts < 1 || d->num_experts % d->e != 0)
    return fail(MOE_ERR_INVALID_ARGUMENT, "ctx_create: E must be a positive multiple of e");
  if (d->top_k < 1 || d->top_k > d->num_experts)
    return fail(MOE_ERR_INVALID_ARGUMENT, "ctx_create: need 1 <= k <= E");
  if (d->tokens < 0 || d->hidden < 1)
    return fail(MOE_ERR_INVALID_ARGUMENT, "ctx_create: bad token/hidden sizes");
  if (dtype_size(d->dtype) == 0 || dtype_size(d->out_dtype) == 0)
    return fail(MOE_ERR_INVALID_ARGUMENT, "ctx_create: bad dtype");
  if (d->logit_dtype != MOE_F32 && d->logit_dtype != MOE_F64)
    return fail(MOE_ERR_INVALID_ARGUMENT, "ctx_create: logits must be f32 or f64");
  if (d->max_chunks < 1) return fail(MOE_ERR_INVALID_ARGUMENT, "ctx_create: max_chunks >= 1");
  return MOE_OK;
}

}  // namespace monta

using namespace monta;

extern "C" moe_status moe_ctx_create(const moe_layer_desc* desc, int device, int rank,
                                     int world_size, moe_ctx** out) {
  if (!out) return fail(MOE_ERR_INVALID_ARGUMENT, "ctx_create: null out");
  *out = nullptr;
  if (moe_status st = validate_desc(desc)) return st;
  const int cards = desc->e * desc->t;
  if (!(world_size == 1 || world_size == cards))
    return fail(MOE_ERR_UNSUPPORTED, "ctx_create: world_size must be 1 or e*t (%d), got %d", cards,
                world_size);
  if (rank < 0 || rank >= world_size) return fail(MOE_ERR_INVALID_ARGUMENT, "ctx_create: bad rank");
  MONTA_CUDA(cudaSetDevice(device));
  moe_ctx* c = new moe_ctx();
  c->d = *desc;
  c->L = desc->num_experts / desc->e;
  c->cards = cards;
  c->device = device;
  c->rank = rank;
  c->world = world_size;
  cudaDeviceGetAttribute(&c->sms, cudaDevAttrMultiProcessorCount, device);
  c->xb = dtype_size(desc->dtype);
  c->lb = dtype_size(desc->logit_dtype);
  c->ob = dtype_size(desc->out_dtype);
  c->R = desc->tokens * desc->top_k;
  c->row_bytes = desc->hidden * int64_t(c->xb);
  c->recv_cap = int64_t(desc->e) * desc->tokens * std::min<int64_t>(desc->top_k, c->L);
  c->n_flag_sigs = kSigChunkBase + kNumPhaseSignals * desc->max_chunks + 2;  // + autotune, layer-backward signals
  c->lay = make_layout(c);
  const int first = world_size == 1 ? 0 : rank;
  const int nlocal = world_size == 1 ? cards : 1;
  for (int i = 0; i < nlocal; ++i) {
    Card cd;
    cd.id = first + i;
    cd.node = cd.id / desc->t;
    cd.rho = cd.id % desc->t;
    cudaError_t err = cudaMalloc(&cd.slab, c->lay.total);
    if (err != cudaSuccess) {
      for (auto& o : c->local) cudaFree(o.slab);
      delete c;
      return cuda_fail(err, "ctx_create: slab allocation");
    }
    cudaMemset(cd.slab, 0, c->lay.total);
    bind_card(c, cd);
    launch_fill_ones(desc->logit_dtype, cd.ones, desc->tokens * desc->top_k, nullptr);
    c->local.push_back(cd);
    set_peer(c, cd.id, cd.slab);
  }
  // default token ids: i + node * 100000 (dataplane::make_batch, dataplane.hpp:48-57)
  {
    std::vector<int32_t> ids(size_t(desc->tokens));
    for (auto& cd : c->local) {
      for (int64_t i = 0; i < desc->tokens; ++i) ids[size_t(i)] = int32_t(i + cd.node * 100000);
      if (desc->tokens > 0)
        cudaMemcpy(cd.v.token_ids, ids.data(), ids.size() * 4, cudaMemcpyHostToDevice);
    }
  }
  int lo = 0, hi = 0;
  cudaDeviceGetStreamPriorityRange(&lo, &hi);  // hi is the numerically smallest (highest) priority
  // the AllToAll legs are EP traffic: the top of the EP > PP > CP > DP order
  // (monta.h 1d), above any PP/CP/DP stream a caller makes with moe_comm_stream_create
  moe_comm_stream_priority(MOE_COMM_EP, device, &hi);
  cudaStreamCreateWithPriority(&c->s_aa, cudaStreamNonBlocking, hi);
  cudaStreamCreateWithPriority(&c->s_ag, cudaStreamNonBlocking, lo);
  cudaStreamCreateWithPriority(&c->s_d2d, cudaStreamNonBlocking, lo);
  cudaStreamCreateWithFlags(&c->s_cap, cudaStreamNonBlocking);
  cudaStreamCreateWithFlags(&c->s_h2d, cudaStreamNonBlocking);
  cudaStreamCreateWithFlags(&c->s_d2h, cudaStreamNonBlocking);
  if (moe_status st = configure_front(desc->num_experts, desc->logit_dtype)) {
    moe_ctx_destroy(c);
    return st;
  }
  cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming);
  cudaEventCreateWithFlags(&c->ev_join_aa, cudaEventDisableTiming);
  cudaEventCreateWithFlags(&c->ev_join_ag, cudaEventDisableTiming);
  cudaEventCreateWithFlags(&c->ev_join_d2d, cudaEventDisableTiming);
  c->ev_aa.resize(size_t(desc->max_chunks));
  c->ev_ag.resize(size_t(desc->max_chunks));
  for (int j = 0; j < desc->max_chunks; ++j) {
    cudaEventCreateWithFlags(&c->ev_aa[j], cudaEventDisableTiming);
    cudaEventCreateWithFlags(&c->ev_ag[j], cudaEventDisableTiming);
  }
  c->ev_h2d.resize(size_t(desc->max_chunks));
  c->ev_d2h.resize(size_t(desc->max_chunks));
  for (int j = 0; j < desc->max_chunks; ++j) {
    cudaEventCreateWithFlags(&c->ev_h2d[j], cudaEventDisableTiming);
    cudaEventCreateWithFlags(&c->ev_d2h[j], cudaEventDisableTiming);
  }
  cudaEventCreateWithFlags(&c->ev_join_d2h, cudaEventDisableTiming);
  cudaEventCreate(&c->ev_base);
  cudaError_t err = cudaDeviceSynchronize();
  if (err != cudaSuccess) {
    moe_ctx_destroy(c);
    return cuda_fail(err, "ctx_create");
  }
  c->connected = world_size == 1;
  *out = c;
  return MOE_OK;
}

extern "C" moe_status moe_ctx_destroy(moe_ctx* c) {
  if (!c) return MOE_OK;
  cudaSetDevice(c->device);
  cudaDeviceSynchronize();
  for (void* p : c->opened) cudaIpcCloseMemHandle(p);
  if (c->xfer_list) cudaFree(c->xfer_list);
  if (c->xfer_host) cudaFreeHost(c->xfer_host);
  for (auto& cd : c->local) {
    cudaFree(cd.slab);
    if (cd.ffn_ws) cudaFree(cd.ffn_ws);
  }
  for (auto& sp : c->spans) {
    cudaEventDestroy(sp.a);
    cudaEventDestroy(sp.b);
  }
  for (auto ev : c->ev_aa) cudaEventDestroy(ev);
  for (auto ev : c->ev_ag) cudaEventDestroy(ev);
  if (c->ev_base) cudaEventDestroy(c->ev_base);
  if (c->ev_fork) cudaEventDestroy(c->ev_fork);
  if (c->ev_join_aa) cudaEventDestroy(c->ev_join_aa);
  if (c->ev_join_ag) cudaEventDestroy(c->ev_join_ag);
  if (c->ev_join_d2d) cudaEventDestroy(c->ev_join_d2d);
  if (c->s_aa) cudaStreamDestroy(c->s_aa);
  if (c->s_ag) cudaStreamDestroy(c->s_ag);
  if (c->s_d2d) cudaStreamDestroy(c->s_d2d);
  if (c->s_cap) cudaStreamDestroy(c->s_cap);
  for (auto ev : c->ev_h2d) cudaEventDestroy(ev);
  for (auto ev : c->ev_d2h) cudaEventDestroy(ev);
  if (c->ev_join_d2h) cudaEventDestroy(c->ev_join_d2h);
  if (c->s_h2d) cudaStreamDestroy(c->s_h2d);
  if (c->s_d2h) cudaStreamDestroy(c->s_d2h);
  for (auto& g : c->graphs)
    if (g.exec) cudaGraphExecDestroy(g.exec);
  delete c;
  return MOE_OK;
}

extern "C" moe_status moe_ctx_card_view(moe_ctx* c, int card, moe_card_view* out) {
  if (!c || !out) return fail(MOE_ERR_INVALID_ARGUMENT, "card_view: null argument");
  for (auto& cd : c->local)
    if (cd.id == card) {
      *out = cd.v;
      return MOE_OK;
    }
  return fail(MOE_ERR_INVALID_ARGUMENT, "card_view: card %d is not local to this context", card);
}

extern "C" int moe_ctx_num_local_cards(const moe_ctx* c) { return c ? int(c->local.size()) : 0; }
extern "C" int moe_ctx_first_card(const moe_ctx* c) { return c && !c->local.empty() ? c->local[0].id : -1; }

extern "C" moe_status moe_ctx_bind_experts(moe_ctx* c, int card, const void* w13, const void* w2, int64_t ffn) {
  if (!c) return fail(MOE_ERR_INVALID_ARGUMENT, "bind_experts: null ctx");
  for (auto& cd : c->local) {
    if (cd.id != card) continue;
    MONTA_CUDA(cudaSetDevice(c->device));
    // a captured graph holds the old expert launches (or none): drop them
    for (auto& g : c->graphs)
      if (g.exec) cudaGraphExecDestroy(g.exec);
    c->graphs.clear();
    if (!w13) {
      cd.w13 = cd.w2 = nullptr;
      cd.ffn = 0;
      return MOE_OK;
    }
    if (!w2) return fail(MOE_ERR_INVALID_ARGUMENT, "bind_experts: null w2");
    if (c->d.dtype != MOE_BF16) return fail(MOE_ERR_INVALID_ARGUMENT, "bind_experts: experts need a bf16 payload");
    if (c->d.hidden % 128)
      return fail(MOE_ERR_INVALID_ARGUMENT, "bind_experts: hidden must be a multiple of 128");
    if (ffn < MOE_W13_BLOCK || ffn % MOE_W13_BLOCK)
      return fail(MOE_ERR_INVALID_ARGUMENT, "bind_experts: ffn must be a positive multiple of %d", MOE_W13_BLOCK);
    if (moe_status st = configure_grouped_gemm()) return st;
    const size_t need = size_t(std::max<int64_t>(c->recv_cap, 1)) * size_t(ffn) * 2;
    if (need > cd.ffn_ws_bytes) {
      if (cd.ffn_ws) cudaFree(cd.ffn_ws);
      cd.ffn_ws = nullptr;
      cd.ffn_ws_bytes = 0;
      MONTA_CUDA(cudaMalloc(&cd.ffn_ws, need));
      cd.ffn_ws_bytes = need;
    }
    cd.w13 = w13;
    cd.w2 = w2;
    cd.ffn = ffn;
    return MOE_OK;
  }
  return fail(MOE_ERR_INVALID_ARGUMENT, "bind_experts: card %d is not local", card);
}

extern "C" moe_status moe_ctx_bind_expert_out(moe_ctx* c, int card, void* expert_out) {
  if (!c) return fail(MOE_ERR_INVALID_ARGUMENT, "bind_expert_out: null ctx");
  for (auto& cd : c->local)
    if (cd.id == card) {
      cd.v.expert_out = expert_out ? expert_out : cd.v.recv;
      return MOE_OK;
    }
  return fail(MOE_ERR_INVALID_ARGUMENT, "bind_expert_out: card %d is not local", card);
}

// ---- IPC -----------------------------------------------------------------
namespace {
struct IpcBlob {
  uint32_t magic;
  int32_t card;
  uint64_t slab_bytes;
  cudaIpcMemHandle_t handle;
  char pad[128 - 16 - sizeof(cudaIpcMemHandle_t)];
};
static_assert(sizeof(IpcBlob) == 128, "ipc blob");
constexpr uint32_t kMagic = 0x4d4f4e54;  // "MONT"
}  // namespace

extern "C" size_t moe_ctx_ipc_handle_size(void) { return sizeof(IpcBlob); }

extern "C" moe_status moe_ctx_ipc_export(moe_ctx* c, void* blob) {
  if (!c || !blob) return fail(MOE_ERR_INVALID_ARGUMENT, "ipc_export: null argument");
  if (c->local.size() != 1) return fail(MOE_ERR_INVALID_ARGUMENT, "ipc_export: multi-process contexts only");
  MONTA_CUDA(cudaSetDevice(c->device));
  IpcBlob b{};
  b.magic = kMagic;
  b.card = c->local[0].id;
  b.slab_bytes = c->lay.total;
  MONTA_CUDA(cudaIpcGetMemHandle(&b.handle, c->local[0].slab));
  std::memcpy(blob, &b, sizeof(b));
  return MOE_OK;
}

extern "C" moe_status moe_ctx_ipc_connect(moe_ctx* c, const void* all_blobs) {
  if (!c || !all_blobs) return fail(MOE_ERR_INVALID_ARGUMENT, "ipc_connect: null argument");
  if (c->world == 1) return MOE_OK;
  MONTA_CUDA(cudaSetDevice(c->device));
  const IpcBlob* blobs = static_cast<const IpcBlob*>(all_blobs);
  for (int r = 0; r < c->world; ++r) {
    const IpcBlob& b = blobs[r];
    if (b.magic != kMagic || b.card != r || b.slab_bytes != c->lay.total)
      return fail(MOE_ERR_TRANSPORT, "ipc_connect: blob %d does not describe card %d of this layer", r, r);
    if (r == c->rank) continue;
    void* p = nullptr;
    cudaError_t err = cudaIpcOpenMemHandle(&p, b.handle, cudaIpcMemLazyEnablePeerAccess);
    if (err != cudaSuccess) return cuda_fail(err, "ipc_connect: cudaIpcOpenMemHandle");
    c->opened.push_back(p);
    set_peer(c, r, static_cast<char*>(p));
  }
  c->connected = true;
  return MOE_OK;
}

// ===========================================================================
// phases
// ===========================================================================
namespace {

moe_status check_ready(moe_ctx* c) {
  if (!c) return fail(MOE_ERR_INVALID_ARGUMENT, "null context");
  if (!c->connected) return fail(MOE_ERR_TRANSPORT, "context not connected (call moe_ctx_ipc_connect)");
  return MOE_OK;
}

moe_status do_route(moe_ctx* c, cudaStream_t s) {
  for (auto& cd : c->local) {
    size_t sl;
    span_begin(c, MOE_STAGE_ROUTE, 0, s, &sl);
    if (moe_status st = route_topk(cd.v.logits, c->d.logit_dtype, c->d.tokens, c->d.num_experts,
                                   c->d.top_k, cd.v.experts, cd.v.probs, s))
      return st;
    span_end(c, sl, s);
    ++c->launches;
  }
  return MOE_OK;
}

bool xchg_eligible(moe_ctx* c, int level);

bool node_dedup_ok(const moe_ctx* c, int level, int n, int landing);

PlanArgs make_plan_args(moe_ctx* c, Card& cd, int level, int n, int landing) {
  const moe_layer_desc& d = c->d;
  PlanArgs a{};
  a.count_table = cd.count_table;
  a.e = d.e;
  a.t = d.t;
  a.E = d.num_experts;
  a.L = c->L;
  a.n = n;
  a.max_chunks = d.max_chunks;
  a.node = cd.node;
  a.rho = cd.rho;
  a.level = level;
  a.landing = landing;
  a.row_bytes = c->row_bytes;
  a.seg_cap = d.num_experts;
  a.lists = cd.lists;
  a.local_delta = cd.local_delta;
  // the per-expert destination table feeds only the token-side AA kernel
  // (per-launch path and node dedup); the persistent exchange reads the
  // segment lists instead
  a.aa_table = xchg_eligible(c, level) && !node_dedup_ok(c, level, n, landing) ? nullptr : cd.aa_table;
  a.recv_rows = cd.recv_rows;
  a.recv_offs = cd.v.recv_expert_offsets;
  a.err = cd.err;
  a.wait = no_wait();
  a.wait.epoch_ptr = cd.epoch_dev;
  // multi-GPU: the peers' count blocks are self-validating {count | epoch}
  // words, polled by the plan — no flag and no system fence on that path
  a.poll_peers = !is_virtual(c) && d.e > 1 ? 1 : 0;
  return a;
}

// Front end of a dispatch: (route) + index + epoch bump + count exchange +
// plan.  Multi-GPU: one fused launch per card.  Virtual mode: every card's
// counts must land before any card plans, so the plan runs as a second
// lockstep launch.
moe_status do_front(moe_ctx* c, bool route, int level, int n, int landing, cudaStream_t s) {
  const moe_layer_desc& d = c->d;
  // one local card: nothing to wait for between the count push and the plan
  const bool fused_plan = !is_virtual(c) || c->local.size() == 1;
  for (auto& cd : c->local) {
    FrontArgs f{};
    f.logits = cd.v.logits;
    f.route = route ? 1 : 0;
    f.T = d.tokens;
    f.E = d.num_experts;
    f.k = d.top_k;
    f.n = n;
    f.experts = cd.v.experts;
    f.probs = cd.v.probs;
    f.perm_src = cd.v.perm_src;
    f.expert_of = cd.v.expert_of;
    f.slot_pos = cd.v.slot_pos;
    f.counts = cd.v.counts;
    f.expert_offsets = cd.v.expert_offsets;
    f.err = cd.err;
    f.tile_tokens = front_tile_tokens(d.num_experts, d.tokens, n);
    f.n_tiles = int32_t((d.tokens + f.tile_tokens - 1) / f.tile_tokens);
    f.aligned = (d.tokens / n) % f.tile_tokens == 0 ? 1 : 0;
    f.tile_hist = cd.tile_hist;
    f.tile_base = cd.tile_base;
    f.counts_acc = cd.counts_acc;
    f.arrive = cd.arrive;
    f.ready = cd.ready;
    f.epoch_dev = cd.epoch_dev;
    f.node = cd.node;
    f.max_chunks = d.max_chunks;
    f.n_dst = 0;
    for (int x = 0; x < d.e; ++x) {
      const int dst = card_of(c, x, cd.rho);
      f.dst_tables[f.n_dst++] = c->peer[dst].count_table;
    }
    // a lone card with final landing needs no plan: its final layout is the permuted order
    const bool identity = d.e == 1 && d.t == 1 && landing == MOE_LAND_FINAL && d.top_k <= 16;
    f.do_plan = fused_plan ? (identity ? 2 : 1) : 0;
    f.plan = make_plan_args(c, cd, level, n, landing);
    f.plan_scratch = cd.scratch;
    f.plan_in_smem = plan_fits_smem(d.e, d.num_experts, n) ? 1 : 0;
    f.dbg = c->debug ? cd.dbg : nullptr;
    f.plan.dbg = f.dbg;
    size_t sl;
    span_begin(c, route ? MOE_STAGE_ROUTE : MOE_STAGE_INDEX, 0, s, &sl);
    if (moe_status st = launch_front(f, d.logit_dtype, s)) return st;
    span_end(c, sl, s);
    ++c->launches;
  }
  if (!fused_plan)
    for (auto& cd : c->local) {
      PlanArgs a = make_plan_args(c, cd, level, n, landing);
      size_t sl;
      span_begin(c, MOE_STAGE_INDEX, 0, s, &sl);
      MONTA_CUDA(launch_plan_with_scratch(a, cd.scratch, s));
      span_end(c, sl, s);
      ++c->launches;
    }
  return MOE_OK;
}

moe_status do_index(moe_ctx* c, int n, cudaStream_t s) {
  for (auto& cd : c->local) {
    if (moe_status st = build_index(cd.v.experts, c->d.tokens, c->d.top_k, c->d.num_experts, n, cd.v.perm_src,
                                    cd.v.expert_of, cd.v.slot_pos, cd.v.counts, cd.v.expert_offsets, cd.err, s))
      return st;
    ++c->launches;
  }
  return MOE_OK;
}

int copy_vec(const moe_ctx* c, bool dedup) {
  return vec_bytes(c->row_bytes, dedup ? c->row_bytes / c->d.t : c->row_bytes);
}

// One chunk of the fused permute + AllToAll, for one card.
// Bulk kernels never spin: a kernel that consumes remote data is preceded
// on its stream by a one-CTA wait kernel.  (A spinning bulk grid can occupy
// every SM and starve the local producer another GPU is waiting for.)
moe_status hoist_wait(moe_ctx* c, WaitList& w, int32_t* err, cudaStream_t s) {
  if (w.n == 0) return MOE_OK;
  MONTA_CUDA(launch_wait(w, err, s));
  ++c->launches;
  w.n = 0;
  return MOE_OK;
}

// Work items per row for the copy kernel.
int items_per_row(int vec, int64_t max_width) {
  const int64_t ib = copy_item_bytes(vec);
  return int((max_width + ib - 1) / ib);
}

// One chunk of the fused permute + AllToAll, for one card.  Cross-node legs
// (NVLink) and own-node legs (HBM, full rows) are separate lists run by
// disjoint CTA sets, sized so both finish together.
moe_status launch_aa(moe_ctx* c, Card& cd, int level, int j, int landing, cudaStream_t s, bool concurrent) {
  const moe_layer_desc& d = c->d;
  const bool dedup = level != MOE_BASELINE && d.t > 1;
  if (d.top_k <= 16) {  // token-side: each row read once, stored to its k destinations
    TokArgs t{};
    t.x = static_cast<const char*>(cd.v.x);
    t.row_bytes = c->row_bytes;
    t.experts = cd.v.experts;
    t.slot_pos = cd.v.slot_pos;
    t.token_ids = cd.v.token_ids;
    t.source_card = card_of(c, cd.node, 0);
    t.table = cd.aa_table;
    t.E = d.num_experts;
    t.k = d.top_k;
    t.n = c->last_n;
    t.j = j;
    t.staged = landing == MOE_LAND_STAGED ? 1 : 0;
    const int64_t ct = d.tokens / std::max(1, c->last_n);
    t.tok_begin = int64_t(j) * ct;
    t.tok_end = t.tok_begin + ct;
    t.dst_stride = c->row_bytes;
    for (int q = 0; q < c->cards; ++q) {
      if (!c->peer[q].slab) continue;
      t.dst[q] = t.staged ? c->peer[q].pre : c->peer[q].recv;
      t.dst_tags[q] = t.staged ? c->peer[q].pre_tags : c->peer[q].recv_tags;
      t.dst_pre[q] = c->peer[q].pre;
      t.dst_scale[q] = c->peer[q].wscale;
    }
    t.fp8 = c->wire == MOE_WIRE_FP8 ? 1 : 0;
    if (c->pace_bpus && d.e > 1) {  // the cross-node legs of this chunk set the pace
      t.pace_list = list_of(c, cd, kPhaseAA, j);
      t.pace_bpus = c->pace_bpus;
    }
    t.node = cd.node;
    t.t = d.t;
    t.blocks_per_row = int(std::max<int64_t>(1, d.hidden / 128));
    t.sig = no_signal();
    t.sig.epoch_ptr = cd.epoch_dev;
    t.sig.done = cd.done + kPsAA * d.max_chunks + j;
    if (!is_virtual(c))
      for (int x = 0; x < d.e; ++x)
        if (x != cd.node) t.sig.flags[t.sig.n++] = flag_at(c, card_of(c, x, cd.rho), sig_chunk(c, kPsAA, j), cd.id);
    t.err = cd.err;
    t.local_dst = is_virtual(c) ? 1 : 0;
    if (c->node_dedup_now) {
      t.nslot = cd.nslot;
      t.e = d.e;
      for (int q = 0; q < c->cards; ++q)
        if (c->peer[q].slab) t.stage[q] = c->peer[q].stage + size_t(cd.node) * d.tokens * c->row_bytes;
    }
    // four resident CTAs (32 warps) per SM, at most one item (token x 2 KiB piece) per warp
    const int64_t items = ct * ((c->row_bytes + 2047) / 2048);
    int grid = int(std::min<int64_t>((items + 7) / 8, int64_t(c->sms) * (concurrent ? 2 : 4)));
    grid = std::max(grid, 1);
    size_t sl;
    span_begin(c, MOE_STAGE_AA, j, s, &sl);
    MONTA_CUDA(launch_aa_token(t, copy_vec(c, dedup), grid, s));
    span_end(c, sl, s);
    ++c->launches;
    return MOE_OK;
  }
  CopyArgs a{};
  const int grid = copy_grid(c, concurrent, true);
  if (d.e > 1) {
    a.list = list_of(c, cd, kPhaseAA, j);
    a.list2 = list_of(c, cd, kPhaseAAL, j);
    a.pace_bpus = c->pace_bpus;  // the cross-node list
    // time(local) / time(remote) ~= (full / width) * 0.2 / (e - 1)  (HBM copy vs NVLink store)
    const double r = (dedup ? double(d.t) : 1.0) * 0.2 / double(d.e - 1);
    const double frac = std::min(0.5, std::max(0.1, r / (1.0 + r)));
    a.split = std::max(1, grid - std::max(1, int(grid * frac + 0.5)));
  } else {
    a.list = list_of(c, cd, kPhaseAAL, j);
    a.list2 = nullptr;
    a.split = grid;
  }
  a.src = static_cast<const char*>(cd.v.x);
  a.src_stride = c->row_bytes;
  a.gather = cd.v.perm_src;
  a.src_tags = nullptr;
  a.token_ids = cd.v.token_ids;
  a.source_card = card_of(c, cd.node, 0);
  a.synth_tags = 1;
  a.dst_stride = c->row_bytes;
  a.dst_mask = 0;
  for (int q = 0; q < c->cards; ++q) {
    if (!c->peer[q].slab) continue;
    a.dst[q] = landing == MOE_LAND_STAGED ? c->peer[q].pre : c->peer[q].recv;
    a.dst_tags[q] = landing == MOE_LAND_STAGED ? c->peer[q].pre_tags : c->peer[q].recv_tags;
  }
  const int vec = copy_vec(c, dedup);
  a.chunks_per_row = items_per_row(vec, c->row_bytes);
  a.wait = no_wait();
  a.sig = no_signal();
  a.sig.epoch_ptr = cd.epoch_dev;
  a.sig.done = cd.done + kPsAA * d.max_chunks + j;
  if (!is_virtual(c))
    for (int x = 0; x < d.e; ++x)
      if (x != cd.node) a.sig.flags[a.sig.n++] = flag_at(c, card_of(c, x, cd.rho), sig_chunk(c, kPsAA, j), cd.id);
  a.err = cd.err;
  size_t sl;
  span_begin(c, MOE_STAGE_AA, j, s, &sl);
  MONTA_CUDA(launch_seg_copy(a, vec, grid, s));
  span_end(c, sl, s);
  ++c->launches;
  return MOE_OK;
}

// One chunk of the intra-node AllGather (forward this rank's slice of the
// rows that arrived from other nodes to every TP peer).
// fp8 wire, receive side: the rows of chunk j (j < 0: every chunk) that came
// from another node, this card's columns, e4m3 + scales (pre, wscale) -> bf16 recv.
moe_status wire_dequant(moe_ctx* c, Card& cd, int level, int j, cudaStream_t s) {
  if (c->wire != MOE_WIRE_FP8 || c->d.e == 1) return MOE_OK;
  const moe_layer_desc& d = c->d;
  const bool dedup = level != MOE_BASELINE && d.t > 1;
  const int64_t w = dedup ? d.hidden / d.t : d.hidden;
  const int64_t ct = d.tokens / std::max(1, c->last_n);
  const int64_t p0 = j < 0 ? 0 : int64_t(j) * ct, p1 = j < 0 ? d.tokens : p0 + ct;
  MONTA_CUDA(launch_wire_dequant(static_cast<char*>(cd.v.recv), cd.v.recv_tags, cd.recv_rows, c->recv_cap,
                                 static_cast<const char*>(cd.v.pre), c->peer[cd.id].wscale, c->row_bytes,
                                 int(std::max<int64_t>(1, d.hidden / 128)), cd.node, d.t,
                                 dedup ? int64_t(cd.rho) * w : 0, w, p0, p1, s));
  ++c->launches;
  return MOE_OK;
}

moe_status launch_ag(moe_ctx* c, Card& cd, int j, int landing, cudaStream_t s, bool concurrent) {
  const moe_layer_desc& d = c->d;
  CopyArgs a{};
  a.list = list_of(c, cd, kPhaseAG, j);
  const bool staged = landing == MOE_LAND_STAGED;
  a.src = staged ? static_cast<const char*>(cd.v.pre) : static_cast<const char*>(cd.v.recv);
  a.src_stride = c->row_bytes;
  a.gather = nullptr;
  a.src_tags = staged ? cd.v.pre_tags : cd.v.recv_tags;
  a.synth_tags = 0;
  a.dst_stride = c->row_bytes;
  a.dst_mask = 0;
  for (int r = 0; r < d.t; ++r) {
    const int q = card_of(c, cd.node, r);
    if (q == cd.id) continue;
    a.dst_mask |= 1ull << q;
    a.dst[q] = staged ? c->peer[q].pre : c->peer[q].recv;
    a.dst_tags[q] = staged ? c->peer[q].pre_tags : c->peer[q].recv_tags;
  }
  a.chunks_per_row = items_per_row(copy_vec(c, true), c->row_bytes / d.t);
  a.split = copy_grid(c, concurrent, false);
  a.wait = no_wait();
  a.wait.epoch_ptr = cd.epoch_dev;
  a.sig = no_signal();
  a.sig.epoch_ptr = cd.epoch_dev;
  a.sig.done = cd.done + kPsAG * d.max_chunks + j;
  if (!is_virtual(c)) {
    for (int g = 0; g < d.e; ++g)
      if (g != cd.node) a.wait.flags[a.wait.n++] = flag_at(c, cd.id, sig_chunk(c, kPsAA, j), card_of(c, g, cd.rho));
    for (int r = 0; r < d.t; ++r)
      if (r != cd.rho) a.sig.flags[a.sig.n++] = flag_at(c, card_of(c, cd.node, r), sig_chunk(c, kPsAG, j), cd.id);
  }
  a.err = cd.err;
  if (moe_status st = hoist_wait(c, a.wait, cd.err, s)) return st;
  if (!is_virtual(c))  // this chunk's cross-node rows arrived (fp8 wire): decode before forwarding
    if (moe_status st = wire_dequant(c, cd, MOE_O1, j, s)) return st;
  size_t sl;
  span_begin(c, MOE_STAGE_AG, j, s, &sl);
  MONTA_CUDA(launch_seg_copy(a, copy_vec(c, true), copy_grid(c, concurrent, false), s));
  span_end(c, sl, s);
  ++c->launches;
  return MOE_OK;
}

moe_status launch_d2d(moe_ctx* c, Card& cd, int level, int j, cudaStream_t s, bool concurrent) {
  const moe_layer_desc& d = c->d;
  const bool dedup = level != MOE_BASELINE && d.t > 1;
  CopyArgs a{};
  a.list = list_of(c, cd, kPhaseD2D, j);
  a.src = static_cast<const char*>(cd.v.pre);
  a.src_stride = c->row_bytes;
  a.src_tags = cd.v.pre_tags;
  a.synth_tags = 0;
  a.dst_stride = c->row_bytes;
  a.dst[cd.id] = static_cast<char*>(cd.v.recv);
  a.dst_tags[cd.id] = cd.v.recv_tags;
  a.chunks_per_row = items_per_row(copy_vec(c, false), c->row_bytes);
  a.split = copy_grid(c, concurrent, false);
  a.wait = no_wait();
  a.wait.epoch_ptr = cd.epoch_dev;
  if (!is_virtual(c)) {
    for (int g = 0; g < d.e; ++g)
      if (g != cd.node) a.wait.flags[a.wait.n++] = flag_at(c, cd.id, sig_chunk(c, kPsAA, j), card_of(c, g, cd.rho));
    if (dedup)
      for (int r = 0; r < d.t; ++r)
        if (r != cd.rho) a.wait.flags[a.wait.n++] = flag_at(c, cd.id, sig_chunk(c, kPsAG, j), card_of(c, cd.node, r));
  }
  a.sig = no_signal();
  a.err = cd.err;
  if (moe_status st = hoist_wait(c, a.wait, cd.err, s)) return st;
  size_t sl;
  span_begin(c, MOE_STAGE_D2D, j, s, &sl);
  MONTA_CUDA(launch_seg_copy(a, copy_vec(c, false), copy_grid(c, concurrent, false), s));
  span_end(c, sl, s);
  ++c->launches;
  return MOE_OK;
}

// Wait (on stream s) until every remote contribution of the dispatch landed.
moe_status dispatch_tail_wait(moe_ctx* c, Card& cd, int level, int n, int landing, cudaStream_t s) {
  if (is_virtual(c)) return MOE_OK;
  const moe_layer_desc& d = c->d;
  const bool dedup = level != MOE_BASELINE && d.t > 1;
  if (landing == MOE_LAND_STAGED) return MOE_OK;  // every D2D already waited
  WaitList w = no_wait();
  w.epoch_ptr = cd.epoch_dev;
  for (int j = 0; j < n; ++j) {
    const int need = dedup ? d.t - 1 : d.e - 1;
    if (w.n + need > kMaxCards) {
      MONTA_CUDA(launch_wait(w, cd.err, s));
      ++c->launches;
      w.n = 0;
    }
    if (dedup) {
      for (int r = 0; r < d.t; ++r)
        if (r != cd.rho) w.flags[w.n++] = flag_at(c, cd.id, sig_chunk(c, kPsAG, j), card_of(c, cd.node, r));
    } else {
      for (int g = 0; g < d.e; ++g)
        if (g != cd.node) w.flags[w.n++] = flag_at(c, cd.id, sig_chunk(c, kPsAA, j), card_of(c, g, cd.rho));
    }
  }
  if (w.n) {
    MONTA_CUDA(launch_wait(w, cd.err, s));
    ++c->launches;
  }
  return MOE_OK;
}

// Whole chunked dispatch of this card in one persistent cooperative launch
// (xchg.cu).  CTAs are split across roles in proportion to the expected
// bytes each moves (uniform routing): NVLink legs ~8x slower per byte than
// local HBM copies.
// The persistent dispatch runs (and declines nothing later) when the rows
// take 4+-byte vectors and 16+ CTAs are co-resident (four roles of >= 4).
bool xchg_eligible(moe_ctx* c, int level) {
  if (!c->use_xchg || c->aa_ctas > 0 || c->wire != MOE_WIRE_BF16 || is_virtual(c)) return false;
  const bool dedup = level != MOE_BASELINE && c->d.t > 1;
  const int vec = copy_vec(c, dedup);
  return vec >= 4 && xchg_max_ctas(vec) >= 16;
}

moe_status launch_dispatch_xchg(moe_ctx* c, Card& cd, int level, int n, int landing, cudaStream_t s, bool* done) {
  *done = false;
  const moe_layer_desc& d = c->d;
  const bool dedup = level != MOE_BASELINE && d.t > 1;
  const bool staged = landing == MOE_LAND_STAGED;
  const int vec = copy_vec(c, dedup);
  if (!xchg_eligible(c, level)) return MOE_OK;
  const int max_ctas = xchg_max_ctas(vec);
  XchgArgs x{};
  x.d2d_in_ag = (staged && dedup && level == MOE_O2) ? 1 : 0;
  // Role sizes from measured per-CTA rates (calibration, profiles/r01):
  // an NVLink-store CTA moves ~4 GB/s, an HBM-copy CTA ~20 GB/s.
  const double row = double(c->row_bytes), rem = (d.e - 1.0) / d.e, loc = 1.0 / d.e;
  const double kNv = 1.0 / 4.0, kHbm = 1.0 / 20.0;
  const bool nv_needed = d.e > 1 || dedup;
  const double w_aa = d.e > 1 ? rem * (dedup ? row / d.t : row) * kNv : 0.0;
  const double w_ag = (dedup ? (d.t - 1.0) * rem * (row / d.t) * kNv : 0.0) + (x.d2d_in_ag ? row * 2.0 * kHbm : 0.0);
  // chunked + dedup: the AllGather gets its own CTAs so it overlaps the next
  // chunks' AllToAll; unchunked, the AA CTAs run both legs back to back
  const bool split_ag = dedup && n > 1 && d.e > 1;
  const double w_nv = split_ag ? w_aa : w_aa + w_ag;
  const double w_loc = loc * row * 2.0 * kHbm;
  const double w_d2d = (staged && !x.d2d_in_ag) ? row * 2.0 * kHbm : 0.0;
  const double wsum = w_nv + (split_ag ? w_ag : 0.0) + w_loc + w_d2d;
  const int G = max_ctas;
  auto share = [&](double w, bool needed) {
    if (!needed) return 0;
    return std::max(4, int(G * w / wsum + 0.5));
  };
  x.r_aa = share(w_nv, nv_needed);
  x.r_ag = share(w_ag, split_ag);
  x.r_aal = share(w_loc, true);
  x.r_d2d = share(w_d2d, staged && !x.d2d_in_ag);
  while (x.r_aa + x.r_ag + x.r_aal + x.r_d2d > max_ctas) {  // trim the largest role
    int* big = &x.r_aa;
    for (int* r : {&x.r_ag, &x.r_aal, &x.r_d2d})
      if (*r > *big) big = r;
    if (*big <= 4) return MOE_OK;
    --*big;
  }
  CopyArgs& a = x.cp;
  a.pace_bpus = c->pace_bpus;  // applied by the AllToAll role only
  a.src = static_cast<const char*>(cd.v.x);
  a.src_stride = c->row_bytes;
  a.gather = cd.v.perm_src;
  a.token_ids = cd.v.token_ids;
  a.source_card = card_of(c, cd.node, 0);
  a.synth_tags = 1;
  a.dst_stride = c->row_bytes;
  for (int q = 0; q < c->cards; ++q) {
    if (!c->peer[q].slab) continue;
    a.dst[q] = staged ? c->peer[q].pre : c->peer[q].recv;
    a.dst_tags[q] = staged ? c->peer[q].pre_tags : c->peer[q].recv_tags;
    x.flags[q] = c->peer[q].flags;
  }
  a.err = cd.err;
  x.lists = cd.lists;
  x.seg_cap = d.num_experts;
  x.max_chunks = d.max_chunks;
  x.n = n;
  x.me = cd.id;
  x.node = cd.node;
  x.rho = cd.rho;
  x.e = d.e;
  x.t = d.t;
  x.dedup = dedup ? 1 : 0;
  x.staged = staged ? 1 : 0;
  x.cpr_full = items_per_row(vec, c->row_bytes);
  x.cpr_slice = items_per_row(vec, c->row_bytes / d.t);
  x.recv_local = static_cast<char*>(cd.v.recv);
  x.recv_tags_local = cd.v.recv_tags;
  x.pre_local = static_cast<char*>(cd.v.pre);
  x.pre_tags_local = cd.v.pre_tags;
  x.d2d_dst[cd.id] = static_cast<char*>(cd.v.recv);
  x.d2d_dst_tags[cd.id] = cd.v.recv_tags;
  for (int r = 0; r < d.t; ++r) {
    const int q = card_of(c, cd.node, r);
    if (q == cd.id) continue;
    x.ag_mask |= 1ull << q;
    x.ag_dst[q] = staged ? c->peer[q].pre : c->peer[q].recv;
    x.ag_dst_tags[q] = staged ? c->peer[q].pre_tags : c->peer[q].recv_tags;
  }
  x.epoch_ptr = cd.epoch_dev;
  x.counters = cd.xchg_counters;
  x.local_flags = cd.xchg_flags;
  x.err = cd.err;
  x.dbg = c->debug ? cd.dbg + 16 : nullptr;
  if (c->timing) {
    x.trace = cd.xtrace;
    MONTA_CUDA(cudaMemsetAsync(cd.xtrace, 0xff, size_t(4) * d.max_chunks * 2 * 8, s));
  }
  size_t sl;
  span_begin(c, MOE_STAGE_AA, -1, s, &sl);
  MONTA_CUDA(launch_xchg(x, vec, s));
  span_end(c, sl, s);
  ++c->launches;
  *done = true;
  return MOE_OK;
}

moe_status validate_dispatch(moe_ctx* c, int level, int n, int landing) {
  const moe_layer_desc& d = c->d;
  if (level == MOE_BASELINE) {
    if (n != 1) return fail(MOE_ERR_INVALID_ARGUMENT, "dispatch_monolithic is unchunked (n = 1)");
  } else {
    if (level != MOE_O1 && level != MOE_O2 && level != MOE_O3)
      return fail(MOE_ERR_INVALID_ARGUMENT, "dispatch_chunked: level must be O1, O2 or O3");
    if (n < 1) return fail(MOE_ERR_INVALID_ARGUMENT, "dispatch_chunked: n must be >= 1");
    if (level == MOE_O1 && n != 1)
      return fail(MOE_ERR_INVALID_ARGUMENT, "dispatch_chunked: O1 is unchunked (n = 1)");
  }
  if (n > d.max_chunks)
    return fail(MOE_ERR_INVALID_ARGUMENT, "dispatch: n = %d exceeds the context's max_chunks %d", n, d.max_chunks);
  if (d.tokens % n != 0) return fail(MOE_ERR_INVALID_ARGUMENT, "dispatch_chunked: n does not divide the sequence");
  if (level != MOE_BASELINE && d.hidden % d.t != 0)
    return fail(MOE_ERR_INVALID_ARGUMENT, "dispatch_chunked: tensor group must evenly split the payload");
  if (landing != MOE_LAND_FINAL && landing != MOE_LAND_STAGED)
    return fail(MOE_ERR_INVALID_ARGUMENT, "dispatch: bad landing mode");
  if (c->wire == MOE_WIRE_FP8 && landing == MOE_LAND_STAGED && level != MOE_BASELINE)
    return fail(MOE_ERR_INVALID_ARGUMENT, "dispatch: the fp8 wire lands in pre: FINAL landing only");
  return MOE_OK;
}

}  // namespace

extern "C" moe_status moe_ctx_route(moe_ctx* c, void* stream) {
  if (moe_status st = check_ready(c)) return st;
  MONTA_CUDA(cudaSetDevice(c->device));
  return do_route(c, static_cast<cudaStream_t>(stream));
}

extern "C" moe_status moe_ctx_permute(moe_ctx* c, int32_t n, void* stream) {
  if (moe_status st = check_ready(c)) return st;
  MONTA_CUDA(cudaSetDevice(c->device));
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (n < 1 || n > c->d.max_chunks || c->d.tokens % n != 0)
    return fail(MOE_ERR_INVALID_ARGUMENT, "permute: bad chunk count %d", n);
  if (moe_status st = do_index(c, n, s)) return st;
  for (auto& cd : c->local) {
    MONTA_CUDA(launch_gather_rows(cd.v.x, c->row_bytes, 0, c->row_bytes, cd.v.perm_src, c->R, cd.v.permuted,
                                  c->row_bytes, s));
    ++c->launches;
  }
  return MOE_OK;
}

namespace {

// Node dedup for EP-only topologies (t == 1): with k slots spread over e
// nodes a token reaches several experts on one remote node, and the plain
// AllToAll sends its row once per such expert.  Here it crosses once per
// (token, remote node): k_node_slots claims a staging slot on the receiver
// (one atomic per warp and node) and writes the slot's descriptor (token id,
// position, the k destination rows on that node, the experts); the token
// kernel stores own-node rows as before and each remote row once into the
// receiver's staging block; after the chunk flags the receiver's
// k_node_fanout copies every staged row to its destination rows and writes
// their tags.  The recv layout is the plain dispatch's, row for row.
bool node_dedup_ok(const moe_ctx* c, int level, int n, int landing) {
  static const int env = [] {  // MONTA_NODE_DEDUP=0 overrides (A/B)
    const char* e = std::getenv("MONTA_NODE_DEDUP");
    return e ? std::atoi(e) : 1;
  }();
  const moe_layer_desc& d = c->d;
  // under TP: the deduplicated levels stage this rank's slice and exchange
  // it between the receiving node's ranks; the naive level stages full rows
  // between same-rank cards (each rank still receives every row it needs)
  (void)level;
  // auto: a token reaches ~k/e experts per node; below two the saved rows do
  // not pay for the staging pass (2x2 Mixtral k = 2: 160.6 -> 172.4 us)
  const bool want = c->node_dedup == 1 || (c->node_dedup == 2 && d.top_k >= 2 * d.e);
  return env != 0 && want && !is_virtual(c) && d.e > 1 && n == 1 && landing == MOE_LAND_FINAL &&
         c->wire == MOE_WIRE_BF16 && !c->pace_bpus && c->aa_ctas == 0 && d.top_k <= 16 && c->row_bytes % 16 == 0 &&
         (c->row_bytes / d.t) % 16 == 0 && d.t <= 9 &&  // 16-byte slices; k_stage_ag's peer table
         c->local.size() == 1;  // (the staging regions exist exactly when e > 1 and world > 1)
}

moe_status dispatch_node_dedup(moe_ctx* c, Card& cd, int level, int landing, cudaStream_t s) {
  const moe_layer_desc& d = c->d;
  const int dw = 2 + 2 * d.top_k;
  MONTA_CUDA(cudaMemsetAsync(c->peer[cd.id].scount, 0, size_t(kMaxCards) * 4, s));
  NodeSlotArgs ns{};
  ns.experts = cd.v.experts;
  ns.slot_pos = cd.v.slot_pos;
  ns.token_ids = cd.v.token_ids;
  ns.table = cd.aa_table;
  ns.T = d.tokens;
  ns.E = d.num_experts;
  ns.k = d.top_k;
  ns.e = d.e;
  ns.t = d.t;
  ns.node = cd.node;
  ns.rho = cd.rho;
  ns.scount = c->peer[cd.id].scount;
  ns.nslot = cd.nslot;
  ns.bcnt = cd.bcnt;
  for (int g = 0; g < d.e; ++g)
    if (g != cd.node) {
      const int q = card_of(c, g, cd.rho);
      ns.sdesc[q] = c->peer[q].sdesc + size_t(cd.node) * d.tokens * dw;
    }
  MONTA_CUDA(launch_node_slots(ns, s));
  ++c->launches;
  c->node_dedup_now = true;
  moe_status st = launch_aa(c, cd, level, 0, landing, s, false);
  c->node_dedup_now = false;
  if (st != MOE_OK) return st;
  const bool dedup = level != MOE_BASELINE && d.t > 1;
  {  // every remote sender's rows (this rank's slice under TP) are staged here
    WaitList w = no_wait();
    w.epoch_ptr = cd.epoch_dev;
    for (int g = 0; g < d.e; ++g)
      if (g != cd.node) w.flags[w.n++] = flag_at(c, cd.id, sig_chunk(c, kPsAA, 0), card_of(c, g, cd.rho));
    MONTA_CUDA(launch_wait(w, cd.err, s));
    ++c->launches;
  }
  FanoutArgs fa{};
  for (int g = 0; g < d.e; ++g) {
    if (g == cd.node) continue;
    const int q = card_of(c, g, cd.rho);
    const int i = fa.nsend++;
    fa.stage[i] = c->peer[cd.id].stage + size_t(g) * d.tokens * c->row_bytes;
    fa.sdesc[i] = c->peer[cd.id].sdesc + size_t(g) * d.tokens * dw;
    fa.count[i] = c->peer[q].scount + cd.id;
    fa.source_card[i] = card_of(c, g, 0);  // the tag names the source node's first card (as the token kernel does)
  }
  fa.row_bytes = c->row_bytes;
  fa.col_lo = 0;
  fa.col_hi = c->row_bytes;
  fa.k = d.top_k;
  fa.recv = static_cast<char*>(cd.v.recv);
  fa.recv_tags = cd.v.recv_tags;
  if (dedup) {
    // the staged rows carry this rank's slice; the TP peers staged the same
    // tokens at the same slots (deterministic slots): exchange the slices at
    // the staging level, then every card fans out whole rows
    StageAgArgs ga{};
    ga.nsend = fa.nsend;
    for (int i = 0; i < fa.nsend; ++i) {
      ga.stage[i] = fa.stage[i];
      ga.count[i] = fa.count[i];
    }
    for (int r = 0; r < d.t; ++r) {
      const int q = card_of(c, cd.node, r);
      if (q == cd.id) continue;
      int i = 0;
      for (int g = 0; g < d.e; ++g)
        if (g != cd.node) ga.peer_stage[ga.npeer][i++] = c->peer[q].stage + size_t(g) * d.tokens * c->row_bytes;
      ++ga.npeer;
    }
    if (ga.npeer > 8) return fail(MOE_ERR_UNSUPPORTED, "node dedup: at most 9 TP ranks");
    ga.row_bytes = c->row_bytes;
    ga.col_lo = int64_t(cd.rho) * (c->row_bytes / d.t);
    ga.col_hi = ga.col_lo + c->row_bytes / d.t;
    ga.sig = no_signal();
    ga.sig.epoch_ptr = cd.epoch_dev;
    ga.sig.done = cd.done + kPsAG * d.max_chunks + 0;
    for (int r = 0; r < d.t; ++r)
      if (r != cd.rho) ga.sig.flags[ga.sig.n++] = flag_at(c, card_of(c, cd.node, r), sig_chunk(c, kPsAG, 0), cd.id);
    MONTA_CUDA(launch_stage_ag(ga, d.tokens, s));
    ++c->launches;
    if (moe_status st4 = dispatch_tail_wait(c, cd, level, 1, landing, s)) return st4;  // the peers' slices
  }
  MONTA_CUDA(launch_node_fanout(fa, d.tokens, 16, s));
  ++c->launches;
  return MOE_OK;
}

moe_status dispatch_impl(moe_ctx* c, int level, int n, int landing, cudaStream_t s, bool route) {
  const moe_layer_desc& d = c->d;
  if (level == MOE_BASELINE) landing = MOE_LAND_FINAL;
  const bool dedup = level != MOE_BASELINE && d.t > 1;
  const bool staged = landing == MOE_LAND_STAGED;
  c->last_level = level;
  c->last_n = n;
  c->last_landing = landing;
  c->combine_ready = true;
  if (c->timing && !c->in_forward) {
    c->span_used = 0;
    record_timing(c->ev_base, s);
  }
  if (c->checks)  // poisoned tags: a row that never lands fails verify_dispatch
    for (auto& cd : c->local) MONTA_CUDA(cudaMemsetAsync(cd.v.recv_tags, 0xff, size_t(c->recv_cap) * 16, s));
  if (moe_status st = do_front(c, route, level, n, landing, s)) return st;

  if (is_virtual(c)) {
    for (int j = 0; j < n; ++j) {
      for (auto& cd : c->local)
        if (moe_status st = launch_aa(c, cd, level, j, landing, s, false)) return st;
      for (auto& cd : c->local)
        if (moe_status st = wire_dequant(c, cd, level, j, s)) return st;
      if (dedup)
        for (auto& cd : c->local)
          if (moe_status st = launch_ag(c, cd, j, landing, s, false)) return st;
      if (staged)
        for (auto& cd : c->local)
          if (moe_status st = launch_d2d(c, cd, level, j, s, false)) return st;
    }
    return MOE_OK;
  }
  // multi-GPU: one card per rank; AllToAll on the high-priority stream,
  // AllGather on its own stream, reorder copies on the AllGather stream (O2)
  // or their own (O3).
  Card& cd = c->local[0];
  if (node_dedup_ok(c, level, n, landing)) return dispatch_node_dedup(c, cd, level, landing, s);
  if (c->use_xchg) {
    bool done = false;
    if (moe_status st = launch_dispatch_xchg(c, cd, level, n, landing, s, &done)) return st;
    if (done) return MOE_OK;
  }
  cudaStream_t s_d2d = level == MOE_O3 ? c->s_d2d : c->s_ag;
  MONTA_CUDA(cudaEventRecord(c->ev_fork, s));
  MONTA_CUDA(cudaStreamWaitEvent(c->s_aa, c->ev_fork, 0));
  MONTA_CUDA(cudaStreamWaitEvent(c->s_ag, c->ev_fork, 0));
  MONTA_CUDA(cudaStreamWaitEvent(c->s_d2d, c->ev_fork, 0));
  for (int j = 0; j < n; ++j) {
    if (c->pipe) MONTA_CUDA(cudaStreamWaitEvent(c->s_aa, c->ev_h2d[j], 0));  // this chunk's x is on the card
    if (moe_status st = launch_aa(c, cd, level, j, landing, c->s_aa, true)) return st;
    MONTA_CUDA(cudaEventRecord(c->ev_aa[j], c->s_aa));
    if (dedup) {
      if (moe_status st = launch_ag(c, cd, j, landing, c->s_ag, true)) return st;
      MONTA_CUDA(cudaEventRecord(c->ev_ag[j], c->s_ag));
    }
    if (staged) {
      MONTA_CUDA(cudaStreamWaitEvent(s_d2d, c->ev_aa[j], 0));
      if (dedup) MONTA_CUDA(cudaStreamWaitEvent(s_d2d, c->ev_ag[j], 0));
      if (moe_status st = launch_d2d(c, cd, level, j, s_d2d, true)) return st;
    }
  }
  MONTA_CUDA(cudaEventRecord(c->ev_join_aa, c->s_aa));
  MONTA_CUDA(cudaEventRecord(c->ev_join_ag, c->s_ag));
  MONTA_CUDA(cudaEventRecord(c->ev_join_d2d, c->s_d2d));
  MONTA_CUDA(cudaStreamWaitEvent(s, c->ev_join_aa, 0));
  MONTA_CUDA(cudaStreamWaitEvent(s, c->ev_join_ag, 0));
  MONTA_CUDA(cudaStreamWaitEvent(s, c->ev_join_d2d, 0));
  if (moe_status st = dispatch_tail_wait(c, cd, level, n, landing, s)) return st;
  if (!dedup) return wire_dequant(c, cd, level, -1, s);  // (deduplicated: decoded per chunk before the AllGather)
  return MOE_OK;
}

}  // namespace

extern "C" moe_status moe_ctx_dispatch(moe_ctx* c, int level, int32_t n, int landing, void* stream) {
  if (moe_status st = check_ready(c)) return st;
  if (moe_status st = validate_dispatch(c, level, n, landing)) return st;
  MONTA_CUDA(cudaSetDevice(c->device));
  return dispatch_impl(c, level, n, landing, static_cast<cudaStream_t>(stream), false);
}

namespace {

// The reverse AllToAll of chunk j.  With l0 >= 0 only the rows of local
// experts [l0, l1) (a contiguous final-layout range) move, and `signal`
// says whether this launch releases the chunk's flags (the last group's).
moe_status launch_caa(moe_ctx* c, Card& cd, int level, int j, cudaStream_t s, bool concurrent, int l0 = -1,
                      int l1 = -1, bool signal = true, int grid_cap = 0) {
  const moe_layer_desc& d = c->d;
  if (d.e == 1) return MOE_OK;  // no other node: the un-permute reads every row in place
  const bool dedup = level != MOE_BASELINE && d.t > 1;
  if (c->wire == MOE_WIRE_FP8) {  // the reverse AllToAll on the fp8 wire too
    CaaFp8Args f{};
    f.list = list_of(c, cd, kPhaseCAA, j);
    f.src = static_cast<const char*>(cd.v.expert_out);
    f.row_bytes = c->row_bytes;
    f.blocks_per_row = int(std::max<int64_t>(1, d.hidden / 128));
    for (int q = 0; q < c->cards; ++q)
      if (c->peer[q].slab) {
        f.dst_wire[q] = c->peer[q].cwire;
        f.dst_scale[q] = c->peer[q].cscale;
      }
    f.pace_bpus = c->pace_bpus;
    f.sig = no_signal();
    f.sig.epoch_ptr = cd.epoch_dev;
    f.sig.done = cd.done + kPsCAA * d.max_chunks + j;
    if (!is_virtual(c))
      for (int g = 0; g < d.e; ++g)
        if (g != cd.node) f.sig.flags[f.sig.n++] = flag_at(c, card_of(c, g, cd.rho), sig_chunk(c, kPsCAA, j), cd.id);
    size_t sl;
    span_begin(c, MOE_STAGE_CAA, j, s, &sl);
    MONTA_CUDA(launch_caa_fp8(f, copy_grid(c, concurrent, true), s));
    span_end(c, sl, s);
    ++c->launches;
    return MOE_OK;
  }
  CopyArgs a{};
  a.list = list_of(c, cd, kPhaseCAA, j);
  a.pace_bpus = c->pace_bpus;
  a.src = static_cast<const char*>(cd.v.expert_out);
  a.src_stride = c->row_bytes;
  a.synth_tags = 0;
  a.dst_stride = c->row_bytes;
  for (int q = 0; q < c->cards; ++q)
    if (c->peer[q].slab) a.dst[q] = c->peer[q].comb;
  a.chunks_per_row = items_per_row(copy_vec(c, dedup), dedup ? c->row_bytes / d.t : c->row_bytes);
  a.split = copy_grid(c, concurrent, true);
  a.wait = no_wait();
  a.sig = no_signal();
  a.sig.epoch_ptr = cd.epoch_dev;
  a.sig.done = cd.done + kPsCAA * d.max_chunks + j;
  if (!is_virtual(c))
    for (int g = 0; g < d.e; ++g)
      if (g != cd.node) a.sig.flags[a.sig.n++] = flag_at(c, card_of(c, g, cd.rho), sig_chunk(c, kPsCAA, j), cd.id);
  a.err = cd.err;
  if (l0 >= 0) {
    a.bounds = cd.v.recv_expert_offsets;
    a.b_lo = l0;
    a.b_hi = l1;
  }
  if (!signal) a.sig.n = 0;
  size_t sl;
  span_begin(c, MOE_STAGE_CAA, j, s, &sl);
  int grid = copy_grid(c, concurrent, true);
  if (grid_cap > 0) grid = std::min(grid, grid_cap);
  a.split = grid;
  MONTA_CUDA(launch_seg_copy(a, copy_vec(c, dedup), grid, s));
  span_end(c, sl, s);
  ++c->launches;
  return MOE_OK;
}

moe_status launch_unperm(moe_ctx* c, Card& cd, int level, int n, int j, cudaStream_t s, bool concurrent) {
  const moe_layer_desc& d = c->d;
  const bool dedup = level != MOE_BASELINE && d.t > 1;
  UnpermArgs a{};
  a.comb = static_cast<const char*>(cd.v.comb);
  a.local_y = static_cast<const char*>(cd.v.expert_out);
  a.local_delta = cd.local_delta;
  a.local_lo = cd.node * c->L;
  a.local_hi = (cd.node + 1) * c->L;
  a.y_stride = c->row_bytes;
  a.slot_pos = cd.v.slot_pos;
  a.experts = cd.v.experts;
  a.probs = c->unit_probs ? cd.ones : cd.v.probs;
  a.k = d.top_k;
  const int64_t ct = d.tokens / n;
  a.tok_begin = int64_t(j) * ct;
  a.tok_end = a.tok_begin + ct;
  a.col_begin = dedup ? int64_t(cd.rho) * (d.hidden / d.t) : 0;
  a.cols = dedup ? d.hidden / d.t : d.hidden;
  a.out_stride = d.hidden * int64_t(c->ob);
  a.n_out = 0;
  if (dedup) {
    for (int r = 0; r < d.t; ++r) a.out[a.n_out++] = c->peer[card_of(c, cd.node, r)].out;
  } else {
    a.out[a.n_out++] = static_cast<char*>(cd.v.out);
  }
  a.wait = no_wait();
  a.wait.epoch_ptr = cd.epoch_dev;
  a.sig = no_signal();
  a.sig.epoch_ptr = cd.epoch_dev;
  a.sig.done = cd.done + kPsCAG * d.max_chunks + j;
  if (!is_virtual(c)) {
    for (int x = 0; x < d.e; ++x)
      if (x != cd.node) a.wait.flags[a.wait.n++] = flag_at(c, cd.id, sig_chunk(c, kPsCAA, j), card_of(c, x, cd.rho));
    if (dedup)
      for (int r = 0; r < d.t; ++r)
        if (r != cd.rho) a.sig.flags[a.sig.n++] = flag_at(c, card_of(c, cd.node, r), sig_chunk(c, kPsCAG, j), cd.id);
  }
  a.err = cd.err;
  {
    // a lone card's un-permute reads the rows its permute just wrote: newest
    // (highest tokens) first, while they are still in L2 (MONTA_UNPERM_REV
    // overrides, A/B)
    static const int rev = [] {
      const char* e = std::getenv("MONTA_UNPERM_REV");
      return e ? std::atoi(e) : -1;
    }();
    a.reverse = rev >= 0 ? rev : (is_virtual(c) && c->local.size() == 1 ? 1 : 0);
  }
  // resident CTAs (2 per SM at 256 threads); the launcher clamps to the item count
  const int grid = concurrent ? c->sms / 2 : c->sms;  // SM budget (the launcher sizes per kernel)
  if (moe_status st = hoist_wait(c, a.wait, cd.err, s)) return st;
  if (c->wire == MOE_WIRE_FP8 && d.e > 1) {  // decode this chunk's cross-node slots (fp8 combine leg)
    MONTA_CUDA(launch_comb_dequant(static_cast<char*>(cd.v.comb), c->peer[cd.id].cwire, c->peer[cd.id].cscale,
                                   cd.v.slot_pos, cd.v.experts, a.tok_begin, a.tok_end, d.top_k, c->L, cd.node,
                                   c->row_bytes, int(std::max<int64_t>(1, d.hidden / 128)), a.col_begin, a.cols, s));
    ++c->launches;
  }
  size_t sl;
  span_begin(c, MOE_STAGE_UNPERMUTE, j, s, &sl);
  bool ok = true;
  MONTA_CUDA(launch_unpermute(a, d.dtype, d.logit_dtype, d.out_dtype, grid, s, &ok));
  if (!ok) return fail(MOE_ERR_UNSUPPORTED, "combine: unsupported dtype combination (payload %d -> out %d)",
                       d.dtype, d.out_dtype);
  span_end(c, sl, s);
  ++c->launches;
  return MOE_OK;
}

// Whole combine of this card in one persistent cooperative launch: CAA role
// (reverse AllToAll per chunk) and UNP role (wait, un-permute + output
// all-gather store per chunk).  *done stays false when no persistent
// instantiation fits (dtype combination / alignment): per-launch path.
moe_status launch_combine_persistent(moe_ctx* c, Card& cd, int level, int n, cudaStream_t s, bool* done) {
  *done = false;
  const moe_layer_desc& d = c->d;
  const bool dedup = level != MOE_BASELINE && d.t > 1;
  const int vec = copy_vec(c, dedup);
  CombArgs x{};
  UnpermArgs& u = x.up;
  u.comb = static_cast<const char*>(cd.v.comb);
  u.local_y = static_cast<const char*>(cd.v.expert_out);
  u.local_delta = cd.local_delta;
  u.local_lo = cd.node * c->L;
  u.local_hi = (cd.node + 1) * c->L;
  u.y_stride = c->row_bytes;
  u.slot_pos = cd.v.slot_pos;
  u.experts = cd.v.experts;
  u.probs = c->unit_probs ? cd.ones : cd.v.probs;
  u.k = d.top_k;
  u.col_begin = dedup ? int64_t(cd.rho) * (d.hidden / d.t) : 0;
  u.cols = dedup ? d.hidden / d.t : d.hidden;
  u.out_stride = d.hidden * int64_t(c->ob);
  if (dedup) {
    for (int r = 0; r < d.t; ++r) u.out[u.n_out++] = c->peer[card_of(c, cd.node, r)].out;
  } else {
    u.out[u.n_out++] = static_cast<char*>(cd.v.out);
  }
  u.err = cd.err;
  CopyArgs& a = x.cp;
  a.pace_bpus = c->pace_bpus;  // applied by the reverse AllToAll only
  a.src = static_cast<const char*>(cd.v.expert_out);
  a.src_stride = c->row_bytes;
  a.dst_stride = c->row_bytes;
  for (int q = 0; q < c->cards; ++q) {
    if (!c->peer[q].slab) continue;
    a.dst[q] = c->peer[q].comb;
    x.flags[q] = c->peer[q].flags;
  }
  a.err = cd.err;
  x.lists = cd.lists;
  x.seg_cap = d.num_experts;
  x.max_chunks = d.max_chunks;
  x.n = n;
  x.me = cd.id;
  x.node = cd.node;
  x.rho = cd.rho;
  x.e = d.e;
  x.t = d.t;
  x.dedup = dedup ? 1 : 0;
  x.cpr = items_per_row(vec, dedup ? c->row_bytes / d.t : c->row_bytes);
  x.T = d.tokens;
  x.epoch_ptr = cd.epoch_dev;
  x.counters = cd.xchg_counters + 4 * d.max_chunks * 17;
  x.err = cd.err;
  x.dbg = c->debug ? cd.dbg + 18 : nullptr;
  if (c->timing) {
    x.trace = cd.xtrace + size_t(4) * d.max_chunks * 2;
    MONTA_CUDA(cudaMemsetAsync(x.trace, 0xff, size_t(4) * d.max_chunks * 2 * 8, s));
  }
  int max_ctas = 0;
  if (launch_combine_xchg(x, d.dtype, d.logit_dtype, d.out_dtype, vec, s, &max_ctas) != cudaSuccess) {
    cudaGetLastError();
    return MOE_OK;
  }
  if (max_ctas < 8) return MOE_OK;
  x.r_caa = 0;
  x.r_unp = max_ctas;  // every CTA runs both legs, software-pipelined over chunks
  size_t sl;
  span_begin(c, MOE_STAGE_UNPERMUTE, -1, s, &sl);
  const cudaError_t err = launch_combine_xchg(x, d.dtype, d.logit_dtype, d.out_dtype, vec, s, nullptr);
  if (err == cudaErrorNotSupported) {
    cudaGetLastError();
    return MOE_OK;
  }
  MONTA_CUDA(err);
  span_end(c, sl, s);
  ++c->launches;
  *done = true;
  return MOE_OK;
}

}  // namespace

namespace {

moe_status combine_impl(moe_ctx* c, int level, int n, cudaStream_t s) {
  if (c->last_level < 0 || !c->combine_ready)
    return fail(MOE_ERR_INVALID_ARGUMENT, "combine: no pending dispatch to mirror (one combine per dispatch)");
  if (n != c->last_n) return fail(MOE_ERR_INVALID_ARGUMENT, "combine: n = %d differs from the dispatch's %d", n, c->last_n);
  const bool dedup_d = c->last_level != MOE_BASELINE && c->d.t > 1;
  const bool dedup = level != MOE_BASELINE && c->d.t > 1;
  if (dedup != dedup_d)
    return fail(MOE_ERR_INVALID_ARGUMENT, "combine: level must mirror the dispatch (baseline vs deduplicated)");
  const moe_layer_desc& d = c->d;
  c->combine_ready = false;
  if (is_virtual(c)) {
    for (int j = 0; j < n; ++j) {
      for (auto& cd : c->local)
        if (moe_status st = launch_caa(c, cd, level, j, s, false)) return st;
      for (auto& cd : c->local)
        if (moe_status st = launch_unperm(c, cd, level, n, j, s, false)) return st;
    }
    return MOE_OK;
  }
  Card& cd = c->local[0];
  if (dedup && d.e == 1) {
    // Nothing orders a TP peer's output stores after this rank's previous
    // read of `out` when there is no cross-node leg: barrier the node.
    SignalList sg = no_signal();
    sg.epoch_ptr = cd.epoch_dev;
    WaitList w = no_wait();
    w.epoch_ptr = cd.epoch_dev;
    for (int r = 0; r < d.t; ++r)
      if (r != cd.rho) {
        sg.flags[sg.n++] = flag_at(c, card_of(c, cd.node, r), kSigBarrier, cd.id);
        w.flags[w.n++] = flag_at(c, cd.id, kSigBarrier, card_of(c, cd.node, r));
      }
    MONTA_CUDA(launch_signal(sg, s));
    MONTA_CUDA(launch_wait(w, cd.err, s));
    c->launches += 2;
  }
  // Unchunked without TP dedup, nothing overlaps the reverse AllToAll and the
  // un-permute writes only local HBM: a separate launch of the top-k item
  // kernel (3-4 CTAs per SM) beats the persistent kernel's register-capped
  // un-permute, so only chunked or deduplicated combines go persistent.
  if (c->use_xchg && c->aa_ctas == 0 && c->wire == MOE_WIRE_BF16 && (n > 1 || dedup)) {
    bool done = false;
    if (moe_status st = launch_combine_persistent(c, cd, level, n, s, &done)) return st;
    if (done) return MOE_OK;
  }
  MONTA_CUDA(cudaEventRecord(c->ev_fork, s));
  MONTA_CUDA(cudaStreamWaitEvent(c->s_aa, c->ev_fork, 0));
  MONTA_CUDA(cudaStreamWaitEvent(c->s_ag, c->ev_fork, 0));
  if (c->pipe) {
    MONTA_CUDA(cudaEventRecord(c->ev_fork, s));
    MONTA_CUDA(cudaStreamWaitEvent(c->s_d2h, c->ev_fork, 0));
  }
  const size_t crow = size_t(d.hidden) * c->ob;
  const int64_t ct = d.tokens / n;
  for (int j = 0; j < n; ++j) {
    if (moe_status st = launch_caa(c, cd, level, j, c->s_aa, true)) return st;
    if (moe_status st = launch_unperm(c, cd, level, n, j, c->s_ag, true)) return st;
    if (c->pipe) {  // chunk j's output rows leave for the host as soon as they are complete
      MONTA_CUDA(cudaEventRecord(c->ev_d2h[j], c->s_ag));
      MONTA_CUDA(cudaStreamWaitEvent(c->s_d2h, c->ev_d2h[j], 0));
      if (dedup) {  // the TP peers' slices of chunk j (their un-permute stores into this card's out)
        WaitList w = no_wait();
        w.epoch_ptr = cd.epoch_dev;
        for (int r = 0; r < d.t; ++r)
          if (r != cd.rho) w.flags[w.n++] = flag_at(c, cd.id, sig_chunk(c, kPsCAG, j), card_of(c, cd.node, r));
        MONTA_CUDA(launch_wait(w, cd.err, c->s_d2h));
        ++c->launches;
      }
      MONTA_CUDA(cudaMemcpyAsync(c->pipe_ho + size_t(j) * ct * crow, static_cast<const char*>(cd.v.out) +
                                 size_t(j) * ct * crow, size_t(ct) * crow, cudaMemcpyDeviceToHost, c->s_d2h));
    }
  }
  MONTA_CUDA(cudaEventRecord(c->ev_join_aa, c->s_aa));
  MONTA_CUDA(cudaEventRecord(c->ev_join_ag, c->s_ag));
  MONTA_CUDA(cudaStreamWaitEvent(s, c->ev_join_aa, 0));
  MONTA_CUDA(cudaStreamWaitEvent(s, c->ev_join_ag, 0));
  if (c->pipe) {
    MONTA_CUDA(cudaEventRecord(c->ev_join_d2h, c->s_d2h));
    MONTA_CUDA(cudaStreamWaitEvent(s, c->ev_join_d2h, 0));
  }
  if (dedup) {
    WaitList w = no_wait();
    w.epoch_ptr = cd.epoch_dev;
    for (int j = 0; j < n; ++j) {
      if (w.n + d.t - 1 > kMaxCards) {
        MONTA_CUDA(launch_wait(w, cd.err, s));
        ++c->launches;
        w.n = 0;
      }
      for (int r = 0; r < d.t; ++r)
        if (r != cd.rho) w.flags[w.n++] = flag_at(c, cd.id, sig_chunk(c, kPsCAG, j), card_of(c, cd.node, r));
    }
    if (w.n) {
      MONTA_CUDA(launch_wait(w, cd.err, s));
      ++c->launches;
    }
  }
  return MOE_OK;
}

}  // namespace

namespace {
moe_status experts_impl(moe_ctx* c, cudaStream_t s);
}  // namespace

extern "C" moe_status moe_ctx_experts(moe_ctx* c, void* stream) {
  if (moe_status st = check_ready(c)) return st;
  MONTA_CUDA(cudaSetDevice(c->device));
  return experts_impl(c, static_cast<cudaStream_t>(stream));
}

extern "C" moe_status moe_ctx_combine(moe_ctx* c, int level, int32_t n, void* stream) {
  if (moe_status st = check_ready(c)) return st;
  MONTA_CUDA(cudaSetDevice(c->device));
  return combine_impl(c, level, n, static_cast<cudaStream_t>(stream));
}

namespace {

// route + dispatch + combine, optionally wrapped in host<->device copies.
// Single-card end to end with host buffers, pipelined per token chunk: the
// host->device copy of chunk j+1, the layer of chunk j (its rows never leave
// the chunk on one card: AA(j) then un-permute(j)) and the device->host copy
// of chunk j-1 run concurrently (copy engines both ways + SMs).  The result
// is identical to the unpipelined path; only the schedule differs.
moe_status forward_host_pipelined(moe_ctx* c, int level, int landing, const void* hx, const void* hl, void* ho,
                                  cudaStream_t s) {
  const moe_layer_desc& d = c->d;
  Card& cd = c->local[0];
  int P = std::min(16, d.max_chunks);
  while (P > 1 && d.tokens % P) --P;
  const int64_t ct = d.tokens / P;
  const size_t xrow = size_t(c->row_bytes), orow = size_t(d.hidden) * c->ob;
  const size_t lbytes = size_t(d.tokens) * d.num_experts * c->lb;
  MONTA_CUDA(cudaMemcpyAsync(cd.v.logits, hl, lbytes, cudaMemcpyHostToDevice, s));
  // x chunks on the copy-in stream
  MONTA_CUDA(cudaEventRecord(c->ev_fork, s));
  MONTA_CUDA(cudaStreamWaitEvent(c->s_aa, c->ev_fork, 0));
  MONTA_CUDA(cudaStreamWaitEvent(c->s_d2d, c->ev_fork, 0));
  for (int j = 0; j < P; ++j) {
    MONTA_CUDA(cudaMemcpyAsync(static_cast<char*>(cd.v.x) + size_t(j) * ct * xrow,
                               static_cast<const char*>(hx) + size_t(j) * ct * xrow, size_t(ct) * xrow,
                               cudaMemcpyHostToDevice, c->s_aa));
    MONTA_CUDA(cudaEventRecord(c->ev_aa[j], c->s_aa));
  }
  c->last_level = level;
  c->last_n = P;
  c->last_landing = MOE_LAND_FINAL;
  if (moe_status st = do_front(c, true, level, P, MOE_LAND_FINAL, s)) return st;
  for (int j = 0; j < P; ++j) {
    MONTA_CUDA(cudaStreamWaitEvent(s, c->ev_aa[j], 0));
    if (moe_status st = launch_aa(c, cd, level, j, MOE_LAND_FINAL, s, false)) return st;
    if (moe_status st = launch_unperm(c, cd, level, P, j, s, false)) return st;
    MONTA_CUDA(cudaEventRecord(c->ev_ag[j], s));
    MONTA_CUDA(cudaStreamWaitEvent(c->s_d2d, c->ev_ag[j], 0));
    MONTA_CUDA(cudaMemcpyAsync(static_cast<char*>(ho) + size_t(j) * ct * orow,
                               static_cast<const char*>(cd.v.out) + size_t(j) * ct * orow, size_t(ct) * orow,
                               cudaMemcpyDeviceToHost, c->s_d2d));
  }
  MONTA_CUDA(cudaEventRecord(c->ev_join_d2d, c->s_d2d));
  MONTA_CUDA(cudaEventRecord(c->ev_join_aa, c->s_aa));
  MONTA_CUDA(cudaStreamWaitEvent(s, c->ev_join_d2d, 0));
  MONTA_CUDA(cudaStreamWaitEvent(s, c->ev_join_aa, 0));
  c->combine_ready = false;
  return MOE_OK;
}

// Routing check of the last dispatch (checks enabled): every landed row's
// tags against the receiving node's reference layout (verify.cu).
moe_status verify_dispatch(moe_ctx* c, cudaStream_t s) {
  if (!c->checks) return MOE_OK;
  if (!is_virtual(c))
    if (moe_status st = dispatch_tail_wait(c, c->local[0], c->last_level, c->last_n, MOE_LAND_FINAL, s)) return st;
  for (auto& cd : c->local) {
    MONTA_CUDA(launch_verify_recv(cd.v.recv_tags, cd.recv_rows, cd.v.recv_expert_offsets, c->L, cd.node, c->d.e,
                                  c->d.t, c->d.tokens, c->recv_cap, cd.err, s));
    ++c->launches;
  }
  return MOE_OK;
}

// Bound experts between dispatch and combine.  Multi-GPU:
// the persistent dispatch returns before the peers' rows have landed, so the
// experts first wait for every incoming chunk (the flags the combine would
// wait on); then the SwiGLU FFN over the card's expert-major recv segments.
moe_status experts_impl(moe_ctx* c, cudaStream_t s) {
  bool any = false;
  for (auto& cd : c->local) any |= cd.w13 != nullptr;
  if (!any) return MOE_OK;
  if (c->last_level < 0 || !c->combine_ready)
    return fail(MOE_ERR_INVALID_ARGUMENT, "experts: no dispatched rows to compute on");
  if (!is_virtual(c))
    if (moe_status st = dispatch_tail_wait(c, c->local[0], c->last_level, c->last_n, MOE_LAND_FINAL, s)) return st;
  const int64_t h = c->d.hidden;
  for (auto& cd : c->local) {
    if (!cd.w13) continue;
    size_t sl;
    span_begin(c, MOE_STAGE_EXPERTS, -1, s, &sl);
    // under TP dedup the combine reads only this card's 1/t column slice
    const bool slice = c->last_level != MOE_BASELINE && c->d.t > 1 && (h / c->d.t) % 128 == 0;
    const int64_t oc0 = slice ? int64_t(cd.rho) * (h / c->d.t) : 0, ocn = slice ? h / c->d.t : h;
    if (moe_status st = expert_ffn_fused(cd.v.recv, h, c->recv_cap, cd.w13, cd.w2, cd.v.recv_expert_offsets, c->L, h,
                                         cd.ffn, cd.ffn_ws, cd.v.expert_out, h, nullptr, 0, 0, oc0, ocn, s))
      return st;
    span_end(c, sl, s);
    c->launches += 2;
  }
  return MOE_OK;
}

// Expert compute fused with the reverse AllToAll (the
// reference gates its expert task on the dispatch terminals and its combine
// on the expert task, pipesim.hpp:102).  The down-projection GEMM's epilogue
// stores every finished 128-row tile to this card's expert outputs AND, for
// rows whose source sits on another node, straight into that source card's
// landing buffer (`comb`) over NVLink — the reverse AllToAll leaves tile by
// tile while the tensor cores work on the next tiles, in one kernel (the row
// addresses come from the chunk CAA lists, k_rowdst).  One signal kernel then
// releases every chunk's CAA flags and the un-permute runs as in the
// per-launch combine.  Results are identical to experts-then-combine.
bool overlap_experts(const moe_ctx* c) {
  if (is_virtual(c) || !c->expert_fused || c->d.e < 2 || c->wire != MOE_WIRE_BF16 || c->pace_bpus) return false;
  return c->local.size() == 1 && c->local[0].w13 != nullptr;
}

moe_status experts_combine_fused(moe_ctx* c, int level, int n, cudaStream_t s) {
  const moe_layer_desc& d = c->d;
  Card& cd = c->local[0];
  if (c->last_level < 0 || !c->combine_ready)
    return fail(MOE_ERR_INVALID_ARGUMENT, "experts: no dispatched rows to compute on");
  if (n != c->last_n) return fail(MOE_ERR_INVALID_ARGUMENT, "combine: n = %d differs from the dispatch's %d", n, c->last_n);
  if ((level != MOE_BASELINE && d.t > 1) != (c->last_level != MOE_BASELINE && d.t > 1))
    return fail(MOE_ERR_INVALID_ARGUMENT, "combine: level must mirror the dispatch (baseline vs deduplicated)");
  const bool dedup = level != MOE_BASELINE && d.t > 1;
  if (moe_status st = dispatch_tail_wait(c, cd, c->last_level, c->last_n, MOE_LAND_FINAL, s)) return st;
  PeerRows comb{};
  for (int q = 0; q < c->cards; ++q)
    if (c->peer[q].slab) comb.base[q] = c->peer[q].comb;
  MONTA_CUDA(launch_rowdst(list_of(c, cd, kPhaseCAA, 0), seglist_bytes(d.num_experts), n, d.num_experts, comb,
                           c->row_bytes, cd.rowdst, c->recv_cap, s));
  ++c->launches;
  // the CAA column window of this card: its 1/t slice under TP dedup, else the row
  const int32_t col_lo = dedup ? int32_t(int64_t(cd.rho) * (c->row_bytes / d.t)) : 0;
  const int32_t col_hi = dedup ? int32_t(col_lo + c->row_bytes / d.t) : int32_t(c->row_bytes);
  size_t sl;
  span_begin(c, MOE_STAGE_EXPERTS, -1, s, &sl);
  // under TP dedup this card's combine reads only its 1/t column slice of
  // the expert outputs (local rows in place, remote rows via the fused
  // stores): the down-projection computes just that slice
  const bool slice = dedup && (d.hidden / d.t) % 128 == 0;  // the GEMM's 128-column blocks
  const int64_t oc0 = slice ? int64_t(cd.rho) * (d.hidden / d.t) : 0;
  const int64_t ocn = slice ? d.hidden / d.t : d.hidden;
  if (moe_status st = expert_ffn_fused(cd.v.recv, d.hidden, c->recv_cap, cd.w13, cd.w2, cd.v.recv_expert_offsets, c->L,
                                       d.hidden, cd.ffn, cd.ffn_ws, cd.v.expert_out, d.hidden, cd.rowdst, col_lo, col_hi,
                                       oc0, ocn, s))
    return st;
  span_end(c, sl, s);
  c->launches += 2;
  c->combine_ready = false;
  // every chunk's rows have left: release the sources' CAA flags
  SignalList sg = no_signal();
  sg.epoch_ptr = cd.epoch_dev;
  for (int j = 0; j < n; ++j)
    for (int g = 0; g < d.e; ++g) {
      if (g == cd.node) continue;
      if (sg.n == kMaxCards) {
        MONTA_CUDA(launch_signal(sg, s));
        ++c->launches;
        sg.n = 0;
      }
      sg.flags[sg.n++] = flag_at(c, card_of(c, g, cd.rho), sig_chunk(c, kPsCAA, j), cd.id);
    }
  if (sg.n) {
    MONTA_CUDA(launch_signal(sg, s));
    ++c->launches;
  }
  for (int j = 0; j < n; ++j)
    if (moe_status st = launch_unperm(c, cd, level, n, j, s, false)) return st;
  if (dedup) {
    WaitList w = no_wait();
    w.epoch_ptr = cd.epoch_dev;
    for (int j = 0; j < n; ++j) {
      if (w.n + d.t - 1 > kMaxCards) {
        MONTA_CUDA(launch_wait(w, cd.err, s));
        ++c->launches;
        w.n = 0;
      }
      for (int r = 0; r < d.t; ++r)
        if (r != cd.rho) w.flags[w.n++] = flag_at(c, cd.id, sig_chunk(c, kPsCAG, j), card_of(c, cd.node, r));
    }
    if (w.n) {
      MONTA_CUDA(launch_wait(w, cd.err, s));
      ++c->launches;
    }
  }
  return MOE_OK;
}

// forward_host on a multi-GPU rank, pipelined per token chunk: the x rows of
// chunk j go up on their own stream while the front routes (it needs only
// the logits), the chunk's AllToAll waits for them, and the chunk's output
// rows go down as soon as its un-permute (and, under TP dedup, the peers'
// slices of it) landed.  The final layout does not depend on the chunk count,
// so the result equals the caller's schedule; the exchange runs on the
// per-launch kernels (the persistent ones cannot wait for copies).
bool host_pipeline_ok(const moe_ctx* c, int landing) {
  // EP-only topologies (t == 1): under TP the 2x2 run measured no gain (4 GPUs
  // share the host's copy bandwidth: 5.5 -> 5.1 ms, and 7.8 ms replayed as a
  // graph against 5.5 ms for the persistent exchange)
  static const int env = [] {  // 0: off, 2: also under TP (diagnosis)
    const char* e = std::getenv("MONTA_HOST_PIPE");
    return e ? std::atoi(e) : 1;
  }();
  if (env == 0 || (c->d.t != 1 && env != 2)) return false;
  return !(is_virtual(c) || c->local.size() != 1 || c->timing || landing != MOE_LAND_FINAL || c->local[0].w13 ||
           c->wire != MOE_WIRE_BF16 || c->pace_bpus || c->d.tokens <= 0);
}

moe_status forward_impl(moe_ctx* c, int level, int n, int landing, const void* hx, const void* hl, void* ho,
                        cudaStream_t s);

moe_status forward_host_multi(moe_ctx* c, int level, const void* hx, const void* hl, void* ho, cudaStream_t s) {
  const moe_layer_desc& d = c->d;
  Card& cd = c->local[0];
  int P = std::min(8, d.max_chunks);
  while (P > 1 && d.tokens % P) --P;
  const int64_t ct = d.tokens / P;
  const size_t xrow = size_t(c->row_bytes);
  MONTA_CUDA(cudaMemcpyAsync(cd.v.logits, hl, size_t(d.tokens) * d.num_experts * c->lb, cudaMemcpyHostToDevice, s));
  MONTA_CUDA(cudaEventRecord(c->ev_fork, s));
  MONTA_CUDA(cudaStreamWaitEvent(c->s_h2d, c->ev_fork, 0));
  for (int j = 0; j < P; ++j) {
    MONTA_CUDA(cudaMemcpyAsync(static_cast<char*>(cd.v.x) + size_t(j) * ct * xrow,
                               static_cast<const char*>(hx) + size_t(j) * ct * xrow, size_t(ct) * xrow,
                               cudaMemcpyHostToDevice, c->s_h2d));
    MONTA_CUDA(cudaEventRecord(c->ev_h2d[j], c->s_h2d));
  }
  // chunked O3 with final landing (rows at their final offsets, no reorder
  // copies): the only chunked schedule the reference's levels allow with
  // final landing; every level's combine gives the same output rows
  (void)level;
  const int lv = MOE_O3;
  const bool saved = c->use_xchg;
  c->use_xchg = false;
  c->pipe = true;
  c->pipe_ho = static_cast<char*>(ho);
  moe_status st = forward_impl(c, lv, P, MOE_LAND_FINAL, nullptr, nullptr, nullptr, s);
  c->pipe = false;
  c->pipe_ho = nullptr;
  c->use_xchg = saved;
  return st;
}

moe_status forward_impl(moe_ctx* c, int level, int n, int landing, const void* hx, const void* hl, void* ho,
                        cudaStream_t s) {
  const moe_layer_desc& d = c->d;
  // a lone card with FINAL landing: its result does not depend on the chunk
  // count, so forward_host picks its own (pipelining) chunking; STAGED
  // landing (pre/pre_tags populated per the caller's n) takes the plain path
  if (hx && is_virtual(c) && c->local.size() == 1 && !c->timing && c->d.tokens > 0 && landing == MOE_LAND_FINAL &&
      !c->local[0].w13)  // bound experts need every chunk's rows before they run
    return forward_host_pipelined(c, level, landing, hx, hl, ho, s);
  const size_t xbytes = size_t(d.tokens) * c->row_bytes;
  const size_t lbytes = size_t(d.tokens) * d.num_experts * c->lb;
  const size_t obytes = size_t(d.tokens) * d.hidden * c->ob;
  if (hx && ho && host_pipeline_ok(c, landing))
    return forward_host_multi(c, level, hx, hl, ho, s);
  if (hx)
    for (size_t i = 0; i < c->local.size(); ++i) {
      MONTA_CUDA(cudaMemcpyAsync(c->local[i].v.x, static_cast<const char*>(hx) + i * xbytes, xbytes,
                                 cudaMemcpyHostToDevice, s));
      MONTA_CUDA(cudaMemcpyAsync(c->local[i].v.logits, static_cast<const char*>(hl) + i * lbytes, lbytes,
                                 cudaMemcpyHostToDevice, s));
    }
  if (c->timing) {
    c->span_used = 0;
    record_timing(c->ev_base, s);
  }
  c->in_forward = true;
  moe_status st = dispatch_impl(c, level, n, landing, s, true);
  c->in_forward = false;
  if (st != MOE_OK) return st;
  if (moe_status st0 = verify_dispatch(c, s)) return st0;
  if (overlap_experts(c)) {
    if (moe_status st1 = experts_combine_fused(c, level, n, s)) return st1;
  } else {
    if (moe_status st1 = experts_impl(c, s)) return st1;
    if (moe_status st2 = combine_impl(c, level, n, s)) return st2;
  }
  if (ho)
    for (size_t i = 0; i < c->local.size(); ++i)
      MONTA_CUDA(cudaMemcpyAsync(static_cast<char*>(ho) + i * obytes, c->local[i].v.out, obytes,
                                 cudaMemcpyDeviceToHost, s));
  return MOE_OK;
}

// CUDA-graph path: the whole step (every stream of it) is captured once per
// (level, n, landing, host buffers) and replayed; flags carry the device
// epoch, so replays stay in lockstep across ranks.
moe_status backward_impl(moe_ctx* c, int level, int n, cudaStream_t s);

moe_status forward_graph(moe_ctx* c, int level, int n, int landing, const void* hx, const void* hl, void* ho,
                         cudaStream_t s, int kind = 0) {
  auto run = [&](cudaStream_t st) {
    return kind ? backward_impl(c, level, n, st) : forward_impl(c, level, n, landing, hx, hl, ho, st);
  };
  for (auto& g : c->graphs)
    if (g.kind == kind && g.level == level && g.n == n && g.landing == landing && g.hx == hx && g.hl == hl &&
        g.ho == ho && g.timed == c->timing) {
      if (!g.exec) return run(s);
      if (g.timed) {  // the replay re-records the captured events: restore their labels
        c->span_used = g.span_labels.size();
        for (size_t i = 0; i < g.span_labels.size(); ++i) {
          c->spans[i].stage = g.span_labels[i].first;
          c->spans[i].chunk = g.span_labels[i].second;
        }
      }
      c->last_level = level;
      c->last_n = n;
      c->last_landing = level == MOE_BASELINE ? MOE_LAND_FINAL : landing;
      c->combine_ready = false;
      MONTA_CUDA(cudaGraphLaunch(g.exec, s));
      c->launches += g.kernels;
      return MOE_OK;
    }
  // capture on the context's own stream (the legacy stream cannot be captured)
  moe_ctx::GraphEntry e{kind, level, n, landing, hx, hl, ho, nullptr, 0, c->timing, {}};
  const int64_t before = c->launches;
  MONTA_CUDA(cudaStreamBeginCapture(c->s_cap, cudaStreamCaptureModeThreadLocal));
  moe_status st = run(c->s_cap);
  cudaGraph_t graph = nullptr;
  cudaError_t err = cudaStreamEndCapture(c->s_cap, &graph);
  e.kernels = c->launches - before;
  c->launches = before;
  if (e.timed)
    for (size_t i = 0; i < c->span_used; ++i) e.span_labels.emplace_back(c->spans[i].stage, c->spans[i].chunk);
  if (st != MOE_OK) {
    if (graph) cudaGraphDestroy(graph);
    return st;
  }
  if (err != cudaSuccess || !graph || cudaGraphInstantiate(&e.exec, graph, 0) != cudaSuccess) {
    cudaGetLastError();  // capture unsupported here (e.g. pageable host memory): run eagerly from now on
    if (graph) cudaGraphDestroy(graph);
    e.exec = nullptr;
    c->graphs.push_back(e);
    return run(s);
  }
  cudaGraphDestroy(graph);
  c->graphs.push_back(e);
  return forward_graph(c, level, n, landing, hx, hl, ho, s, kind);
}

}  // namespace

extern "C" moe_status moe_ctx_set_link_rate(moe_ctx* c, double gbps) {
  if (moe_status st = check_ready(c)) return st;
  if (!(gbps >= 0.0) || gbps > 4.0e6) return fail(MOE_ERR_INVALID_ARGUMENT, "set_link_rate: bad rate %g GB/s", gbps);
  const uint32_t bpus = uint32_t(gbps * 1000.0 + 0.5);
  if (bpus != c->pace_bpus) {
    for (auto& g : c->graphs)
      if (g.exec) cudaGraphExecDestroy(g.exec);
    c->graphs.clear();
  }
  c->pace_bpus = bpus;
  return MOE_OK;
}

extern "C" moe_status moe_ctx_set_wire(moe_ctx* c, int wire) {
  if (moe_status st = check_ready(c)) return st;
  if (wire != MOE_WIRE_BF16 && wire != MOE_WIRE_FP8) return fail(MOE_ERR_INVALID_ARGUMENT, "set_wire: unknown format %d", wire);
  const moe_layer_desc& d = c->d;
  if (wire == MOE_WIRE_FP8 && (d.dtype != MOE_BF16 || d.hidden % 128 || (d.hidden / d.t) % 128 || d.top_k > 16))
    return fail(MOE_ERR_INVALID_ARGUMENT,
                "set_wire: the fp8 wire needs a bf16 payload, hidden and hidden/t multiples of 128, top_k <= 16");
  if (c->wire != wire) {
    for (auto& g : c->graphs)
      if (g.exec) cudaGraphExecDestroy(g.exec);
    c->graphs.clear();
  }
  c->wire = wire;
  return MOE_OK;
}

extern "C" moe_status moe_ctx_enable_checks(moe_ctx* c, int enable) {
  if (moe_status st = check_ready(c)) return st;
  if (c->checks != (enable != 0)) {
    for (auto& g : c->graphs)
      if (g.exec) cudaGraphExecDestroy(g.exec);
    c->graphs.clear();
  }
  c->checks = enable != 0;
  return MOE_OK;
}

extern "C" moe_status moe_ctx_verify(moe_ctx* c, void* stream) {
  if (moe_status st = check_ready(c)) return st;
  if (!c->checks) return fail(MOE_ERR_INVALID_ARGUMENT, "verify: checks not enabled (moe_ctx_enable_checks)");
  MONTA_CUDA(cudaSetDevice(c->device));
  return verify_dispatch(c, static_cast<cudaStream_t>(stream));
}

extern "C" moe_status moe_ctx_forward(moe_ctx* c, int level, int32_t n, int landing, void* stream) {
  if (moe_status st = check_ready(c)) return st;
  if (moe_status st = validate_dispatch(c, level, n, landing)) return st;
  MONTA_CUDA(cudaSetDevice(c->device));
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (c->use_graphs) return forward_graph(c, level, n, landing, nullptr, nullptr, nullptr, s);
  return forward_impl(c, level, n, landing, nullptr, nullptr, nullptr, s);
}

// In-place schedule selection: every candidate (level, n, landing) runs
// `steps` timed forwards through this context (after two warm-ups); on a
// multi-GPU context the per-candidate times are max-reduced over the ranks
// through the peers' slabs (stores + epoch flags), so every rank picks the
// same schedule.  The reference's select_strategy stays exact; this is the
// measured decision (SURVEY §8(a) planner row on one NVSwitch box).
extern "C" moe_status moe_ctx_autotune(moe_ctx* c, moe_schedule* cand, int32_t count, int32_t steps, void* stream,
                                       int32_t* best) {
  if (moe_status st = check_ready(c)) return st;
  if (!cand || !best || count < 1 || count > kMaxTune || steps < 1)
    return fail(MOE_ERR_INVALID_ARGUMENT, "autotune: need 1..%d candidates, steps >= 1, outputs", kMaxTune);
  for (int i = 0; i < count; ++i)
    if (moe_status st = validate_dispatch(c, cand[i].level, cand[i].n_chunks, cand[i].landing)) return st;
  MONTA_CUDA(cudaSetDevice(c->device));
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  cudaEvent_t e0, e1;
  MONTA_CUDA(cudaEventCreate(&e0));
  MONTA_CUDA(cudaEventCreate(&e1));
  std::vector<double> local(size_t(kMaxTune), 0.0);
  moe_status st = MOE_OK;
  for (int i = 0; i < count && st == MOE_OK; ++i) {
    for (int w = 0; w < 2 + steps && st == MOE_OK; ++w) {
      if (w == 2) cudaEventRecord(e0, s);
      st = moe_ctx_forward(c, cand[i].level, cand[i].n_chunks, cand[i].landing, stream);
    }
    cudaEventRecord(e1, s);
    if (cudaEventSynchronize(e1) != cudaSuccess) st = cuda_fail(cudaGetLastError(), "autotune");
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    local[size_t(i)] = double(ms) * 1e3 / steps;
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  if (st != MOE_OK) return st;
  if (moe_status s2 = moe_ctx_sync(c)) return s2;
  std::vector<double> worst(local.begin(), local.begin() + count);
  if (!is_virtual(c)) {
    Card& cd = c->local[0];
    const uint64_t epoch = ++c->tune_epoch;
    for (int q = 0; q < c->cards; ++q)  // my times into every card's [me] row (mine included)
      if (c->peer[q].slab)
        MONTA_CUDA(cudaMemcpyAsync(c->peer[q].slab + c->lay.tune + size_t(cd.id) * kMaxTune * 8, local.data(),
                                   size_t(count) * 8, cudaMemcpyHostToDevice, s));
    SignalList sg = no_signal();
    sg.epoch = epoch;
    WaitList w = no_wait();
    w.epoch = epoch;
    for (int q = 0; q < c->cards; ++q)
      if (q != cd.id && c->peer[q].slab) {
        sg.flags[sg.n++] = flag_at(c, q, sig_tune(c), cd.id);
        w.flags[w.n++] = flag_at(c, cd.id, sig_tune(c), q);
      }
    MONTA_CUDA(launch_signal(sg, s));
    MONTA_CUDA(launch_wait(w, cd.err, s));
    std::vector<double> all(size_t(c->cards) * kMaxTune);
    MONTA_CUDA(cudaMemcpyAsync(all.data(), cd.slab + c->lay.tune, all.size() * 8, cudaMemcpyDeviceToHost, s));
    MONTA_CUDA(cudaStreamSynchronize(s));
    if (moe_status s3 = moe_ctx_sync(c)) return s3;
    for (int q = 0; q < c->cards; ++q)
      for (int i = 0; i < count; ++i) worst[size_t(i)] = std::max(worst[size_t(i)], all[size_t(q) * kMaxTune + i]);
  }
  int b = 0;
  for (int i = 0; i < count; ++i) {
    cand[i].us = worst[size_t(i)];
    if (worst[size_t(i)] < worst[size_t(b)]) b = i;  // ties keep the earlier candidate
  }
  *best = b;
  return MOE_OK;
}

// ---------------------------------------------------------------------------
// Layer backward on the device (the reference has none).
namespace {

// recv <-> pre in every local view and every peer pointer: the gradient
// dispatch lands in the `pre` memory (FINAL landing never stages), so the
// forward's dispatched rows / expert outputs in recv stay intact.
void swap_recv_pre(moe_ctx* c) {
  for (auto& cd : c->local) {
    const bool eo = cd.v.expert_out == cd.v.recv;
    std::swap(cd.v.recv, cd.v.pre);
    std::swap(cd.v.recv_tags, cd.v.pre_tags);
    if (eo) cd.v.expert_out = cd.v.recv;
  }
  for (int q = 0; q < c->cards; ++q) {
    std::swap(c->peer[q].recv, c->peer[q].pre);
    std::swap(c->peer[q].recv_tags, c->peer[q].pre_tags);
  }
}

BwdPeers bwd_peers(moe_ctx* c) {
  BwdPeers pe{};
  for (int q = 0; q < c->cards; ++q) {
    pe.experts[q] = c->peer[q].experts;
    pe.probs[q] = c->peer[q].probs;
    pe.parts[q] = c->peer[q].parts;
  }
  return pe;
}

// combine adjoint: grad_out (each card's x buffer) -> the forward's dispatch
// (same level / n, FINAL landing into `pre`) -> per landed row g:
// grad_y = p * g in place in `pre`, partial <g, y> over the card's column
// slice -> every TP card of the source node -> grad_probs -> grad_logits.
moe_status backward_combine_impl(moe_ctx* c, int level, int n, cudaStream_t s) {
  const moe_layer_desc& d = c->d;
  if (d.dtype == MOE_I64) return fail(MOE_ERR_INVALID_ARGUMENT, "backward: integer payloads have no gradient");
  swap_recv_pre(c);
  moe_status st = dispatch_impl(c, level, n, MOE_LAND_FINAL, s, false);
  if (st == MOE_OK && !is_virtual(c)) st = dispatch_tail_wait(c, c->local[0], level, n, MOE_LAND_FINAL, s);
  swap_recv_pre(c);
  if (st != MOE_OK) return st;
  const BwdPeers pe = bwd_peers(c);
  const int64_t h = d.hidden, w = d.hidden / d.t;
  const size_t es = c->xb;
  const int ydt = d.dtype, pdt = d.logit_dtype;
  for (auto& cd : c->local) {
    MONTA_CUDA(launch_row_meta(pdt, cd.v.pre_tags, cd.recv_rows, c->recv_cap, d.t, cd.rho, d.top_k, pe, cd.prow,
                               cd.rowpos, cd.rowslot, cd.err, s));
    // partial dot over this card's column slice first (needs g), then grad_y = p * g in place
    const size_t off = size_t(cd.rho) * size_t(w) * es;
    if (moe_status s1 = moe_combine_backward(static_cast<char*>(cd.v.pre) + off, ydt, h,
                                             static_cast<const char*>(cd.v.expert_out) + off, ydt, h, w, cd.rowpos,
                                             cd.prow, pdt, c->recv_cap, 1, nullptr, h, cd.dot, s))
      return s1;
    if (moe_status s2 = moe_combine_backward(cd.v.pre, ydt, h, nullptr, ydt, h, h, cd.rowpos, cd.prow, pdt,
                                             c->recv_cap, 1, cd.v.pre, h, nullptr, s))
      return s2;
    MONTA_CUDA(launch_scatter_parts(pdt, cd.v.pre_tags, cd.recv_rows, c->recv_cap, d.t, cd.rho, d.top_k,
                                    cd.rowslot, cd.dot, pe, s));
    c->launches += 4;
  }
  if (!is_virtual(c)) {  // every card's partials landed (stores into this card) before the sums
    Card& cd = c->local[0];
    SignalList sg = no_signal();
    sg.epoch_ptr = cd.epoch_dev;
    WaitList wl = no_wait();
    wl.epoch_ptr = cd.epoch_dev;
    for (int q = 0; q < c->cards; ++q)
      if (q != cd.id) {
        sg.flags[sg.n++] = flag_at(c, q, sig_bwd(c), cd.id);
        wl.flags[wl.n++] = flag_at(c, cd.id, sig_bwd(c), q);
      }
    MONTA_CUDA(launch_signal(sg, s));
    MONTA_CUDA(launch_wait(wl, cd.err, s));
    c->launches += 2;
  }
  for (auto& cd : c->local) {
    MONTA_CUDA(launch_sum_parts(pdt, cd.parts, cd.v.experts, d.tokens * d.top_k, d.t, cd.v.grad_probs, s));
    if (moe_status s3 = moe_route_backward(cd.v.logits, pdt, d.tokens, d.num_experts, d.top_k, cd.v.experts,
                                           cd.v.grad_probs, cd.v.grad_logits, s))
      return s3;
    c->launches += 2;
  }
  return MOE_OK;
}

// dispatch adjoint: grad_x = the forward combine with unit weights over the
// gradient rows in `pre` (grad_y, or the caller's expert-input gradient).
moe_status backward_dispatch_impl(moe_ctx* c, int level, int n, cudaStream_t s) {
  std::vector<void*> saved;
  for (auto& cd : c->local) {
    saved.push_back(cd.v.expert_out);
    cd.v.expert_out = cd.v.pre;
  }
  c->unit_probs = true;
  const moe_status st = combine_impl(c, level, n, s);
  c->unit_probs = false;
  for (size_t i = 0; i < c->local.size(); ++i) c->local[i].v.expert_out = saved[i];
  return st;
}

}  // namespace

extern "C" moe_status moe_ctx_backward_combine(moe_ctx* c, int level, int32_t n, void* stream) {
  if (moe_status st = check_ready(c)) return st;
  if (moe_status st = validate_dispatch(c, level, n, MOE_LAND_FINAL)) return st;
  MONTA_CUDA(cudaSetDevice(c->device));
  return backward_combine_impl(c, level, n, static_cast<cudaStream_t>(stream));
}

extern "C" moe_status moe_ctx_backward_dispatch(moe_ctx* c, int level, int32_t n, void* stream) {
  if (moe_status st = check_ready(c)) return st;
  MONTA_CUDA(cudaSetDevice(c->device));
  return backward_dispatch_impl(c, level, n, static_cast<cudaStream_t>(stream));
}

namespace {
moe_status backward_impl(moe_ctx* c, int level, int n, cudaStream_t s) {
  if (moe_status st = backward_combine_impl(c, level, n, s)) return st;
  return backward_dispatch_impl(c, level, n, s);
}
}  // namespace

extern "C" moe_status moe_ctx_backward(moe_ctx* c, int level, int32_t n, void* stream) {
  if (moe_status st = check_ready(c)) return st;
  if (moe_status st = validate_dispatch(c, level, n, MOE_LAND_FINAL)) return st;
  MONTA_CUDA(cudaSetDevice(c->device));
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (c->use_graphs)  // the whole backward replays as one CUDA graph
    return forward_graph(c, level, n, MOE_LAND_FINAL, nullptr, nullptr, nullptr, s, 1);
  return backward_impl(c, level, n, s);
}

extern "C" moe_status moe_ctx_forward_host(moe_ctx* c, int level, int32_t n, int landing, const void* host_x,
                                           const void* host_logits, void* host_out, void* stream) {
  if (moe_status st = check_ready(c)) return st;
  if (!host_x || !host_logits || !host_out) return fail(MOE_ERR_INVALID_ARGUMENT, "forward_host: null buffer");
  if (moe_status st = validate_dispatch(c, level, n, landing)) return st;
  MONTA_CUDA(cudaSetDevice(c->device));
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (c->use_graphs) return forward_graph(c, level, n, landing, host_x, host_logits, host_out, s);
  return forward_impl(c, level, n, landing, host_x, host_logits, host_out, s);
}

extern "C" moe_status moe_ctx_enable_graphs(moe_ctx* c, int enable) {
  if (!c) return fail(MOE_ERR_INVALID_ARGUMENT, "enable_graphs: null ctx");
  c->use_graphs = enable != 0;
  return MOE_OK;
}

extern "C" moe_status moe_ctx_recv_rows(moe_ctx* c, int card, int64_t* rows) {
  if (!c || !rows) return fail(MOE_ERR_INVALID_ARGUMENT, "recv_rows: null argument");
  MONTA_CUDA(cudaSetDevice(c->device));
  for (auto& cd : c->local)
    if (cd.id == card) {
      MONTA_CUDA(cudaDeviceSynchronize());
      MONTA_CUDA(cudaMemcpy(rows, cd.recv_rows, 8, cudaMemcpyDeviceToHost));
      return MOE_OK;
    }
  return fail(MOE_ERR_INVALID_ARGUMENT, "recv_rows: card %d is not local", card);
}

extern "C" moe_status moe_ctx_sync(moe_ctx* c) {
  if (!c) return fail(MOE_ERR_INVALID_ARGUMENT, "sync: null ctx");
  MONTA_CUDA(cudaSetDevice(c->device));
  MONTA_CUDA(cudaDeviceSynchronize());
  // every card's error word is read and cleared; the first error is reported
  int32_t e = 0;
  int first = -1;
  for (auto& cd : c->local) {
    int32_t ec = 0;
    MONTA_CUDA(cudaMemcpy(&ec, cd.err, 4, cudaMemcpyDeviceToHost));
    if (ec != 0) {
      const int32_t zero = 0;
      cudaMemcpy(cd.err, &zero, 4, cudaMemcpyHostToDevice);
      if (first < 0) {
        first = cd.id;
        e = ec;
      }
    }
  }
  if (first < 0) return MOE_OK;
  if (e == MOE_ERR_TIMEOUT) return fail(MOE_ERR_TIMEOUT, "card %d: cross-GPU flag wait timed out", first);
  if (e == MOE_ERR_INVALID_ARGUMENT)
    return fail(MOE_ERR_INVALID_ARGUMENT, "card %d: expert id out of range in the routing", first);
  if (e == MOE_ERR_CORRUPT_ROUTING)
    return fail(MOE_ERR_CORRUPT_ROUTING, "card %d: a dispatched row is missing or out of place (tag check)", first);
  return fail(moe_status(e), "card %d: device error %d", first, e);
}

extern "C" moe_status moe_ctx_enable_timing(moe_ctx* c, int enable) {
  if (!c) return fail(MOE_ERR_INVALID_ARGUMENT, "enable_timing: null ctx");
  c->timing = enable != 0;
  c->span_used = 0;
  return MOE_OK;
}

extern "C" moe_status moe_ctx_spans(moe_ctx* c, moe_span* spans, int32_t capacity, int32_t* n_spans) {
  if (!c || !n_spans) return fail(MOE_ERR_INVALID_ARGUMENT, "spans: null argument");
  *n_spans = 0;
  if (!c->timing) return MOE_OK;
  MONTA_CUDA(cudaSetDevice(c->device));
  MONTA_CUDA(cudaDeviceSynchronize());
  for (size_t i = 0; i < c->span_used && int32_t(i) < capacity; ++i) {
    const Span& sp = c->spans[i];
    float a = 0, b = 0;
    MONTA_CUDA(cudaEventElapsedTime(&a, c->ev_base, sp.a));
    MONTA_CUDA(cudaEventElapsedTime(&b, c->ev_base, sp.b));
    spans[i] = moe_span{sp.stage, sp.chunk, a, b};
    ++*n_spans;
  }
  return MOE_OK;
}

extern "C" moe_status moe_ctx_set_aa_ctas(moe_ctx* c, int32_t ctas) {
  if (!c || ctas < 0) return fail(MOE_ERR_INVALID_ARGUMENT, "set_aa_ctas: bad argument");
  c->aa_ctas = ctas;
  return MOE_OK;
}

extern "C" moe_status moe_ctx_xfer(moe_ctx* c, const int64_t* rows_per_card, int32_t row_bytes, int32_t grid,
                                   void* stream) {
  if (!c || !rows_per_card) return fail(MOE_ERR_INVALID_ARGUMENT, "xfer: null argument");
  if (c->local.size() != 1) return fail(MOE_ERR_UNSUPPORTED, "xfer: one local card per context only");
  if (row_bytes <= 0 || row_bytes > c->row_bytes) return fail(MOE_ERR_INVALID_ARGUMENT, "xfer: bad row width");
  if (!c->connected) return fail(MOE_ERR_TRANSPORT, "xfer: context not connected");
  MONTA_CUDA(cudaSetDevice(c->device));
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  Card& cd = c->local[0];
  if (!c->xfer_list) {
    MONTA_CUDA(cudaMalloc(&c->xfer_list, seglist_bytes(kMaxCards)));
    MONTA_CUDA(cudaHostAlloc(&c->xfer_host, seglist_bytes(kMaxCards), cudaHostAllocDefault));
    std::memset(c->xfer_host, 0, seglist_bytes(kMaxCards));
    c->xfer_host->nseg = -1;
  }
  // Build the list on the host; upload only when it changed (so repeated
  // calls time the copy kernel alone).
  SegList* L = c->xfer_host;
  std::vector<Seg> segs;
  int64_t total = 0;
  for (int q = 0; q < c->cards; ++q) {
    if (rows_per_card[q] <= 0) continue;
    if (!c->peer[q].slab) return fail(MOE_ERR_TRANSPORT, "xfer: card %d is not mapped", q);
    if (rows_per_card[q] > c->recv_cap) return fail(MOE_ERR_INVALID_ARGUMENT, "xfer: too many rows for card %d", q);
    Seg sg{};
    sg.row_begin = total;
    sg.src_row = total;
    sg.dst_row = 0;
    sg.rows = int32_t(rows_per_card[q]);
    sg.dst = q;
    sg.col_off = 0;
    sg.width = row_bytes;
    sg.expert = 0;
    segs.push_back(sg);
    total += rows_per_card[q];
  }
  if (total > c->recv_cap) return fail(MOE_ERR_INVALID_ARGUMENT, "xfer: %lld rows exceed the buffer", (long long)total);
  const bool same = L->nseg == int32_t(segs.size()) && L->total_rows == total &&
                    std::memcmp(L->segs, segs.data(), segs.size() * sizeof(Seg)) == 0;
  if (!same) {
    MONTA_CUDA(cudaStreamSynchronize(s));  // the pinned staging may still feed a previous upload
    L->nseg = int32_t(segs.size());
    L->total_rows = total;
    if (!segs.empty()) std::memcpy(L->segs, segs.data(), segs.size() * sizeof(Seg));
    MONTA_CUDA(cudaMemcpyAsync(c->xfer_list, L, seglist_bytes(L->nseg), cudaMemcpyHostToDevice, s));
  }
  CopyArgs a{};
  a.list = c->xfer_list;
  a.src = static_cast<const char*>(cd.v.recv);
  a.src_stride = c->row_bytes;
  a.dst_stride = c->row_bytes;
  for (int q = 0; q < c->cards; ++q) {
    if (!c->peer[q].slab) continue;
    a.dst[q] = q == cd.id ? static_cast<char*>(cd.v.pre) : c->peer[q].recv;
  }
  a.wait = no_wait();
  a.sig = no_signal();
  a.err = cd.err;
  const int g = grid > 0 ? grid : c->sms * 2;
  const int vec = vec_bytes(row_bytes, c->row_bytes);
  a.chunks_per_row = items_per_row(vec, row_bytes);
  a.split = g;
  MONTA_CUDA(launch_seg_copy(a, vec, g, s));
  ++c->launches;
  return MOE_OK;
}

extern "C" int64_t moe_ctx_launch_count(const moe_ctx* c) { return c ? c->launches : 0; }

extern "C" moe_status moe_ctx_debug_front(moe_ctx* c, int enable, int card, uint64_t* out20) {
  if (!c) return fail(MOE_ERR_INVALID_ARGUMENT, "debug_front: null ctx");
  c->debug = enable != 0;
  MONTA_CUDA(cudaSetDevice(c->device));
  if (!out20) {
    for (auto& cd : c->local) MONTA_CUDA(cudaMemset(cd.dbg, 0, 20 * sizeof(uint64_t)));
    return MOE_OK;
  }
  for (auto& cd : c->local)
    if (cd.id == card) {
      MONTA_CUDA(cudaDeviceSynchronize());
      MONTA_CUDA(cudaMemcpy(out20, cd.dbg, 160, cudaMemcpyDeviceToHost));
      MONTA_CUDA(cudaMemset(cd.dbg + 16, 0, 4 * sizeof(uint64_t)));  // the per-launch min/max stamps
      return MOE_OK;
    }
  return fail(MOE_ERR_INVALID_ARGUMENT, "debug_front: card %d is not local", card);
}

extern "C" moe_status moe_ctx_set_node_dedup(moe_ctx* c, int32_t enable) {
  if (!c) return fail(MOE_ERR_INVALID_ARGUMENT, "set_node_dedup: null ctx");
  if (enable < 0 || enable > 2) return fail(MOE_ERR_INVALID_ARGUMENT, "set_node_dedup: mode must be 0, 1 or 2");
  if (c->node_dedup != enable) {
    MONTA_CUDA(cudaSetDevice(c->device));
    for (auto& g : c->graphs)
      if (g.exec) cudaGraphExecDestroy(g.exec);
    c->graphs.clear();
  }
  c->node_dedup = enable;
  return MOE_OK;
}

extern "C" moe_status moe_ctx_set_expert_overlap(moe_ctx* c, int32_t enable) {
  if (!c) return fail(MOE_ERR_INVALID_ARGUMENT, "set_expert_overlap: null ctx");
  if (c->expert_fused != (enable != 0)) {
    MONTA_CUDA(cudaSetDevice(c->device));
    for (auto& g : c->graphs)
      if (g.exec) cudaGraphExecDestroy(g.exec);
    c->graphs.clear();
  }
  c->expert_fused = enable != 0;
  return MOE_OK;
}

extern "C" moe_status moe_ctx_set_persistent(moe_ctx* c, int enable) {
  if (!c) return fail(MOE_ERR_INVALID_ARGUMENT, "set_persistent: null ctx");
  c->use_xchg = enable != 0;
  return MOE_OK;
}

extern "C" moe_status moe_ctx_xchg_trace(moe_ctx* c, int card, uint64_t* out, int32_t capacity, int32_t* max_chunks) {
  if (!c || !out || !max_chunks) return fail(MOE_ERR_INVALID_ARGUMENT, "xchg_trace: null argument");
  *max_chunks = c->d.max_chunks;
  const int32_t need = 2 * 4 * c->d.max_chunks * 2;
  if (capacity < need) return fail(MOE_ERR_INVALID_ARGUMENT, "xchg_trace: need capacity %d", need);
  MONTA_CUDA(cudaSetDevice(c->device));
  for (auto& cd : c->local)
    if (cd.id == card) {
      MONTA_CUDA(cudaDeviceSynchronize());
      MONTA_CUDA(cudaMemcpy(out, cd.xtrace, size_t(need) * 8, cudaMemcpyDeviceToHost));
      return MOE_OK;
    }
  return fail(MOE_ERR_INVALID_ARGUMENT, "xchg_trace: card %d is not local", card);
}

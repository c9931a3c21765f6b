// Data structures shared by the layer context (ctx.cu) and the movement /
// combine kernels (copy.cu, combine.cu, plan.cu).
#pragma once

#include "common.cuh"

namespace monta {

// One contiguous run of rows moved by a copy kernel.  A list of these (built
// on the device by the plan kernel from the exchanged counts) describes one
// (phase, chunk) of the exchange, so no host round trip is needed to learn
// the dynamic row counts.
struct Seg {
  int64_t row_begin;  // exclusive prefix of `rows` over the list
  int64_t src_row;    // first source row (AA: index into the sender's permuted order)
  int64_t dst_row;    // first destination row
  int32_t rows;
  int32_t dst;        // destination card id, or -1: every card in dst_mask
  int32_t col_off;    // byte offset of the moved column slice
  int32_t width;      // bytes moved per row
  int32_t expert;     // global expert id (tag synthesis)
  int32_t pad;
};
static_assert(sizeof(Seg) == 48, "Seg layout");

struct SegList {
  int32_t nseg;
  int32_t pad;
  int64_t total_rows;
  Seg segs[1];  // [capacity]
};
__host__ __device__ inline size_t seglist_bytes(int cap) { return 16 + size_t(cap) * sizeof(Seg); }

// AA = cross-node legs of the fused permute+AllToAll, AAL = its local
// (own-node, full-row) legs — separate lists so the copy kernel can run them
// on disjoint CTA sets and overlap NVLink with HBM traffic.
enum SegPhase { kPhaseAA = 0, kPhaseAG = 1, kPhaseD2D = 2, kPhaseCAA = 3, kPhaseAAL = 4, kNumPhases = 5 };

// Signals carried in each card's flag array: flags[(sig) * kMaxCards + sender].
enum Signal {
  kSigCounts = 0,     // unused since the count words carry their epoch (slot kept: flag layout)
  kSigBarrier = 1,
  kSigChunkBase = 2,  // + phase_signal * max_chunks + j
};
enum PhaseSignal { kPsAA = 0, kPsAG = 1, kPsCAA = 2, kPsCAG = 3, kNumPhaseSignals = 4 };

struct CopyArgs {
  const SegList* list;
  const SegList* list2;      // optional second list, run by CTAs [split, grid)
  int32_t split;             // CTAs [0, split) run `list`
  int32_t chunks_per_row;    // work items per row (kItemBytes each)
  const char* src;
  int64_t src_stride;        // bytes per source row
  const int32_t* gather;     // AA: perm_src; row = gather[seg.src_row + i]
  const int32_t* src_tags;   // int4 per source row (COPY), or null
  const int32_t* token_ids;  // AA tag synthesis
  int32_t source_card;       // AA tag synthesis
  int32_t synth_tags;        // 1: AA synthesises tags, 0: copy src_tags (if any)
  int64_t dst_stride;        // bytes per destination row
  uint64_t dst_mask;         // seg.dst == -1 targets
  char* dst[kMaxCards];
  int32_t* dst_tags[kMaxCards];
  WaitList wait;
  SignalList sig;
  int32_t* err;
  uint32_t pace_bpus;        // emulated inter-node link (moe_ctx_set_link_rate): bytes per us, 0 = off
  // optional source-row filter: only segments with bounds[b_lo] <= src_row <
  // bounds[b_hi] are copied (the reverse AllToAll of one expert group)
  const int32_t* bounds;
  int32_t b_lo, b_hi;
};

struct UnpermArgs {
  const char* comb;          // [R, h] landing buffer (sender-permuted order)
  const char* local_y;       // expert outputs of this card's own node (final layout), or null
  const int32_t* local_delta;  // [E] row delta permuted->final for own-node experts, or null
  int32_t local_lo, local_hi;  // own-node experts [lo, hi)
  int64_t y_stride;          // bytes per row (comb and local_y)
  const int32_t* slot_pos;   // [T, k]
  const int32_t* experts;    // [T, k]
  const void* probs;         // [T, k]
  int32_t k;
  int64_t tok_begin, tok_end;
  int64_t col_begin, cols;   // element columns to produce
  int64_t out_stride;        // bytes per output row
  int32_t n_out;
  int32_t reverse;           // k_unpermute_rows: tokens in descending order
  char* out[kMaxCards];      // every destination (fused all-gather)
  WaitList wait;
  SignalList sig;
  int32_t* err;
};

// Launchers (return cudaGetLastError()).
cudaError_t launch_seg_copy(const CopyArgs& a, int vec, int grid, cudaStream_t s);
int copy_item_bytes(int vec);  // bytes one warp moves per work item
cudaError_t launch_gather_rows(const void* src, int64_t src_stride, int64_t col_off, int64_t width,
                               const int32_t* perm, int64_t R, void* out, int64_t out_stride,
                               cudaStream_t s);
cudaError_t launch_unpermute(const UnpermArgs& a, int y_dtype, int probs_dtype, int out_dtype,
                             int grid, cudaStream_t s, bool* supported);
cudaError_t launch_wait(const WaitList& w, int32_t* err, cudaStream_t s);
cudaError_t launch_signal(const SignalList& sg, cudaStream_t s);

// Token-side fused permute + AllToAll (aa.cu): one warp per token reads the
// row once and stores it (or this rank's 1/t slice of it) to each of its k
// destinations; dst row = table base of its expert + its permuted position.
struct TokArgs {
  const char* x;
  int64_t row_bytes;
  const int32_t* experts;   // [T, k]
  const int32_t* slot_pos;  // [T, k]
  const int32_t* token_ids;
  int32_t source_card;
  const int32_t* table;     // PlanArgs::aa_table
  int32_t E, k, n, j, staged;
  int64_t tok_begin, tok_end;
  int64_t dst_stride;
  char* dst[kMaxCards];
  int32_t* dst_tags[kMaxCards];
  // fp8 wire (moe_ctx_set_wire): cross-node legs store e4m3 bytes + one fp32
  // scale per 128 elements into the receiver's pre / wscale instead of bf16
  int32_t fp8, node, t, blocks_per_row;
  char* dst_pre[kMaxCards];
  float* dst_scale[kMaxCards];
  // emulated inter-node link: the chunk's cross-node list (kPhaseAA) paces the kernel's release
  const SegList* pace_list;
  uint32_t pace_bpus;
  SignalList sig;
  int32_t* err;
  // every destination is in this GPU's own memory (a lone card, or virtual
  // cards on one GPU): the TMA bulk-copy form may run (aa.cu k_aa_bulk)
  int32_t local_dst;
  // node dedup (EP only): a remote card gets the token's row once, into its
  // staging block for this node at slot nslot[i * e + node]; the receiver
  // fans it out (k_node_fanout).  null: every (token, expert) row crosses.
  const int32_t* nslot;
  int32_t e;
  char* stage[kMaxCards];
};
// Node dedup: staging slots + descriptors (sender), fan-out (receiver).
struct NodeSlotArgs {
  const int32_t* experts;    // [T, k]
  const int32_t* slot_pos;   // [T, k]
  const int32_t* token_ids;  // [T]
  const int32_t* table;      // aa_table: [0, E) card, [E, 2E) row base
  int64_t T;
  int32_t E, k, e, t, node, rho;
  uint32_t* scount;          // this card's [kMaxCards] staged-row counts
  int32_t* nslot;            // [T][e] staging slot, or -1
  int32_t* bcnt;             // [e][ceil(T / 1024)] per-block counts (deterministic slot scan)
  int32_t* sdesc[kMaxCards]; // each card's descriptor block for this node
};
cudaError_t launch_node_slots(const NodeSlotArgs& a, cudaStream_t s);
struct FanoutArgs {
  int32_t nsend;                     // remote senders
  const char* stage[kMaxCards];      // this card's staging block of sender i
  const int32_t* sdesc[kMaxCards];   // its descriptors
  const uint32_t* count[kMaxCards];  // rows sender i staged to this card (sender's scount[this card])
  int32_t source_card[kMaxCards];
  int64_t row_bytes;
  int64_t col_lo, col_hi;            // byte window of a row this card owns (its 1/t slice under TP)
  int32_t k;
  char* recv;
  int32_t* recv_tags;
};
cudaError_t launch_node_fanout(const FanoutArgs& a, int64_t max_rows, int vec, cudaStream_t s);
struct StageAgArgs {
  int32_t nsend;                          // remote sender nodes
  int32_t npeer;                          // TP peers of this card
  const char* stage[kMaxCards];           // this card's staging block of sender i
  char* peer_stage[8][kMaxCards];         // [peer][sender i]: the same block on TP peer p (t <= 9)
  const uint32_t* count[kMaxCards];       // rows sender i staged (to this card and, equally, to the peers)
  int64_t row_bytes, col_lo, col_hi;      // this rank's slice of a staged row
  SignalList sig;
};
cudaError_t launch_stage_ag(const StageAgArgs& a, int64_t max_rows, cudaStream_t s);
// Fused combine (experts.cu + ctx.cu): rowdst[r] = the address of final-layout
// row r's reverse-AllToAll destination row (a peer's comb) from the CAA lists
// of chunks [0, n), null for rows that stay on this node.
struct PeerRows {
  char* base[kMaxCards];
};
cudaError_t launch_rowdst(const SegList* lists, size_t list_stride, int n, int nseg_cap, const PeerRows& comb,
                          int64_t row_bytes, char** rowdst, int64_t cap, cudaStream_t s);
// SwiGLU expert FFN whose down-projection computes output columns
// [out_col0, out_col0 + out_cols) only (a TP rank's combine slice) and whose
// epilogue also stores each row's bytes [col_lo, col_hi) to rowdst[r] (when
// rowdst and the entry are non-null): the reverse AllToAll issued tile by
// tile from the GEMM (experts.cu).
moe_status expert_ffn_fused(const void* x, int64_t ldx, int64_t x_rows, const void* w13, const void* w2,
                            const int32_t* offs, int L, int64_t hidden, int64_t ffn, void* workspace, void* y,
                            int64_t ldy, char* const* rowdst, int32_t col_lo, int32_t col_hi, int64_t out_col0,
                            int64_t out_cols, cudaStream_t s);
cudaError_t launch_aa_token(const TokArgs& a, int vec, int grid, cudaStream_t s);
// fp8 wire, combine leg (aa.cu): the reverse AllToAll of one chunk (CAA
// segment list) quantised into each source card's cwire / cscale; the
// source decodes its cross-node slots into comb before the un-permute.
struct CaaFp8Args {
  const SegList* list;
  const char* src;        // expert outputs (bf16 rows, row_bytes apart)
  int64_t row_bytes;
  int32_t blocks_per_row;
  char* dst_wire[kMaxCards];
  float* dst_scale[kMaxCards];
  uint32_t pace_bpus;
  SignalList sig;
};
cudaError_t launch_caa_fp8(const CaaFp8Args& a, int grid, cudaStream_t s);
cudaError_t launch_comb_dequant(char* comb, const char* wire, const float* scales, const int32_t* slot_pos,
                                const int32_t* experts, int64_t tok_begin, int64_t tok_end, int k, int L, int node,
                                int64_t row_bytes, int blocks_per_row, int64_t col0, int64_t width, cudaStream_t s);
// fp8 wire receive side (aa.cu): rows of this card that came from another
// node with source position in [p0, p1): columns [col0, col0 + width) of
// recv (bf16) = dequant(pre (e4m3), wscale)
cudaError_t launch_wire_dequant(char* recv, const int32_t* tags, const int64_t* recv_rows, int64_t cap,
                                const char* pre, const float* scales, int64_t row_bytes, int blocks_per_row,
                                int node, int t, int64_t col0, int64_t width, int64_t p0, int64_t p1,
                                cudaStream_t s);

// Persistent exchange (xchg.cu): the whole chunked dispatch of one card in
// one cooperative launch.  CTA roles, in order: AA (cross-node legs), AAL
// (own-node legs), AG (dedup forward to TP peers; under O2 staged it also
// runs the reorder), D2D (staged reorder, O3).  Per chunk, each role's last
// CTA publishes a flag; consumers wait in-kernel (every CTA is co-resident).
struct XchgArgs {
  CopyArgs cp;                  // gather/src/dst/tags (src = node batch for AA/AAL)
  SegList* lists;               // [kNumPhases][max_chunks]
  int32_t seg_cap, max_chunks, n;
  int32_t me, node, rho, e, t;
  int32_t dedup, staged, d2d_in_ag;
  int32_t r_aa, r_aal, r_ag, r_d2d;  // CTAs per role (AA | AAL | AG | D2D)
  int32_t cpr_full, cpr_slice;
  char* recv_local;             // AG source (FINAL) / D2D destination
  int32_t* recv_tags_local;
  char* pre_local;              // AG source (STAGED) / D2D source
  int32_t* pre_tags_local;
  char* ag_dst[kMaxCards];      // AG destinations (peer recv or pre)
  int32_t* ag_dst_tags[kMaxCards];
  char* d2d_dst[kMaxCards];     // reorder destination: [me] = recv_local
  int32_t* d2d_dst_tags[kMaxCards];
  uint64_t ag_mask;             // TP peers
  uint64_t* flags[kMaxCards];   // every card's flag array (peer-mapped)
  const uint64_t* epoch_ptr;
  unsigned int* counters;       // [4][max_chunks] per-role chunk completion (local, zero)
  uint64_t* local_flags;        // [max_chunks] own-node copy of chunk j finished (epoch)
  unsigned long long* trace;    // optional [4 roles][max_chunks][2] (ns)
  unsigned long long* dbg;      // optional {kernel start, kernel end} stamps (ns, debug)
  int32_t* err;
};
cudaError_t launch_xchg(const XchgArgs& a, int vec, cudaStream_t s);
int xchg_max_ctas(int vec);

// Persistent combine (combine.cu): roles CAA (reverse AllToAll of the expert
// outputs, per chunk) | UNP (wait CAA[j], weighted un-permute of chunk j's
// tokens, output slice stored to every TP peer = the output AllGather).
struct CombArgs {
  UnpermArgs up;
  CopyArgs cp;
  SegList* lists;
  int32_t seg_cap, max_chunks, n;
  int32_t me, node, rho, e, t, dedup;
  int32_t r_caa, r_unp, cpr;
  int64_t T;
  uint64_t* flags[kMaxCards];
  const uint64_t* epoch_ptr;
  unsigned int* counters;  // [2][max_chunks]
  unsigned long long* trace;  // optional [2 roles][max_chunks][2] (ns)
  unsigned long long* dbg;    // optional {kernel start, kernel end} stamps (ns, debug)
  int32_t* err;
};
// Returns cudaErrorNotSupported when no persistent instantiation fits.
cudaError_t launch_combine_xchg(const CombArgs& a, int y_dtype, int probs_dtype, int out_dtype, int vec,
                                cudaStream_t s, int* max_ctas_out);

// Plan kernel (plan.cu).
struct PlanArgs {
  const uint64_t* count_table;  // [e][max_chunks][E] words {count (low 32) | epoch (high 32)}
  int32_t e, t, E, L, n, max_chunks;
  int32_t node, rho;
  int32_t level, landing;
  int64_t row_bytes;           // full row bytes (h * elem)
  int32_t seg_cap;             // capacity of each list
  SegList* lists;              // [kNumPhases][max_chunks] lists, stride seglist_bytes(seg_cap)
  int32_t* local_delta;        // [E]
  int32_t* aa_table;           // [4][E] {card, base_final, col_off, width} + [n][E] base_staged
  int64_t* recv_rows;          // [1]
  int32_t* recv_offs;          // [L + 1] this node's local-expert row offsets in recv (final layout)
  WaitList wait;
  int32_t poll_peers;          // wait until every peer node's count words carry this epoch
  int32_t* err;
  unsigned long long* dbg;     // optional step timestamps (front kernel debug)
};
size_t plan_scratch_ints(int e, int E, int max_chunks);
moe_status configure_grouped_gemm();  // experts.cu
// layer backward (layer_bwd.cu): every card's routing and grad-prob partials by card id
struct BwdPeers {
  const int32_t* experts[kMaxCards];
  const void* probs[kMaxCards];
  void* parts[kMaxCards];
};
cudaError_t launch_row_meta(int logit_dtype, const int32_t* tags, const int64_t* recv_rows, int64_t cap, int t,
                            int rho, int k, const BwdPeers& pe, void* prow, int32_t* rowpos, int32_t* rowslot,
                            int32_t* err, cudaStream_t s);
cudaError_t launch_scatter_parts(int logit_dtype, const int32_t* tags, const int64_t* recv_rows, int64_t cap, int t,
                                 int rho, int k, const int32_t* rowslot, const void* dot, const BwdPeers& pe,
                                 cudaStream_t s);
cudaError_t launch_sum_parts(int logit_dtype, const void* parts, const int32_t* experts, int64_t Tk, int t,
                             void* gprobs, cudaStream_t s);
cudaError_t launch_fill_ones(int logit_dtype, void* p, int64_t n, cudaStream_t s);
cudaError_t launch_verify_recv(const int32_t* tags, const int64_t* recv_rows, const int32_t* offs, int L, int node,
                               int e, int t, int64_t T, int64_t cap, int32_t* err, cudaStream_t s);  // verify.cu
bool plan_fits_smem(int e, int E, int n);
moe_status configure_plan();
cudaError_t launch_plan_with_scratch(const PlanArgs& a, int32_t* scratch, cudaStream_t s);
// Index-build shared memory (ints): hist [nwarps][E] | offs [E+1] | counts [n][E]
inline size_t index_smem_ints(int nwarps, int E, int n, bool count_in_smem) {
  return size_t(nwarps) * E + E + 1 + (count_in_smem ? size_t(n) * E : 0);
}
// Fused front end (front.cu), one cooperative launch over token tiles:
// route each tile, histogram it, elect the last CTA to scan tile bases /
// offsets / chunk counts, bump the device epoch and push this node's counts
// to its expert-parallel peers (NVLink stores + flags), release the grid,
// rank every tile's pairs in parallel, then (do_plan) plan.
struct FrontArgs {
  const void* logits;   // [T, E] (route != 0)
  int32_t route;
  int64_t T;
  int32_t E, k, n;
  int32_t* experts;     // [T, k]
  void* probs;          // [T, k]
  int32_t* perm_src;
  int32_t* expert_of;
  int32_t* slot_pos;
  int32_t* counts;      // [n, E]
  int32_t* expert_offsets;
  int32_t* err;
  int32_t tile_tokens;  // tokens per tile (= kFrontThreads / G when routing)
  int32_t n_tiles;
  int32_t aligned;      // (T / n) % tile_tokens == 0: chunk counts from tile histograms
  int32_t* tile_hist;   // [n_tiles][E]
  int32_t* tile_base;   // [n_tiles][E]
  int32_t* counts_acc;  // [2][max_chunks][E] chunk counts accumulated by the tile CTAs; buffer epoch & 1
                        // is this launch's, the other is zeroed for the next
  unsigned int* arrive; // grid-barrier arrival counter (zero between launches)
  unsigned long long* ready;  // grid-barrier release flag (= epoch)
  uint64_t* epoch_dev;  // bumped once per dispatch
  int32_t node, max_chunks;
  int32_t n_dst;
  uint64_t* dst_tables[kMaxCards];  // count words stored into every EP peer's table
  int32_t do_plan;      // 0: none (separate plan launch), 1: plan_block, 2: identity plan (lone card, final landing)
  PlanArgs plan;        // its wait list is satisfied at the bumped epoch
  int32_t* plan_scratch;
  int32_t plan_in_smem; // plan tables in (reused) dynamic shared memory
  unsigned long long* dbg;  // optional phase timestamps [8] (globaltimer ns)
};
constexpr int kFrontThreads = 512;
// Front CTA size: wide expert sets (a whole warp per token, >= 3 scores per
// lane: E > 64) route 32 tokens per pass with 1024 threads — half the
// dependent top-k rounds per warp of a 512-thread CTA on the same tiles.
__host__ __device__ constexpr int front_threads(int G, int PER) { return (G == 32 && PER >= 3) ? 1024 : kFrontThreads; }
moe_status launch_front(const FrontArgs& a, int logit_dtype, cudaStream_t s);
// Set the front kernel's shared-memory attribute ahead of graph capture.
moe_status configure_front(int E, int logit_dtype);
// Router tokens per front CTA, and the index tile length for (E, T, n).
int front_router_tokens(int E);
int front_tile_tokens(int E, int64_t T, int n);
moe_status check_route_args(int64_t T, int E, int k);

moe_status route_topk(const void* logits, int logit_dtype, int64_t T, int E, int k, int32_t* experts,
                      void* probs, cudaStream_t stream);
moe_status build_index(const int32_t* experts, int64_t T, int k, int E, int n_chunks,
                       int32_t* perm_src, int32_t* expert_of, int32_t* slot_pos, int32_t* counts,
                       int32_t* expert_offsets, int32_t* dev_error, cudaStream_t stream);

}  // namespace monta

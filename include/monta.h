/*
 * monta.h — C ABI of the B200-native MoNTA dispatch/combine path.
 *
 * This is the drop-in boundary for the reference's operator API
 * (/root/reference/proj/include/moeplan/{dataplane,commcost,chunkopt,strategy,
 * calibrate,pipesim,config}.hpp).  The reference is a header-only C++20
 * library with value semantics and exceptions; here every entry point is a
 * plain `extern "C"` function over device/host pointers and sizes that
 * returns a moe_status.  Exceptions map to status codes:
 *
 *   std::invalid_argument                 -> MOE_ERR_INVALID_ARGUMENT
 *   dataplane::CorruptRoutingError        -> MOE_ERR_CORRUPT_ROUTING   (dataplane.hpp:18-20)
 *   StrategyInapplicableError             -> MOE_ERR_STRATEGY_INAPPLICABLE (chunkopt.hpp:11-13)
 *   CalibrationError                      -> MOE_ERR_CALIBRATION       (calibrate.hpp:12-14)
 *   pipesim::InvalidGraphError            -> MOE_ERR_INVALID_GRAPH     (pipesim.hpp:65-67)
 *
 * The message of the last failure on the calling thread is moe_last_error().
 *
 * Three families of entry points:
 *   1. stateless device ops (router, index build, permute, un-permute combine)
 *      that work on caller-owned device pointers and a caller stream;
 *   2. a layer context (moe_ctx) that owns the per-card HBM layout, the
 *      NVLink peer mappings, prioritised streams and cross-GPU flags, and runs
 *      the TP-deduplicated chunked dispatch and the mirrored combine;
 *   3. the host planner (cost model, chunk search, strategy selection,
 *      calibration, pipeline simulator) in double precision.
 *
 * Streams are passed as `void*` (a cudaStream_t); NULL is the legacy stream.
 */
#ifndef MONTA_H_
#define MONTA_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MONTA_ABI_VERSION 2

typedef enum moe_status {
  MOE_OK = 0,
  MOE_ERR_INVALID_ARGUMENT = 1,
  MOE_ERR_CORRUPT_ROUTING = 2,
  MOE_ERR_STRATEGY_INAPPLICABLE = 3,
  MOE_ERR_CALIBRATION = 4,
  MOE_ERR_INVALID_GRAPH = 5,
  MOE_ERR_CUDA = 6,
  MOE_ERR_TRANSPORT = 7, /* peer mapping failed / peer not reachable */
  MOE_ERR_TIMEOUT = 8,   /* a cross-GPU flag wait timed out */
  MOE_ERR_UNSUPPORTED = 9
} moe_status;

/* Mirrors moeplan::StrategyLevel (commcost.hpp:11).  BASELINE is the
 * monolithic TP-redundant AllToAll (dataplane::dispatch_monolithic). */
typedef enum moe_level { MOE_BASELINE = 0, MOE_O1 = 1, MOE_O2 = 2, MOE_O3 = 3 } moe_level;

typedef enum moe_dtype {
  MOE_F32 = 0,
  MOE_BF16 = 1,
  MOE_F16 = 2,
  MOE_F64 = 3,
  MOE_I64 = 4 /* the reference's payload type (dataplane.hpp:39) */
} moe_dtype;

/* Where the chunked exchange lands rows on the receiving card.
 *   FINAL : senders know every offset after the count exchange and write
 *           straight into the source-major final layout (no reorder copy).
 *   STAGED: rows land chunk-major (the reference's ChunkedDispatchTrace::pre_copy
 *           layout, dataplane.hpp:260-261) and a D2D reorder copy moves them
 *           to the final layout (dataplane.hpp:263-274), as MoNTA does. */
typedef enum moe_landing { MOE_LAND_FINAL = 0, MOE_LAND_STAGED = 1 } moe_landing;

const char* moe_last_error(void);
int moe_abi_version(void);
size_t moe_dtype_size(int dtype);

/* Page-locked host buffers for moe_ctx_forward_host (cudaHostAlloc, portable
 * across contexts), for hosts without another pinned allocator.
 * Errors: null out pointer -> MOE_ERR_INVALID_ARGUMENT. */
moe_status moe_host_alloc(size_t bytes, void** ptr);
moe_status moe_host_free(void* ptr);

/* ------------------------------------------------------------------------
 * 1. Stateless device ops
 * ------------------------------------------------------------------------ */

/* dataplane::route_topk (dataplane.hpp:72-106).
 * logits [T, E] row-major in `logit_dtype` (MOE_F32 or MOE_F64).  Softmax in
 * that precision (max-subtract, exp, sum, divide); the k largest RAW scores
 * win, lower expert index on ties; experts written ascending; probs are the
 * softmax values of the selected experts (not renormalised), same dtype as
 * the logits.  T == 0 is allowed (no launch).
 * Errors: k < 1, E < 1 (empty row), k > E -> MOE_ERR_INVALID_ARGUMENT. */
moe_status moe_route_topk(const void* logits, int logit_dtype, int64_t T, int32_t E, int32_t k,
                          int32_t* experts, void* probs, void* stream);

/* Stable counting sort of the (token, slot) pairs by expert — the index
 * form of dataplane::permute (dataplane.hpp:118-140).
 *   experts     [T, k]   expert of each pair, 0 <= x < E
 *   perm_src    [T*k]    source token of permuted row r
 *   expert_of   [T*k]    expert of permuted row r           (PermutedBatch::expert_of)
 *   slot_pos    [T, k]   permuted row of pair (i, s)       (PermutedBatch::inverse_map
 *                        when the token's experts ascend, which route_topk guarantees)
 *   counts      [n, E]   rows of expert x whose token falls in chunk j = i / (T/n)
 *   expert_offsets [E+1] exclusive scan of rows per expert
 *   dev_error   device int32 set to MOE_ERR_INVALID_ARGUMENT if an expert id
 *               is out of range (may be NULL).
 * Ordering is expert-major, token-ascending, with no atomics in the ordering.
 * Errors: n < 1, T % n != 0 -> MOE_ERR_INVALID_ARGUMENT. */
moe_status moe_build_index(const int32_t* experts, int64_t T, int32_t k, int32_t E, int32_t n_chunks,
                           int32_t* perm_src, int32_t* expert_of, int32_t* slot_pos,
                           int32_t* counts, int32_t* expert_offsets, int32_t* dev_error,
                           void* stream);

/* Gather-permute: out[r, 0:width) = src[perm_src[r], col_off:col_off+width)
 * (bytes).  16-byte vectorised when every size/stride/offset allows. */
moe_status moe_permute_rows(const void* src, int64_t src_row_bytes, int64_t col_off_bytes,
                            int64_t width_bytes, const int32_t* perm_src, int64_t R, void* out,
                            int64_t out_row_bytes, void* stream);

/* Weighted un-permute (the arithmetic of dataplane::combine_unpermute,
 * dataplane.hpp:325-342):  out[i, q] = sum_s probs[i,s] * y[slot_pos[i,s], q],
 * accumulated from 0 in ascending slot order.  Accumulation is fp32 for
 * f32/bf16/f16 inputs and fp64 for f64/i64 inputs.  `probs_dtype` is MOE_F32
 * or MOE_F64.  out_dtype: MOE_F32/MOE_BF16/MOE_F16/MOE_F64. */
moe_status moe_unpermute_combine(const void* y, int y_dtype, int64_t y_row_elems, int64_t width,
                                 const int32_t* slot_pos, const void* probs, int probs_dtype,
                                 int64_t T, int32_t k, void* out, int out_dtype,
                                 int64_t out_row_elems, void* stream);

/* ------------------------------------------------------------------------
 * 1b. Backward of the stateless ops.  The reference
 * has no backward; these are the adjoints of moe_unpermute_combine,
 * moe_permute_rows and moe_route_topk so a training step can run through the
 * same index.  On a multi-card layer the cross-card legs of the backward are
 * the forward exchanges in the opposite direction; these are the per-card
 * kernels either side of them.
 * ------------------------------------------------------------------------ */

/* Adjoint of moe_unpermute_combine:
 *   grad_y[slot_pos[i,s], 0:width) = probs[i,s] * grad_out[i, 0:width)   (y's dtype)
 *   grad_probs[i,s]                = sum_q grad_out[i,q] * y[slot_pos[i,s], q]  (probs' dtype)
 * fp32 arithmetic (fp64 if any operand is f64).  grad_y or grad_probs may be
 * NULL to skip that output; grad_probs needs y.  Dtypes: grad_out and y
 * f32/bf16/f16/f64, probs f32/f64.  1 <= k <= 64. */
moe_status moe_combine_backward(const void* grad_out, int grad_dtype, int64_t grad_row_elems,
                                const void* y, int y_dtype, int64_t y_row_elems, int64_t width,
                                const int32_t* slot_pos, const void* probs, int probs_dtype,
                                int64_t T, int32_t k, void* grad_y, int64_t grad_y_row_elems,
                                void* grad_probs, void* stream);

/* Adjoint of the dispatch gather (moe_permute_rows through slot_pos):
 *   grad_x[i, 0:width) = sum_s grad_rows[slot_pos[i,s], 0:width)
 * accumulated from zero in ascending slot order, fp32 (fp64 if f64).
 * 1 <= k <= 64. */
moe_status moe_dispatch_backward(const void* grad_rows, int rows_dtype, int64_t row_elems, int64_t width,
                                 const int32_t* slot_pos, int64_t T, int32_t k, void* grad_x,
                                 int out_dtype, int64_t out_row_elems, void* stream);

/* Adjoint of moe_route_topk with respect to the logits (the selection is
 * piecewise constant):  grad_logits[i,e] = P_e * (G_e - sum_s g_s P_{x_s})
 * where P = softmax(logits[i]), g = grad_probs[i], G_e = g_s if e == x_s.
 * logits, grad_probs and grad_logits share logit_dtype (MOE_F32 or MOE_F64). */
moe_status moe_route_backward(const void* logits, int logit_dtype, int64_t T, int32_t E, int32_t k,
                              const int32_t* experts, const void* grad_probs, void* grad_logits,
                              void* stream);

/* ------------------------------------------------------------------------
 * 1d. Communication priorities (conflict.hpp:40-50,
 * PAPER.md "Communication Conflict": EP > PP > CP > DP on the shared
 * inter-node fabric).  On B200 every group's traffic is issued by kernels on
 * CUDA streams (this library's exchange kernels for EP, NCCL kernels on the
 * caller's streams for PP/CP/DP), so the resolution priority becomes the
 * stream priority: the block scheduler starts a higher-priority stream's
 * pending CTAs first whenever the groups' kernels contend for SMs.
 * ------------------------------------------------------------------------ */
#define MOE_COMM_TP_SP 0
#define MOE_COMM_EP 1
#define MOE_COMM_PP 2
#define MOE_COMM_CP 3
#define MOE_COMM_DP 4
/* The reference's resolution priority (EP 3, PP 2, CP 1, DP 0, TP/SP -1). */
int moe_comm_priority(int group);
/* CUDA stream priority for a group on `device`: the groups' order spread over
 * the device's range (EP = greatest, TP/SP = least; distinct levels when the
 * range allows). */
moe_status moe_comm_stream_priority(int group, int device, int* cuda_priority);
/* A non-blocking stream on the current device with that priority. */
moe_status moe_comm_stream_create(int group, void** stream);
moe_status moe_comm_stream_destroy(void* stream);
/* Measured on a B200 box (scripts/micro/priority_bench.py): stream priority
 * orders CTA scheduling, not the shared NVLink ports — a concurrent DP
 * all-reduce slows the EP layer the same at either priority; sequencing the
 * lower-priority traffic after the EP phase (resolve_by_priority) is the
 * caller's stream order. */

/* ------------------------------------------------------------------------
 * 1e. NVSwitch multicast (NVLS) for the intra-node AllGather (SURVEY.md §8(f)
 * item 3; replaces the TP-shard gather of dataplane.hpp:243-256): one
 * multimem.st reaches every device bound to a multicast object, so a TP rank
 * sends its slice once instead of t - 1 times.  Multi-process setup: the
 * group leader creates the object and exports a POSIX fd (the caller passes
 * it to the other processes, e.g. SCM_RIGHTS over a Unix socket), the others
 * import it; every process adds its device, then (after a group barrier)
 * binds: a physical buffer of `bytes` on its device (local_va) bound into the
 * object, and the object's multicast address (mc_va).  `bytes` must be a
 * multiple of moe_mc_granularity.
 * ------------------------------------------------------------------------ */
typedef struct moe_mc moe_mc;
moe_status moe_mc_supported(int device, int* supported);
moe_status moe_mc_granularity(int ndev, size_t bytes, size_t* granularity);
moe_status moe_mc_create(int ndev, size_t bytes, int* fd_out, moe_mc** out);
moe_status moe_mc_import(int fd, int ndev, size_t bytes, moe_mc** out);
moe_status moe_mc_add_device(moe_mc* mc, int device);
moe_status moe_mc_bind(moe_mc* mc, void** local_va, void** mc_va);
/* Store `bytes` (16-byte multiple) from src through the multicast address
 * mc_dst on `grid` CTAs (0 = default): lands at the same offset in every
 * bound device's buffer, the storing device's own included. */
moe_status moe_mc_store(const void* src, void* mc_dst, size_t bytes, int32_t grid, void* stream);
moe_status moe_mc_destroy(moe_mc* mc);

/* ------------------------------------------------------------------------
 * 1c. Expert compute between dispatch and combine (
 * the reference's expert task gated on the dispatch terminals,
 * pipesim.hpp:102 — the reference models it, it computes nothing).
 * ------------------------------------------------------------------------
 * Grouped bf16 GEMM over expert-major rows (tcgen05.mma + TMEM accumulators,
 * TMA-fed, fp32 accumulation, bf16 out): for expert l in [0, num_experts),
 *   y[r, :] = x[r, :] . w[l]^T   for r in [expert_offsets[l], expert_offsets[l+1])
 * w is [num_experts][n][k] bf16 (nn.Linear layout, k contiguous).  x has
 * x_rows addressable rows (>= expert_offsets[num_experts]; rows past an
 * expert's end are read but never written), row stride ldx elements; y row
 * stride ldy.  k % 64 == 0, n % 128 == 0, 16-byte aligned rows.
 * act == MOE_ACT_SWIGLU: w holds gate and up rows tile-interleaved
 * (moe_interleave_w13) and y gets n/2 columns silu(gate) * up. */
#define MOE_ACT_NONE 0
#define MOE_ACT_SWIGLU 1
#define MOE_W13_BLOCK 128 /* features per gate/up block of an interleaved w13 */
moe_status moe_grouped_gemm(const void* x, int64_t ldx, int64_t x_rows, const void* w,
                            const int32_t* expert_offsets, int32_t num_experts, int64_t n, int64_t k,
                            void* y, int64_t ldy, int act, void* stream);
/* w13[l] = blocks of MOE_W13_BLOCK gate rows then the matching up rows:
 * rows [256 b, 256 b + 128) = gate[l][128 b ..], [256 b + 128, 256 b + 256) =
 * up[l][128 b ..].  gate/up [num_experts][ffn][hidden], ffn % 128 == 0. */
moe_status moe_interleave_w13(const void* w_gate, const void* w_up, int32_t num_experts, int64_t ffn,
                              int64_t hidden, void* w13, void* stream);
/* SwiGLU expert FFN (Mixtral / DeepSeek experts):
 *   y = (silu(x . Wg^T) * (x . Wu^T)) . W2^T  per expert segment,
 * w13 from moe_interleave_w13 ([E][2 ffn][hidden]), w2 [E][hidden][ffn];
 * workspace >= x_rows * ffn bf16.  y may alias x (x is fully consumed by the
 * first GEMM before the second writes y). */
moe_status moe_expert_ffn(const void* x, int64_t ldx, int64_t x_rows, const void* w13, const void* w2,
                          const int32_t* expert_offsets, int32_t num_experts, int64_t hidden, int64_t ffn,
                          void* workspace, void* y, int64_t ldy, void* stream);

/* ------------------------------------------------------------------------
 * 2. Layer context: one MoE layer's dispatch + combine over e x t cards
 * ------------------------------------------------------------------------
 * Topology (dataplane::VirtualTopology, dataplane.hpp:25-33): card c =
 * node*t + rho; node x hosts experts [x*L, (x+1)*L) with L = E/e, sharded over
 * its t cards; the e cards with equal rho form an expert-parallel group.
 *
 * world_size == 1        : every card lives on `device` (virtual mode; the
 *                          reference's single-process emulation).
 * world_size == e*t      : one card per process, card == rank; peers are
 *                          mapped over NVLink with CUDA IPC (moe_ctx_ipc_*).
 */
typedef struct moe_layer_desc {
  int32_t e;           /* node groups (expert parallel degree)            */
  int32_t t;           /* tensor-parallel ranks per node                  */
  int32_t num_experts; /* E, a multiple of e                              */
  int32_t top_k;       /* k                                               */
  int64_t tokens;      /* T per node group                                */
  int64_t hidden;      /* h payload elements per row                      */
  int32_t dtype;       /* payload dtype (any; dispatch moves bytes)       */
  int32_t logit_dtype; /* MOE_F32 or MOE_F64                              */
  int32_t out_dtype;   /* combine output dtype                            */
  int32_t max_chunks;  /* upper bound on n                                */
} moe_layer_desc;

typedef struct moe_ctx moe_ctx;

/* Device pointers of one card (all owned by the context). */
typedef struct moe_card_view {
  void* x;                 /* [T, h] node batch (replicated across the node's TP ranks) */
  void* logits;            /* [T, E]                                              */
  int32_t* token_ids;      /* [T]   TokenRecord::token_id (default i + node*100000) */
  int32_t* experts;        /* [T, k] routing (route output or caller-provided)    */
  void* probs;             /* [T, k] logit dtype                                  */
  int32_t* perm_src;       /* [T*k]                                               */
  int32_t* expert_of;      /* [T*k]                                               */
  int32_t* slot_pos;       /* [T, k]                                              */
  int32_t* counts;         /* [max_chunks, E] (first n rows valid)               */
  int32_t* expert_offsets; /* [E+1]                                               */
  void* permuted;          /* [T*k, h] permute output (moe_ctx_permute)           */
  void* recv;              /* [recv_cap, h] dispatched rows, final layout         */
  int32_t* recv_tags;      /* [recv_cap, 4] {token_id, source_card, source_position, expert} */
  void* pre;               /* [recv_cap, h] staged chunk-major layout (pre_copy)  */
  int32_t* pre_tags;       /* [recv_cap, 4]                                       */
  void* expert_out;        /* [recv_cap, h] expert outputs read by combine (== recv unless rebound) */
  void* comb;              /* [T*k, h] combine landing, sender-permuted order     */
  void* out;               /* [T, h] combined output in out_dtype                 */
  int64_t rows_permuted;   /* T*k                                                 */
  int64_t recv_cap;        /* e*T*min(k, L)                                       */
  int32_t* recv_expert_offsets; /* [L + 1] row offsets of this node's local experts in
                                 * recv after a FINAL-landing dispatch (expert-major) */
  void* grad_probs;        /* [T, k] logit dtype: moe_ctx_backward's d loss / d probs   */
  void* grad_logits;       /* [T, E] logit dtype: moe_ctx_backward's d loss / d logits  */
} moe_card_view;

moe_status moe_ctx_create(const moe_layer_desc* desc, int device, int rank, int world_size,
                          moe_ctx** out);
moe_status moe_ctx_destroy(moe_ctx* ctx);
moe_status moe_ctx_card_view(moe_ctx* ctx, int card, moe_card_view* out);
int moe_ctx_num_local_cards(const moe_ctx* ctx);
int moe_ctx_first_card(const moe_ctx* ctx);

/* Multi-process wiring: export this rank's IPC handle blob, then import the
 * blobs of all ranks (concatenated in rank order). */
size_t moe_ctx_ipc_handle_size(void);
moe_status moe_ctx_ipc_export(moe_ctx* ctx, void* blob);
moe_status moe_ctx_ipc_connect(moe_ctx* ctx, const void* all_blobs);

/* Expert outputs: by default the combine reads `recv` (identity experts, or
 * an expert computed in place).  Rebind to any [recv_cap, h] buffer. */
moe_status moe_ctx_bind_expert_out(moe_ctx* ctx, int card, void* expert_out);

/* Expert FFN of a card's local experts, run between dispatch and combine by
 * moe_ctx_forward (or explicitly with moe_ctx_experts): SwiGLU experts over
 * the card's recv rows, segment l = [recv_expert_offsets[l], [l+1]) uses
 * expert l's weights; output into expert_out (in place over recv by
 * default).  w13 [L][2 ffn][h] from moe_interleave_w13, w2 [L][h][ffn], bf16,
 * owned by the caller; the context allocates a [recv_cap, ffn] workspace.
 * Under TP (t > 1) every rank of a node holds the node's full rows after the
 * AllGather and runs the gate/up projection on all of them; with TP dedup
 * (level != MOE_BASELINE) the down-projection computes only the rank's 1/t
 * output column slice — the only columns its combine reads — so expert_out
 * columns outside the slice are left untouched.  Pass
 * w13 == NULL to unbind (identity experts).  Needs dtype bf16, h % 64 == 0,
 * ffn % 128 == 0. */
moe_status moe_ctx_bind_experts(moe_ctx* ctx, int card, const void* w13, const void* w2, int64_t ffn);
/* Run the bound experts of every local card on the rows of the last
 * dispatch (waits for every incoming row first).  No-op when none bound. */
moe_status moe_ctx_experts(moe_ctx* ctx, void* stream);
/* Bound experts fused with the reverse AllToAll inside moe_ctx_forward
 * (multi-GPU, bf16 wire, no link pacing): the down-projection GEMM's epilogue
 * stores every finished tile row both to expert_out and, when the row's
 * source card sits on another node, straight into that card's landing buffer
 * over NVLink (the reference's expert task feeding its combine,
 * pipesim.hpp:102) — the reverse AllToAll overlaps the tensor-core tiles in
 * one kernel.  enable = 0: experts, then the combine's own AllToAll.
 * Default on.  Results are identical either way. */
moe_status moe_ctx_set_expert_overlap(moe_ctx* ctx, int32_t enable);
/* Node dedup of the cross-node AllToAll (multi-GPU, unchunked, final
 * landing, bf16 wire; EP-only, or a TP-deduplicated level): a token's row
 * (this rank's 1/t slice under TP) crosses to a remote node once, however
 * many of its experts live there, into a staging block the receiving card
 * fans out to the experts' rows before the AllGather (the recv layout and
 * tags are the plain dispatch's, row for row).  mode 0: one row per (token,
 * expert) as the reference's dispatch does; 1: node dedup; 2 (default):
 * node dedup when top_k >= 2 e (a token reaches ~k/e experts per node). */
moe_status moe_ctx_set_node_dedup(moe_ctx* ctx, int32_t mode);

/* Route every local card (moe_route_topk on its logits). */
moe_status moe_ctx_route(moe_ctx* ctx, void* stream);
/* Materialise the permuted batch of every local card (dataplane::permute). */
moe_status moe_ctx_permute(moe_ctx* ctx, int32_t n_chunks, void* stream);
/* Dispatch (dataplane::dispatch_monolithic when level == MOE_BASELINE,
 * dataplane::dispatch_chunked otherwise).  Builds the index, exchanges the
 * per-chunk counts, and moves rows.  Validation mirrors dataplane.hpp:190-216. */
moe_status moe_ctx_dispatch(moe_ctx* ctx, int level, int32_t n_chunks, int landing, void* stream);
/* Second AllToAll + weighted un-permute (dataplane::combine_unpermute),
 * mirrored per level: BASELINE returns full rows; O1/O2/O3 return the
 * receiving rank's 1/t slice, un-permute it and all-gather the output
 * slices inside the node.  Must follow a dispatch with the same n. */
moe_status moe_ctx_combine(moe_ctx* ctx, int level, int32_t n_chunks, void* stream);
/* route + dispatch + (bound experts) + combine. */
moe_status moe_ctx_forward(moe_ctx* ctx, int level, int32_t n_chunks, int landing, void* stream);
/* Measured schedule choice (the planner's candidates checked in place):
 * each candidate runs `steps` timed forwards through this context; times
 * (us/layer, written back into .us) are max-reduced over the ranks of a
 * multi-GPU context through peer memory, so all ranks return the same
 * *best (index of the fastest; ties keep the earlier).  Every rank must call
 * it with the same candidates. */
typedef struct moe_schedule {
  int32_t level, n_chunks, landing;
  double us;
} moe_schedule;
moe_status moe_ctx_autotune(moe_ctx* ctx, moe_schedule* candidates, int32_t count, int32_t steps,
                            void* stream, int32_t* best);
/* End-to-end from HOST buffers: H2D of x/logits for every local card
 * (node-major [local cards][T][...]), forward, D2H of `out`.  Host buffers
 * should be pinned for async copies.  A lone card (1x1 context) with
 * MOE_LAND_FINAL picks its own token chunking to overlap the copies with the
 * layer (the result does not depend on n there); STAGED landing honours
 * n_chunks and populates pre/pre_tags like moe_ctx_forward. */
moe_status moe_ctx_forward_host(moe_ctx* ctx, int level, int32_t n_chunks, int landing,
                                const void* host_x, const void* host_logits, void* host_out,
                                void* stream);
/* Layer backward on the device (the reference has no backward; these are
 * the adjoints of combine_unpermute / dispatch routed through the forward's
 * own exchanges).  After a forward with the same
 * level and n (the routing must still be in the context):
 *   moe_ctx_backward_combine: d loss / d out is read from each card's x
 *     buffer (payload dtype; equal on a node's TP cards); it is dispatched
 *     with the forward's plan into each card's `pre` buffer (recv — the
 *     forward's rows / expert outputs — is left intact), then on every expert
 *     card pre[r] := p_r * g[r] (d loss / d expert output), and the partial
 *     <g[r], y[r]> of each TP card's column slice goes to every TP card of
 *     the source node, summed there in fixed order into grad_probs [T, k];
 *     grad_logits [T, E] follows (softmax adjoint).  No host round trip.
 *   moe_ctx_backward_dispatch: d loss / d x into `out` — the forward combine
 *     with unit weights over the gradient rows in `pre` (grad_y, or the
 *     expert-input gradient a caller's expert backward wrote there).
 *   moe_ctx_backward: both (identity experts). */
moe_status moe_ctx_backward_combine(moe_ctx* ctx, int level, int32_t n_chunks, void* stream);
moe_status moe_ctx_backward_dispatch(moe_ctx* ctx, int level, int32_t n_chunks, void* stream);
moe_status moe_ctx_backward(moe_ctx* ctx, int level, int32_t n_chunks, void* stream);
/* Emulated inter-node link (the paper's B1 << B2 regime, PAPER.md:183-184,
 * on one NVSwitch box): every cross-node leg — the dispatch AllToAll and the
 * combine's reverse AllToAll, naive or deduplicated — completes no sooner
 * than its bytes / gbps (GB/s per card), while the intra-node AllGather and
 * local copies run at NVLink / HBM speed.  0 = off.  Applies to every
 * exchange path (persistent kernels and per-leg launches); with the fp8 wire
 * a leg is paced on its fp8 bytes + scales. */
moe_status moe_ctx_set_link_rate(moe_ctx* ctx, double gbps);
/* Dispatch wire format of the cross-node (AllToAll) legs (SURVEY.md §8(f)
 * item 3).  MOE_WIRE_BF16 (default): rows move bit-exactly.  MOE_WIRE_FP8:
 * the sender quantises each 128-element block of a cross-node row slice to
 * e4m3 (x / scale, scale = amax / 448, round to nearest, saturating) with
 * that fp32 scale and
 * stores bytes + scales into the receiver's pre / scale buffers — half the
 * AllToAll bytes; the receiver decodes them into recv before the intra-node
 * AllGather forwards its slice (bf16).  The combine's reverse AllToAll uses
 * the same format (expert outputs -> the source's fp8 landing, decoded per
 * chunk before the un-permute).  Own-node rows stay bf16.  Lossy by
 * design (one e4m3 rounding, <= 2^-4 relative per element); needs a bf16
 * payload, hidden and hidden/t multiples of 128, top_k <= 16, FINAL landing;
 * runs the per-leg launches. */
#define MOE_WIRE_BF16 0
#define MOE_WIRE_FP8 1
moe_status moe_ctx_set_wire(moe_ctx* ctx, int wire);
/* Routing checks (the reference's CorruptRoutingError, dataplane.hpp:18-20):
 * when enabled, every dispatch first poisons the receive tags, and
 * moe_ctx_forward (or moe_ctx_verify after moe_ctx_dispatch) checks every
 * landed row's tags {source card, position, expert} against the receiving
 * node's reference layout (expert-major, sources ascending, positions
 * ascending) on the device; a lost, duplicated or misplaced row raises
 * MOE_ERR_CORRUPT_ROUTING at the next moe_ctx_sync. */
moe_status moe_ctx_enable_checks(moe_ctx* ctx, int enable);
moe_status moe_ctx_verify(moe_ctx* ctx, void* stream);
/* Rows in card's recv buffer after the last dispatch (synchronises). */
moe_status moe_ctx_recv_rows(moe_ctx* ctx, int card, int64_t* rows);
/* Synchronise the context's streams and report device-side errors
 * (corrupt routing, out-of-range experts, flag timeouts). */
moe_status moe_ctx_sync(moe_ctx* ctx);
/* Per-stage timing of the last dispatch/combine (ms, from CUDA events
 * recorded when enabled).  stage ids: see moe_stage.  Returns MOE_OK with
 * *n_spans == 0 when timing is disabled. */
typedef enum moe_stage {
  MOE_STAGE_ROUTE = 0,
  MOE_STAGE_INDEX = 1,
  MOE_STAGE_AA = 2,
  MOE_STAGE_AG = 3,
  MOE_STAGE_D2D = 4,
  MOE_STAGE_CAA = 5,
  MOE_STAGE_UNPERMUTE = 6,
  MOE_STAGE_TOTAL = 7,
  MOE_STAGE_EXPERTS = 8
} moe_stage;
typedef struct moe_span {
  int32_t stage;
  int32_t chunk;
  float start_ms; /* relative to the dispatch start event */
  float end_ms;
} moe_span;
moe_status moe_ctx_enable_timing(moe_ctx* ctx, int enable);
/* Replay moe_ctx_forward / moe_ctx_forward_host as CUDA graphs: each
 * (level, n, landing, host buffers) is captured once (every stream of the
 * step) and replayed; flags carry a device-resident epoch so replays stay in
 * lockstep across ranks.  Ignored while timing is enabled. */
moe_status moe_ctx_enable_graphs(moe_ctx* ctx, int enable);
moe_status moe_ctx_spans(moe_ctx* ctx, moe_span* spans, int32_t capacity, int32_t* n_spans);
/* Cap the CTAs of the cross-group (AllToAll, dispatch and combine) copy
 * kernels, emulating a slow inter-node link — the paper's B2/B1 >> 1 regime
 * on one NVSwitch box.  While capped the context runs the
 * per-leg launches (AllToAll on the high-priority stream, AllGather and
 * reorder copies on their own at full width), so only the cross-node legs
 * are throttled.  0 = no cap (persistent exchange kernels). */
moe_status moe_ctx_set_aa_ctas(moe_ctx* ctx, int32_t ctas);
/* Transport primitive (calibration / microbenchmarks, config 5): card-local
 * rows [0, sum) of this card's `recv` buffer are stored, rows_per_card[c]
 * of them to card c (consecutive source rows per destination), each row
 * `row_bytes` wide, with the exchange's copy kernel on `grid` CTAs
 * (0 = default).  A peer destination receives into its `recv` buffer over
 * NVLink; this card itself receives into its `pre` buffer (a local D2D
 * copy).  Only local + peer-mapped cards may be named. */
moe_status moe_ctx_xfer(moe_ctx* ctx, const int64_t* rows_per_card, int32_t row_bytes, int32_t grid,
                        void* stream);
/* Debug: record phase timestamps of the fused front kernel and the start /
 * end of the persistent exchange kernels (enable != 0); with out20 != NULL,
 * synchronise and copy the card's 20 globaltimer stamps (ns): [0..15] front,
 * [16..17] dispatch kernel start/end, [18..19] combine kernel start/end. */
moe_status moe_ctx_debug_front(moe_ctx* ctx, int enable, int card, uint64_t* out20);
/* Multi-GPU contexts run each phase (dispatch, combine) as ONE persistent,
 * role-specialised cooperative kernel with per-chunk flags (default on);
 * enable = 0 selects one launch per (leg, chunk) on prioritised streams. */
moe_status moe_ctx_set_persistent(moe_ctx* ctx, int enable);
/* Role trace of the last persistent dispatch/combine (timing enabled):
 * out[((kernel * 4 + role) * max_chunks + j) * 2 + {0,1}] = globaltimer ns of
 * the first CTA starting / the last CTA finishing chunk j of the role;
 * kernel 0 = dispatch (roles AA, AAL, AG, D2D), 1 = combine (CAA, UNP).
 * Unused entries hold UINT64_MAX / 0xff.. patterns. */
moe_status moe_ctx_xchg_trace(moe_ctx* ctx, int card, uint64_t* out, int32_t capacity, int32_t* max_chunks);
/* Number of kernels this context launched since creation. */
int64_t moe_ctx_launch_count(const moe_ctx* ctx);

/* ------------------------------------------------------------------------
 * 3. Planner (host, fp64)
 * ------------------------------------------------------------------------ */
typedef struct moe_model_spec { /* config.hpp:14-24 */
  int64_t b, s, h, a, l, k, p1, p2;
  int32_t bpe;
} moe_model_spec;
typedef struct moe_parallel_spec { /* config.hpp:26-32 */
  int32_t d, p, t, e, cp;
} moe_parallel_spec;
typedef struct moe_cluster_spec { /* config.hpp:34-42 */
  int32_t nodes, gpus_per_node;
  double b1, b2, b3, peak_flops;
  int64_t switch_capacity;
} moe_cluster_spec;
typedef struct moe_curve { /* EfficiencyCurve, config.hpp:49-61; volumes strictly increasing */
  const double* volume;
  const double* efficiency;
  int32_t n_points;
  double i_minimal;
} moe_curve;
typedef struct moe_curve_set {
  moe_curve alltoall, allgather, d2d;
} moe_curve_set;
typedef struct moe_overhead { /* OverheadModel, commcost.hpp:24-27 */
  double alpha_comm, alpha_copy;
} moe_overhead;
typedef struct moe_chunk_timing { /* ChunkTiming, commcost.hpp:30-36 */
  double aa, ag, d2d;
  int32_t n;
  double volume;
} moe_chunk_timing;
typedef struct moe_chunk_search_result { /* ChunkSearchResult, chunkopt.hpp:26-31 */
  int32_t n_opt;
  double t_pred;
  moe_chunk_timing per_chunk;
  int32_t feasible;
} moe_chunk_search_result;
typedef struct moe_strategy_alt {
  int32_t level;
  double t_pred;
  int32_t n;
} moe_strategy_alt;
typedef struct moe_strategy_decision { /* StrategyDecision, strategy.hpp:13-18 */
  int32_t level;
  int32_t n;
  double t_pred;
  int32_t n_alternatives;
  moe_strategy_alt alternatives[3];
} moe_strategy_decision;
typedef struct moe_perf_report {
  double step_latency, throughput, mfu;
} moe_perf_report;

moe_status moe_lookup_efficiency(const moe_curve* curve, double volume, double* out);
double moe_traffic_volume(const moe_model_spec* m);
moe_status moe_chunk_alltoall_time(double volume, int32_t n, int32_t t, int32_t e, double b1,
                                   const moe_curve* curve, const moe_overhead* ov, double* out);
moe_status moe_chunk_allgather_time(double volume, int32_t n, int32_t t, double b2,
                                    const moe_curve* curve, const moe_overhead* ov, double* out);
moe_status moe_chunk_d2d_time(double volume, int32_t n, double b3, const moe_curve* curve,
                              const moe_overhead* ov, double* out);
moe_status moe_baseline_time(double volume, int32_t e, double b1, const moe_curve* curve,
                             const moe_overhead* ov, double* out);
moe_status moe_o1_time(double volume, int32_t t, int32_t e, double b1, double b2,
                       const moe_curve_set* curves, const moe_overhead* ov, double* out);
double moe_o2_score(double aa, double ag, double d2d, int32_t n);
double moe_o3_score(double aa, double ag, double d2d, int32_t n);
moe_status moe_o2_search(const moe_model_spec* m, const moe_parallel_spec* par,
                         const moe_cluster_spec* cl, const moe_curve_set* curves,
                         const moe_overhead* ov, int32_t n_cap, moe_chunk_search_result* out);
moe_status moe_o3_search(const moe_model_spec* m, const moe_parallel_spec* par,
                         const moe_cluster_spec* cl, const moe_curve_set* curves,
                         const moe_overhead* ov, int32_t n_cap, moe_chunk_search_result* out);
moe_status moe_asymptotic_speedup(int32_t t, int32_t e, double b1, double b2, double r1,
                                  double r2, double* out);
moe_status moe_select_strategy(const moe_model_spec* m, const moe_parallel_spec* par,
                               const moe_cluster_spec* cl, const moe_curve_set* curves,
                               const moe_overhead* ov, int32_t n_cap, moe_strategy_decision* out);
/* B200 variant of select_strategy.  shared_egress == 0: exactly
 * moe_select_strategy (the reference's separate inter-/intra-node links).
 * shared_egress != 0 (every card on one NVSwitch domain, no AllToAll cap):
 * both legs leave through the same NVLink egress, so chunking cannot
 * overlap them, and the engine lands rows at their final offsets (no reorder
 * copy): O2/O3 score aa(n=1) + ag(n=1) + (n - 1) alpha_comm — same
 * candidates, gates, search and tie order as the reference. */
moe_status moe_select_strategy_b200(const moe_model_spec* m, const moe_parallel_spec* par,
                                    const moe_cluster_spec* cl, const moe_curve_set* curves,
                                    const moe_overhead* ov, int32_t n_cap, int32_t shared_egress,
                                    moe_strategy_decision* out);
moe_status moe_estimate_performance(const moe_strategy_decision* d, const moe_model_spec* m,
                                    const moe_parallel_spec* par, const moe_cluster_spec* cl,
                                    int32_t moe_layer_count, double non_comm_time,
                                    moe_perf_report* out);

/* calibrate (calibrate.hpp:84-118).  primitive: 0 alltoall, 1 allgather, 2 d2d.
 * Output curves are written into caller arrays of capacity `count` each
 * (volumes/efficiencies per primitive), with point counts in n_points[3]. */
typedef struct moe_bench_sample {
  int32_t primitive;
  double volume;
  double seconds;
} moe_bench_sample;
moe_status moe_calibrate(const moe_bench_sample* samples, int32_t count,
                         const moe_cluster_spec* cl, double* volumes /*[3][count]*/,
                         double* efficiencies /*[3][count]*/, int32_t* n_points /*[3]*/,
                         moe_overhead* overhead);

/* pipesim::build_pipeline + pipesim::simulate (pipesim.hpp:91-173).
 * Streams: 0 alltoall, 1 allgather, 2 d2d, 3 compute.  Task ids follow the
 * reference ("dispatch_aa_1", ...) and are written as `kind` codes:
 * kind = phase*8 + {0 aa, 1 ag, 2 d2d, 3 expert}; chunk is 1-based. */
typedef struct moe_sim_span {
  int32_t kind;
  int32_t chunk;
  int32_t stream;
  double start, end;
} moe_sim_span;
moe_status moe_simulate_pipeline(int level, int32_t n, const moe_chunk_timing* timing,
                                 double expert_time, int32_t phases, moe_sim_span* spans,
                                 int32_t capacity, int32_t* n_spans, double* makespan);
/* General list scheduler over an explicit task graph (pipesim::simulate).
 * deps are indices into the task array, flattened with offsets. */
typedef struct moe_sim_task {
  int32_t stream;
  double duration;
  int32_t dep_begin, dep_end; /* range into deps[] */
} moe_sim_task;
moe_status moe_simulate_graph(const moe_sim_task* tasks, int32_t count, const int32_t* deps,
                              double* start, double* end, double* makespan);
/* pipesim::build_pipeline (pipesim.hpp:91-105) as an explicit task graph:
 * tasks[i] {stream, duration, dep range into deps}, kinds[i] (as in
 * moe_sim_span), chunks[i] (1-based).  tasks == NULL: *count only. */
moe_status moe_build_pipeline(int level, int32_t n, const moe_chunk_timing* timing, double expert_time,
                              int32_t phases, moe_sim_task* tasks, int32_t* kinds, int32_t* chunks,
                              int32_t capacity, int32_t* deps, int32_t dep_capacity, int32_t* count);

/* config.hpp check(ModelSpec|ParallelSpec|ClusterSpec) and validate()
 * (config.hpp:89-158): one message per violated rule, '\n'-separated into
 * buf (truncated to capacity; *bytes_needed = full size + 1). */
#define MOE_CHECK_MODEL 0
#define MOE_CHECK_PARALLEL 1
#define MOE_CHECK_CLUSTER 2
#define MOE_CHECK_PLACEMENT 3
moe_status moe_check_specs(int which, const moe_model_spec* m, const moe_parallel_spec* p,
                           const moe_cluster_spec* c, char* buf, int64_t capacity, int32_t* n_messages,
                           int64_t* bytes_needed);

#ifdef __cplusplus
} /* extern "C" */
#endif
#endif /* MONTA_H_ */

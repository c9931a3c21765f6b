// Weighted un-permute: the arithmetic of dataplane::combine_unpermute
// (reference dataplane.hpp:317-344):  out[i,q] = sum_s probs[i,s] * y(i,s)[q],
// accumulated from zero in ascending slot order.
//
// y(i,s) is the expert output row of token i's s-th expert.  Rows that came
// back over the reverse AllToAll sit in `comb` at the sender-permuted
// position slot_pos[i,s]; rows whose expert lives on this card's own node are
// read in place from the node's final-layout expert outputs (local_y), which
// saves the local half of the reverse exchange.  Output rows (or this rank's
// 1/t column slice of them) are written to every card of `out[]` — in the
// TP-deduplicated combine that store IS the intra-node all-gather.
//
// One warp per token; each lane owns 16-byte column vectors; fp32
// accumulation for 16/32-bit inputs, fp64 for f64/i64 (the reference's
// double arithmetic, without FMA contraction).
#include <algorithm>
#include <cstdlib>

#include "copy.cuh"

namespace monta {
namespace {

constexpr int kThreads = 256;
constexpr int kMaxK = 32;

template <class T, int N> struct alignas(sizeof(T) * N) Pack { T v[N]; };

template <class TAcc> __device__ __forceinline__ TAcc madd(TAcc acc, TAcc p, TAcc y);
template <> __device__ __forceinline__ float madd<float>(float acc, float p, float y) {
  return fmaf(p, y, acc);
}
template <> __device__ __forceinline__ double madd<double>(double acc, double p, double y) {
  return __dadd_rn(acc, __dmul_rn(p, y));  // reference: acc += p * double(y), unfused
}

template <class TIn, class TAcc> __device__ __forceinline__ TAcc widen(TIn v) { return TAcc(v); }
template <> __device__ __forceinline__ float widen<__nv_bfloat16, float>(__nv_bfloat16 v) {
  return __bfloat162float(v);
}
template <> __device__ __forceinline__ float widen<__half, float>(__half v) { return __half2float(v); }
template <> __device__ __forceinline__ double widen<int64_t, double>(int64_t v) { return double(v); }

template <class TAcc, class TOut> __device__ __forceinline__ TOut narrow(TAcc v) { return TOut(v); }
template <> __device__ __forceinline__ __nv_bfloat16 narrow<float, __nv_bfloat16>(float v) {
  return __float2bfloat16_rn(v);
}
template <> __device__ __forceinline__ __half narrow<float, __half>(float v) { return __float2half_rn(v); }

constexpr int kDeltaSmem = 1024;  // own-node expert deltas staged in shared memory up to this many

// Column vectors per lane per work item.
template <int N> constexpr int unperm_uv() { return N >= 8 ? 4 : 2; }

// Tokens [tok_begin, tok_end) by a group of warps.  Work item = (token,
// column batch of 32*UV vectors); warp (warp0 + w) of `nwarps` takes items
// warp0 + w, strided by nwarps, so the grid balances at sub-token grain.
// Per-warp pipeline: while item i is computed, the row addresses of item i+1
// are staged and the index entries (slot, expert, weight) of item i+2 are in
// flight.  Own-node expert deltas sit in shared memory, so a row address is
// one dependent load away from its index.
template <class TIn, class TAcc, class TOut, class TProb, int N, int UV = unperm_uv<N>()>
__device__ __forceinline__ void unpermute_tokens(const UnpermArgs& a, int64_t tok_begin, int64_t tok_end,
                                                 int64_t warp0, int64_t nwarps) {
  // Per-warp staging (double-buffered) of an item's k source rows and weights:
  // the column loop below has a lane-dependent trip count, so no shuffles in it.
  __shared__ const char* s_row[2][kThreads / 32][kMaxK];
  __shared__ TAcc s_p[2][kThreads / 32][kMaxK];
  __shared__ int s_delta[kDeltaSmem];
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  const TProb* probs = static_cast<const TProb*>(a.probs);
  const int64_t nvec = a.cols / N;
  const int64_t nb = (nvec + 32 * UV - 1) / (32 * UV);
  const int64_t n_items = (tok_end - tok_begin) * nb;
  const int nloc = a.local_y ? a.local_hi - a.local_lo : 0;
  const bool delta_smem = nloc <= kDeltaSmem;
  if (delta_smem)
    for (int l = threadIdx.x; l < nloc; l += blockDim.x) s_delta[l] = __ldg(a.local_delta + a.local_lo + l);
  __syncthreads();
  int pos = -1, x = -1;
  TAcc p = TAcc(0);
  auto load_index = [&](int64_t item) {
    if (item < n_items && lane < a.k) {
      const int64_t q = (tok_begin + item / nb) * a.k + lane;
      pos = __ldg(a.slot_pos + q);
      x = __ldg(a.experts + q);
      p = TAcc(__ldg(probs + q));
    }
  };
  // rows of `item` from the index registers into staging buffer `buf`
  auto stage = [&](int buf) {
    if (lane < a.k) {
      s_p[buf][wib][lane] = p;
      const char* row;
      if (pos < 0) {
        row = nullptr;  // empty slot (negative expert id)
      } else if (nloc && x >= a.local_lo && x < a.local_hi) {
        const int d = delta_smem ? s_delta[x - a.local_lo] : __ldg(a.local_delta + x);
        row = a.local_y + (int64_t(pos) + d) * a.y_stride;
      } else {
        row = a.comb + int64_t(pos) * a.y_stride;
      }
      s_row[buf][wib][lane] = row;
    }
  };
  int64_t it = warp0 + wib;
  int buf = 0;
  load_index(it);
  if (it < n_items) stage(0);
  load_index(it + nwarps);
  for (; it < n_items; it += nwarps, buf ^= 1) {
    __syncwarp();
    if (it + nwarps < n_items) stage(buf ^ 1);
    load_index(it + 2 * nwarps);
    const int64_t i = tok_begin + it / nb;
    const int64_t v0 = (it % nb) * (32 * UV) + lane;
    // slots in groups of SG: all SG*UV loads of a group are issued before its
    // first multiply-add (the slot loop has a runtime trip count, so without
    // the grouping each slot's loads would wait for the previous slot's math);
    // accumulation stays in ascending slot order
    constexpr int SG = 2;
    TAcc acc[UV][N];
#pragma unroll
    for (int w = 0; w < UV; ++w)
#pragma unroll
      for (int u = 0; u < N; ++u) acc[w][u] = TAcc(0);
    for (int s0 = 0; s0 < a.k; s0 += SG) {
      const char* rows[SG];
      Pack<TIn, N> y[SG][UV];
#pragma unroll
      for (int g = 0; g < SG; ++g) {
        rows[g] = s0 + g < a.k ? s_row[buf][wib][s0 + g] : nullptr;
#pragma unroll
        for (int w = 0; w < UV; ++w) {
          const int64_t v = v0 + w * 32;
          if (rows[g] && v < nvec)
            y[g][w] = *reinterpret_cast<const Pack<TIn, N>*>(rows[g] + (a.col_begin + v * N) * sizeof(TIn));
        }
      }
#pragma unroll
      for (int g = 0; g < SG; ++g) {
        if (!rows[g]) continue;
        const TAcc ps = s_p[buf][wib][s0 + g];
#pragma unroll
        for (int w = 0; w < UV; ++w)
#pragma unroll
          for (int u = 0; u < N; ++u) acc[w][u] = madd<TAcc>(acc[w][u], ps, widen<TIn, TAcc>(y[g][w].v[u]));
      }
    }
#pragma unroll
    for (int w = 0; w < UV; ++w) {
      const int64_t v = v0 + w * 32;
      if (v >= nvec) continue;
      const int64_t col = a.col_begin + v * N;
      Pack<TOut, N> o;
#pragma unroll
      for (int u = 0; u < N; ++u) o.v[u] = narrow<TAcc, TOut>(acc[w][u]);
      for (int d = 0; d < a.n_out; ++d)
        *reinterpret_cast<Pack<TOut, N>*>(a.out[d] + i * a.out_stride + col * sizeof(TOut)) = o;
    }
    __syncwarp();
  }
}

// Lean top-1/top-2 un-permute (16-byte vectors, fp32 accumulation): warp per
// item of (token, 32*UV vectors); both slots' UV loads are in flight at once;
// row addresses and weights are broadcast by shuffle from lanes 0..k-1 (no
// staging); 32-bit item arithmetic keeps registers low — occupancy is what
// keeps the gather at HBM speed (scripts/micro/gather_bench.cu: 5.7 TB/s at
// 16 warps/SM, 6.3 TB/s at 32 warps/SM for the same bytes in flight).  The
// bf16 top-2 launch runs 2 KiB items at 3 CTAs/SM (80 registers): 1 KiB items
// at 4 CTAs/SM measured slower, and 2 KiB items under the 64-register cap of
// 4 CTAs/SM spill (ptxas: 72 B of spill stores).
template <class TIn, class TOut, class TProb, int UV, int MinB, int KMAX = 2>
__global__ void __launch_bounds__(kThreads, MinB) k_unpermute_k2(const __grid_constant__ UnpermArgs a) {
  constexpr int N = 16 / sizeof(TIn);
  __shared__ int s_delta[kDeltaSmem];
  if (!cta_wait(a.wait, a.err)) return;
  const int lane = threadIdx.x & 31;
  const int nvec = int(a.cols / N);
  const int nb = nvec / (32 * UV);  // launcher: nvec % (32*UV) == 0
  const int n_items = int(a.tok_end - a.tok_begin) * nb;
  const int nloc = a.local_y ? a.local_hi - a.local_lo : 0;
  const bool delta_smem = nloc <= kDeltaSmem;
  if (delta_smem)
    for (int l = threadIdx.x; l < nloc; l += blockDim.x) s_delta[l] = __ldg(a.local_delta + a.local_lo + l);
  __syncthreads();
  const TProb* probs = static_cast<const TProb*>(a.probs);
  const int k = a.k;
  const int warps = int(gridDim.x) * (kThreads / 32);
  const uint64_t pol = l2_evict_first_policy();
  for (int it = int(blockIdx.x) * (kThreads / 32) + (threadIdx.x >> 5); it < n_items; it += warps) {
    const int64_t i = a.reverse ? a.tok_end - 1 - it / nb : a.tok_begin + it / nb;  // newest rows first (L2)
    const int cv = (it % nb) * (32 * UV);  // first vector of the item
    const char* row = nullptr;
    float p = 0.f;
    if (lane < k) {
      const int64_t q = i * k + lane;
      const int pos = __ldg(a.slot_pos + q);
      const int x = __ldg(a.experts + q);
      p = float(__ldg(probs + q));
      if (pos >= 0) {
        if (nloc && x >= a.local_lo && x < a.local_hi) {
          const int d = delta_smem ? s_delta[x - a.local_lo] : __ldg(a.local_delta + x);
          row = a.local_y + (int64_t(pos) + d) * a.y_stride;
        } else {
          row = a.comb + int64_t(pos) * a.y_stride;
        }
        row += (a.col_begin + int64_t(cv) * N) * int64_t(sizeof(TIn));  // the item's first vector
      }
    }
    // slot rows (null: empty slot or k == 1) broadcast from lanes 0 and 1
    const char* r0 = reinterpret_cast<const char*>(__shfl_sync(0xffffffffu, reinterpret_cast<uintptr_t>(row), 0));
    const char* r1 = reinterpret_cast<const char*>(__shfl_sync(0xffffffffu, reinterpret_cast<uintptr_t>(row), 1));
    const float p0 = __shfl_sync(0xffffffffu, p, 0), p1 = __shfl_sync(0xffffffffu, p, 1);
    if (KMAX < 2 || k < 2) r1 = nullptr;  // KMAX == 1: top-1 instance, wider items instead of a second slot
    Pack<TIn, N> y0[UV], y1[UV];
#pragma unroll
    for (int w = 0; w < UV; ++w) {  // rows are read once: L2 evict-first (1% per layer, A/B)
      if (r0) {
        const int4 q = ld_stream_ef(reinterpret_cast<const int4*>(r0 + w * 512 + lane * 16), pol);
        y0[w] = *reinterpret_cast<const Pack<TIn, N>*>(&q);
      }
      if (r1) {
        const int4 q = ld_stream_ef(reinterpret_cast<const int4*>(r1 + w * 512 + lane * 16), pol);
        y1[w] = *reinterpret_cast<const Pack<TIn, N>*>(&q);
      }
    }
    const int64_t obase = i * a.out_stride + (a.col_begin + int64_t(cv + lane) * N) * int64_t(sizeof(TOut));
#pragma unroll
    for (int w = 0; w < UV; ++w) {
      float acc[N];
#pragma unroll
      for (int u = 0; u < N; ++u) acc[u] = 0.f;
      if (r0)
#pragma unroll
        for (int u = 0; u < N; ++u) acc[u] = madd<float>(acc[u], p0, widen<TIn, float>(y0[w].v[u]));
      if (r1)
#pragma unroll
        for (int u = 0; u < N; ++u) acc[u] = madd<float>(acc[u], p1, widen<TIn, float>(y1[w].v[u]));
      Pack<TOut, N> o;
#pragma unroll
      for (int u = 0; u < N; ++u) o.v[u] = narrow<float, TOut>(acc[u]);
      for (int d = 0; d < a.n_out; ++d)
        *reinterpret_cast<Pack<TOut, N>*>(a.out[d] + obase + w * 32 * N * int(sizeof(TOut))) = o;
    }
  }
  cta_signal(a.sig);
}

// Un-permute for any k with 16-bit rows: CTA per token (the layout of the
// dispatch backward, backward.cu, which runs the same k-row gather-sum at
// 0.95 of the HBM peak).  The CTA is sized so every round of U 16-byte
// vectors per thread covers the row (DeepSeek h = 5120: 160 threads x 2 x 2
// rounds);
// threads 0..k-1 resolve the token's slot rows and weights into shared
// memory (double-buffered: one barrier per token); SG slots' loads are in
// flight before their multiply-adds, which stay in ascending slot order
// (bit-identical to k_unpermute).  Many small CTAs per SM keep the gather
// saturated without a per-warp index pipeline.
constexpr int kRowThreads = 256;
template <class TIn, class TOut, class TProb, int U, int SG, int MinB>
__global__ void __launch_bounds__(kRowThreads, MinB) k_unpermute_rows(const __grid_constant__ UnpermArgs a) {
  constexpr int N = 16 / sizeof(TIn);
  __shared__ const char* s_row[2][kMaxK];
  __shared__ float s_p[2][kMaxK];
  __shared__ int s_delta[kDeltaSmem];
  if (!cta_wait(a.wait, a.err)) return;
  const int nloc = a.local_y ? a.local_hi - a.local_lo : 0;
  const bool delta_smem = nloc <= kDeltaSmem;
  if (delta_smem)
    for (int l = threadIdx.x; l < nloc; l += blockDim.x) s_delta[l] = __ldg(a.local_delta + a.local_lo + l);
  __syncthreads();  // threads 0..k-1 read the deltas before the token loop's barrier
  const TProb* probs = static_cast<const TProb*>(a.probs);
  const int k = a.k;
  const int nvec = int(a.cols / N);
  const uint64_t pol = l2_evict_first_policy();
  int buf = 0;
  for (int64_t it = a.tok_begin + blockIdx.x; it < a.tok_end; it += gridDim.x, buf ^= 1) {
    // newest rows first: the permute wrote tokens in ascending order, so the
    // highest tokens' rows are the ones still in L2
    const int64_t i = a.reverse ? a.tok_end - 1 - (it - a.tok_begin) : it;
    if (threadIdx.x < k) {
      const int64_t q = i * k + threadIdx.x;
      const int pos = __ldg(a.slot_pos + q);
      const int x = __ldg(a.experts + q);
      const char* row = nullptr;
      if (pos >= 0) {
        if (nloc && x >= a.local_lo && x < a.local_hi) {
          const int d = delta_smem ? s_delta[x - a.local_lo] : __ldg(a.local_delta + x);
          row = a.local_y + (int64_t(pos) + d) * a.y_stride;
        } else {
          row = a.comb + int64_t(pos) * a.y_stride;
        }
        row += a.col_begin * int64_t(sizeof(TIn));
      }
      s_row[buf][threadIdx.x] = row;
      s_p[buf][threadIdx.x] = float(__ldg(probs + q));
    }
    __syncthreads();
    for (int c0 = threadIdx.x; c0 < nvec; c0 += blockDim.x * U) {
      float acc[U][N];
#pragma unroll
      for (int u = 0; u < U; ++u)
#pragma unroll
        for (int j = 0; j < N; ++j) acc[u][j] = 0.f;
      for (int s0 = 0; s0 < k; s0 += SG) {
        int4 v[SG][U];
        const char* rows[SG];
#pragma unroll
        for (int g = 0; g < SG; ++g) {
          rows[g] = s0 + g < k ? s_row[buf][s0 + g] : nullptr;
#pragma unroll
          for (int u = 0; u < U; ++u) {
            const int c = c0 + u * int(blockDim.x);
            if (rows[g] && c < nvec) v[g][u] = ld_stream_ef(reinterpret_cast<const int4*>(rows[g]) + c, pol);
          }
        }
#pragma unroll
        for (int g = 0; g < SG; ++g) {
          if (!rows[g]) continue;
          const float ps = s_p[buf][s0 + g];
#pragma unroll
          for (int u = 0; u < U; ++u) {
            const Pack<TIn, N> y = *reinterpret_cast<const Pack<TIn, N>*>(&v[g][u]);
#pragma unroll
            for (int j = 0; j < N; ++j) acc[u][j] = madd<float>(acc[u][j], ps, widen<TIn, float>(y.v[j]));
          }
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int c = c0 + u * int(blockDim.x);
        if (c >= nvec) continue;
        Pack<TOut, N> o;
#pragma unroll
        for (int j = 0; j < N; ++j) o.v[j] = narrow<float, TOut>(acc[u][j]);
        const int64_t off = i * a.out_stride + (a.col_begin + int64_t(c) * N) * int64_t(sizeof(TOut));
        for (int d = 0; d < a.n_out; ++d) *reinterpret_cast<Pack<TOut, N>*>(a.out[d] + off) = o;
      }
    }
  }
  cta_signal(a.sig);
}

// MinB: resident CTAs per SM the register budget must allow (occupancy, not
// per-warp depth, is what keeps enough gather loads in flight on B200:
// scripts/micro/gather_bench.cu measured 5.7 TB/s at 16 warps/SM vs 6.3 TB/s
// at 32 warps/SM for the same bytes in flight).
template <class TIn, class TAcc, class TOut, class TProb, int N, int UV = unperm_uv<N>(), int MinB = 2>
__global__ void __launch_bounds__(kThreads, MinB) k_unpermute(const __grid_constant__ UnpermArgs a) {
  if (!cta_wait(a.wait, a.err)) return;
  const int64_t wpc = blockDim.x / 32;
  unpermute_tokens<TIn, TAcc, TOut, TProb, N, UV>(a, a.tok_begin, a.tok_end, int64_t(blockIdx.x) * wpc,
                                                      int64_t(gridDim.x) * wpc);
  cta_signal(a.sig);
}

__device__ __forceinline__ SegList* comb_list(const CombArgs& a, int j) {
  char* base = reinterpret_cast<char*>(a.lists);
  return reinterpret_cast<SegList*>(base + (size_t(kPhaseCAA) * a.max_chunks + j) * seglist_bytes(a.seg_cap));
}
__device__ __forceinline__ uint64_t* comb_flag(const CombArgs& a, int owner, int ps, int j, int sender) {
  return a.flags[owner] + size_t(kSigChunkBase + ps * a.max_chunks + j) * kMaxCards + sender;
}

// Persistent combine, software-pipelined over chunks in every CTA: step s
// runs the reverse AllToAll of chunk s (CAA[s] released at the source
// cards), then waits for every remote CAA[s-1] and un-permutes chunk s-1
// (output slice stored to every TP peer; CAG[s-1] released at them).
template <class TIn, class TAcc, class TOut, class TProb, int N, int V>
__global__ void __launch_bounds__(kThreads, 2) k_combine_xchg(const __grid_constant__ CombArgs a) {
  __shared__ int s_ok;
  __shared__ unsigned long long s_epoch;
  if (threadIdx.x == 0) {
    s_epoch = *a.epoch_ptr;
    if (a.dbg && blockIdx.x == 0) a.dbg[0] = globaltimer();
  }
  __syncthreads();
  const uint64_t epoch = s_epoch;
  const int c = blockIdx.x;
  const int ctas = gridDim.x;
  const int n = a.n;
  const int64_t wpc = blockDim.x / 32;
  const int64_t ct = a.T / n;
  for (int s = 0; s <= n; ++s) {
    if (s < n && a.e > 1) {
      trace_start(a.trace, 0, a.max_chunks, s);
      const unsigned long long t0 = globaltimer();
      copy_items<V, false, false>(view_of(a.cp), comb_list(a, s), a.cpr, c, ctas);
      pace_list(comb_list(a, s), t0, a.cp.pace_bpus);
      chunk_done(a.counters + s * 17, ctas, c, [&] {
        trace_end(a.trace, 0, a.max_chunks, s);
        for (int x = 0; x < a.e; ++x)
          if (x != a.node) st_release_sys(comb_flag(a, x * a.t + a.rho, kPsCAA, s, a.me), epoch);
      });
    }
    const int j = s - 1;
    if (j < 0) continue;
    if (threadIdx.x == 0) {
      s_ok = 1;
      for (int x = 0; x < a.e && s_ok; ++x)
        if (x != a.node) s_ok = wait_flag(comb_flag(a, a.me, kPsCAA, j, x * a.t + a.rho), epoch, a.err);
    }
    __syncthreads();
    if (!s_ok) return;
    trace_start(a.trace, 1, a.max_chunks, j);
    // UV 2: the persistent kernel also carries the copy engine within 128 registers
    unpermute_tokens<TIn, TAcc, TOut, TProb, N, 2>(a.up, int64_t(j) * ct, int64_t(j + 1) * ct, int64_t(c) * wpc,
                                                   int64_t(ctas) * wpc);
    chunk_done(a.counters + (a.max_chunks + j) * 17, ctas, c, [&] {
      trace_end(a.trace, 1, a.max_chunks, j);
      if (a.dedup)
        for (int r = 0; r < a.t; ++r)
          if (r != a.rho) st_release_sys(comb_flag(a, a.node * a.t + r, kPsCAG, j, a.me), epoch);
    });
  }
  if (c == 0 && threadIdx.x == 0) {
    if (a.dedup) {  // tail: every TP peer's output slice landed here
      bool ok = true;
      for (int j = 0; j < n && ok; ++j)
        for (int r = 0; r < a.t && ok; ++r)
          if (r != a.rho) ok = wait_flag(comb_flag(a, a.me, kPsCAG, j, a.node * a.t + r), epoch, a.err);
    }
    if (a.dbg) a.dbg[1] = globaltimer();
  }
}

}  // namespace

template <class TIn, class TAcc, class TOut, class TProb, int N>
static cudaError_t launch_comb_n(const CombArgs& a, cudaStream_t s, int* max_ctas_out) {
  auto fn = k_combine_xchg<TIn, TAcc, TOut, TProb, N, 16>;
  int dev = 0, sms = 0, per_sm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, kThreads, 0);
  if (max_ctas_out) {
    *max_ctas_out = per_sm * sms;
    return cudaSuccess;
  }
  void* args[] = {const_cast<CombArgs*>(&a)};
  return cudaLaunchCooperativeKernel((const void*)fn, dim3(a.r_unp), dim3(kThreads), args, 0, s);
}

template <class TIn, class TAcc, class TOut, class TProb>
static cudaError_t launch_comb(const CombArgs& a, cudaStream_t s, int* max_ctas_out) {
  constexpr int N16 = 16 / sizeof(TIn) > 0 ? 16 / sizeof(TIn) : 1;
  const UnpermArgs& u = a.up;
  uintptr_t addr_bits = reinterpret_cast<uintptr_t>(u.comb) | reinterpret_cast<uintptr_t>(u.local_y);
  for (int d = 0; d < u.n_out; ++d) addr_bits |= reinterpret_cast<uintptr_t>(u.out[d]);
  const int64_t ib = int64_t(N16) * sizeof(TIn), ob = int64_t(N16) * sizeof(TOut);
  const bool fits = u.cols % N16 == 0 && (u.col_begin * int64_t(sizeof(TIn))) % ib == 0 &&
                    (u.col_begin * int64_t(sizeof(TOut))) % ob == 0 && u.y_stride % ib == 0 &&
                    u.out_stride % ob == 0 && addr_bits % (ib > ob ? ib : ob) == 0 && ob <= 16;
  if (!fits) return cudaErrorNotSupported;
  return launch_comb_n<TIn, TAcc, TOut, TProb, N16>(a, s, max_ctas_out);
}

cudaError_t launch_combine_xchg(const CombArgs& a, int y_dtype, int probs_dtype, int out_dtype, int vec,
                                cudaStream_t s, int* max_ctas_out) {
  if (vec != 16 || a.up.k > kMaxK || probs_dtype != MOE_F32) return cudaErrorNotSupported;
  if (y_dtype == MOE_BF16 && out_dtype == MOE_BF16) return launch_comb<__nv_bfloat16, float, __nv_bfloat16, float>(a, s, max_ctas_out);
  if (y_dtype == MOE_BF16 && out_dtype == MOE_F32) return launch_comb<__nv_bfloat16, float, float, float>(a, s, max_ctas_out);
  if (y_dtype == MOE_F32 && out_dtype == MOE_F32) return launch_comb<float, float, float, float>(a, s, max_ctas_out);
  if (y_dtype == MOE_F16 && out_dtype == MOE_F16) return launch_comb<__half, float, __half, float>(a, s, max_ctas_out);
  return cudaErrorNotSupported;
}

// A/B switch for the k > 2 un-permute (read once): MONTA_UNPERM_ROWS=0
// selects the warp-per-item kernel.
static bool unperm_rows_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("MONTA_UNPERM_ROWS");
    return !(e && e[0] == '0');
  }();
  return on;
}

// any k, 16-bit rows: CTA per token, sized so each round of U = 2 vectors
// per thread covers the row in the fewest rounds of <= 160 threads, two
// slots' loads in flight, <= 48 registers (8 CTAs of 160 threads per SM).
// Measured on the N=1 DeepSeek layer (MONTA_UNPERM_* A/B runs): 100.8 us
// against 105.6 (U = 4, one slot, 64 registers), 106.3 (U = 2, one slot),
// 101.6 (U = 2, three slots) and 113.8 for the warp-per-item k_unpermute;
// 16 CTAs per SM of grid (8: same, one token per CTA: 104.2).
template <class TIn, class TAcc, class TOut, class TProb>
static void launch_rows(const UnpermArgs& a, int grid, cudaStream_t s) {
  if constexpr (sizeof(TIn) == 2 && sizeof(TAcc) == 4) {
    const int64_t nvec = a.cols / 8;
    auto block_of = [&](int U) {
      const int64_t rounds = (nvec + int64_t(160) * U - 1) / (int64_t(160) * U);
      const int b = int(((nvec + U * rounds - 1) / (U * rounds) + 31) / 32 * 32);
      return std::min(std::max(b, 32), kRowThreads);
    };
    const int64_t toks = a.tok_end - a.tok_begin;
    const int rows_grid = int(std::max<int64_t>(1, std::min<int64_t>(toks, int64_t(grid) * 16)));
    apply_carveout(k_unpermute_rows<TIn, TOut, TProb, 2, 2, 5>);
    k_unpermute_rows<TIn, TOut, TProb, 2, 2, 5><<<rows_grid, block_of(2), 0, s>>>(a);
  }
}

template <class TIn, class TAcc, class TOut, class TProb>
static cudaError_t launch_n(const UnpermArgs& a, int grid, cudaStream_t s) {
  // Vector of N elements: as wide as 16 bytes of input allows and the column
  // range / addresses divide.
  constexpr int N16 = 16 / sizeof(TIn) > 0 ? 16 / sizeof(TIn) : 1;
  uintptr_t addr_bits = reinterpret_cast<uintptr_t>(a.comb) |
                        reinterpret_cast<uintptr_t>(a.local_y);
  for (int d = 0; d < a.n_out; ++d) addr_bits |= reinterpret_cast<uintptr_t>(a.out[d]);
  auto fits = [&](int n) {
    const int64_t ib = int64_t(n) * sizeof(TIn), ob = int64_t(n) * sizeof(TOut);
    return a.cols % n == 0 && (a.col_begin * int64_t(sizeof(TIn))) % ib == 0 &&
           (a.col_begin * int64_t(sizeof(TOut))) % ob == 0 && a.y_stride % ib == 0 &&
           a.out_stride % ob == 0 && addr_bits % (ib > ob ? ib : ob) == 0 && ob <= 16;
  };
  // grid: at most one item per warp (items = tokens x column batches)
  // grid: `grid` is the SM budget; resident CTAs per SM of the chosen
  // kernel, capped at one item per warp (items = tokens x column batches)
  auto g = [&](int n, int uv, int per_sm = 2) {
    const int64_t nb = (a.cols / n + 32 * uv - 1) / (32 * uv);
    const int64_t need = ((a.tok_end - a.tok_begin) * nb + kThreads / 32 - 1) / (kThreads / 32);
    return int(std::max<int64_t>(1, std::min<int64_t>(int64_t(grid) * per_sm, need)));
  };
  if (N16 >= 8 && fits(8) && a.k <= 2 && sizeof(TAcc) == 4 && (a.cols / 8) % (32 * 4) == 0 &&
      (a.tok_end - a.tok_begin) * (a.cols / 8) < (int64_t(1) << 31)) {
    // top-1/top-2: lean kernel, both slots' loads in flight (2 KiB items, 3 CTAs/SM;
    // 1 KiB items at 4 CTAs/SM measured slower)
    if (a.k == 1 && (a.cols / 8) % (32 * 8) == 0)  // top-1: 4 KiB items keep as many bytes in flight per warp
      k_unpermute_k2<TIn, TOut, TProb, 8, 3, 1><<<g(8, 8, 3), kThreads, 0, s>>>(a);
    else
      k_unpermute_k2<TIn, TOut, TProb, 4, 3><<<g(8, 4, 3), kThreads, 0, s>>>(a);
  } else if (N16 == 8 && sizeof(TAcc) == 4 && fits(8) && unperm_rows_enabled()) {
    launch_rows<TIn, TAcc, TOut, TProb>(a, grid, s);
  } else if (N16 >= 8 && fits(8)) {
    k_unpermute<TIn, TAcc, TOut, TProb, 8><<<g(8, unperm_uv<8>()), kThreads, 0, s>>>(a);
  } else if (N16 >= 4 && fits(4)) {
    k_unpermute<TIn, TAcc, TOut, TProb, 4><<<g(4, unperm_uv<4>()), kThreads, 0, s>>>(a);
  } else if (N16 >= 2 && fits(2)) {
    k_unpermute<TIn, TAcc, TOut, TProb, 2><<<g(2, unperm_uv<2>()), kThreads, 0, s>>>(a);
  } else {
    k_unpermute<TIn, TAcc, TOut, TProb, 1><<<g(1, unperm_uv<1>()), kThreads, 0, s>>>(a);
  }
  return cudaGetLastError();
}

template <class TIn, class TAcc, class TOut>
static cudaError_t launch_p(const UnpermArgs& a, int probs_dtype, int grid, cudaStream_t s) {
  if (probs_dtype == MOE_F64) return launch_n<TIn, TAcc, TOut, double>(a, grid, s);
  return launch_n<TIn, TAcc, TOut, float>(a, grid, s);
}

cudaError_t launch_unpermute(const UnpermArgs& a, int y_dtype, int probs_dtype, int out_dtype,
                             int grid, cudaStream_t s, bool* supported) {
  *supported = true;
  if (a.k > kMaxK) { *supported = false; return cudaSuccess; }
  switch (y_dtype) {
    case MOE_F32:
      if (out_dtype == MOE_F32) return launch_p<float, float, float>(a, probs_dtype, grid, s);
      if (out_dtype == MOE_BF16) return launch_p<float, float, __nv_bfloat16>(a, probs_dtype, grid, s);
      if (out_dtype == MOE_F16) return launch_p<float, float, __half>(a, probs_dtype, grid, s);
      if (out_dtype == MOE_F64) return launch_p<float, double, double>(a, probs_dtype, grid, s);
      break;
    case MOE_BF16:
      if (out_dtype == MOE_BF16) return launch_p<__nv_bfloat16, float, __nv_bfloat16>(a, probs_dtype, grid, s);
      if (out_dtype == MOE_F32) return launch_p<__nv_bfloat16, float, float>(a, probs_dtype, grid, s);
      break;
    case MOE_F16:
      if (out_dtype == MOE_F16) return launch_p<__half, float, __half>(a, probs_dtype, grid, s);
      if (out_dtype == MOE_F32) return launch_p<__half, float, float>(a, probs_dtype, grid, s);
      break;
    case MOE_F64:
      if (out_dtype == MOE_F64) return launch_p<double, double, double>(a, probs_dtype, grid, s);
      break;
    case MOE_I64:
      if (out_dtype == MOE_F64) return launch_p<int64_t, double, double>(a, probs_dtype, grid, s);
      break;
  }
  *supported = false;
  return cudaSuccess;
}

}  // namespace monta

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

// Tokens [tok_begin, tok_end) by a group of warps: warp (warp0 + w) of
// `nwarps` takes tokens tok_begin + warp0 + w, strided by nwarps.
template <class TIn, class TAcc, class TOut, class TProb, int N>
__device__ __forceinline__ void unpermute_tokens(const UnpermArgs& a, int64_t tok_begin, int64_t tok_end,
                                                 int64_t warp0, int64_t nwarps) {
  // Per-warp staging of the token's k source rows and weights: the column
  // loop below has a lane-dependent trip count, so no shuffles inside it.
  __shared__ const char* s_row[kThreads / 32][kMaxK];
  __shared__ TAcc s_p[kThreads / 32][kMaxK];
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  const int64_t warps = nwarps;
  const TProb* probs = static_cast<const TProb*>(a.probs);
  const int64_t nvec = a.cols / N;
  for (int64_t i = tok_begin + warp0 + (threadIdx.x >> 5); i < tok_end; i += warps) {
    if (lane < a.k) {
      const int64_t q = i * a.k + lane;
      const int pos = __ldg(a.slot_pos + q);
      const int x = __ldg(a.experts + q);
      s_p[wib][lane] = TAcc(__ldg(probs + q));
      if (pos < 0) {
        s_row[wib][lane] = nullptr;  // empty slot (negative expert id)
      } else if (a.local_y && x >= a.local_lo && x < a.local_hi) {
        s_row[wib][lane] = a.local_y + (int64_t(pos) + __ldg(a.local_delta + x)) * a.y_stride;
      } else {
        s_row[wib][lane] = a.comb + int64_t(pos) * a.y_stride;
      }
    }
    __syncwarp();
    // UV column vectors per lane per batch; for every slot the UV loads are
    // independent, and no store intervenes, so k*UV loads are in flight.
    constexpr int UV = N >= 8 ? 8 : 2;
    for (int64_t v0 = lane; v0 < nvec; v0 += 32 * UV) {
      TAcc acc[UV][N];
#pragma unroll
      for (int w = 0; w < UV; ++w)
#pragma unroll
        for (int u = 0; u < N; ++u) acc[w][u] = TAcc(0);
      for (int s = 0; s < a.k; ++s) {
        const TAcc p = s_p[wib][s];
        const char* row = s_row[wib][s];
        if (!row) continue;
        Pack<TIn, N> y[UV];
#pragma unroll
        for (int w = 0; w < UV; ++w) {
          const int64_t v = v0 + w * 32;
          if (v < nvec) y[w] = *reinterpret_cast<const Pack<TIn, N>*>(row + (a.col_begin + v * N) * sizeof(TIn));
        }
#pragma unroll
        for (int w = 0; w < UV; ++w)
#pragma unroll
          for (int u = 0; u < N; ++u) acc[w][u] = madd<TAcc>(acc[w][u], p, widen<TIn, TAcc>(y[w].v[u]));
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
    }
    __syncwarp();
  }
}

template <class TIn, class TAcc, class TOut, class TProb, int N>
__global__ void __launch_bounds__(kThreads) k_unpermute(const __grid_constant__ UnpermArgs a) {
  if (!cta_wait(a.wait, a.err)) return;
  const int64_t wpc = blockDim.x / 32;
  unpermute_tokens<TIn, TAcc, TOut, TProb, N>(a, a.tok_begin, a.tok_end, int64_t(blockIdx.x) * wpc,
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
  if (threadIdx.x == 0) s_epoch = *a.epoch_ptr;
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
      copy_items<V>(view_of(a.cp), comb_list(a, s), a.cpr, c, ctas);
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
    unpermute_tokens<TIn, TAcc, TOut, TProb, N>(a.up, int64_t(j) * ct, int64_t(j + 1) * ct, int64_t(c) * wpc,
                                                int64_t(ctas) * wpc);
    chunk_done(a.counters + (a.max_chunks + j) * 17, ctas, c, [&] {
      trace_end(a.trace, 1, a.max_chunks, j);
      if (a.dedup)
        for (int r = 0; r < a.t; ++r)
          if (r != a.rho) st_release_sys(comb_flag(a, a.node * a.t + r, kPsCAG, j, a.me), epoch);
    });
  }
  if (c == 0 && threadIdx.x == 0 && a.dedup) {  // tail: every TP peer's output slice landed here
    bool ok = true;
    for (int j = 0; j < n && ok; ++j)
      for (int r = 0; r < a.t && ok; ++r)
        if (r != a.rho) ok = wait_flag(comb_flag(a, a.me, kPsCAG, j, a.node * a.t + r), epoch, a.err);
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
  if (N16 >= 8 && fits(8)) {
    k_unpermute<TIn, TAcc, TOut, TProb, 8><<<grid, kThreads, 0, s>>>(a);
  } else if (N16 >= 4 && fits(4)) {
    k_unpermute<TIn, TAcc, TOut, TProb, 4><<<grid, kThreads, 0, s>>>(a);
  } else if (N16 >= 2 && fits(2)) {
    k_unpermute<TIn, TAcc, TOut, TProb, 2><<<grid, kThreads, 0, s>>>(a);
  } else {
    k_unpermute<TIn, TAcc, TOut, TProb, 1><<<grid, kThreads, 0, s>>>(a);
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

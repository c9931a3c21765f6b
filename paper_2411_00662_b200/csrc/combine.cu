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
#include "engine.cuh"

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

template <class TIn, class TAcc, class TOut, class TProb, int N>
__global__ void __launch_bounds__(kThreads) k_unpermute(const UnpermArgs a) {
  if (!cta_wait(a.wait, a.err)) return;
  // Per-warp staging of the token's k source rows and weights: the column
  // loop below has a lane-dependent trip count, so no shuffles inside it.
  __shared__ const char* s_row[kThreads / 32][kMaxK];
  __shared__ TAcc s_p[kThreads / 32][kMaxK];
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  const int64_t warps = int64_t(gridDim.x) * (blockDim.x / 32);
  const TProb* probs = static_cast<const TProb*>(a.probs);
  const int64_t nvec = a.cols / N;
  for (int64_t i = a.tok_begin + (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) / 32; i < a.tok_end;
       i += warps) {
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
    constexpr int UV = N >= 8 ? 4 : 2;
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
  cta_signal(a.sig);
}

}  // namespace

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

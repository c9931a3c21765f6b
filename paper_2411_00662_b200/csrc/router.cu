// Top-k gating router: dataplane::route_topk (reference dataplane.hpp:72-106).
//
// One sub-warp group of G lanes per token (G = next power of two >= E, capped
// at 32), so small expert counts pack several tokens per warp and every warp
// load is a contiguous run of the [T, E] logits.  Per token:
//   softmax   : row max, exp(s - max), sum, divide — in the logit precision;
//   selection : k rounds of a group argmax over the RAW scores with the lower
//               index winning ties (== the reference's stable_sort by score);
//   output    : experts ascending, probs = softmax of the selected experts
//               (not renormalised over the top-k).
#include "common.cuh"

namespace monta {
namespace {

template <class T> __device__ __forceinline__ T dev_exp(T x);
template <> __device__ __forceinline__ float dev_exp<float>(float x) { return expf(x); }
template <> __device__ __forceinline__ double dev_exp<double>(double x) { return exp(x); }

template <class T> __device__ __forceinline__ T neg_inf();
template <> __device__ __forceinline__ float neg_inf<float>() { return -INFINITY; }
template <> __device__ __forceinline__ double neg_inf<double>() { return -(double)INFINITY; }

// G lanes per token, PER elements per lane (E <= G * PER).
template <class T, int G, int PER>
__global__ void __launch_bounds__(256) k_route_topk(const T* __restrict__ logits, int64_t T_tokens,
                                                    int E, int k, int32_t* __restrict__ experts,
                                                    T* __restrict__ probs) {
  constexpr int kGroupsPerWarp = kWarp / G;
  const int lane = threadIdx.x & (kWarp - 1);
  const int sub = lane % G;  // lane within the token group
  const int64_t warp_global = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) / kWarp;
  const int64_t token = warp_global * kGroupsPerWarp + lane / G;
  const bool active = token < T_tokens;
  // Group mask: the G consecutive lanes of this token.
  const unsigned gmask =
      (G == 32) ? 0xffffffffu : (((1u << G) - 1u) << ((lane / G) * G));

  T v[PER];
  const T* row = logits + (active ? token : 0) * int64_t(E);
#pragma unroll
  for (int m = 0; m < PER; ++m) {
    const int x = sub + m * G;
    v[m] = (active && x < E) ? row[x] : neg_inf<T>();
  }
  // Row max.
  T mx = v[0];
#pragma unroll
  for (int m = 1; m < PER; ++m) mx = v[m] > mx ? v[m] : mx;
#pragma unroll
  for (int off = G / 2; off > 0; off >>= 1) {
    const T o = __shfl_xor_sync(gmask, mx, off, G);
    mx = o > mx ? o : mx;
  }
  // exp and sum.
  T ex[PER];
  T sum = T(0);
#pragma unroll
  for (int m = 0; m < PER; ++m) {
    const int x = sub + m * G;
    ex[m] = (x < E) ? dev_exp<T>(v[m] - mx) : T(0);
    sum += ex[m];
  }
#pragma unroll
  for (int off = G / 2; off > 0; off >>= 1) sum += __shfl_xor_sync(gmask, sum, off, G);

  // k rounds of argmax over raw scores; ties -> lower index.
  unsigned taken = 0;  // bit m: element m of this lane already selected
  int my_sel = -1;     // lane `sub` < k keeps the sub-th selected expert
  T my_soft = T(0);
  for (int s = 0; s < k; ++s) {
    T bv = neg_inf<T>();
    int bi = 0x7fffffff;
    T bs = T(0);
#pragma unroll
    for (int m = 0; m < PER; ++m) {
      const int x = sub + m * G;
      if (x < E && !((taken >> m) & 1u)) {
        if (v[m] > bv || (v[m] == bv && x < bi) || bi == 0x7fffffff) {
          bv = v[m];
          bi = x;
          bs = ex[m];
        }
      }
    }
#pragma unroll
    for (int off = G / 2; off > 0; off >>= 1) {
      const T ov = __shfl_xor_sync(gmask, bv, off, G);
      const int oi = __shfl_xor_sync(gmask, bi, off, G);
      const T os = __shfl_xor_sync(gmask, bs, off, G);
      const bool take = (oi != 0x7fffffff) &&
                        (bi == 0x7fffffff || ov > bv || (ov == bv && oi < bi));
      if (take) {
        bv = ov;
        bi = oi;
        bs = os;
      }
    }
    // Owner marks the element taken.
    if (bi != 0x7fffffff && (bi % G) == sub) taken |= 1u << (bi / G);
    if (sub == s) {
      my_sel = bi;
      my_soft = bs / sum;
    }
  }
  // Ascending order of the k selected experts: rank = #selected smaller ids.
  int rank = 0;
  for (int s = 0; s < k; ++s) {
    const int other = __shfl_sync(gmask, my_sel, (lane / G) * G + s, kWarp);
    if (other < my_sel) ++rank;
  }
  if (active && sub < k) {
    experts[token * k + rank] = my_sel;
    probs[token * k + rank] = my_soft;
  }
}

template <class T, int G, int PER>
cudaError_t launch(const T* logits, int64_t tokens, int E, int k, int32_t* experts, T* probs,
                   cudaStream_t stream) {
  constexpr int kThreads = 256;
  constexpr int kTokensPerCta = kThreads / G;
  const int64_t blocks = (tokens + kTokensPerCta - 1) / kTokensPerCta;
  k_route_topk<T, G, PER><<<unsigned(blocks), kThreads, 0, stream>>>(logits, tokens, E, k, experts,
                                                                      probs);
  return cudaGetLastError();
}

template <class T>
cudaError_t route_dispatch(const T* logits, int64_t tokens, int E, int k, int32_t* experts, T* probs,
                           cudaStream_t s) {
  if (E <= 1) return launch<T, 1, 1>(logits, tokens, E, k, experts, probs, s);
  if (E <= 2) return launch<T, 2, 1>(logits, tokens, E, k, experts, probs, s);
  if (E <= 4) return launch<T, 4, 1>(logits, tokens, E, k, experts, probs, s);
  if (E <= 8) return launch<T, 8, 1>(logits, tokens, E, k, experts, probs, s);
  if (E <= 16) return launch<T, 16, 1>(logits, tokens, E, k, experts, probs, s);
  if (E <= 32) return launch<T, 32, 1>(logits, tokens, E, k, experts, probs, s);
  if (E <= 64) return launch<T, 32, 2>(logits, tokens, E, k, experts, probs, s);
  if (E <= 128) return launch<T, 32, 4>(logits, tokens, E, k, experts, probs, s);
  if (E <= 256) return launch<T, 32, 8>(logits, tokens, E, k, experts, probs, s);
  if (E <= 512) return launch<T, 32, 16>(logits, tokens, E, k, experts, probs, s);
  return launch<T, 32, 32>(logits, tokens, E, k, experts, probs, s);
}

}  // namespace

moe_status route_topk(const void* logits, int logit_dtype, int64_t T, int E, int k, int32_t* experts,
                      void* probs, cudaStream_t stream) {
  if (k < 1) return fail(MOE_ERR_INVALID_ARGUMENT, "route_topk: k must be >= 1");
  if (E < 1 && T > 0) return fail(MOE_ERR_INVALID_ARGUMENT, "route_topk: empty gate score row");
  if (k > E && T > 0) return fail(MOE_ERR_INVALID_ARGUMENT, "route_topk: k exceeds the expert count");
  if (T == 0) return MOE_OK;
  if (E > 1024) return fail(MOE_ERR_UNSUPPORTED, "route_topk: at most 1024 experts");
  if (k > 32) return fail(MOE_ERR_UNSUPPORTED, "route_topk: at most k = 32");
  if (!logits || !experts || !probs) return fail(MOE_ERR_INVALID_ARGUMENT, "route_topk: null pointer");
  cudaError_t err;
  if (logit_dtype == MOE_F32) {
    err = route_dispatch<float>(static_cast<const float*>(logits), T, E, k, experts,
                                static_cast<float*>(probs), stream);
  } else if (logit_dtype == MOE_F64) {
    err = route_dispatch<double>(static_cast<const double*>(logits), T, E, k, experts,
                                 static_cast<double*>(probs), stream);
  } else {
    return fail(MOE_ERR_INVALID_ARGUMENT, "route_topk: logits must be f32 or f64");
  }
  if (err != cudaSuccess) return cuda_fail(err, "route_topk launch");
  return MOE_OK;
}

}  // namespace monta

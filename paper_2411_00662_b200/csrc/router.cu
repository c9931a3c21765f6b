// Top-k gating router: dataplane::route_topk (reference dataplane.hpp:72-106).
// One sub-warp group of G lanes per token (G = next power of two >= E, capped
// at 32), so small expert counts pack several tokens per warp and every warp
// load is a contiguous run of the [T, E] logits.  The arithmetic lives in
// front.cuh (route_tokens), shared with the fused front kernel.
#include "front.cuh"

namespace monta {
namespace {

template <class T, int G, int PER>
__global__ void __launch_bounds__(256) k_route_topk(const T* __restrict__ logits, int64_t T_tokens, int E, int k,
                                                    int32_t* __restrict__ experts, T* __restrict__ probs) {
  const int64_t token = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) / G;
  route_tokens<T, G, PER>(logits, T_tokens, E, k, experts, probs, token);
}

template <class T, int G, int PER>
cudaError_t launch(const T* logits, int64_t tokens, int E, int k, int32_t* experts, T* probs, cudaStream_t stream) {
  constexpr int kThreads = 256;
  constexpr int kTokensPerCta = kThreads / G;
  const int64_t blocks = (tokens + kTokensPerCta - 1) / kTokensPerCta;
  k_route_topk<T, G, PER><<<unsigned(blocks), kThreads, 0, stream>>>(logits, tokens, E, k, experts, probs);
  return cudaGetLastError();
}

template <class T>
cudaError_t route_dispatch(const T* logits, int64_t tokens, int E, int k, int32_t* experts, T* probs, cudaStream_t s) {
  if (E <= 1) return launch<T, 1, 1>(logits, tokens, E, k, experts, probs, s);
  if (E <= 2) return launch<T, 2, 1>(logits, tokens, E, k, experts, probs, s);
  if (E <= 4) return launch<T, 4, 1>(logits, tokens, E, k, experts, probs, s);
  if (E <= 8) return launch<T, 8, 1>(logits, tokens, E, k, experts, probs, s);
  if (E <= 16) return launch<T, 16, 1>(logits, tokens, E, k, experts, probs, s);
  if (E <= 32) return launch<T, 32, 1>(logits, tokens, E, k, experts, probs, s);
  if (E <= 64) return launch<T, 32, 2>(logits, tokens, E, k, experts, probs, s);
  if (E <= 96) return launch<T, 32, 3>(logits, tokens, E, k, experts, probs, s);
  if (E <= 128) return launch<T, 32, 4>(logits, tokens, E, k, experts, probs, s);
  if (E <= 160) return launch<T, 32, 5>(logits, tokens, E, k, experts, probs, s);
  if (E <= 192) return launch<T, 32, 6>(logits, tokens, E, k, experts, probs, s);
  if (E <= 224) return launch<T, 32, 7>(logits, tokens, E, k, experts, probs, s);
  if (E <= 256) return launch<T, 32, 8>(logits, tokens, E, k, experts, probs, s);
  if (E <= 512) return launch<T, 32, 16>(logits, tokens, E, k, experts, probs, s);
  return launch<T, 32, 32>(logits, tokens, E, k, experts, probs, s);
}

}  // namespace

moe_status check_route_args(int64_t T, int E, int k) {
  if (k < 1) return fail(MOE_ERR_INVALID_ARGUMENT, "route_topk: k must be >= 1");
  if (E < 1 && T > 0) return fail(MOE_ERR_INVALID_ARGUMENT, "route_topk: empty gate score row");
  if (k > E && T > 0) return fail(MOE_ERR_INVALID_ARGUMENT, "route_topk: k exceeds the expert count");
  if (E > 1024) return fail(MOE_ERR_UNSUPPORTED, "route_topk: at most 1024 experts");
  if (k > 32) return fail(MOE_ERR_UNSUPPORTED, "route_topk: at most k = 32");
  return MOE_OK;
}

moe_status route_topk(const void* logits, int logit_dtype, int64_t T, int E, int k, int32_t* experts, void* probs,
                      cudaStream_t stream) {
  if (moe_status st = check_route_args(T, E, k)) return st;
  if (T == 0) return MOE_OK;
  if (!logits || !experts || !probs) return fail(MOE_ERR_INVALID_ARGUMENT, "route_topk: null pointer");
  cudaError_t err;
  if (logit_dtype == MOE_F32) {
    err = route_dispatch<float>(static_cast<const float*>(logits), T, E, k, experts, static_cast<float*>(probs), stream);
  } else if (logit_dtype == MOE_F64) {
    err = route_dispatch<double>(static_cast<const double*>(logits), T, E, k, experts, static_cast<double*>(probs),
                                 stream);
  } else {
    return fail(MOE_ERR_INVALID_ARGUMENT, "route_topk: logits must be f32 or f64");
  }
  if (err != cudaSuccess) return cuda_fail(err, "route_topk launch");
  return MOE_OK;
}

}  // namespace monta

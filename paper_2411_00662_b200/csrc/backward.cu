// Backward pass of the lone-card data path.
//
// The reference has no backward (it is a planner + data-plane simulator); these
// are the adjoints of the three forward ops this library exports, so a
// training step can run router -> dispatch -> experts -> combine and back:
//
//   combine    out[i]  = sum_s p[i,s] * y[pos[i,s]]          (dataplane.hpp:325-342)
//     grad_y[pos[i,s]] = p[i,s] * grad_out[i]
//     grad_p[i,s]      = <grad_out[i], y[pos[i,s]]>
//   dispatch   rows[pos[i,s]] = x[i]                          (dataplane.hpp:118-140)
//     grad_x[i]        = sum_s grad_rows[pos[i,s]]             (un-permute with unit weights)
//   route      p[i,s]  = softmax(z[i])[x_s]  (not renormalised, dataplane.hpp:72-106)
//     grad_z[i,e]      = P_e * (G_e - sum_s g_s P_{x_s}),  G_e = g_s if e == x_s else 0
//
// On a multi-card layer the cross-card legs of the backward are the forward
// exchanges run in the opposite direction (combine backward = dispatch of the
// weighted gradient rows, dispatch backward = combine's reverse AllToAll); the
// kernels here are the per-card compute either side of them.
//
// All three are HBM-bound streaming kernels (CTA per token for the row
// kernels, warp per token for the router), 8-element
// packs moved with 16-byte vector accesses (bf16/f16: one int4, f32: two,
// f64: four), fp32 accumulation (fp64 for f64), no atomics: every output
// element has exactly one writer.
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <type_traits>

#include "common.cuh"

namespace monta {
namespace {

// fp32 accumulation unless any operand is fp64.
template <class... T> struct AccOf {
  using type = std::conditional_t<(std::is_same_v<T, double> || ...), double, float>;
};

template <class A, class T> __device__ __forceinline__ A cvt_in(T v) { return A(to_f32(v)); }
template <> __device__ __forceinline__ double cvt_in<double, double>(double v) { return v; }

template <class T, class A> __device__ __forceinline__ T cvt_out(A v) { return from_f32<T>(float(v)); }
template <> __device__ __forceinline__ double cvt_out<double, double>(double v) { return v; }
template <> __device__ __forceinline__ float cvt_out<float, double>(double v) { return float(v); }

// N consecutive elements of T, loaded/stored with 16-byte accesses when N == 8
// (8 * sizeof(T) is a multiple of 16 for every supported dtype) and the
// caller guaranteed alignment; N == 1 is the scalar fallback.
template <class T, int N> struct Pack {
  static_assert(N == 1 || N == 8, "pack of 1 or 8");
  static constexpr int kVec = N == 8 ? int(8 * sizeof(T) / 16) : 1;  // int4 accesses per pack of 8
  // A pack as loaded (kept in this form while other loads are in flight, so
  // the in-flight registers are the bytes, not their fp32 expansion).
  union Raw {
    int4 v[kVec];
    T e[N];
  };
  __device__ __forceinline__ static void load_raw(const T* p, Raw& r) {
    if constexpr (N == 1) {
      r.e[0] = *p;
    } else {
#pragma unroll
      for (int j = 0; j < kVec; ++j) r.v[j] = ld_stream(reinterpret_cast<const int4*>(p) + j);
    }
  }
  template <class A> __device__ __forceinline__ static void load(const T* p, A* out) {
    if constexpr (N == 1) {
      out[0] = cvt_in<A>(*p);
    } else {
      constexpr int kVec = int(8 * sizeof(T) / 16);  // int4 accesses per pack of 8
      union { int4 v[kVec]; T e[8]; } u;
#pragma unroll
      for (int j = 0; j < kVec; ++j) u.v[j] = ld_stream(reinterpret_cast<const int4*>(p) + j);
#pragma unroll
      for (int j = 0; j < 8; ++j) out[j] = cvt_in<A>(u.e[j]);
    }
  }
  template <class A> __device__ __forceinline__ static void store(T* p, const A* in) {
    if constexpr (N == 1) {
      *p = cvt_out<T>(in[0]);
    } else {
      constexpr int kVec = int(8 * sizeof(T) / 16);  // int4 accesses per pack of 8
      union { int4 v[kVec]; T e[8]; } u;
#pragma unroll
      for (int j = 0; j < 8; ++j) u.e[j] = cvt_out<T>(in[j]);
#pragma unroll
      for (int j = 0; j < kVec; ++j) st_vec(reinterpret_cast<int4*>(p) + j, u.v[j]);
    }
  }
};

template <class A> __device__ __forceinline__ A warp_sum(A v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

template <class P> __device__ __forceinline__ double load_p(const P* p) { return double(*p); }

// Both streaming kernels give each token to one CTA whose threads split its
// row: thread t owns packs t, t + blockDim.x, ...  and keeps unroll_for() of
// them in flight.  The host sizes the CTA so that every round is full (the
// fewest rounds of <= 160 threads, then the fewest warps covering the row in
// that many rounds: Mixtral 128, DeepSeek 160, 2x70B 128 threads x 2
// rounds), and small layers (toy: T = 2048) still spread over the SMs.
constexpr int kMaxThreads = 256;
constexpr int kSizingThreads = 160;
constexpr int kMaxSlots = 64;  // combine backward keeps per-slot partial dots in shared memory

// Packs in flight per thread and stream: 64 bytes (4 for 16-bit types, 2 for
// f32, 1 for f64), so the raw in-flight bytes fit the register budget of
// 16 resident CTAs per SM.
template <class T, int N> __host__ __device__ constexpr int unroll_for() { return N == 1 ? 4 : int(64 / (8 * sizeof(T))); }
template <class TG, class TY, int N> __host__ __device__ constexpr int combine_unroll() {
  return unroll_for<TG, N>() < unroll_for<TY, N>() ? unroll_for<TG, N>() : unroll_for<TY, N>();
}

inline int block_for(int64_t packs, int unroll) {
  // Fewest rounds of at most 160 threads, then the fewest whole warps that
  // cover the row in that many rounds.
  const int64_t per_round = int64_t(kSizingThreads) * unroll;
  const int64_t rounds = packs <= 0 ? 1 : (packs + per_round - 1) / per_round;
  int64_t t = (packs + unroll * rounds - 1) / (unroll * rounds);
  t = (t + 31) / 32 * 32;
  return int(t < 32 ? 32 : (t > kMaxThreads ? kMaxThreads : t));
}

// combine backward: per round the CTA loads its slice of the token's
// gradient row once into registers, then for each slot streams the expert
// output row, writes p * grad into the expert-gradient row and reduces the
// dot product for grad_probs in a fixed order (lanes, then rounds, then
// warps): deterministic, no atomics.  Every thread runs the same number of
// rounds so the warp reductions inside them stay converged.
template <class TG, class TY, class PT, int N>
__global__ void __launch_bounds__(kMaxThreads) k_combine_bwd(const TG* __restrict__ g, int64_t g_stride,
                                                          const TY* __restrict__ y, int64_t y_stride,
                                                          int64_t width, const int32_t* __restrict__ pos,
                                                          const PT* __restrict__ probs, int64_t T, int k,
                                                          TY* __restrict__ gy, int64_t gy_stride,
                                                          PT* __restrict__ gp) {
  using A = typename AccOf<TG, TY, PT>::type;
  using PG = Pack<TG, N>;
  using PY = Pack<TY, N>;
  constexpr int U = combine_unroll<TG, TY, N>();
  __shared__ A part[kMaxSlots][kMaxThreads / 32];
  const int warps = blockDim.x >> 5;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t packs = width / N;
  const int64_t step = int64_t(blockDim.x) * U;
  for (int64_t i = blockIdx.x; i < T; i += gridDim.x) {
    const TG* grow = g + i * g_stride;
    for (int64_t base = 0; base < packs; base += step) {
      typename PG::Raw gv[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t c = base + threadIdx.x + int64_t(u) * blockDim.x;
        if (c < packs) PG::load_raw(grow + c * N, gv[u]);
      }
      for (int s = 0; s < k; ++s) {
        // an empty slot (r < 0, no expert: front.cuh index_block) has no row:
        // nothing to read or write, and its grad_prob is 0.  r is uniform over
        // the CTA, so the warp reductions below stay converged.
        const int64_t r = pos[i * k + s];
        const bool live = r >= 0;
        const A p = live ? A(load_p(probs + i * k + s)) : A(0);
        A dot = 0;
        typename PY::Raw yv[U];
        if (gp && live) {
#pragma unroll
          for (int u = 0; u < U; ++u) {
            const int64_t c = base + threadIdx.x + int64_t(u) * blockDim.x;
            if (c < packs) PY::load_raw(y + r * y_stride + c * N, yv[u]);
          }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int64_t c = base + threadIdx.x + int64_t(u) * blockDim.x;
          if (c < packs && live) {
            if (gp) {
#pragma unroll
              for (int j = 0; j < N; ++j) dot += cvt_in<A>(gv[u].e[j]) * cvt_in<A>(yv[u].e[j]);
            }
            if (gy) {
              A ov[N];
#pragma unroll
              for (int j = 0; j < N; ++j) ov[j] = p * cvt_in<A>(gv[u].e[j]);
              PY::store(gy + r * gy_stride + c * N, ov);
            }
          }
        }
        if (gp) {
          dot = warp_sum(dot);
          if (lane == 0) part[s][warp] = base == 0 ? dot : part[s][warp] + dot;
        }
      }
    }
    if (gp) {
      __syncthreads();
      if (threadIdx.x < k) {
        A sum = 0;
        for (int w = 0; w < warps; ++w) sum += part[threadIdx.x][w];
        gp[i * k + threadIdx.x] = PT(sum);
      }
      __syncthreads();  // part[] is reused by the next token
    }
  }
}

// dispatch backward: grad_x[i] = sum_s grad_rows[pos[i,s]], accumulated from
// zero in ascending slot order (the order of a sequential CPU sum).
template <class TI, class TO, int N>
__global__ void __launch_bounds__(kMaxThreads) k_dispatch_bwd(const TI* __restrict__ rows, int64_t in_stride,
                                                           int64_t width, const int32_t* __restrict__ pos,
                                                           int64_t T, int k, TO* __restrict__ out,
                                                           int64_t out_stride) {
  using A = typename AccOf<TI, TO>::type;
  using PI = Pack<TI, N>;
  constexpr int U = unroll_for<TI, N>();
  const int64_t packs = width / N;
  for (int64_t i = blockIdx.x; i < T; i += gridDim.x) {
    for (int64_t c0 = threadIdx.x; c0 < packs; c0 += int64_t(blockDim.x) * U) {
      A acc[U][N];
#pragma unroll
      for (int u = 0; u < U; ++u)
#pragma unroll
        for (int j = 0; j < N; ++j) acc[u][j] = 0;
      for (int s = 0; s < k; ++s) {
        const int64_t r = pos[i * k + s];
        if (r < 0) continue;  // empty slot: contributes nothing
        typename PI::Raw v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int64_t c = c0 + int64_t(u) * blockDim.x;
          if (c < packs) PI::load_raw(rows + r * in_stride + c * N, v[u]);
        }
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
          for (int j = 0; j < N; ++j) acc[u][j] += cvt_in<A>(v[u].e[j]);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t c = c0 + int64_t(u) * blockDim.x;
        if (c < packs) Pack<TO, N>::store(out + i * out_stride + c * N, acc[u]);
      }
    }
  }
}

// route backward: warp per token, softmax recomputed in the logit dtype with
// the forward's recipe (max-subtract, exp, sum, divide).
template <class F>
__global__ void __launch_bounds__(256) k_route_bwd(const F* __restrict__ z, int64_t T, int E, int k,
                                                   const int32_t* __restrict__ experts,
                                                   const F* __restrict__ gp, F* __restrict__ gz) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = int64_t(gridDim.x) * (blockDim.x >> 5);
  for (int64_t i = int64_t(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5); i < T; i += warps) {
    const F* zr = z + i * E;
    F m = -INFINITY;
    for (int e = lane; e < E; e += 32) m = fmax(m, zr[e]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    F sum = 0;
    for (int e = lane; e < E; e += 32) sum += exp(zr[e] - m);
    sum = warp_sum(sum);
    // S = sum_s g_s * P_{x_s}
    F S = 0;
    for (int s = lane; s < k; s += 32)
      if (experts[i * k + s] >= 0) S += gp[i * k + s] * (exp(zr[experts[i * k + s]] - m) / sum);
    S = warp_sum(S);
    for (int e = lane; e < E; e += 32) {
      F G = 0;
      for (int s = 0; s < k; ++s)
        if (experts[i * k + s] == e) G = gp[i * k + s];
      const F P = exp(zr[e] - m) / sum;
      gz[i * E + e] = P * (G - S);
    }
  }
}

int sm_count() {
  static int sms[16] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  int& n = sms[dev & 15];
  if (n == 0) {
    n = 148;
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  }
  return n;
}

// Streaming kernels: one CTA per token, at most 16 resident CTAs per SM.
int stream_grid(int64_t T) {
  const int64_t cap = int64_t(sm_count()) * 16;
  return int(T < cap ? (T < 1 ? 1 : T) : cap);
}

// Warp-per-token kernels (route backward): 8 warps per CTA, up to 8 CTAs per SM.
int grid_for(int64_t T) {
  const int64_t want = (T + 7) / 8;
  const int64_t cap = int64_t(sm_count()) * 8;
  return int(want < cap ? (want < 1 ? 1 : want) : cap);
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

template <class TG, class TY, class PT>
cudaError_t launch_cbwd(const void* g, int64_t gs, const void* y, int64_t ys, int64_t w, const int32_t* pos,
                        const void* p, int64_t T, int k, void* gy, int64_t gys, void* gp, cudaStream_t st) {
  const bool vec = w % 8 == 0 && gs % 8 == 0 && ys % 8 == 0 && gys % 8 == 0 && aligned16(g) &&
                   (!y || aligned16(y)) && (!gy || aligned16(gy));
  const int grid = stream_grid(T);
  const int block = vec ? block_for(w / 8, combine_unroll<TG, TY, 8>()) : block_for(w, combine_unroll<TG, TY, 1>());
  if (vec)
    k_combine_bwd<TG, TY, PT, 8><<<grid, block, 0, st>>>(
        static_cast<const TG*>(g), gs, static_cast<const TY*>(y), ys, w, pos, static_cast<const PT*>(p), T, k,
        static_cast<TY*>(gy), gys, static_cast<PT*>(gp));
  else
    k_combine_bwd<TG, TY, PT, 1><<<grid, block, 0, st>>>(
        static_cast<const TG*>(g), gs, static_cast<const TY*>(y), ys, w, pos, static_cast<const PT*>(p), T, k,
        static_cast<TY*>(gy), gys, static_cast<PT*>(gp));
  return cudaGetLastError();
}

template <class TG, class TY>
cudaError_t cbwd_p(int pdt, const void* g, int64_t gs, const void* y, int64_t ys, int64_t w, const int32_t* pos,
                   const void* p, int64_t T, int k, void* gy, int64_t gys, void* gp, cudaStream_t st) {
  if (pdt == MOE_F64) return launch_cbwd<TG, TY, double>(g, gs, y, ys, w, pos, p, T, k, gy, gys, gp, st);
  return launch_cbwd<TG, TY, float>(g, gs, y, ys, w, pos, p, T, k, gy, gys, gp, st);
}

template <class TG>
cudaError_t cbwd_y(int ydt, int pdt, const void* g, int64_t gs, const void* y, int64_t ys, int64_t w,
                   const int32_t* pos, const void* p, int64_t T, int k, void* gy, int64_t gys, void* gp,
                   cudaStream_t st) {
  switch (ydt) {
    case MOE_F32: return cbwd_p<TG, float>(pdt, g, gs, y, ys, w, pos, p, T, k, gy, gys, gp, st);
    case MOE_BF16: return cbwd_p<TG, __nv_bfloat16>(pdt, g, gs, y, ys, w, pos, p, T, k, gy, gys, gp, st);
    case MOE_F16: return cbwd_p<TG, __half>(pdt, g, gs, y, ys, w, pos, p, T, k, gy, gys, gp, st);
    default: return cbwd_p<TG, double>(pdt, g, gs, y, ys, w, pos, p, T, k, gy, gys, gp, st);
  }
}

template <class TI, class TO>
cudaError_t launch_dbwd(const void* in, int64_t is, int64_t w, const int32_t* pos, int64_t T, int k, void* out,
                        int64_t os, cudaStream_t st) {
  const bool vec = w % 8 == 0 && is % 8 == 0 && os % 8 == 0 && aligned16(in) && aligned16(out);
  const int grid = stream_grid(T);
  const int block = vec ? block_for(w / 8, unroll_for<TI, 8>()) : block_for(w, unroll_for<TI, 1>());
  if (vec)
    k_dispatch_bwd<TI, TO, 8><<<grid, block, 0, st>>>(static_cast<const TI*>(in), is, w, pos, T, k,
                                                    static_cast<TO*>(out), os);
  else
    k_dispatch_bwd<TI, TO, 1><<<grid, block, 0, st>>>(static_cast<const TI*>(in), is, w, pos, T, k,
                                                    static_cast<TO*>(out), os);
  return cudaGetLastError();
}

template <class TI>
cudaError_t dbwd_o(int odt, const void* in, int64_t is, int64_t w, const int32_t* pos, int64_t T, int k,
                   void* out, int64_t os, cudaStream_t st) {
  switch (odt) {
    case MOE_F32: return launch_dbwd<TI, float>(in, is, w, pos, T, k, out, os, st);
    case MOE_BF16: return launch_dbwd<TI, __nv_bfloat16>(in, is, w, pos, T, k, out, os, st);
    case MOE_F16: return launch_dbwd<TI, __half>(in, is, w, pos, T, k, out, os, st);
    default: return launch_dbwd<TI, double>(in, is, w, pos, T, k, out, os, st);
  }
}

bool float_dtype(int dt) { return dt == MOE_F32 || dt == MOE_BF16 || dt == MOE_F16 || dt == MOE_F64; }

}  // namespace
}  // namespace monta

using namespace monta;

extern "C" moe_status moe_combine_backward(const void* grad_out, int grad_dtype, int64_t grad_row_elems,
                                           const void* y, int y_dtype, int64_t y_row_elems, int64_t width,
                                           const int32_t* slot_pos, const void* probs, int probs_dtype,
                                           int64_t T, int32_t k, void* grad_y, int64_t grad_y_row_elems,
                                           void* grad_probs, void* stream) {
  if (T < 0 || k < 1 || k > kMaxSlots || width < 0 || width > grad_row_elems || (y && width > y_row_elems) ||
      (grad_y && width > grad_y_row_elems))
    return fail(MOE_ERR_INVALID_ARGUMENT, "combine_backward: bad geometry (1 <= k <= 64)");
  if (probs_dtype != MOE_F32 && probs_dtype != MOE_F64)
    return fail(MOE_ERR_INVALID_ARGUMENT, "combine_backward: probs must be f32 or f64");
  if (!float_dtype(grad_dtype) || !float_dtype(y_dtype))
    return fail(MOE_ERR_INVALID_ARGUMENT, "combine_backward: gradient and expert rows must be f32/bf16/f16/f64");
  if (grad_probs && !y)
    return fail(MOE_ERR_INVALID_ARGUMENT, "combine_backward: grad_probs needs the expert rows y");
  if (T == 0 || (!grad_y && !grad_probs)) return MOE_OK;
  if (!grad_out || !slot_pos || !probs) return fail(MOE_ERR_INVALID_ARGUMENT, "combine_backward: null pointer");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  cudaError_t err;
  switch (grad_dtype) {
    case MOE_F32:
      err = cbwd_y<float>(y_dtype, probs_dtype, grad_out, grad_row_elems, y, y_row_elems, width, slot_pos, probs, T,
                          k, grad_y, grad_y_row_elems, grad_probs, st);
      break;
    case MOE_BF16:
      err = cbwd_y<__nv_bfloat16>(y_dtype, probs_dtype, grad_out, grad_row_elems, y, y_row_elems, width, slot_pos,
                                  probs, T, k, grad_y, grad_y_row_elems, grad_probs, st);
      break;
    case MOE_F16:
      err = cbwd_y<__half>(y_dtype, probs_dtype, grad_out, grad_row_elems, y, y_row_elems, width, slot_pos, probs,
                           T, k, grad_y, grad_y_row_elems, grad_probs, st);
      break;
    default:
      err = cbwd_y<double>(y_dtype, probs_dtype, grad_out, grad_row_elems, y, y_row_elems, width, slot_pos, probs,
                           T, k, grad_y, grad_y_row_elems, grad_probs, st);
  }
  if (err != cudaSuccess) return cuda_fail(err, "combine_backward launch");
  return MOE_OK;
}

extern "C" moe_status moe_dispatch_backward(const void* grad_rows, int rows_dtype, int64_t row_elems, int64_t width,
                                            const int32_t* slot_pos, int64_t T, int32_t k, void* grad_x,
                                            int out_dtype, int64_t out_row_elems, void* stream) {
  if (T < 0 || k < 1 || k > kMaxSlots || width < 0 || width > row_elems || width > out_row_elems)
    return fail(MOE_ERR_INVALID_ARGUMENT, "dispatch_backward: bad geometry (1 <= k <= 64)");
  if (!float_dtype(rows_dtype) || !float_dtype(out_dtype))
    return fail(MOE_ERR_INVALID_ARGUMENT, "dispatch_backward: dtypes must be f32/bf16/f16/f64");
  if (T == 0 || width == 0) return MOE_OK;
  if (!grad_rows || !slot_pos || !grad_x) return fail(MOE_ERR_INVALID_ARGUMENT, "dispatch_backward: null pointer");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  cudaError_t err;
  switch (rows_dtype) {
    case MOE_F32: err = dbwd_o<float>(out_dtype, grad_rows, row_elems, width, slot_pos, T, k, grad_x, out_row_elems, st); break;
    case MOE_BF16: err = dbwd_o<__nv_bfloat16>(out_dtype, grad_rows, row_elems, width, slot_pos, T, k, grad_x, out_row_elems, st); break;
    case MOE_F16: err = dbwd_o<__half>(out_dtype, grad_rows, row_elems, width, slot_pos, T, k, grad_x, out_row_elems, st); break;
    default: err = dbwd_o<double>(out_dtype, grad_rows, row_elems, width, slot_pos, T, k, grad_x, out_row_elems, st);
  }
  if (err != cudaSuccess) return cuda_fail(err, "dispatch_backward launch");
  return MOE_OK;
}

extern "C" moe_status moe_route_backward(const void* logits, int logit_dtype, int64_t T, int32_t E, int32_t k,
                                         const int32_t* experts, const void* grad_probs, void* grad_logits,
                                         void* stream) {
  if (T < 0 || E < 1 || k < 1 || k > E) return fail(MOE_ERR_INVALID_ARGUMENT, "route_backward: need 1 <= k <= E");
  if (logit_dtype != MOE_F32 && logit_dtype != MOE_F64)
    return fail(MOE_ERR_INVALID_ARGUMENT, "route_backward: logits must be f32 or f64");
  if (T == 0) return MOE_OK;
  if (!logits || !experts || !grad_probs || !grad_logits)
    return fail(MOE_ERR_INVALID_ARGUMENT, "route_backward: null pointer");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int grid = grid_for(T);
  if (logit_dtype == MOE_F64)
    k_route_bwd<double><<<grid, 256, 0, st>>>(static_cast<const double*>(logits), T, E, k, experts,
                                              static_cast<const double*>(grad_probs),
                                              static_cast<double*>(grad_logits));
  else
    k_route_bwd<float><<<grid, 256, 0, st>>>(static_cast<const float*>(logits), T, E, k, experts,
                                             static_cast<const float*>(grad_probs),
                                             static_cast<float*>(grad_logits));
  const cudaError_t err = cudaGetLastError();
  if (err != cudaSuccess) return cuda_fail(err, "route_backward launch");
  return MOE_OK;
}

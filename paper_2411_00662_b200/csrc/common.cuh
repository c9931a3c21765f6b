// Shared device/host helpers for the MoNTA dispatch/combine kernels (sm_100a).
#pragma once

#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdlib>

#include "monta.h"

namespace monta {
// Diagnosis: MONTA_CARVEOUT=<0..100> sets every data-path kernel's preferred
// shared-memory carveout (read once; unset leaves the driver's choice).
inline int carveout_env() {
  static const int v = [] {
    const char* e = std::getenv("MONTA_CARVEOUT");
    return e ? std::atoi(e) : -1;
  }();
  return v;
}
template <class F> inline void apply_carveout(F* fn) {
  if (carveout_env() >= 0) cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout, carveout_env());
}


constexpr int kMaxCards = 64;     // e*t cards per layer context
constexpr int kWarp = 32;

// ---------------------------------------------------------------------------
// Error plumbing (host).  Every ABI entry point funnels through fail() so the
// message survives for moe_last_error().
moe_status fail(moe_status st, const char* fmt, ...);
moe_status cuda_fail(cudaError_t err, const char* what);

#define MONTA_CUDA(expr)                                   \
  do {                                                     \
    cudaError_t _e = (expr);                               \
    if (_e != cudaSuccess) return ::monta::cuda_fail(_e, #expr); \
  } while (0)

#define MONTA_CHECK_LAUNCH(what)                           \
  do {                                                     \
    cudaError_t _e = cudaGetLastError();                   \
    if (_e != cudaSuccess) return ::monta::cuda_fail(_e, what); \
  } while (0)

inline size_t dtype_size(int dt) {
  switch (dt) {
    case MOE_F32: return 4;
    case MOE_BF16: return 2;
    case MOE_F16: return 2;
    case MOE_F64: return 8;
    case MOE_I64: return 8;
  }
  return 0;
}

// Largest power-of-two vector width (<= 16 bytes) dividing every argument.
inline int vec_bytes(int64_t a, int64_t b = 16, int64_t c = 16, int64_t d = 16, int64_t e = 16) {
  int64_t g = a | b | c | d | e;
  int v = 16;
  while (v > 1 && (g % v) != 0) v >>= 1;
  return v;
}

inline int ceil_div(int64_t a, int64_t b) { return int((a + b - 1) / b); }

// ---------------------------------------------------------------------------
// Vector memory primitives.  Sources are streamed once: non-coherent loads
// that do not allocate in L1.  Destinations may be NVLink peer addresses.
template <int V> struct VecT;
template <> struct VecT<16> { using type = int4; };
template <> struct VecT<8> { using type = int2; };
template <> struct VecT<4> { using type = int; };
template <> struct VecT<2> { using type = short; };
template <> struct VecT<1> { using type = char; };

__device__ __forceinline__ int4 ld_stream(const int4* p) {
  int4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}
// Read-once source rows that should not displace data a later kernel of the
// step re-reads from L2 (L2 evict-first policy).
__device__ __forceinline__ uint64_t l2_evict_first_policy() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ int4 ld_stream_ef(const int4* p, uint64_t pol) {
  int4 r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.s32 {%0,%1,%2,%3}, [%4], %5;"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p), "l"(pol));
  return r;
}
__device__ __forceinline__ int2 ld_stream(const int2* p) {
  int2 r;
  asm volatile("ld.global.nc.L1::no_allocate.v2.s32 {%0,%1}, [%2];" : "=r"(r.x), "=r"(r.y) : "l"(p));
  return r;
}
__device__ __forceinline__ int ld_stream(const int* p) {
  int r;
  asm volatile("ld.global.nc.L1::no_allocate.s32 %0, [%1];" : "=r"(r) : "l"(p));
  return r;
}
__device__ __forceinline__ short ld_stream(const short* p) { return *p; }
__device__ __forceinline__ char ld_stream(const char* p) { return *p; }
template <class V> __device__ __forceinline__ V ld_stream_ef(const V* p, uint64_t) { return ld_stream(p); }

// Plain (coherent) loads for buffers another GPU may have written during
// this launch's lifetime window (after an acquire).
template <class T> __device__ __forceinline__ T ld_plain(const T* p) { return *p; }

__device__ __forceinline__ void st_vec(int4* p, const int4& v) {
  asm volatile("st.global.v4.s32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z),
               "r"(v.w)
               : "memory");
}
__device__ __forceinline__ void st_vec(int2* p, const int2& v) { *p = v; }
__device__ __forceinline__ void st_vec(int* p, const int& v) { *p = v; }
__device__ __forceinline__ void st_vec(short* p, const short& v) { *p = v; }
__device__ __forceinline__ void st_vec(char* p, const char& v) { *p = v; }

// ---------------------------------------------------------------------------
// Cross-GPU signalling.  Each card owns a flag array that peers write over
// NVLink: flags[signal * kMaxCards + sender] = epoch.  Epochs only grow, so
// no flag is ever reset.  A kernel that consumes remote data waits (thread 0
// of every CTA, bounded by a timeout) before touching it; a kernel that
// produces remote data has its LAST CTA publish the flags after a
// system-scope fence.
// The epoch is read from device memory (`epoch_ptr`, bumped once per
// dispatch by the front kernel) so a captured CUDA graph replays correctly;
// `epoch` is used when epoch_ptr is null.
struct WaitList {
  const uint64_t* flags[kMaxCards];  // local flag words to watch
  int n;
  uint64_t epoch;
  const uint64_t* epoch_ptr;
};
struct SignalList {
  uint64_t* flags[kMaxCards];  // peer (or local) flag words to set
  int n;
  uint64_t epoch;
  const uint64_t* epoch_ptr;
  unsigned int* done;  // per-launch CTA completion counter (local, zeroed)
};

constexpr unsigned long long kWaitTimeoutNs = 20ull * 1000ull * 1000ull * 1000ull;  // 20 s

__device__ __forceinline__ uint64_t ld_acquire_sys(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys(uint64_t* p, uint64_t v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Returns false (and records MOE_ERR_TIMEOUT in *err) when the wait timed out.
__device__ __forceinline__ bool cta_wait(const WaitList& w, int* err) {
  __shared__ int ok;
  if (threadIdx.x == 0) {
    ok = 1;
    if (w.n > 0) {
      const uint64_t epoch = w.epoch_ptr ? *w.epoch_ptr : w.epoch;
      const unsigned long long t0 = globaltimer();
      for (int i = 0; i < w.n; ++i) {
        while (ld_acquire_sys(w.flags[i]) < epoch) {
          if (globaltimer() - t0 > kWaitTimeoutNs) {
            atomicExch(err, (int)MOE_ERR_TIMEOUT);
            ok = 0;
            break;
          }
          __nanosleep(128);
        }
        if (!ok) break;
      }
    }
  }
  __syncthreads();
  return ok != 0;
}

__device__ __forceinline__ void cta_signal(const SignalList& s) {
  if (s.n == 0) return;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence_system();
    const unsigned int prev = atomicAdd(s.done, 1u);
    if (prev == gridDim.x - 1) {
      __threadfence_system();
      const uint64_t epoch = s.epoch_ptr ? *s.epoch_ptr : s.epoch;
      for (int i = 0; i < s.n; ++i) st_release_sys(s.flags[i], epoch);
      *s.done = 0u;  // ready for the next launch that reuses this counter
    }
  }
}

// ---------------------------------------------------------------------------
// Value conversion for the combine arithmetic.
template <class T> __device__ __forceinline__ float to_f32(T v);
template <> __device__ __forceinline__ float to_f32<float>(float v) { return v; }
template <> __device__ __forceinline__ float to_f32<__nv_bfloat16>(__nv_bfloat16 v) {
  return __bfloat162float(v);
}
template <> __device__ __forceinline__ float to_f32<__half>(__half v) { return __half2float(v); }

template <class T> __device__ __forceinline__ T from_f32(float v);
template <> __device__ __forceinline__ float from_f32<float>(float v) { return v; }
template <> __device__ __forceinline__ __nv_bfloat16 from_f32<__nv_bfloat16>(float v) {
  return __float2bfloat16_rn(v);
}
template <> __device__ __forceinline__ __half from_f32<__half>(float v) { return __float2half_rn(v); }
template <> __device__ __forceinline__ double from_f32<double>(float v) { return double(v); }

}  // namespace monta

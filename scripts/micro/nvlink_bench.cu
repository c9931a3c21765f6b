// Micro-benchmark (dev tool): peer-store throughput over NVLink/NVSwitch for
// the exchange legs, every GPU writing `bytes` to its partner (g ^ 1) at the
// same time (the 2x2 AllToAll leg pattern), single process, peer access on.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 nvlink_bench.cu
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

// register copy: warp per item of 32*U int4
template <int U>
__global__ void __launch_bounds__(256) k_st(const int4* __restrict__ src, int4* __restrict__ dst, int64_t n) {
  const int lane = threadIdx.x & 31;
  const int64_t w = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5, nw = (int64_t(gridDim.x) * blockDim.x) >> 5;
  for (int64_t base = w * 32 * U; base < n; base += nw * 32 * U) {
    int4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t i = base + u * 32 + lane;
      if (i < n) v[u] = src[i];
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t i = base + u * 32 + lane;
      if (i < n) dst[i] = v[u];
    }
  }
}

// contiguous-chunk variant: CTA c copies a contiguous 1/grid share (long runs per CTA)
template <int U>
__global__ void __launch_bounds__(256) k_st_chunk(const int4* __restrict__ src, int4* __restrict__ dst, int64_t n) {
  const int64_t per = (n + gridDim.x - 1) / gridDim.x;
  const int64_t lo = blockIdx.x * per, hi = lo + per < n ? lo + per : n;
  for (int64_t base = lo + threadIdx.x; base < hi; base += int64_t(blockDim.x) * U) {
    int4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t i = base + u * blockDim.x;
      if (i < hi) v[u] = src[i];
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t i = base + u * blockDim.x;
      if (i < hi) dst[i] = v[u];
    }
  }
}

__device__ __forceinline__ uint32_t sa(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
// TMA bulk: local global -> smem (bulk load, mbarrier) -> peer global (bulk store), one thread per CTA drives
__global__ void k_bulk(const char* __restrict__ src, char* __restrict__ dst, int64_t bytes, int seg, int stages) {
  extern __shared__ __align__(128) char ring[];
  __shared__ uint64_t bar[16];
  if (threadIdx.x != 0) return;
  for (int s = 0; s < stages; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bar[s])) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  const int64_t nseg = bytes / seg;
  auto load = [&](int64_t it, int st) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&bar[st])), "r"(seg) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(sa(ring + size_t(st) * seg)),
                 "l"(src + it * seg), "r"(seg), "r"(sa(&bar[st])) : "memory");
  };
  int m = 0;
  for (int s = 0; s < stages; ++s) {
    const int64_t it = blockIdx.x + int64_t(s) * gridDim.x;
    if (it < nseg) load(it, s);
  }
  for (int64_t it = blockIdx.x; it < nseg; it += gridDim.x, ++m) {
    const int st = m % stages;
    const unsigned ph = (m / stages) & 1;
    asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n" ::"r"(sa(&bar[st])), "r"(ph) : "memory");
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst + it * seg), "r"(sa(ring + size_t(st) * seg)), "r"(seg) : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    const int64_t nxt = it + int64_t(stages) * gridDim.x;
    if (nxt < nseg) {
      asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");  // this stage's store has read smem
      load(nxt, st);
    }
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}


// chunked copy with per-chunk completion: every CTA copies its share of chunk
// s, then (mode 0) no fence, (1) __threadfence_system + gpu atomic,
// (2) __threadfence (gpu scope) + gpu atomic, the last arriver fences at
// system scope; the last CTA bumps a per-chunk counter (a flag stand-in).
__global__ void __launch_bounds__(256) k_chunked(const int4* __restrict__ src, int4* __restrict__ dst, int64_t n, int chunks,
                                                 unsigned* counters, int mode) {
  const int lane = threadIdx.x & 31;
  const int64_t per = n / chunks;
  for (int s = 0; s < chunks; ++s) {
    const int64_t lo = s * per;
    const int64_t w = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5, nw = (int64_t(gridDim.x) * blockDim.x) >> 5;
    for (int64_t base = lo + w * 128; base < lo + per; base += nw * 128) {
      int4 v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) { const int64_t i = base + u * 32 + lane; if (i < lo + per) v[u] = src[i]; }
#pragma unroll
      for (int u = 0; u < 4; ++u) { const int64_t i = base + u * 32 + lane; if (i < lo + per) dst[i] = v[u]; }
    }
    if (mode == 0) continue;
    __syncthreads();
    if (threadIdx.x == 0) {
      if (mode == 1) __threadfence_system(); else __threadfence();
      const unsigned prev = atomicAdd(counters + s, 1u);
      if (prev == gridDim.x - 1) { __threadfence_system(); atomicExch(counters + 64 + s, 1u); counters[s] = 0; }
    }
  }
}

int main() {
  int ng = 0;
  CK(cudaGetDeviceCount(&ng));
  if (ng < 2) { printf("need >= 2 GPUs\n"); return 0; }
  ng = ng >= 4 ? 4 : 2;
  const size_t maxb = size_t(256) << 20;
  std::vector<char*> src(ng), dst(ng);
  std::vector<cudaStream_t> st(ng);
  std::vector<cudaEvent_t> e0(ng), e1(ng);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int g = 0; g < ng; ++g) {
    CK(cudaSetDevice(g));
    for (int p = 0; p < ng; ++p)
      if (p != g) cudaDeviceEnablePeerAccess(p, 0);
    cudaGetLastError();
    CK(cudaMalloc(&src[g], maxb));
    CK(cudaMalloc(&dst[g], maxb));
    CK(cudaMemset(src[g], g + 1, maxb));
    CK(cudaStreamCreateWithFlags(&st[g], cudaStreamNonBlocking));
    CK(cudaEventCreate(&e0[g]));
    CK(cudaEventCreate(&e1[g]));
    cudaFuncSetAttribute(k_bulk, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  }
  auto run = [&](const char* name, size_t bytes, auto launch) {
    float tot = 0;
    for (int rep = 0; rep < 8; ++rep) {
      for (int g = 0; g < ng; ++g) { cudaSetDevice(g); cudaDeviceSynchronize(); }
      for (int g = 0; g < ng; ++g) {
        cudaSetDevice(g);
        cudaEventRecord(e0[g], st[g]);
        launch(g, dst[g ^ 1], bytes);
        cudaEventRecord(e1[g], st[g]);
      }
      float mx = 0;
      for (int g = 0; g < ng; ++g) {
        cudaSetDevice(g);
        cudaEventSynchronize(e1[g]);
        float ms;
        cudaEventElapsedTime(&ms, e0[g], e1[g]);
        mx = ms > mx ? ms : mx;
      }
      if (rep >= 2) tot += mx;
    }
    const float ms = tot / 6;
    printf("%-44s %6zu MiB %8.2f us %7.0f GB/s per GPU\n", name, bytes >> 20, ms * 1e3, bytes / (ms * 1e-3) / 1e9);
  };
  std::vector<unsigned*> cnt(ng);
  for (int g = 0; g < ng; ++g) { cudaSetDevice(g); CK(cudaMalloc(&cnt[g], 4096)); CK(cudaMemset(cnt[g], 0, 4096)); }
  for (int chunks : {1, 4, 16})
    for (int mode : {0, 1, 2})
      for (int per_sm : {1, 2}) {
        char nm[64];
        snprintf(nm, sizeof nm, "chunked n=%d mode=%d grid=%d/SM", chunks, mode, per_sm);
        run(nm, size_t(16) << 20, [&](int g, char* d, size_t b) { k_chunked<<<sms * per_sm, 256, 0, st[g]>>>((const int4*)src[g], (int4*)d, b / 16, chunks, cnt[g], mode); });
      }
  if (getenv("CHUNKED_ONLY")) return 0;
  for (size_t mb : {4, 16, 64, 256}) {
    const size_t bytes = mb << 20;
    run("cudaMemcpyPeerAsync (copy engine)", bytes, [&](int g, char* d, size_t b) { cudaMemcpyPeerAsync(d, g ^ 1, src[g], g, b, st[g]); });
    for (int per_sm : {1, 2, 4}) {
      char nm[64];
      snprintf(nm, sizeof nm, "reg U=4 grid=%d/SM", per_sm);
      run(nm, bytes, [&](int g, char* d, size_t b) { k_st<4><<<sms * per_sm, 256, 0, st[g]>>>((const int4*)src[g], (int4*)d, b / 16); });
      snprintf(nm, sizeof nm, "reg U=8 grid=%d/SM", per_sm);
      run(nm, bytes, [&](int g, char* d, size_t b) { k_st<8><<<sms * per_sm, 256, 0, st[g]>>>((const int4*)src[g], (int4*)d, b / 16); });
      snprintf(nm, sizeof nm, "reg-chunk U=4 grid=%d/SM", per_sm);
      run(nm, bytes, [&](int g, char* d, size_t b) { k_st_chunk<4><<<sms * per_sm, 256, 0, st[g]>>>((const int4*)src[g], (int4*)d, b / 16); });
    }
    for (int seg : {8192, 16384, 32768})
      for (int per_sm : {1, 2}) {
        const int stages = int((96 * 1024) / seg) > 8 ? 8 : int((96 * 1024) / seg);
        char nm[64];
        snprintf(nm, sizeof nm, "tma bulk seg=%d stages=%d grid=%d/SM", seg, stages, per_sm);
        run(nm, bytes, [&](int g, char* d, size_t b) { k_bulk<<<sms * per_sm, 32, size_t(seg) * stages, st[g]>>>(src[g], d, b, seg, stages); });
      }
  }
  for (int g = 0; g < ng; ++g) { cudaSetDevice(g); CK(cudaDeviceSynchronize()); }
  return 0;
}

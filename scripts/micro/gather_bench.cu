// Micro-benchmark (dev tool): row-gather throughput on B200 for the copy
// engines the un-permute / permute kernels can use.
//   y[i] = x[perm[i]]   (R rows of `row` bytes; 2*R*row bytes of traffic)
// Variants: register gather (warp per row, U 16-byte loads per lane in
// flight), TMA bulk load -> smem -> st.global, TMA bulk load -> smem -> TMA
// bulk store.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 gather_bench.cu
#include <cstdio>
#include <cstdint>
#include <vector>
#include <random>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

__global__ void k_read(const int4* p, size_t n, int* sink) {
  int acc = 0;
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x) acc ^= p[i].x;
  if (acc == 0x7fffffff) *sink = acc;
}

template <int U>
__global__ void __launch_bounds__(256) k_reg(const char* __restrict__ x, const int* __restrict__ perm, char* __restrict__ y,
                                            int R, int row) {
  const int lane = threadIdx.x & 31;
  const int wg = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
  const int per = row / 16;  // vectors per row
  const int items_per_row = per / (32 * U);
  for (int it = wg; it < R * items_per_row; it += nw) {
    const int r = it / items_per_row, c = it % items_per_row;
    const int src = __ldg(perm + r);
    const int4* s = reinterpret_cast<const int4*>(x + int64_t(src) * row) + c * 32 * U + lane;
    int4* d = reinterpret_cast<int4*>(y + int64_t(r) * row) + c * 32 * U + lane;
    int4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = s[u * 32];
#pragma unroll
    for (int u = 0; u < U; ++u) d[u * 32] = v[u];
  }
}

__device__ __forceinline__ uint32_t sa(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void mb_init(uint64_t* b, unsigned c) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa(b)), "r"(c) : "memory"); }
__device__ __forceinline__ void mb_expect(uint64_t* b, unsigned n) { asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(b)), "r"(n) : "memory"); }
__device__ __forceinline__ void mb_arrive(uint64_t* b) { asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sa(b)) : "memory"); }
__device__ __forceinline__ void mb_wait(uint64_t* b, unsigned ph) {
  asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n" ::"r"(sa(b)), "r"(ph) : "memory");
}
__device__ __forceinline__ void g2s(void* d, const void* s, unsigned n, uint64_t* b) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(sa(d)), "l"(s), "r"(n), "r"(sa(b)) : "memory");
}
__device__ __forceinline__ void s2g(void* d, const void* s, unsigned n) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(d), "r"(sa(s)), "r"(n) : "memory");
}

// TMA bulk gather: warp 0 lane 0 produces; `cons` consumer warps either copy
// smem -> global with 16-byte stores (store_tma = 0) or one elected thread per
// stage issues a bulk store (store_tma = 1).
template <int kMaxStages>
__global__ void k_bulk(const char* __restrict__ x, const int* __restrict__ perm, char* __restrict__ y, int R, int row,
                       int seg, int stages, int store_tma) {
  extern __shared__ __align__(128) char ring[];
  __shared__ uint64_t full[kMaxStages], empty[kMaxStages];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int cons = blockDim.x / 32 - 1;
  const int segs = row / seg;
  const int items = R * segs;
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) { mb_init(&full[s], 1); mb_init(&empty[s], store_tma ? 1 : cons); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (warp == cons) {
    // the whole warp loads the source rows of 32 items per round trip
    for (int m0 = 0;; m0 += 32) {
      const int my = blockIdx.x + (m0 + lane) * gridDim.x;
      if (blockIdx.x + m0 * gridDim.x >= items) break;
      const int src = my < items ? __ldg(perm + my / segs) : 0;
      for (int b = 0; b < 32; ++b) {
        const int m = m0 + b;
        const int it = blockIdx.x + m * gridDim.x;
        if (it >= items) break;
        const int st = m % stages;
        const int s_b = __shfl_sync(0xffffffffu, src, b);
        if (lane == 0) {
          if (m >= stages) mb_wait(&empty[st], ((m / stages) & 1) ^ 1);
          const int c = it % segs;
          mb_expect(&full[st], seg);
          g2s(ring + size_t(st) * seg, x + int64_t(s_b) * row + int64_t(c) * seg, seg, &full[st]);
        }
        __syncwarp();
      }
    }
  } else if (store_tma) {
    if (warp == 0 && lane == 0) {
      int m = 0;
      for (int it = blockIdx.x; it < items; it += gridDim.x, ++m) {
        const int st = m % stages;
        mb_wait(&full[st], (m / stages) & 1);
        const int r = it / segs, c = it % segs;
        s2g(y + int64_t(r) * row + int64_t(c) * seg, ring + size_t(st) * seg, seg);
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");  // smem read done -> stage free
        mb_arrive(&empty[st]);
      }
      asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    }
  } else {
    int m = 0;
    for (int it = blockIdx.x; it < items; it += gridDim.x, ++m) {
      const int st = m % stages;
      mb_wait(&full[st], (m / stages) & 1);
      const int r = it / segs, c = it % segs;
      const int4* s = reinterpret_cast<const int4*>(ring + size_t(st) * seg);
      int4* d = reinterpret_cast<int4*>(y + int64_t(r) * row + int64_t(c) * seg);
      for (int v = warp * 32 + lane; v < seg / 16; v += cons * 32) d[v] = s[v];
      __syncwarp();
      if (lane == 0) mb_arrive(&empty[st]);
    }
  }
}

int main() {
  const int R = 8192, row = 8192;
  const size_t bytes = size_t(R) * row;
  char *x, *y, *flush, *flush2;
  int* sink;
  int* perm;
  CK(cudaMalloc(&x, bytes * 2));  // source pool twice the gathered rows
  CK(cudaMalloc(&y, bytes));
  CK(cudaMalloc(&flush, 256 << 20));
  CK(cudaMalloc(&flush2, 256 << 20));
  CK(cudaMalloc(&sink, 4));
  CK(cudaMemset(flush2, 0, 256 << 20));
  CK(cudaMalloc(&perm, R * sizeof(int)));
  std::vector<int> h(R);
  std::mt19937 g(1);
  for (int i = 0; i < R; ++i) h[i] = int(g() % (2 * R));
  CK(cudaMemcpy(perm, h.data(), R * 4, cudaMemcpyHostToDevice));
  CK(cudaMemset(x, 1, bytes * 2));
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  int clean = 1;
  auto timeit = [&](auto launch) {
    float best = 1e9, tot = 0;
    for (int rep = 0; rep < 12; ++rep) {
      cudaMemsetAsync(flush, rep, 256 << 20);
      if (clean) k_read<<<sms * 4, 512>>>(reinterpret_cast<const int4*>(flush2), (256u << 20) / 16, sink);
      cudaEventRecord(a);
      launch();
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      if (rep >= 2) { best = ms < best ? ms : best; tot += ms; }
    }
    return tot / 10;
  };
  auto report = [&](const char* name, float ms) {
    printf("%-48s %8.2f us  %7.0f GB/s\n", name, ms * 1e3, 2.0 * bytes / (ms * 1e-3) / 1e9);
  };
  report("cudaMemcpy D2D (same bytes)", timeit([&] { cudaMemcpyAsync(y, x, bytes, cudaMemcpyDeviceToDevice); }));
  for (int per_sm : {1, 2, 4, 8}) {
    char nm[96];
    snprintf(nm, sizeof nm, "reg U=16 grid=%d/SM", per_sm);
    report(nm, timeit([&] { k_reg<16><<<sms * per_sm, 256>>>(x, perm, y, R, row); }));
    snprintf(nm, sizeof nm, "reg U=8 grid=%d/SM", per_sm);
    report(nm, timeit([&] { k_reg<8><<<sms * per_sm, 256>>>(x, perm, y, R, row); }));
    snprintf(nm, sizeof nm, "reg U=4 grid=%d/SM", per_sm);
    report(nm, timeit([&] { k_reg<4><<<sms * per_sm, 256>>>(x, perm, y, R, row); }));
  }
  cudaFuncSetAttribute(k_bulk<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  for (int store_tma : {0, 1})
    for (int seg : {2048, 4096, 8192})
      for (int stages : {2, 4, 8, 16})
        for (int per_sm : {1, 2, 3}) {
          const size_t smem = size_t(seg) * stages;
          if (smem * per_sm > 200 * 1024) continue;
          char nm[96];
          snprintf(nm, sizeof nm, "bulk %s seg=%d stages=%d cta/SM=%d", store_tma ? "tma-store" : "st.global", seg, stages, per_sm);
          report(nm, timeit([&] { k_bulk<16><<<sms * per_sm, store_tma ? 64 : 288, smem>>>(x, perm, y, R, row, seg, stages, store_tma); }));
          CK(cudaGetLastError());
        }
  // verify last
  std::vector<char> out(row);
  CK(cudaMemcpy(out.data(), y + row, row, cudaMemcpyDeviceToHost));
  printf("check %d\n", int(out[5]));
  return 0;
}

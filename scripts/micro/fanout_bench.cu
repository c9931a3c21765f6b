// Micro-benchmark (dev tool): does a GPU push more bytes per second over
// NVSwitch when it writes to two peers at once than to one?  4 GPUs, one
// process, peer access on; every GPU runs the same pattern at the same time
// (cards c = node * 2 + rho of a 2x2 layout):
//   one-peer   B bytes to c ^ 2                      (naive AllToAll leg)
//   serial     B/2 to c ^ 2, then B/2 to c ^ 1       (dedup AllToAll, then AllGather)
//   fan-out    B/2 to c ^ 2 and B/2 to c ^ 3 at once  (slices straight to both cards of the other node)
//   two-legs   B/2 to c ^ 2 and B/2 to c ^ 1 at once  (AllToAll and AllGather legs concurrently)
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 fanout_bench.cu -o fanout_bench
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

// warp per item of 32*4 int4; CTAs [0, split) write dst0, the rest dst1
__global__ void __launch_bounds__(256) k_st2(const int4* __restrict__ src, int4* __restrict__ dst0, int4* __restrict__ dst1,
                                             int64_t n0, int64_t n1, int split) {
  constexpr int U = 4;
  const int lane = threadIdx.x & 31;
  const bool second = int(blockIdx.x) >= split;
  const int cta = second ? blockIdx.x - split : blockIdx.x;
  const int ctas = second ? gridDim.x - split : split;
  int4* dst = second ? dst1 : dst0;
  const int64_t n = second ? n1 : n0;
  const int4* s = second ? src + n0 : src;
  const int64_t w = (int64_t(cta) * blockDim.x + threadIdx.x) >> 5, nw = (int64_t(ctas) * blockDim.x) >> 5;
  for (int64_t base = w * 32 * U; base < n; base += nw * 32 * U) {
    int4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t i = base + u * 32 + lane;
      if (i < n) v[u] = s[i];
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t i = base + u * 32 + lane;
      if (i < n) dst[i] = v[u];
    }
  }
}

int main() {
  int ng = 0;
  CK(cudaGetDeviceCount(&ng));
  if (ng < 4) { printf("needs 4 GPUs\n"); return 0; }
  const int G = 4;
  const size_t maxb = size_t(256) << 20;
  std::vector<char*> src(G), dst(G);
  std::vector<cudaStream_t> st(G);
  std::vector<cudaEvent_t> e0(G), e1(G);
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  for (int g = 0; g < G; ++g) {
    CK(cudaSetDevice(g));
    for (int p = 0; p < G; ++p)
      if (p != g) cudaDeviceEnablePeerAccess(p, 0);
    cudaGetLastError();
    CK(cudaMalloc(&src[g], maxb));
    CK(cudaMalloc(&dst[g], 2 * maxb));  // halves: [0, maxb) from one sender, [maxb, 2maxb) from another
    CK(cudaMemset(src[g], g, maxb));
    CK(cudaStreamCreateWithFlags(&st[g], cudaStreamNonBlocking));
    CK(cudaEventCreate(&e0[g]));
    CK(cudaEventCreate(&e1[g]));
  }
  // receiver slot: a sender writes into the first half of its partner across nodes (c^2)
  // and into the second half of any other peer, so concurrent senders never overlap
  auto run = [&](const char* name, size_t B, int mode) -> int {
    float best = 1e30f;
    for (int rep = 0; rep < 7; ++rep) {
      for (int g = 0; g < G; ++g) { CK(cudaSetDevice(g)); CK(cudaDeviceSynchronize()); }
      for (int g = 0; g < G; ++g) {
        CK(cudaSetDevice(g));
        CK(cudaEventRecord(e0[g], st[g]));
        const int4* s = reinterpret_cast<const int4*>(src[g]);
        int4* a = reinterpret_cast<int4*>(dst[g ^ 2]);
        int4* b1 = reinterpret_cast<int4*>(dst[g ^ 1] + maxb);
        int4* b3 = reinterpret_cast<int4*>(dst[g ^ 3] + maxb);
        const int grid = sms * 4;
        const int64_t n = int64_t(B / 16), h = n / 2;
        if (mode == 0) k_st2<<<grid, 256, 0, st[g]>>>(s, a, a, n, 0, grid);
        if (mode == 1) {
          k_st2<<<grid, 256, 0, st[g]>>>(s, a, a, h, 0, grid);
          k_st2<<<grid, 256, 0, st[g]>>>(s + h, b1, b1, h, 0, grid);
        }
        if (mode == 2) k_st2<<<grid, 256, 0, st[g]>>>(s, a, b3, h, h, grid / 2);
        if (mode == 3) k_st2<<<grid, 256, 0, st[g]>>>(s, a, b1, h, h, grid / 2);
        CK(cudaEventRecord(e1[g], st[g]));
      }
      float worst = 0.f;
      for (int g = 0; g < G; ++g) {
        CK(cudaSetDevice(g));
        CK(cudaEventSynchronize(e1[g]));
        float ms = 0.f;
        CK(cudaEventElapsedTime(&ms, e0[g], e1[g]));
        worst = ms > worst ? ms : worst;
      }
      if (rep > 1 && worst < best) best = worst;
    }
    printf("%-10s %7.1f MiB per GPU  %8.2f us  %6.0f GB/s egress per GPU\n", name, B / 1048576.0, best * 1e3,
           B / (best * 1e-3) / 1e9);
    return 0;
  };
  for (size_t mb : {8, 16, 32, 64, 128}) {
    const size_t B = mb << 20;
    run("one-peer", B, 0);
    run("serial", B, 1);
    run("fan-out", B, 2);
    run("two-legs", B, 3);
  }
  return 0;
}

// Stable expert-major index build: the index form of dataplane::permute
// (reference dataplane.hpp:118-140) plus the per-chunk segment counts that
// dispatch_chunked derives on the fly (dataplane.hpp:224-240).
//
// The (token, slot) pairs are flattened to p = i*k + s.  Within an expert the
// reference orders records by token, and a token selects an expert at most
// once, so the permuted position of pair p is
//     expert_offset[x] + #{p' < p : experts[p'] == x}
// — a stable counting sort.  One CTA of 32 warps per node batch:
//   pass 1: each warp owns a contiguous pair range; per 32-pair step,
//           __match_any_sync groups lanes by expert and the group leader adds
//           the group size to the warp's histogram row (no atomics);
//   scan  : warp-major exclusive scan per expert, then across experts;
//   pass 2: same walk; rank = popc(peers & lanemask_lt) + running base.
//   counts: rows of expert x in chunk j, by binary search of the chunk
//           boundaries inside x's (token-sorted) segment.
// Nothing in the ordering depends on atomics or scheduling, so the result is
// bit-identical run to run and to the CPU oracle.
#include "common.cuh"

namespace monta {
namespace {

constexpr int kIndexWarps = 32;
constexpr int kUnroll = 8;

__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

__global__ void __launch_bounds__(kIndexWarps * kWarp)
    k_build_index(const int32_t* __restrict__ experts, int64_t T, int k, int E, int n_chunks,
                  int32_t* __restrict__ perm_src, int32_t* __restrict__ expert_of,
                  int32_t* __restrict__ slot_pos, int32_t* __restrict__ counts,
                  int32_t* __restrict__ expert_offsets, int32_t* __restrict__ err) {
  extern __shared__ int smem[];
  int* hist = smem;                       // [kIndexWarps][E]
  int* offs = smem + kIndexWarps * E;     // [E + 1]
  const int tid = threadIdx.x;
  const int lane = tid & 31;
  const int w = tid >> 5;
  const int64_t R = T * k;
  const int64_t per_warp = ((R + kIndexWarps - 1) / kIndexWarps + 31) / 32 * 32;
  const int64_t begin = int64_t(w) * per_warp;
  const int64_t end = begin + per_warp < R ? begin + per_warp : R;

  for (int i = tid; i < kIndexWarps * E + E + 1; i += blockDim.x) smem[i] = 0;
  __syncthreads();

  int* my_hist = hist + w * E;
  // ---- pass 1: per-warp histogram
  for (int64_t base = begin; base < end; base += 32 * kUnroll) {
    int key[kUnroll];
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      const int64_t p = base + u * 32 + lane;
      key[u] = p < end ? __ldg(experts + p) : -1;
    }
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      if (base + u * 32 >= end) break;  // warp-uniform
      int x = key[u];
      if (x >= E || (x < 0 && base + u * 32 + lane < end)) {
        atomicExch(err, (int)MOE_ERR_INVALID_ARGUMENT);
        x = -1;
      }
      const unsigned peers = __match_any_sync(0xffffffffu, x);
      if (x >= 0 && lane == __ffs(peers) - 1) my_hist[x] += __popc(peers);
    }
  }
  __syncthreads();
  // ---- scan: exclusive over warps per expert, totals into offs[x]
  for (int x = tid; x < E; x += blockDim.x) {
    int run = 0;
    for (int ww = 0; ww < kIndexWarps; ++ww) {
      const int c = hist[ww * E + x];
      hist[ww * E + x] = run;
      run += c;
    }
    offs[x] = run;
  }
  __syncthreads();
  // exclusive scan of totals across experts (warp 0)
  if (w == 0) {
    int carry = 0;
    for (int x0 = 0; x0 < E; x0 += 32) {
      const int x = x0 + lane;
      const int v = x < E ? offs[x] : 0;
      int inc = v;
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const int o = __shfl_up_sync(0xffffffffu, inc, off);
        if (lane >= off) inc += o;
      }
      if (x < E) offs[x] = carry + inc - v;
      carry += __shfl_sync(0xffffffffu, inc, 31);
    }
    if (lane == 0) offs[E] = carry;
  }
  __syncthreads();
  for (int i = tid; i < kIndexWarps * E; i += blockDim.x) hist[i] += offs[i % E];
  __syncthreads();
  // ---- pass 2: ranks
  for (int64_t base = begin; base < end; base += 32 * kUnroll) {
    int key[kUnroll];
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      const int64_t p = base + u * 32 + lane;
      key[u] = p < end ? __ldg(experts + p) : -1;
    }
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      if (base + u * 32 >= end) break;
      const int64_t p = base + u * 32 + lane;
      int x = key[u];
      if (x >= E) x = -1;
      const unsigned peers = __match_any_sync(0xffffffffu, x);
      int pos = 0;
      if (x >= 0) pos = my_hist[x] + __popc(peers & lanemask_lt());
      __syncwarp();
      if (x >= 0 && lane == __ffs(peers) - 1) my_hist[x] += __popc(peers);
      __syncwarp();
      if (x >= 0 && p < end) {
        expert_of[pos] = x;
        perm_src[pos] = int32_t(p / k);
        slot_pos[p] = pos;
      } else if (p < end) {
        slot_pos[p] = -1;
      }
    }
  }
  __syncthreads();  // perm_src visible to the whole CTA
  // ---- per-chunk counts: segment x is token-sorted, so the rows of chunk j
  // are [lower_bound(j*ct), lower_bound((j+1)*ct)).
  const int64_t ct = T / n_chunks;
  for (int idx = tid; idx < n_chunks * E; idx += blockDim.x) {
    const int j = idx / E;
    const int x = idx % E;
    const int lo0 = offs[x], hi0 = offs[x + 1];
    auto lower_bound = [&](int64_t tok) {
      int lo = lo0, hi = hi0;
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (perm_src[mid] < tok) lo = mid + 1; else hi = mid;
      }
      return lo;
    };
    counts[idx] = lower_bound(int64_t(j + 1) * ct) - lower_bound(int64_t(j) * ct);
  }
  for (int x = tid; x <= E; x += blockDim.x) expert_offsets[x] = offs[x];
}

}  // namespace

size_t index_smem_bytes(int E) { return size_t(kIndexWarps * E + E + 1) * sizeof(int); }

moe_status build_index(const int32_t* experts, int64_t T, int k, int E, int n_chunks,
                       int32_t* perm_src, int32_t* expert_of, int32_t* slot_pos, int32_t* counts,
                       int32_t* expert_offsets, int32_t* dev_error, cudaStream_t stream) {
  if (k < 1 || E < 1) return fail(MOE_ERR_INVALID_ARGUMENT, "build_index: k and E must be >= 1");
  if (n_chunks < 1) return fail(MOE_ERR_INVALID_ARGUMENT, "build_index: n must be >= 1");
  if (T < 0) return fail(MOE_ERR_INVALID_ARGUMENT, "build_index: negative token count");
  if (T % n_chunks != 0)
    return fail(MOE_ERR_INVALID_ARGUMENT, "build_index: n does not divide the sequence");
  if (T * k > INT32_MAX) return fail(MOE_ERR_UNSUPPORTED, "build_index: more than 2^31 rows");
  const size_t smem = index_smem_bytes(E);
  if (smem > 200 * 1024) return fail(MOE_ERR_UNSUPPORTED, "build_index: too many experts (%d)", E);
  static int configured = 0;
  if (!configured) {
    MONTA_CUDA(cudaFuncSetAttribute(k_build_index, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    200 * 1024));
    configured = 1;
  }
  static int32_t* scratch_err = nullptr;
  if (!dev_error) {
    if (!scratch_err) MONTA_CUDA(cudaMalloc(&scratch_err, sizeof(int32_t)));
    dev_error = scratch_err;
  }
  k_build_index<<<1, kIndexWarps * kWarp, smem, stream>>>(experts, T, k, E, n_chunks, perm_src,
                                                          expert_of, slot_pos, counts,
                                                          expert_offsets, dev_error);
  MONTA_CHECK_LAUNCH("build_index launch");
  return MOE_OK;
}

}  // namespace monta

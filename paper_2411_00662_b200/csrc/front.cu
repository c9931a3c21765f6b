// Fused dispatch front end: route -> index -> epoch bump -> count exchange
// -> plan, in ONE cooperative launch (grid = token tiles, co-resident).
//
//   phase 1 (every CTA, per tile): gate the tile's tokens (dataplane::route_topk,
//            dataplane.hpp:72-106) and histogram its (token, slot) pairs by
//            expert (order-free shared-memory counts);
//   barrier  the last CTA to arrive is elected: it scans the tile histograms
//            into per-tile bases and expert offsets, derives the per-chunk
//            counts (dataplane.hpp:224-240), bumps the device epoch, stores
//            this node's counts into every expert-parallel peer's count table
//            over NVLink, and releases the grid;
//   phase 2 (every CTA, per tile): stable ranks of the tile's pairs — warps own
//            32-pair groups, __match_any_sync ranks lanes with equal experts,
//            a scan over groups orders them — written as the index
//            (dataplane::permute, dataplane.hpp:118-140).  The order depends
//            only on (token, slot), never on atomics or scheduling;
//   plan     the elected CTA waits for its peers' counts and plans
//            (plan_block, front.cuh).
#include <algorithm>
#include <vector>

#include "front.cuh"

namespace monta {
namespace {

constexpr int kFrontSmemMax = 200 * 1024;
constexpr int kScanSmemInts = 48 * 1024;  // tile histograms scanned in shared memory up to 192 KiB

__device__ __forceinline__ unsigned long long ld_acquire_gpu(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_gpu(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

template <class T, int G, int PER>
__global__ void __launch_bounds__(kFrontThreads) k_front(const FrontArgs a) {
  extern __shared__ int smem[];
  __shared__ int s_last;
  __shared__ unsigned long long s_epoch;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, nw = blockDim.x >> 5;
  const int E = a.E, k = a.k;
  const int64_t ct = a.T / a.n;
  if (tid == 0) {
    s_epoch = *a.epoch_dev + 1;  // read before any CTA can arrive: the bump happens after the barrier
    if (a.dbg && blockIdx.x == 0) a.dbg[0] = globaltimer();
  }
  // ---------------- phase 1: route + tile histograms
  for (int b = blockIdx.x; b < a.n_tiles; b += gridDim.x) {
    const int64_t i0 = int64_t(b) * a.tile_tokens;
    const int64_t i1 = i0 + a.tile_tokens < a.T ? i0 + a.tile_tokens : a.T;
    if (a.route)
      for (int64_t r0 = i0; r0 < i1; r0 += kFrontThreads / G)
        route_tokens<T, G, PER>(static_cast<const T*>(a.logits), i1, E, k, a.experts, static_cast<T*>(a.probs),
                                r0 + tid / G);
    int* h = smem;                 // [E]
    int* hc = smem + E;            // [2][E] chunk parts (unaligned only)
    for (int i = tid; i < 3 * E; i += blockDim.x) smem[i] = 0;
    __syncthreads();  // routing of this tile visible; histogram zeroed
    const int64_t np = (i1 - i0) * k;
    const int64_t j0 = i0 / ct;
    for (int64_t q = tid; q < np; q += blockDim.x) {
      const int x = a.experts[i0 * k + q];
      if (x < 0) continue;  // empty slot
      if (x >= E) {
        atomicExch(a.err, (int)MOE_ERR_INVALID_ARGUMENT);
        continue;
      }
      atomicAdd(h + x, 1);
      if (!a.aligned) {
        const int64_t j = (i0 + q / k) / ct;
        if (j - j0 < 2) atomicAdd(hc + (j - j0) * E + x, 1);
        else atomicAdd(a.counts_acc + j * E + x, 1);
      }
    }
    __syncthreads();
    for (int x = tid; x < E; x += blockDim.x) {
      a.tile_hist[int64_t(b) * E + x] = h[x];
      if (!a.aligned) {
        if (hc[x]) atomicAdd(a.counts_acc + j0 * E + x, hc[x]);
        if (hc[E + x]) atomicAdd(a.counts_acc + (j0 + 1) * E + x, hc[E + x]);
      }
    }
    __syncthreads();
  }
  // ---------------- grid barrier: the last CTA to arrive is elected
  if (tid == 0) {
    __threadfence();
    const unsigned prev = atomicAdd(a.arrive, 1u);
    s_last = prev == gridDim.x - 1;
  }
  __syncthreads();
  if (s_last) {
    if (tid == 0) {
      *a.arrive = 0u;
      *a.epoch_dev = s_epoch;
      if (a.dbg) a.dbg[1] = globaltimer();
      __threadfence();
    }
    const int nt = a.n_tiles;
    const int ld = nt + 1;  // padded row: conflict-free column walks
    const bool in_smem = int64_t(E) * ld + E + 1 <= int64_t(kScanSmemInts);
    int* tot = smem;                  // [E+1]
    int* tbs = smem + E + 1;          // [E][ld] tile-local exclusive prefix (x-major)
    auto TB = [&](int b, int x) -> int& { return in_smem ? tbs[x * ld + b] : a.tile_base[int64_t(b) * E + x]; };
    if (in_smem)
      for (int64_t i = tid; i < int64_t(nt) * E; i += blockDim.x) tbs[(i % E) * ld + i / E] = __ldcg(a.tile_hist + i);
    __syncthreads();
    // exclusive scan over tiles, one warp per expert
    for (int x = wid; x < E; x += nw) {
      int carry = 0;
      for (int b0 = 0; b0 < nt; b0 += 32) {
        const int b = b0 + lane;
        int tsum;
        const int v = b < nt ? (in_smem ? TB(b, x) : __ldcg(a.tile_hist + int64_t(b) * E + x)) : 0;
        const int ex = warp_exscan(v, lane, &tsum);
        if (b < nt) TB(b, x) = carry + ex;
        carry += tsum;
      }
      if (lane == 0) tot[x] = carry;
    }
    __syncthreads();
    // per-chunk counts: differences of the tile prefixes at chunk starts
    const int n = a.n;
    if (a.aligned) {
      const int tpc = ct > 0 ? int(ct / a.tile_tokens) : 0;  // tiles per chunk
      for (int q = tid; q < n * E; q += blockDim.x) {
        const int j = q / E, x = q % E;
        const int b_lo = j * tpc, b_hi = (j + 1) * tpc;
        const int lo = b_lo < nt ? TB(b_lo, x) : tot[x];
        const int hi = b_hi < nt ? TB(b_hi, x) : tot[x];
        a.counts[q] = hi - lo;
      }
    } else {
      for (int q = tid; q < n * E; q += blockDim.x) {
        a.counts[q] = __ldcg(a.counts_acc + q);
        a.counts_acc[q] = 0;
      }
    }
    __syncthreads();
    if (wid == 0) {  // expert offsets
      int carry = 0;
      for (int x0 = 0; x0 < E; x0 += 32) {
        const int x = x0 + lane;
        int tsum;
        const int ex = warp_exscan(x < E ? tot[x] : 0, lane, &tsum);
        __syncwarp();
        if (x < E) tot[x] = carry + ex;
        carry += tsum;
      }
      if (lane == 0) tot[E] = carry;
    }
    __syncthreads();
    for (int x = tid; x <= E; x += blockDim.x) a.expert_offsets[x] = tot[x];
    for (int64_t i = tid; i < int64_t(nt) * E; i += blockDim.x) a.tile_base[i] = TB(int(i / E), int(i % E)) + tot[i % E];
    __syncthreads();
    if (tid == 0) {
      __threadfence();
      st_release_gpu(a.ready, s_epoch);  // release the grid: tile bases are final
    }
    __syncthreads();
    // count exchange: this node's [n][E] block of every EP peer's table
    for (int d = 0; d < a.n_dst; ++d) {
      int32_t* dst = a.dst_tables[d] + int64_t(a.node) * a.max_chunks * E;
      for (int i = tid; i < n * E; i += blockDim.x) dst[i] = a.counts[i];
    }
    __syncthreads();
    if (tid == 0) {
      if (a.n_sig > 0) {
        __threadfence_system();
        for (int i = 0; i < a.n_sig; ++i) st_release_sys(a.sig_flags[i], s_epoch);
      }
      if (a.dbg) a.dbg[2] = globaltimer();
    }
  } else if (tid == 0) {
    const unsigned long long t0 = globaltimer();
    while (ld_acquire_gpu(a.ready) < s_epoch) {
      if (globaltimer() - t0 > kWaitTimeoutNs) {
        atomicExch(a.err, (int)MOE_ERR_TIMEOUT);
        break;
      }
      __nanosleep(32);
    }
  }
  __syncthreads();
  // ---------------- plan (elected CTA), overlapping the other CTAs' ranking
  __shared__ int s_ok;
  if (s_last && a.do_plan) {
    if (tid == 0) {
      s_ok = 1;
      if (a.dbg) a.dbg[3] = globaltimer();
      const unsigned long long t0 = globaltimer();
      for (int i = 0; i < a.plan.wait.n && s_ok; ++i)
        while (ld_acquire_sys(a.plan.wait.flags[i]) < s_epoch) {
          if (globaltimer() - t0 > kWaitTimeoutNs) {
            atomicExch(a.err, (int)MOE_ERR_TIMEOUT);
            s_ok = 0;
            break;
          }
          __nanosleep(32);
        }
      if (a.dbg) a.dbg[4] = globaltimer();
    }
    __syncthreads();
    if (s_ok) plan_block(a.plan, plan_tables(a.plan_in_smem ? smem : a.plan_scratch, a.plan.e, a.plan.E, a.plan.n));
    __syncthreads();
    if (a.dbg && tid == 0) a.dbg[5] = globaltimer();
  }
  // ---------------- phase 2: stable ranks of every tile's pairs
  for (int b = blockIdx.x; b < a.n_tiles; b += gridDim.x) {
    const int64_t i0 = int64_t(b) * a.tile_tokens;
    const int64_t i1 = i0 + a.tile_tokens < a.T ? i0 + a.tile_tokens : a.T;
    const int np = int((i1 - i0) * k);
    const int groups = (np + 31) / 32;
    int* hg = smem;  // [groups][E]
    for (int i = tid; i < groups * E; i += blockDim.x) hg[i] = 0;
    __syncthreads();
    for (int g = wid; g < groups; g += nw) {
      const int q = g * 32 + lane;
      int x = q < np ? a.experts[i0 * k + q] : -1;
      if (x >= E || x < 0) x = -1;
      const unsigned peers = __match_any_sync(0xffffffffu, x);
      if (x >= 0 && lane == __ffs(peers) - 1) hg[g * E + x] = __popc(peers);
    }
    __syncthreads();
    for (int x = tid; x < E; x += blockDim.x) {
      int run = __ldcg(a.tile_base + int64_t(b) * E + x);
      for (int g = 0; g < groups; ++g) {
        const int c = hg[g * E + x];
        hg[g * E + x] = run;
        run += c;
      }
    }
    __syncthreads();
    for (int g = wid; g < groups; g += nw) {
      const int q = g * 32 + lane;
      int x = q < np ? a.experts[i0 * k + q] : -1;
      if (x >= E || x < 0) x = -1;
      const unsigned peers = __match_any_sync(0xffffffffu, x);
      if (q < np) {
        if (x >= 0) {
          const int pos = hg[g * E + x] + __popc(peers & lanemask_lt());
          a.expert_of[pos] = x;
          a.perm_src[pos] = int32_t(i0 + q / k);
          a.slot_pos[i0 * k + q] = pos;
        } else {
          a.slot_pos[i0 * k + q] = -1;
        }
      }
    }
    __syncthreads();
  }
}

size_t front_smem_bytes(const FrontArgs* a) {
  const int groups = (a->tile_tokens * a->k + 31) / 32;
  size_t ints = std::max<size_t>(size_t(3) * a->E, size_t(groups) * a->E);
  const size_t scan = size_t(a->E) * (a->n_tiles + 1) + size_t(a->E) + 1;
  ints = std::max<size_t>(ints, scan <= size_t(kScanSmemInts) ? scan : size_t(a->E) + 1);
  if (a->do_plan && a->plan_in_smem) ints = std::max(ints, plan_smem_ints(a->plan.e, a->plan.E, a->plan.n));
  return ints * 4;
}

struct CoopInfo {
  const void* fn;
  int device;
  size_t smem;
  int blocks;
};

template <class T, int G, int PER>
moe_status launch_t(const FrontArgs* a, cudaStream_t s, bool configure) {
  if (configure) {
    MONTA_CUDA(cudaFuncSetAttribute(k_front<T, G, PER>, cudaFuncAttributeMaxDynamicSharedMemorySize, kFrontSmemMax));
    return MOE_OK;
  }
  const size_t smem = front_smem_bytes(a);
  if (smem > size_t(kFrontSmemMax)) return fail(MOE_ERR_UNSUPPORTED, "front: too many experts (%d)", a->E);
  // co-resident grid for the barrier: tiles, capped at the occupancy limit
  static std::vector<CoopInfo> cache;
  int dev = 0;
  cudaGetDevice(&dev);
  int max_blocks = -1;
  for (const auto& ci : cache)
    if (ci.fn == (const void*)k_front<T, G, PER> && ci.device == dev && ci.smem == smem) max_blocks = ci.blocks;
  if (max_blocks < 0) {
    int per_sm = 0, sms = 0;
    MONTA_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_front<T, G, PER>, kFrontThreads, smem));
    MONTA_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    max_blocks = std::max(1, per_sm * sms);
    cache.push_back(CoopInfo{(const void*)k_front<T, G, PER>, dev, smem, max_blocks});
  }
  const int grid = std::max(1, std::min(a->n_tiles, max_blocks));
  void* args[] = {const_cast<FrontArgs*>(a)};
  MONTA_CUDA(cudaLaunchCooperativeKernel((const void*)k_front<T, G, PER>, dim3(grid), dim3(kFrontThreads), args, smem,
                                         s));
  return MOE_OK;
}

template <class T>
moe_status launch_e(const FrontArgs* a, int E, cudaStream_t s, bool configure) {
  if (E <= 1) return launch_t<T, 1, 1>(a, s, configure);
  if (E <= 2) return launch_t<T, 2, 1>(a, s, configure);
  if (E <= 4) return launch_t<T, 4, 1>(a, s, configure);
  if (E <= 8) return launch_t<T, 8, 1>(a, s, configure);
  if (E <= 16) return launch_t<T, 16, 1>(a, s, configure);
  if (E <= 32) return launch_t<T, 32, 1>(a, s, configure);
  if (E <= 64) return launch_t<T, 32, 2>(a, s, configure);
  if (E <= 128) return launch_t<T, 32, 4>(a, s, configure);
  if (E <= 256) return launch_t<T, 32, 8>(a, s, configure);
  if (E <= 512) return launch_t<T, 32, 16>(a, s, configure);
  return launch_t<T, 32, 32>(a, s, configure);
}

}  // namespace

int front_router_tokens(int E) {
  int g = 1;
  while (g < E && g < 32) g <<= 1;
  return kFrontThreads / g;
}

// Index tile: a multiple of the router's tokens per CTA, grown (while it
// still divides the chunk length) until at most 128 tiles remain, so the
// elected CTA's scan stays small and chunk counts come from tile prefixes.
int front_tile_tokens(int E, int64_t T, int n) {
  int tt = front_router_tokens(E);
  const int64_t ct = n > 0 ? T / n : T;
  while ((T + tt - 1) / tt > 128 && ct % (2 * int64_t(tt)) == 0) tt *= 2;
  return tt;
}

moe_status launch_front(const FrontArgs& a, int logit_dtype, cudaStream_t s) {
  if (a.route)
    if (moe_status st = check_route_args(a.T, a.E, a.k)) return st;
  if (a.tile_tokens % front_router_tokens(a.E) != 0) return fail(MOE_ERR_INVALID_ARGUMENT, "front: bad tile size");
  if (logit_dtype == MOE_F64) return launch_e<double>(&a, a.E, s, false);
  return launch_e<float>(&a, a.E, s, false);
}

moe_status configure_front(int E, int logit_dtype) {
  if (moe_status st = configure_plan()) return st;
  if (logit_dtype == MOE_F64) return launch_e<double>(nullptr, E, nullptr, true);
  return launch_e<float>(nullptr, E, nullptr, true);
}

}  // namespace monta

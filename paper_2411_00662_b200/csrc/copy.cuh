// Row-copy device helpers shared by the per-launch copy kernels (copy.cu)
// and the persistent exchange kernels (xchg.cu, combine.cu).
#pragma once

#include "engine.cuh"

namespace monta {

constexpr int kCopyThreads = 256;
constexpr int kSegSmem = 1024;  // segment starts cached in shared memory

template <int V> struct CopyUnroll { static constexpr int value = V >= 8 ? 8 : 4; };

// L2-coherent vector loads, for data other GPUs store during this kernel.
__device__ __forceinline__ int4 ld_cg(const int4* p) { return __ldcg(p); }
__device__ __forceinline__ int2 ld_cg(const int2* p) { return __ldcg(p); }
__device__ __forceinline__ int ld_cg(const int* p) { return __ldcg(p); }
__device__ __forceinline__ short ld_cg(const short* p) { return __ldcg(p); }
__device__ __forceinline__ char ld_cg(const char* p) { return __ldcg(p); }

// One batch per warp: up to U vectors per lane, every load issued before any
// store (predicated, so short rows and tails keep all loads in flight).
// kCG: coherent loads (the source is written by peers during this kernel).
template <int V, bool kCG = false>
__device__ __forceinline__ void copy_bytes(const char* __restrict__ s, char* const* d, int nd, int64_t bytes,
                                           int lane) {
  using Vec = typename VecT<V>::type;
  constexpr int U = CopyUnroll<V>::value;
  const Vec* sv = reinterpret_cast<const Vec*>(s);
  const int64_t nvec = bytes / V;
  for (int64_t i0 = 0; i0 < nvec; i0 += U * 32) {
    Vec r[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t i = i0 + u * 32 + lane;
      if (i < nvec) r[u] = kCG ? ld_cg(sv + i) : ld_stream(sv + i);
    }
    for (int q = 0; q < nd; ++q) {
      Vec* dv = reinterpret_cast<Vec*>(d[q]);
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t i = i0 + u * 32 + lane;
        if (i < nvec) st_vec(dv + i, r[u]);
      }
    }
  }
}

// Work item = (row, chunk of kItemBytes): a wide row is spread over several
// warps, so per-row latency does not serialise small transfers.  CTA `cta`
// of a group of `ctas` CTAs takes items cta*warps+w, strided by the group.
// Ends with __syncthreads() (shared memory reusable afterwards).
// What copy_items needs, by reference into (grid-constant) kernel
// parameters — never a by-value copy of the 64-entry destination tables.
struct CopyView {
  const char* src;
  int64_t src_stride;
  const int32_t* gather;
  const int32_t* src_tags;
  const int32_t* token_ids;
  int32_t source_card;
  int32_t synth_tags;
  int64_t dst_stride;
  uint64_t dst_mask;
  char* const* dst;
  int32_t* const* dst_tags;
  const int32_t* bounds;  // source-row filter (null: none)
  int32_t b_lo, b_hi;
};
__device__ __forceinline__ CopyView view_of(const CopyArgs& a) {
  return CopyView{a.src, a.src_stride, a.gather, a.src_tags, a.token_ids, a.source_card, a.synth_tags,
                  a.dst_stride, a.dst_mask, a.dst, a.dst_tags, a.bounds, a.b_lo, a.b_hi};
}

// kStage: stage the segment starts in shared memory (one CTA barrier).  The
// persistent exchange kernels pass false: a barrier at the start of each
// chunk would make every warp wait for warp 0's system-scope fence of the
// previous chunk (chunk_done), which under a saturated NVLink lasts as long
// as the link queue takes to drain.
template <int V, bool kCG = false, bool kStage = true>
__device__ __forceinline__ void copy_items(const CopyView& a, const SegList* L, int64_t cpr, int64_t cta,
                                           int64_t ctas) {
  constexpr int kItemBytes = 32 * V * CopyUnroll<V>::value;
  __shared__ int64_t sbeg[kStage ? kSegSmem : 1];
  const int nseg = L->nseg;
  cpr = cpr > 0 ? cpr : 1;
  const int64_t total = L->total_rows * cpr;
  const bool cached = kStage && nseg <= kSegSmem;
  if (kStage) {
    if (cached)
      for (int i = threadIdx.x; i < nseg; i += blockDim.x) sbeg[i] = L->segs[i].row_begin;
    __syncthreads();
  }
  const int lane = threadIdx.x & 31;
  const int64_t wpc = blockDim.x / 32;
  // A warp's items visit rows in increasing order, so its segment only moves
  // forward: gallop from the previous one (usually 0-2 probes) instead of a
  // fresh binary search over every segment per item (log2(nseg) dependent
  // loads: 8 for the fine-grained 160-expert lists).
  int cur = 0;
  auto beg = [&](int i) -> int64_t { return cached ? sbeg[i] : L->segs[i].row_begin; };
  const int64_t flo = a.bounds ? int64_t(__ldg(a.bounds + a.b_lo)) : 0;
  const int64_t fhi = a.bounds ? int64_t(__ldg(a.bounds + a.b_hi)) : INT64_MAX;
  for (int64_t item = cta * wpc + (threadIdx.x >> 5); item < total; item += ctas * wpc) {
    const int64_t r = item / cpr;
    const int64_t chunk = item - r * cpr;
    int lo = cur, step = 1;
    while (lo + step < nseg && beg(lo + step) <= r) {
      lo += step;
      step <<= 1;
    }
    int hi = (lo + step < nseg ? lo + step : nseg) - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (beg(mid) <= r) lo = mid; else hi = mid - 1;
    }
    cur = lo;
    const Seg sg = L->segs[lo];
    const int64_t off = chunk * kItemBytes;
    if (off >= sg.width) continue;
    if (sg.src_row < flo || sg.src_row >= fhi) continue;  // another expert group's segment
    const int64_t bytes = sg.width - off < kItemBytes ? sg.width - off : kItemBytes;
    const int64_t i = r - sg.row_begin;
    const int64_t src_row = a.gather ? int64_t(__ldg(a.gather + sg.src_row + i)) : sg.src_row + i;
    const int64_t dst_row = sg.dst_row + i;
    const char* sp = a.src + src_row * a.src_stride + sg.col_off + off;
    char* dps[8];
    int nd = 0;
    if (sg.dst >= 0) {
      dps[nd++] = a.dst[sg.dst] + dst_row * a.dst_stride + sg.col_off + off;
    } else {
      uint64_t m = a.dst_mask;
      while (m && nd < 8) {
        const int c = __ffsll(m) - 1;
        m &= m - 1;
        dps[nd++] = a.dst[c] + dst_row * a.dst_stride + sg.col_off + off;
      }
    }
    copy_bytes<V, kCG>(sp, dps, nd, bytes, lane);
    // tags ride along with the row: {token_id, source_card, source_position, expert}
    if (chunk == 0 && lane == 0) {
      int4 tag;
      bool have = true;
      if (a.synth_tags) {
        tag = make_int4(__ldg(a.token_ids + src_row), a.source_card, int(src_row), sg.expert);
      } else if (a.src_tags) {
        tag = __ldcg(reinterpret_cast<const int4*>(a.src_tags + 4 * (sg.src_row + i)));
      } else {
        have = false;
      }
      if (have) {
        if (sg.dst >= 0) {
          if (a.dst_tags[sg.dst]) *reinterpret_cast<int4*>(a.dst_tags[sg.dst] + 4 * dst_row) = tag;
        } else {
          uint64_t m = a.dst_mask;
          while (m) {
            const int c = __ffsll(m) - 1;
            m &= m - 1;
            if (a.dst_tags[c]) *reinterpret_cast<int4*>(a.dst_tags[c] + 4 * dst_row) = tag;
          }
        }
      }
    }
  }
  __syncthreads();
}

// ---------------------------------------------------------------------------
// Per-chunk flags of the persistent exchange kernels.
// thread 0 spins until *f >= epoch (acquire, system scope); 20 s timeout
__device__ __forceinline__ bool wait_flag(const uint64_t* f, uint64_t epoch, int32_t* err) {
  const unsigned long long t0 = globaltimer();
  while (ld_acquire_sys(f) < epoch) {
    if (globaltimer() - t0 > kWaitTimeoutNs) {
      atomicExch(err, (int)MOE_ERR_TIMEOUT);
      return false;
    }
    __nanosleep(64);
  }
  return true;
}

// Optional role trace: tr[(role * max_chunks + j) * 2 + {0 start, 1 end}]
// (globaltimer ns; start = first CTA to begin the chunk, end = last to finish).
__device__ __forceinline__ void trace_start(unsigned long long* tr, int role, int max_chunks, int j) {
  if (tr && threadIdx.x == 0) atomicMin(tr + (size_t(role) * max_chunks + j) * 2, globaltimer());
}
__device__ __forceinline__ void trace_end(unsigned long long* tr, int role, int max_chunks, int j) {
  if (tr) tr[(size_t(role) * max_chunks + j) * 2 + 1] = globaltimer();
}

// The role's warps count chunk j done; the last one runs `publish`.
// Warp-granular, with no CTA barrier: a warp never waits for another warp's
// stores or fence.  A gpu-scope fence per warp orders its (possibly remote)
// stores before its count; the last arriver's system-scope fence then covers
// every counted warp's stores (fence-fence synchronisation at gpu scope plus
// cumulativity, PTX memory model) before `publish` raises the peers' flags.
// A system-scope fence per CTA and chunk costs a full NVLink queue drain each
// (scripts/micro/nvlink_bench.cu, 16 MiB in 16 chunks by 148 CTAs: 131 us
// with per-CTA system fences, 65 us with gpu-scope ones, 36 us unfenced).
// Two counter levels (kDoneGroups sub-counters, then the root) so ~1000
// warps do not serialise on one L2 atomic: counter[0] = root, counter[1 + g]
// = group g.  Counters are left at zero for the next launch.
constexpr int kDoneGroups = 16;
template <class F>
__device__ __forceinline__ void chunk_done(unsigned int* counter, int role_ctas, int cta, F publish) {
  __syncwarp();
  if ((threadIdx.x & 31) == 0) {
    const int wpc = int(blockDim.x >> 5);
    const int warps = role_ctas * wpc;
    const int w = cta * wpc + int(threadIdx.x >> 5);
    const int groups = warps < kDoneGroups ? warps : kDoneGroups;
    const int g = w % groups;
    const unsigned members = unsigned(warps / groups + (g < warps % groups ? 1 : 0));
    __threadfence();  // this warp's stores (lanes ordered by __syncwarp) before its count
    const unsigned prev = atomicAdd(counter + 1 + g, 1u);
    if (prev == members - 1) {
      counter[1 + g] = 0u;
      __threadfence();
      const unsigned top = atomicAdd(counter, 1u);
      if (top == unsigned(groups) - 1) {
        __threadfence_system();
        publish();
        *counter = 0u;
      }
    }
  }
  __syncwarp();
}

// Emulated slow inter-node link (moe_ctx_set_link_rate): a cross-node leg
// whose bytes would take longer than `bytes / rate` holds its completion
// until then — every CTA of the leg waits out the whole list's time from its
// own start t0, so the leg (and the flag it releases) lands at the emulated
// rate however fast NVLink moved it.
__device__ __forceinline__ void pace_list(const SegList* L, unsigned long long t0, uint32_t bpus, bool fp8 = false) {
  if (!bpus) return;
  __syncthreads();
  if (threadIdx.x == 0) {
    int64_t bytes = 0;
    for (int i = 0; i < L->nseg; ++i)  // fp8 wire: one byte per bf16 element + one fp32 scale per 128
      bytes += int64_t(L->segs[i].rows) * (fp8 ? L->segs[i].width / 2 + L->segs[i].width / 64 : L->segs[i].width);
    const unsigned long long until = t0 + (unsigned long long)(bytes * 1000 / int64_t(bpus));
    while (globaltimer() < until) __nanosleep(256);
  }
  __syncthreads();
}

}  // namespace monta

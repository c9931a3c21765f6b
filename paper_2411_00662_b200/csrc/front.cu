// Fused dispatch front end: route -> index -> epoch bump -> count exchange
// -> plan, in ONE cooperative launch (co-resident grid: token-tile CTAs plus
// one control CTA, the last block).
//
//   phase 1 (tile CTAs): gate the tile's tokens (dataplane::route_topk,
//            dataplane.hpp:72-106) — experts also mirrored in shared memory —
//            and histogram its (token, slot) pairs by expert;
//   barrier  every CTA arrives; the last to arrive bumps the device epoch and
//            releases the grid at once (no scan on the release path);
//   phase 2 (tile CTAs): each CTA sums the tile histograms itself (L2 reads,
//            shared-memory atomics) into expert totals and its own tile's
//            prefix, scans the totals into expert offsets, and ranks its pairs
//            stably — warps own 32-pair groups, __match_any_sync ranks lanes
//            with equal experts, a scan over groups orders them — written as
//            the index (dataplane::permute, dataplane.hpp:118-140).  The order
//            depends only on (token, slot), never on atomics or scheduling;
//   control  (last CTA, concurrently): the same sums give expert offsets and
//            per-chunk counts (dataplane.hpp:224-240); it stores this node's
//            counts into every expert-parallel peer's count table over NVLink
//            as self-validating {count | epoch} words, polls until the peers'
//            words carry this epoch and plans (plan_block) from a shared-memory
//            copy of its arguments prefetched while phase 1 ran.
#include <algorithm>
#include <vector>

#include <cstdlib>

#include "front.cuh"

namespace monta {
namespace {

constexpr int kFrontSmemMax = 200 * 1024;

__device__ __forceinline__ void st_relaxed_sys(unsigned long long* p, unsigned long long v) {
  asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ bool wait_flag_ok(const uint64_t* f, unsigned long long epoch) {
  const unsigned long long t0 = globaltimer();
  while (ld_acquire_sys(f) < epoch) {
    if (globaltimer() - t0 > kWaitTimeoutNs) return false;
    __nanosleep(32);
  }
  return true;
}
__device__ __forceinline__ unsigned long long ld_acquire_gpu(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_gpu(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// Exclusive scan of v[0..n) in shared memory by the whole CTA; v[n] = total.
// Chunks of 32 per warp, then one warp scans the chunk totals (chunk_tot holds
// (n + 31) / 32 <= 33 entries: n <= 1056).
__device__ __forceinline__ void block_exscan(int* v, int n, int* chunk_tot) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int nch = (n + 31) / 32;
  #pragma unroll 1
  for (int c = wid; c < nch; c += nw) {
    const int x = c * 32 + lane;
    int tsum;
    const int ex = warp_exscan(x < n ? v[x] : 0, lane, &tsum);
    if (x < n) v[x] = ex;
    if (lane == 0) chunk_tot[c] = tsum;
  }
  __syncthreads();
  if (wid == 0) {
    int carry = 0;
    #pragma unroll 1
    for (int c0 = 0; c0 < nch; c0 += 32) {
      const int c = c0 + lane;
      int tsum;
      const int ex = warp_exscan(c < nch ? chunk_tot[c] : 0, lane, &tsum);
      if (c < nch) chunk_tot[c] = carry + ex;
      carry += tsum;
    }
    if (lane == 0) v[n] = carry;
  }
  __syncthreads();
  #pragma unroll 1
  for (int x = threadIdx.x; x < n; x += blockDim.x) v[x] += chunk_tot[x / 32];
  __syncthreads();
}

// Sums of the tile histograms [rows][E] (L2-coherent loads, kB in flight per
// thread): tot[x] over all rows, pre[x] over rows < b_pre, cnt[j][x] over the
// rows of chunk j = row / tpc (j < n).  Null targets are skipped; with tot
// null only rows < b_pre are read.  (row, x) advance incrementally — no
// integer division in the loop (it dominated the instruction count).
__device__ __forceinline__ void sum_hists(const int32_t* hist, int rows, int E, int* tot, int* pre, int b_pre,
                                          int* cnt, int tpc, int n) {
  constexpr int kB = 8;
  const int bd = blockDim.x, dq = bd / E, dr = bd - (bd / E) * E;
  const int N = (tot ? rows : b_pre) * E;
  const double inv_tpc = 1.0 / double(tpc);
  int row = threadIdx.x / E, x = threadIdx.x - (threadIdx.x / E) * E;
  if (dq >= 1 && (cnt == nullptr || tpc >= 1)) {
    // common case: the first dq*E threads each keep one expert x (the rest
    // idle, so E need not divide the block); sum in registers (16 loads in
    // flight per thread), fold the lanes of a warp that share x, then one
    // shared atomic per (warp, x) (per-value atomics were 64-way conflicts on
    // E addresses: ~1 us; the per-element path for E = 160 cost ~5 us)
    // Chunk counts (cnt): tiles are chunk-aligned, chunk j = row / tpc; the
    // running count flushes with one atomic when the thread's row crosses a
    // chunk boundary (no division in the loop).
    constexpr int kF = 16;
    const int span = dq * E;
    int st = 0, sp = 0;
    int cj = 0, crun = 0, cnext = tpc;
    if (int(threadIdx.x) < span) {
      if (cnt) {
        cj = row / tpc;
        cnext = (cj + 1) * tpc;
      }
      for (int base = threadIdx.x; base < N; base += kF * span) {
        int v[kF];
#pragma unroll
        for (int u = 0; u < kF; ++u) {
          const int i = base + u * span;
          v[u] = i < N ? __ldcg(hist + i) : 0;
        }
#pragma unroll
        for (int u = 0; u < kF; ++u) {
          st += v[u];
          sp += row < b_pre ? v[u] : 0;
          if (cnt) {
            if (row >= cnext) {
              if (crun && cj < n) atomicAdd(cnt + cj * E + x, crun);
              cj = row / tpc;
              cnext = (cj + 1) * tpc;
              crun = 0;
            }
            crun += v[u];
          }
          row += dq;
        }
      }
      if (cnt && crun && cj < n) atomicAdd(cnt + cj * E + x, crun);
    }
    if (dr == 0 && 32 % E == 0) {  // every lane active: fold lanes sharing x
      for (int off = 16; off >= E; off >>= 1) {
        st += __shfl_xor_sync(0xffffffffu, st, off);
        sp += __shfl_xor_sync(0xffffffffu, sp, off);
      }
      if ((threadIdx.x & 31) >= E) st = sp = 0;
    }
    if (st && tot) atomicAdd(tot + x, st);
    if (sp && pre) atomicAdd(pre + x, sp);
    return;
  }
  for (int base = threadIdx.x; base < N; base += kB * bd) {
    int v[kB];
#pragma unroll
    for (int u = 0; u < kB; ++u) {
      const int i = base + u * bd;
      v[u] = i < N ? __ldcg(hist + i) : 0;
    }
#pragma unroll
    for (int u = 0; u < kB; ++u) {
      if (v[u]) {
        if (tot) atomicAdd(tot + x, v[u]);
        if (pre && row < b_pre) atomicAdd(pre + x, v[u]);
        if (cnt) {
          const int j = n == 1 ? (row < tpc ? 0 : 1) : int((double(row) + 0.5) * inv_tpc);
          if (j < n) atomicAdd(cnt + j * E + x, v[u]);
        }
      }
      row += dq;
      x += dr;
      if (x >= E) {
        x -= E;
        ++row;
      }
    }
  }
}

// Shared-memory layout (ints) of one front CTA.
struct FrontSmem {
  int exp_ints;   // tile experts mirror [tile_tokens * k] (one tile per CTA), else 0
  int work_ints;  // phase-dependent work area
};
__host__ __device__ inline FrontSmem front_smem_layout(int tile_tokens, int k, int E, int n, bool single,
                                                       size_t plan_ints) {
  FrontSmem l;
  l.exp_ints = single ? tile_tokens * k : 0;
  const int groups = (tile_tokens * k + 31) / 32;
  size_t w = size_t(3) * E;                                            // phase 1: h[E] | hc[2][E]
  const size_t p2 = size_t(2 * E + 1 + 33) + size_t(groups) * E;  // phase 2: offs | pre | ctot | hg
  const size_t cc = size_t(E + 1 + 33) + size_t(n) * E;              // control: offs | ctot | cnt
  w = w > p2 ? w : p2;
  w = w > cc ? w : cc;
  w = w > plan_ints ? w : plan_ints;
  l.work_ints = int(w);
  return l;
}

// Control CTA after the barrier: expert offsets, chunk counts, count push,
// plan.
__device__ __forceinline__ void control_tail(const FrontArgs& a, const PlanArgs& p, int* W,
                                             unsigned long long epoch) {
  __shared__ int s_ok;
  const int tid = threadIdx.x;
  const int E = a.E, nt = a.n_tiles, n = a.n;
  const int64_t ct = a.T / n;
  int* offs = W;            // [E+1]
  int* ctot = W + E + 1;    // [33]
  int* cnt = ctot + 33;     // [n][E]
  (void)ct;
  (void)nt;
  // chunk counts: the tile CTAs accumulated them (one atomic per tile and
  // expert) into this launch's parity buffer; the other buffer is zeroed for
  // the next launch (every reader of it finished in the previous one) — all
  // max_chunks of it: the next launch may use more chunks than this one, and
  // a launch with fewer chunks than the one before must not leave that
  // launch's upper chunks behind (n = 4, then 1, then 8 read stale counts)
  const int32_t* acc = a.counts_acc + size_t(epoch & 1ull) * a.max_chunks * E;
  int32_t* other = a.counts_acc + size_t((epoch + 1ull) & 1ull) * a.max_chunks * E;
  #pragma unroll 1
  for (int q = tid; q < n * E; q += blockDim.x) cnt[q] = __ldcg(acc + q);
  #pragma unroll 1
  for (int q = tid; q < a.max_chunks * E; q += blockDim.x) other[q] = 0;
  __syncthreads();
  #pragma unroll 1
  for (int x = tid; x < E; x += blockDim.x) {
    int sum = 0;
    for (int j = 0; j < n; ++j) sum += cnt[j * E + x];
    offs[x] = sum;
  }
  __syncthreads();
  // count exchange: this node's [n][E] block of every EP peer's table, as
  // 8-byte {count | epoch << 32} words — each word is single-copy atomic, so a
  // reader that sees this epoch sees the count, with no flag round trip and
  // no fence waiting for the words' own acknowledgement.  No fence before the
  // push either (a system fence costs ~1.7 us here): a peer that sees these
  // words goes on to STORE into this card's buffers, and every read this card
  // makes of those buffers (the previous combine, the host) was made by a
  // kernel that completed before this one started — all cross-GPU traffic is
  // stores into the receiver, so there is no read left for them to overtake.
  const unsigned long long tag = (unsigned long long)(uint32_t(epoch)) << 32;
  #pragma unroll 1
  for (int d = 0; d < a.n_dst; ++d) {
    unsigned long long* dst =
        reinterpret_cast<unsigned long long*>(a.dst_tables[d]) + int64_t(a.node) * a.max_chunks * E;
    #pragma unroll 1
    for (int q = tid; q < n * E; q += blockDim.x) st_relaxed_sys(dst + q, tag | uint32_t(cnt[q]));
  }
  block_exscan(offs, E, ctot);
  #pragma unroll 1
  for (int x = tid; x <= E; x += blockDim.x)
    a.expert_offsets[x] = offs[x];
  #pragma unroll 1
  for (int q = tid; q < n * E; q += blockDim.x)
    a.counts[q] = cnt[q];
  __syncthreads();
  if (tid == 0 && a.dbg) a.dbg[2] = globaltimer();
  if (!a.do_plan) return;
  if (a.do_plan == 2) {
    // one card holding every expert, final landing: the final layout IS the
    // permuted order (every base 0, full rows, nothing crosses a node)
    for (int x = tid; x <= E; x += blockDim.x)
      if (p.recv_offs) p.recv_offs[x] = offs[x];
    for (int x = tid; x < E; x += blockDim.x) {
      p.local_delta[x] = 0;
      p.aa_table[x] = 0;
      p.aa_table[E + x] = 0;
      p.aa_table[2 * E + x] = 0;
      p.aa_table[3 * E + x] = int(p.row_bytes);
    }
    if (tid == 0) {
      *p.recv_rows = offs[E];
      if (a.dbg) a.dbg[3] = a.dbg[6] = globaltimer();
    }
    return;
  }
  if (tid == 0) s_ok = 1;
  if (p.poll_peers) {  // every peer node's block carries this epoch once it has landed
    const unsigned long long* tbl = reinterpret_cast<const unsigned long long*>(p.count_table);
    const unsigned long long t0 = globaltimer();
    #pragma unroll 1
    for (;;) {
      int missing = 0;
      #pragma unroll 1
      for (int i = tid; i < p.e * n * E; i += blockDim.x) {
        const int g = i / (n * E);
        if (g == p.node) continue;
        const uint64_t v = ld_acquire_sys(reinterpret_cast<const uint64_t*>(tbl) + int64_t(g) * p.max_chunks * E + (i - g * n * E));
        missing |= uint32_t(v >> 32) != uint32_t(epoch);
      }
      if (!__syncthreads_or(missing)) break;
      if (globaltimer() - t0 > kWaitTimeoutNs) {
        if (tid == 0) {
          atomicExch(a.err, (int)MOE_ERR_TIMEOUT);
          s_ok = 0;
        }
        break;
      }
      __nanosleep(64);
    }
  }
  if (tid == 0) {
    #pragma unroll 1
    for (int i = 0; i < p.wait.n && s_ok; ++i)
      if (!wait_flag_ok(p.wait.flags[i], epoch)) {
        atomicExch(a.err, (int)MOE_ERR_TIMEOUT);
        s_ok = 0;
      }
    if (a.dbg) a.dbg[3] = globaltimer();
  }
  __syncthreads();
  if (s_ok) plan_block(p, plan_tables(a.plan_in_smem ? W : a.plan_scratch, p.e, p.E, p.n));
  __syncthreads();
  if (a.dbg && tid == 0) a.dbg[6] = globaltimer();
}

template <class T, int G, int PER>
__global__ void __launch_bounds__(front_threads(G, PER)) k_front(const __grid_constant__ FrontArgs a) {
  extern __shared__ int smem[];
  __shared__ unsigned long long s_epoch;
  __shared__ PlanArgs s_plan;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, nw = blockDim.x >> 5;
  const int E = a.E, k = a.k, nt = a.n_tiles, n = a.n;
  const int64_t ct = a.T / n;
  const int tile_ctas = gridDim.x - 1;
  const bool control = blockIdx.x == tile_ctas;
  const bool single = nt <= tile_ctas;  // at most one tile per CTA: experts stay in shared memory
  const FrontSmem L = front_smem_layout(a.tile_tokens, k, E, n, single, 0);
  int* s_exp = smem;
  int* W = smem + L.exp_ints;
  if (tid == 0) {
    s_epoch = *a.epoch_dev + 1;  // read before this CTA arrives: the bump happens after every arrival
    if (a.dbg) {
      const unsigned long long t = globaltimer();
      if (blockIdx.x == 0) a.dbg[0] = t;
      atomicMax(a.dbg + 16, ~t);  // earliest CTA start (complemented)
      atomicMax(a.dbg + 17, t);   // latest CTA start
    }
    // the CTA's tiles of gate logits are contiguous: one bulk L2 prefetch up
    // front, so the router's passes over a wide tile (E = 160: four passes)
    // do not each wait for HBM
    if (a.route && !control && blockIdx.x < nt) {
      const size_t lb = sizeof(T) * size_t(E);
      const int64_t i0 = int64_t(blockIdx.x) * a.tile_tokens;
      const int64_t i1 = i0 + a.tile_tokens < a.T ? i0 + a.tile_tokens : a.T;
      const uint32_t bytes = uint32_t(size_t(i1 - i0) * lb) & ~15u;
      const char* src = static_cast<const char*>(a.logits) + size_t(i0) * lb;
      if (bytes >= 16 && (reinterpret_cast<uintptr_t>(src) & 15) == 0 && bytes <= (1u << 20))
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
    }
  }
  // this launch's chunk-count buffer (epoch parity; control_tail zeroes the other)
  int32_t* cacc = a.counts_acc + size_t((*a.epoch_dev + 1ull) & 1ull) * a.max_chunks * E;
  // ---------------- phase 1: route + tile histograms (tile CTAs)
  if (!control) {
    for (int b = blockIdx.x; b < nt; b += tile_ctas) {
      const int64_t i0 = int64_t(b) * a.tile_tokens;
      const int64_t i1 = i0 + a.tile_tokens < a.T ? i0 + a.tile_tokens : a.T;
      const int np = int((i1 - i0) * k);
      int* h = W;       // [E]
      int* hc = W + E;  // [2][E] chunk parts (unaligned only)
      for (int i = tid; i < 3 * E; i += blockDim.x) W[i] = 0;
      if (a.route) {
        constexpr int kPass = front_threads(G, PER) / G;  // tokens per pass of the CTA
        if constexpr (sizeof(T) == 4 && G == 32 && PER <= 5) {  // two tokens per warp per pass (E <= 160: no spills)
          for (int64_t r0 = i0; r0 < i1; r0 += 2 * kPass)
            route_tokens_w32x2<PER>(reinterpret_cast<const float*>(a.logits), i1, E, k, a.experts,
                                    reinterpret_cast<float*>(a.probs), r0 + tid / G, r0 + kPass + tid / G,
                                    single ? s_exp : nullptr, i0);
        } else {
          for (int64_t r0 = i0; r0 < i1; r0 += kPass)
            route_tokens<T, G, PER>(static_cast<const T*>(a.logits), i1, E, k, a.experts, static_cast<T*>(a.probs),
                                    r0 + tid / G, single ? s_exp : nullptr, i0);
        }
      } else if (single) {
        for (int q = tid; q < np; q += blockDim.x) s_exp[q] = a.experts[i0 * k + q];
      }
      __syncthreads();  // the tile's experts visible; histogram zeroed
      const int64_t j0 = i0 / ct;
      for (int q = tid; q < np; q += blockDim.x) {
        const int x = single ? s_exp[q] : a.experts[i0 * k + q];
        if (x < 0) continue;  // empty slot
        if (x >= E) {
          atomicExch(a.err, (int)MOE_ERR_INVALID_ARGUMENT);
          continue;
        }
        atomicAdd(h + x, 1);
        if (!a.aligned) {
          const int64_t j = (i0 + q / k) / ct;
          if (j - j0 < 2) atomicAdd(hc + (j - j0) * E + x, 1);
          else atomicAdd(cacc + j * E + x, 1);
        }
      }
      __syncthreads();
      for (int x = tid; x < E; x += blockDim.x) {
        a.tile_hist[int64_t(b) * E + x] = h[x];
        if (!a.aligned) {
          if (hc[x]) atomicAdd(cacc + j0 * E + x, hc[x]);
          if (hc[E + x]) atomicAdd(cacc + (j0 + 1) * E + x, hc[E + x]);
        } else if (h[x]) {
          atomicAdd(cacc + j0 * E + x, h[x]);  // the tile lies inside chunk j0
        }
      }
      __syncthreads();
    }
  } else {
    // control: prefetch the plan arguments (kernel-parameter space) into shared memory
    const int* src = reinterpret_cast<const int*>(&a.plan);
    int* dst = reinterpret_cast<int*>(&s_plan);
    for (int i = tid; i < int(sizeof(PlanArgs) / 4); i += blockDim.x) dst[i] = src[i];
  }
  // ---------------- grid barrier: every CTA arrives; the last one releases
  __shared__ int s_last;
  if (tid == 0) {
    __threadfence();
    const unsigned prev = atomicAdd(a.arrive, 1u);
    s_last = prev == gridDim.x - 1;
    if (s_last) {
      *a.arrive = 0u;
      *a.epoch_dev = s_epoch;
      __threadfence();
      st_release_gpu(a.ready, s_epoch);
      if (a.dbg) a.dbg[1] = globaltimer();
    }
  }
  if (tid == 0 && !s_last) {
    const unsigned long long t0 = globaltimer();
    while (ld_acquire_gpu(a.ready) < s_epoch) {
      if (globaltimer() - t0 > kWaitTimeoutNs) {
        atomicExch(a.err, (int)MOE_ERR_TIMEOUT);
        break;
      }
      __nanosleep(20);
    }
  }
  __syncthreads();
  if (!control) {
    // ---------------- phase 2: expert totals + own tile prefix, then stable ranks
    int* offs = W;               // [E+1] totals -> exclusive offsets
    int* pre = W + E + 1;        // [E] this tile's prefix over earlier tiles
    int* ctot = pre + E;         // [32+1] scan chunk totals
    int* hg = ctot + 33;         // [groups][E]
    bool have_tot = false;
    for (int b = blockIdx.x; b < nt; b += tile_ctas) {
      for (int i = tid; i < (have_tot ? E : 2 * E + 1); i += blockDim.x) (have_tot ? pre : W)[i] = 0;
      __syncthreads();
      if (!have_tot)  // expert totals: column sums of the n x E chunk counts (not every tile histogram)
        for (int x = tid; x < E; x += blockDim.x) {
          int sum = 0;
          for (int j = 0; j < n; ++j) sum += __ldcg(cacc + j * E + x);
          offs[x] = sum;
        }
      sum_hists(a.tile_hist, nt, E, nullptr, pre, b, nullptr, 1, 0);
      __syncthreads();
      if (!have_tot) block_exscan(offs, E, ctot);
      have_tot = true;
      const int64_t i0 = int64_t(b) * a.tile_tokens;
      const int64_t i1 = i0 + a.tile_tokens < a.T ? i0 + a.tile_tokens : a.T;
      const int np = int((i1 - i0) * k);
      const int groups = (np + 31) / 32;
      for (int i = tid; i < groups * E; i += blockDim.x) hg[i] = 0;
      __syncthreads();
      for (int g = wid; g < groups; g += nw) {
        const int q = g * 32 + lane;
        int x = q < np ? (single ? s_exp[q] : a.experts[i0 * k + q]) : -1;
        if (x >= E || x < 0) x = -1;
        const unsigned peers = __match_any_sync(0xffffffffu, x);
        if (x >= 0 && lane == __ffs(peers) - 1) hg[g * E + x] = __popc(peers);
      }
      __syncthreads();
      for (int x = tid; x < E; x += blockDim.x) {
        int run = offs[x] + pre[x];
        for (int g = 0; g < groups; ++g) {
          const int c = hg[g * E + x];
          hg[g * E + x] = run;
          run += c;
        }
      }
      __syncthreads();
      for (int g = wid; g < groups; g += nw) {
        const int q = g * 32 + lane;
        int x = q < np ? (single ? s_exp[q] : a.experts[i0 * k + q]) : -1;
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
    if (a.dbg && tid == 0) {
      if (blockIdx.x == 0) a.dbg[7] = globaltimer();
      atomicMax(a.dbg + 18, globaltimer());  // latest CTA end
    }
    return;
  }
  control_tail(a, s_plan, W, s_epoch);
  if (a.dbg && tid == 0) atomicMax(a.dbg + 19, globaltimer());  // control CTA end
}

size_t front_smem_bytes(const FrontArgs* a, int tile_ctas) {
  const bool single = a->n_tiles <= tile_ctas;
  const size_t plan = a->do_plan && a->plan_in_smem ? plan_smem_ints(a->plan.e, a->plan.E, a->plan.n) : 0;
  const FrontSmem l = front_smem_layout(a->tile_tokens, a->k, a->E, a->n, single, plan);
  return (size_t(l.exp_ints) + size_t(l.work_ints)) * 4;
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
  // co-resident grid for the barrier: tile CTAs (capped at the occupancy
  // limit) plus the control CTA; occupancy is taken at the largest layout
  static std::vector<CoopInfo> cache;
  int dev = 0;
  cudaGetDevice(&dev);
  const size_t smem_max = front_smem_bytes(a, a->n_tiles);  // the one-tile-per-CTA layout is the larger
  if (smem_max > size_t(kFrontSmemMax)) return fail(MOE_ERR_UNSUPPORTED, "front: too many experts (%d)", a->E);
  int max_blocks = -1;
  for (const auto& ci : cache)
    if (ci.fn == (const void*)k_front<T, G, PER> && ci.device == dev && ci.smem == smem_max) max_blocks = ci.blocks;
  if (max_blocks < 0) {
    int per_sm = 0, sms = 0;
    MONTA_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_front<T, G, PER>, front_threads(G, PER),
                                                             smem_max));
    MONTA_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    max_blocks = std::max(2, per_sm * sms);
    cache.push_back(CoopInfo{(const void*)k_front<T, G, PER>, dev, smem_max, max_blocks});
  }
  const int tile_ctas = std::max(1, std::min(a->n_tiles, max_blocks - 1));
  const int grid = tile_ctas + 1;
  const size_t smem = std::min(smem_max, front_smem_bytes(a, tile_ctas));
  void* args[] = {const_cast<FrontArgs*>(a)};
  static const int coop = [] {
    const char* e = std::getenv("MONTA_FRONT_COOP");
    return e ? std::atoi(e) : 1;
  }();
  apply_carveout(k_front<T, G, PER>);
  if (coop)
    MONTA_CUDA(cudaLaunchCooperativeKernel((const void*)k_front<T, G, PER>, dim3(grid), dim3(front_threads(G, PER)),
                                           args, smem, s));
  else
    MONTA_CUDA(cudaLaunchKernel((const void*)k_front<T, G, PER>, dim3(grid), dim3(front_threads(G, PER)), args, smem, s));
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
  if (E <= 96) return launch_t<T, 32, 3>(a, s, configure);
  if (E <= 128) return launch_t<T, 32, 4>(a, s, configure);
  if (E <= 160) return launch_t<T, 32, 5>(a, s, configure);
  if (E <= 192) return launch_t<T, 32, 6>(a, s, configure);
  if (E <= 224) return launch_t<T, 32, 7>(a, s, configure);
  if (E <= 256) return launch_t<T, 32, 8>(a, s, configure);
  if (E <= 512) return launch_t<T, 32, 16>(a, s, configure);
  return launch_t<T, 32, 32>(a, s, configure);
}

}  // namespace

int front_router_tokens(int E) {
  int g = 1;
  while (g < E && g < 32) g <<= 1;
  const int per = g < 32 ? 1 : (E + 31) / 32;
  return front_threads(g, per) / g;
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
  FrontArgs f = a;
  if (f.plan_in_smem && front_smem_bytes(&f, f.n_tiles) > size_t(kFrontSmemMax)) f.plan_in_smem = 0;
  if (logit_dtype == MOE_F64) return launch_e<double>(&f, f.E, s, false);
  return launch_e<float>(&f, f.E, s, false);
}

moe_status configure_front(int E, int logit_dtype) {
  if (moe_status st = configure_plan()) return st;
  if (logit_dtype == MOE_F64) return launch_e<double>(nullptr, E, nullptr, true);
  return launch_e<float>(nullptr, E, nullptr, true);
}

}  // namespace monta

// Token-side fused permute + AllToAll (reference dispatch_monolithic /
// dispatch_chunked data movement, dataplane.hpp:145-283).
//
// The permute-side form gathers each of the R = T*k destination rows from
// its source row (x is read k times).  Here a warp owns an ITEM = (token,
// piece of 32*U vectors): it loads the piece of the token's row once (all U
// loads in flight) and stores it to every destination of the token — the
// final (or staged) row of each selected expert on its card, full width on
// own-node legs, this rank's 1/t column slice on cross-node legs under TP
// dedup (hidden_shard, dataplane.hpp:166-176).  The row index is
// base[expert] + slot_pos: the plan's per-expert table turns the permuted
// position into the receiver's offset.  Lanes 0..k-1 resolve one destination
// each and the store loop takes them by shuffle (no staging).  Tags
// {token_id, source_card, source_position, expert} are written once per
// destination row, by the token's first piece.
//
// Sub-row items and a small register budget (four CTAs, 32 warps per SM) are
// what keep enough loads in flight: the gather micro-benchmark
// (scripts/micro/gather_bench.cu) gains ~10% from 16 to 32 warps per SM at
// equal bytes in flight.
#include <cuda_fp8.h>

#include <algorithm>
#include <cstdlib>

#include "copy.cuh"

namespace monta {
namespace {

constexpr int kTokThreads = 256;
constexpr int kTokMaxK = 16;

template <int V, bool ND = false, bool FP8 = false>
__global__ void __launch_bounds__(kTokThreads, 4) k_aa_token(const __grid_constant__ TokArgs a) {
  using Vec = typename VecT<V>::type;
  constexpr int U = 64 / V > 4 ? 4 : (64 / V < 1 ? 1 : 64 / V);  // 16-byte vectors: 4 per lane (2 KiB pieces)
  constexpr int kPieceVec = 32 * U;
  const int lane = threadIdx.x & 31;
  const int E = a.E, k = a.k;
  const int64_t nvec = a.row_bytes / V;
  const int64_t pieces = (nvec + kPieceVec - 1) / kPieceVec;
  const int64_t n_items = (a.tok_end - a.tok_begin) * pieces;
  const int64_t warps = int64_t(gridDim.x) * (kTokThreads / 32);
  const uint64_t pol = l2_evict_first_policy();  // x is read once: keep L2 for the stored rows
  const unsigned long long t0 = globaltimer();
  for (int64_t it = int64_t(blockIdx.x) * (kTokThreads / 32) + (threadIdx.x >> 5); it < n_items; it += warps) {
    const int64_t i = a.tok_begin + it / pieces;
    const int64_t v0 = (it % pieces) * kPieceVec;
    // lane s < k: destination of slot s (row pointer, byte window [off, end))
    char* dp = nullptr;
    char* qp = nullptr;   // fp8 wire: e4m3 row on the receiver (cross-node legs)
    float* sp = nullptr;  //           its per-128-element scales
    int off = 0, end = 0;
    int rcard = -1;       // node dedup: the remote card this lane's row would cross to
    if (lane < k) {
      const int64_t q = i * k + lane;
      const int x = __ldg(a.experts + q);
      if (x >= 0 && x < E) {
        const int p = __ldg(a.slot_pos + q);
        const int card = __ldg(a.table + x);
        const int base = a.staged ? __ldg(a.table + (4 + a.j) * E + x) : __ldg(a.table + E + x);
        const int64_t row = int64_t(base) + p;
        off = __ldg(a.table + 2 * E + x);
        end = off + __ldg(a.table + 3 * E + x);
        if (ND && card / a.t != a.node) {
          rcard = card;  // staged below, once per (token, card); the receiver writes the tags
        } else {
          dp = a.dst[card] + row * a.dst_stride;
          if (FP8 && card / a.t != a.node) {
            qp = a.dst_pre[card] + row * a.dst_stride;
            sp = a.dst_scale[card] + row * a.blocks_per_row;
          }
          if (v0 == 0 && a.dst_tags[card])
            *reinterpret_cast<int4*>(a.dst_tags[card] + 4 * row) = make_int4(__ldg(a.token_ids + i), a.source_card,
                                                                               int(i), x);
        }
      }
    }
    if constexpr (ND) {  // node dedup
      const unsigned same = __match_any_sync(0xffffffffu, rcard);
      if (rcard >= 0 && (same & ((1u << lane) - 1u)) == 0) {  // the token's first slot on that card
        dp = a.stage[rcard] + int64_t(__ldg(a.nslot + i * a.e + rcard / a.t)) * a.dst_stride;  // same window
      }
    }
    const Vec* src = reinterpret_cast<const Vec*>(a.x + i * a.row_bytes);
    Vec r[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t v = v0 + u * 32 + lane;
      if (v < nvec) r[u] = ld_stream_ef(src + v, pol);
    }
    const int64_t piece_lo = v0 * V, piece_hi = piece_lo + int64_t(kPieceVec) * V;
    for (int s = 0; s < k; ++s) {
      char* d = reinterpret_cast<char*>(__shfl_sync(0xffffffffu, reinterpret_cast<uintptr_t>(dp), s));
      const int o = __shfl_sync(0xffffffffu, off, s), e = __shfl_sync(0xffffffffu, end, s);
      if (!d || e <= piece_lo || o >= piece_hi) continue;  // warp-uniform
      if constexpr (V == 16 && FP8) {  // (the fp8 wire is an instantiation of its own: bf16 rows keep their registers)
        char* q = reinterpret_cast<char*>(__shfl_sync(0xffffffffu, reinterpret_cast<uintptr_t>(qp), s));
        if (q) {  // warp-uniform: the fp8 wire for this cross-node leg
          float* sc = reinterpret_cast<float*>(__shfl_sync(0xffffffffu, reinterpret_cast<uintptr_t>(sp), s));
#pragma unroll
          for (int u = 0; u < U; ++u) {
            const int64_t v = v0 + u * 32 + lane;  // 16 lanes x 8 bf16 = one 128-element block
            const int64_t byte = v * V;
            const bool in = v < nvec && byte >= o && byte < e;
            const __nv_bfloat16* hv = reinterpret_cast<const __nv_bfloat16*>(&r[u]);
            float f[8];
            float amax = 0.f;
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              f[j] = in ? __bfloat162float(hv[j]) : 0.f;
              amax = fmaxf(amax, fabsf(f[j]));
            }
#pragma unroll
            for (int m = 8; m > 0; m >>= 1) amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, m));
            const float scale = amax > 0.f ? amax / 448.f : 1.f;
            if (in) {
              uint32_t w[2];
#pragma unroll
              for (int j = 0; j < 2; ++j) {
                const __nv_fp8x2_storage_t lo = __nv_cvt_float2_to_fp8x2(
                    make_float2(f[4 * j] / scale, f[4 * j + 1] / scale), __NV_SATFINITE, __NV_E4M3);
                const __nv_fp8x2_storage_t hi = __nv_cvt_float2_to_fp8x2(
                    make_float2(f[4 * j + 2] / scale, f[4 * j + 3] / scale), __NV_SATFINITE, __NV_E4M3);
                w[j] = uint32_t(lo) | (uint32_t(hi) << 16);
              }
              *reinterpret_cast<uint2*>(q + v * 8) = make_uint2(w[0], w[1]);
              if ((lane & 15) == 0) sc[v / 16] = scale;
            }
          }
          continue;
        }
      }
      Vec* dv = reinterpret_cast<Vec*>(d);
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t v = v0 + u * 32 + lane;
        const int64_t byte = v * V;
        if (v < nvec && byte >= o && byte < e) st_vec(dv + v, r[u]);
      }
    }
  }
  if (a.pace_list) pace_list(a.pace_list, t0, a.pace_bpus, a.fp8 != 0);
  cta_signal(a.sig);
}

// TMA form of the same permute, for destinations in this GPU's memory (a
// lone card or virtual cards; bf16 wire, no link pacing): one warp per CTA
// streams its tokens through a ring of S whole-row shared-memory stages.
// Lane 0 issues the row load (cp.async.bulk global -> shared, completing on
// the stage's mbarrier, L2 evict-first: x is read once); once it lands, lane
// s < k issues slot s's row store (cp.async.bulk shared -> global, the
// destination's column window) and writes its tag.  Every lane commits one
// bulk group per token, so "at most D groups pending" (wait_group.read D)
// frees the stage of token m - D for token m - D + S: S - D loads and D
// tokens' stores stay in flight with no registers holding row data.
__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__global__ void __launch_bounds__(32) k_aa_bulk(const __grid_constant__ TokArgs a, int stages, int depth) {
  extern __shared__ __align__(128) char smem[];
  const int lane = threadIdx.x;
  const int E = a.E, k = a.k;
  const uint32_t rb = uint32_t(a.row_bytes);
  const uint32_t sb = (rb + 127u) & ~127u;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + size_t(stages) * sb);
  const int64_t first = a.tok_begin + blockIdx.x;
  const int64_t ntok = first < a.tok_end ? (a.tok_end - first + gridDim.x - 1) / gridDim.x : 0;
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  if (lane == 0) {
    for (int q = 0; q < stages; ++q)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(bars + q)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  __syncwarp();
  auto load = [&](int64_t m) {  // lane 0: token m of this CTA into stage m % S
    const int q = int(m % stages);
    const uint32_t bar = smem_addr(bars + q);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(rb) : "memory");
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::
            "r"(smem_addr(smem + size_t(q) * sb)),
        "l"(a.x + (first + m * gridDim.x) * a.row_bytes), "r"(rb), "r"(bar), "l"(pol)
        : "memory");
  };
  if (lane == 0)
    for (int64_t m = 0; m < ntok && m < stages; ++m) load(m);
  for (int64_t m = 0; m < ntok; ++m) {
    const int64_t i = first + m * gridDim.x;
    const int q = int(m % stages);
    // destination of slot `lane` (index loads overlap the row load)
    char* dp = nullptr;
    uint32_t off = 0, len = 0;
    if (lane < k) {
      const int64_t qi = i * k + lane;
      const int x = __ldg(a.experts + qi);
      if (x >= 0 && x < E) {
        const int p = __ldg(a.slot_pos + qi);
        const int card = __ldg(a.table + x);
        const int base = a.staged ? __ldg(a.table + (4 + a.j) * E + x) : __ldg(a.table + E + x);
        const int64_t row = int64_t(base) + p;
        off = uint32_t(__ldg(a.table + 2 * E + x));
        len = uint32_t(__ldg(a.table + 3 * E + x));
        dp = a.dst[card] + row * a.dst_stride;
        if (a.dst_tags[card])
          *reinterpret_cast<int4*>(a.dst_tags[card] + 4 * row) = make_int4(__ldg(a.token_ids + i), a.source_card,
                                                                           int(i), x);
      }
    }
    {  // wait for the row (every lane: the stores below are per lane)
      const uint32_t bar = smem_addr(bars + q), parity = uint32_t((m / stages) & 1);
      uint32_t done;
      do {
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(done)
            : "r"(bar), "r"(parity)
            : "memory");
      } while (!done);
    }
    if (dp && len)
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dp + off),
                   "r"(smem_addr(smem + size_t(q) * sb + off)), "r"(len)
                   : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    // stage of token m - D is free once every lane's stores of it have read smem
    const int64_t r = m - depth;
    if (r >= 0 && r + stages < ntok) {
      switch (depth) {  // wait_group.read takes an immediate
        case 1: asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory"); break;
        case 2: asm volatile("cp.async.bulk.wait_group.read 2;" ::: "memory"); break;
        case 4: asm volatile("cp.async.bulk.wait_group.read 4;" ::: "memory"); break;
        default: asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); break;
      }
      __syncwarp();
      if (lane == 0) load(r + stages);
    }
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  asm volatile("fence.proxy.async.global;" ::: "memory");
  __syncwarp();
  cta_signal(a.sig);
}

// Node dedup, sender pre-pass (two launches, thread per token, 1024-token
// blocks): k_node_count marks the tokens that reach each remote node and
// counts them per block; k_node_slots gives each such token its staging slot
// = earlier blocks' counts + its rank in the block — token order, so the TP
// ranks of a node (same tokens, same routing) stage a token at the same slot
// on their same-rank receivers, which lets the receivers exchange staged
// slices (k_stage_ag) — and writes the descriptor {token id, position, its k
// destination rows on that node (-1: elsewhere), the k experts} to the
// receiver; the last block records the total in scount[card].
__device__ __forceinline__ bool reaches(const NodeSlotArgs& a, int64_t i, int card) {
  bool has = false;
  for (int s = 0; s < a.k; ++s) {
    const int x = __ldg(a.experts + i * a.k + s);
    has |= x >= 0 && x < a.E && __ldg(a.table + x) == card;
  }
  return has;
}

__device__ __forceinline__ int block_rank(bool has, int* warp_tot, int* total) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const unsigned bal = __ballot_sync(0xffffffffu, has);
  if (lane == 0) warp_tot[wid] = __popc(bal);
  __syncthreads();
  int before = 0, tot = 0;
  for (int w = 0; w < nw; ++w) {
    const int c = warp_tot[w];
    before += w < wid ? c : 0;
    tot += c;
  }
  __syncthreads();
  *total = tot;
  return before + __popc(bal & ((1u << lane) - 1u));
}

__global__ void __launch_bounds__(1024) k_node_count(const __grid_constant__ NodeSlotArgs a) {
  __shared__ int warp_tot[32];
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const int nb = gridDim.x;
  for (int g = 0; g < a.e; ++g) {
    if (g == a.node) continue;
    const bool has = i < a.T && reaches(a, i, g * a.t + a.rho);
    if (i < a.T) a.nslot[i * a.e + g] = has ? 0 : -1;
    int tot;
    block_rank(has, warp_tot, &tot);
    if (threadIdx.x == 0) a.bcnt[g * nb + blockIdx.x] = tot;
  }
}

__global__ void __launch_bounds__(1024) k_node_slots(const __grid_constant__ NodeSlotArgs a) {
  __shared__ int warp_tot[32];
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const int nb = gridDim.x;
  const int k = a.k, E = a.E;
  for (int g = 0; g < a.e; ++g) {
    if (g == a.node) continue;
    const int card = g * a.t + a.rho;
    const bool has = i < a.T && __ldg(a.nslot + i * a.e + g) == 0;
    int tot;
    const int r = block_rank(has, warp_tot, &tot);
    int base = 0, all = 0;
    for (int b = 0; b < nb; ++b) {
      const int c = __ldg(a.bcnt + g * nb + b);
      base += b < int(blockIdx.x) ? c : 0;
      all += c;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) a.scount[card] = uint32_t(all);
    if (!has) continue;
    const int slot = base + r;
    a.nslot[i * a.e + g] = slot;
    int32_t* d = a.sdesc[card] + int64_t(slot) * (2 + 2 * k);
    d[0] = __ldg(a.token_ids + i);
    d[1] = int32_t(i);
    for (int s = 0; s < k; ++s) {
      const int x = __ldg(a.experts + i * k + s);
      const bool on = x >= 0 && x < E && __ldg(a.table + x) == card;
      d[2 + s] = on ? __ldg(a.table + E + x) + __ldg(a.slot_pos + i * k + s) : -1;
      d[2 + k + s] = x;
    }
  }
}

// Node dedup under TP, receiver: this rank's slice of every staged row goes
// to the same rows of each TP peer's staging block (the peers hold the same
// tokens at the same slots), so each card ends with whole staged rows and
// fans them out itself — the AllGather moves one slice per (token, node)
// instead of one per (token, expert).  Warp per (staged row, 2 KiB piece).
__global__ void __launch_bounds__(256) k_stage_ag(const __grid_constant__ StageAgArgs a) {
  constexpr int U = 4;
  constexpr int kPieceVec = 32 * U;
  const int lane = threadIdx.x & 31;
  const int gx = int(gridDim.x) / a.nsend;  // one 1-D grid (cta_signal counts gridDim.x): sender = block / gx
  const int y = int(blockIdx.x) / gx, bx = int(blockIdx.x) % gx;
  const int64_t cnt = int64_t(*a.count[y]);
  const int64_t v_lo = a.col_lo / 16, v_hi = a.col_hi / 16;
  const int64_t pieces = (v_hi - v_lo + kPieceVec - 1) / kPieceVec;
  const int64_t warps = int64_t(gx) * (blockDim.x / 32);
  for (int64_t it = int64_t(bx) * (blockDim.x / 32) + (threadIdx.x >> 5); it < cnt * pieces; it += warps) {
    const int64_t q = it / pieces;
    const int64_t v0 = v_lo + (it % pieces) * kPieceVec;
    const int4* src = reinterpret_cast<const int4*>(a.stage[y] + q * a.row_bytes);
    int4 r[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t v = v0 + u * 32 + lane;
      if (v < v_hi) r[u] = ld_stream_ef(src + v, l2_evict_first_policy());
    }
    for (int p = 0; p < a.npeer; ++p) {
      int4* dst = reinterpret_cast<int4*>(a.peer_stage[p][y] + q * a.row_bytes);
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t v = v0 + u * 32 + lane;
        if (v < v_hi) dst[v] = r[u];
      }
    }
  }
  cta_signal(a.sig);
}

// Node dedup, receiver: warp per (staged row, 2 KiB piece) of every remote
// sender (blockIdx.y); the piece is loaded once and stored to each of its
// destination rows on this card, tags written with the first piece.
__global__ void __launch_bounds__(256) k_node_fanout(const __grid_constant__ FanoutArgs a) {
  constexpr int U = 4;
  constexpr int kPieceVec = 32 * U;
  const int lane = threadIdx.x & 31;
  const int y = blockIdx.y;
  const int64_t cnt = int64_t(*a.count[y]);
  const int64_t nvec = a.row_bytes / 16;
  const int64_t pieces = (nvec + kPieceVec - 1) / kPieceVec;
  const int k = a.k;
  const int dw = 2 + 2 * k;
  const uint64_t pol = l2_evict_first_policy();
  const int64_t warps = int64_t(gridDim.x) * (blockDim.x / 32);
  for (int64_t it = int64_t(blockIdx.x) * (blockDim.x / 32) + (threadIdx.x >> 5); it < cnt * pieces; it += warps) {
    const int64_t q = it / pieces;
    const int64_t v0 = (it % pieces) * kPieceVec;
    const int32_t* d = a.sdesc[y] + q * dw;
    int row = -1;
    if (lane < k) {
      row = __ldg(d + 2 + lane);
      if (v0 == 0 && row >= 0)
        *reinterpret_cast<int4*>(a.recv_tags + 4 * int64_t(row)) =
            make_int4(__ldg(d), a.source_card[y], __ldg(d + 1), __ldg(d + 2 + k + lane));
    }
    if (v0 * 16 + kPieceVec * 16 <= a.col_lo || v0 * 16 >= a.col_hi) continue;  // piece outside the window
    const int4* src = reinterpret_cast<const int4*>(a.stage[y] + q * a.row_bytes);
    int4 r[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t v = v0 + u * 32 + lane;
      if (v < nvec && v * 16 >= a.col_lo && v * 16 < a.col_hi) r[u] = ld_stream_ef(src + v, pol);
    }
    for (int s = 0; s < k; ++s) {
      const int rs = __shfl_sync(0xffffffffu, row, s);
      if (rs < 0) continue;
      int4* dst = reinterpret_cast<int4*>(a.recv + int64_t(rs) * a.row_bytes);
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t v = v0 + u * 32 + lane;
        if (v < nvec && v * 16 >= a.col_lo && v * 16 < a.col_hi) dst[v] = r[u];
      }
    }
  }
}

// fp8 wire receive: thread per 8 columns of a row that came cross-node.
__global__ void __launch_bounds__(256) k_wire_dequant(char* __restrict__ recv, const int32_t* __restrict__ tags,
                                                      const int64_t* __restrict__ recv_rows, const char* __restrict__ pre,
                                                      const float* __restrict__ scales, int64_t row_bytes, int bpr,
                                                      int node, int t, int64_t col0, int64_t width, int64_t p0,
                                                      int64_t p1) {
  const int64_t rows = *recv_rows;
  const int64_t per_row = width / 8;
  for (int64_t q = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; q < rows * per_row;
       q += int64_t(gridDim.x) * blockDim.x) {
    const int64_t r = q / per_row, c = col0 + (q - r * per_row) * 8;
    const int4 tg = reinterpret_cast<const int4*>(tags)[r];  // {token_id, source_card, source_position, expert}
    if (tg.y / t == node || tg.z < p0 || tg.z >= p1) continue;
    const uint2 b = *reinterpret_cast<const uint2*>(pre + r * row_bytes + c);
    const float scale = scales[r * bpr + c / 128];
    const uint32_t w[2] = {b.x, b.y};
    __nv_bfloat162 o[4];
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const __half2_raw lo = __nv_cvt_fp8x2_to_halfraw2(__nv_fp8x2_storage_t(w[j] & 0xffffu), __NV_E4M3);
      const __half2_raw hi = __nv_cvt_fp8x2_to_halfraw2(__nv_fp8x2_storage_t(w[j] >> 16), __NV_E4M3);
      const float2 fl = __half22float2(__half2(lo)), fh = __half22float2(__half2(hi));
      o[2 * j] = __floats2bfloat162_rn(fl.x * scale, fl.y * scale);
      o[2 * j + 1] = __floats2bfloat162_rn(fh.x * scale, fh.y * scale);
    }
    *reinterpret_cast<uint4*>(recv + r * row_bytes + c * 2) = *reinterpret_cast<const uint4*>(o);
  }
}

// Combine leg, send: warp per (row of the CAA list, pair of 128-element
// blocks): 16 lanes x 8 bf16 per block, amax over the half-warp, e4m3 bytes
// + fp32 scale into the source card's cwire / cscale at the same row.
__global__ void __launch_bounds__(256) k_caa_fp8(const __grid_constant__ CaaFp8Args a) {
  const int lane = threadIdx.x & 31;
  const SegList* L = a.list;
  const unsigned long long t0 = globaltimer();
  const int64_t total = L->total_rows;
  const int64_t warps = int64_t(gridDim.x) * (blockDim.x / 32);
  for (int64_t q = int64_t(blockIdx.x) * (blockDim.x / 32) + (threadIdx.x >> 5); q < total; q += warps) {
    int lo = 0, hi = L->nseg - 1;  // segment holding list row q
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (L->segs[mid].row_begin <= q) lo = mid;
      else hi = mid - 1;
    }
    const Seg& sg = L->segs[lo];
    const int64_t i = q - sg.row_begin;
    const __nv_bfloat16* src =
        reinterpret_cast<const __nv_bfloat16*>(a.src + (sg.src_row + i) * a.row_bytes + sg.col_off);
    char* wire = a.dst_wire[sg.dst] + (sg.dst_row + i) * (a.row_bytes / 2) + sg.col_off / 2;
    float* sc = a.dst_scale[sg.dst] + (sg.dst_row + i) * a.blocks_per_row + sg.col_off / 256;
    const int nblk = sg.width / 256;  // 128 bf16 per block
    for (int b0 = 0; b0 < nblk; b0 += 2) {
      const int blk = b0 + (lane >> 4);
      const bool in = blk < nblk;
      const int e0 = blk * 128 + (lane & 15) * 8;
      float f[8];
      float amax = 0.f;
      if (in) {
        const uint4 raw = *reinterpret_cast<const uint4*>(src + e0);
        const __nv_bfloat16* hv = reinterpret_cast<const __nv_bfloat16*>(&raw);
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          f[j] = __bfloat162float(hv[j]);
          amax = fmaxf(amax, fabsf(f[j]));
        }
      }
#pragma unroll
      for (int m = 8; m > 0; m >>= 1) amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, m));
      if (in) {
        const float scale = amax > 0.f ? amax / 448.f : 1.f;
        uint32_t w[2];
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          const __nv_fp8x2_storage_t l2 = __nv_cvt_float2_to_fp8x2(make_float2(f[4 * j] / scale, f[4 * j + 1] / scale),
                                                                   __NV_SATFINITE, __NV_E4M3);
          const __nv_fp8x2_storage_t h2 = __nv_cvt_float2_to_fp8x2(
              make_float2(f[4 * j + 2] / scale, f[4 * j + 3] / scale), __NV_SATFINITE, __NV_E4M3);
          w[j] = uint32_t(l2) | (uint32_t(h2) << 16);
        }
        *reinterpret_cast<uint2*>(wire + e0) = make_uint2(w[0], w[1]);
        if ((lane & 15) == 0) sc[blk] = scale;
      }
    }
  }
  pace_list(L, t0, a.pace_bpus, true);
  cta_signal(a.sig);
}

// Combine leg, receive: thread per 8 columns of each (token, slot) of the
// chunk whose expert lives on another node: comb row (bf16) = decode(cwire).
__global__ void __launch_bounds__(256) k_comb_dequant(char* __restrict__ comb, const char* __restrict__ wire,
                                                      const float* __restrict__ scales,
                                                      const int32_t* __restrict__ slot_pos,
                                                      const int32_t* __restrict__ experts, int64_t tok_begin,
                                                      int64_t tok_end, int k, int L, int node, int64_t row_bytes,
                                                      int bpr, int64_t col0, int64_t width) {
  const int64_t per = width / 8;
  const int64_t total = (tok_end - tok_begin) * k * per;
  for (int64_t q = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; q < total; q += int64_t(gridDim.x) * blockDim.x) {
    const int64_t ps = q / per;  // (token, slot) within the chunk
    const int64_t qs = tok_begin * k + ps;
    const int x = experts[qs];
    if (x < 0 || x / L == node) continue;  // own-node slots are read in place by the un-permute
    const int64_t r = slot_pos[qs];
    const int64_t c = col0 + (q - ps * per) * 8;
    const uint2 b = *reinterpret_cast<const uint2*>(wire + r * (row_bytes / 2) + c);
    const float scale = scales[r * bpr + c / 128];
    const uint32_t w[2] = {b.x, b.y};
    __nv_bfloat162 o[4];
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const __half2_raw lo = __nv_cvt_fp8x2_to_halfraw2(__nv_fp8x2_storage_t(w[j] & 0xffffu), __NV_E4M3);
      const __half2_raw hi = __nv_cvt_fp8x2_to_halfraw2(__nv_fp8x2_storage_t(w[j] >> 16), __NV_E4M3);
      const float2 fl = __half22float2(__half2(lo)), fh = __half22float2(__half2(hi));
      o[2 * j] = __floats2bfloat162_rn(fl.x * scale, fl.y * scale);
      o[2 * j + 1] = __floats2bfloat162_rn(fh.x * scale, fh.y * scale);
    }
    *reinterpret_cast<uint4*>(comb + r * row_bytes + c * 2) = *reinterpret_cast<const uint4*>(o);
  }
}

}  // namespace

cudaError_t launch_caa_fp8(const CaaFp8Args& a, int grid, cudaStream_t s) {
  k_caa_fp8<<<grid, 256, 0, s>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_comb_dequant(char* comb, const char* wire, const float* scales, const int32_t* slot_pos,
                                const int32_t* experts, int64_t tok_begin, int64_t tok_end, int k, int L, int node,
                                int64_t row_bytes, int blocks_per_row, int64_t col0, int64_t width, cudaStream_t s) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t work = (tok_end - tok_begin) * k * (width / 8);
  const int grid = int(std::max<int64_t>(1, std::min<int64_t>((work + 255) / 256, int64_t(sms) * 8)));
  k_comb_dequant<<<grid, 256, 0, s>>>(comb, wire, scales, slot_pos, experts, tok_begin, tok_end, k, L, node,
                                      row_bytes, blocks_per_row, col0, width);
  return cudaGetLastError();
}

cudaError_t launch_wire_dequant(char* recv, const int32_t* tags, const int64_t* recv_rows, int64_t cap,
                                const char* pre, const float* scales, int64_t row_bytes, int blocks_per_row,
                                int node, int t, int64_t col0, int64_t width, int64_t p0, int64_t p1,
                                cudaStream_t s) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t work = cap * (width / 8);
  const int grid = int(std::max<int64_t>(1, std::min<int64_t>((work + 255) / 256, int64_t(sms) * 8)));
  k_wire_dequant<<<grid, 256, 0, s>>>(recv, tags, recv_rows, pre, scales, row_bytes, blocks_per_row, node, t, col0,
                                      width, p0, p1);
  return cudaGetLastError();
}

// TMA bulk form (k_aa_bulk) when it applies; MONTA_AA_BULK=0 turns it off
// (A/B), MONTA_AA_STAGES / MONTA_AA_DEPTH / MONTA_AA_CPS tune the ring.
static int env_int(const char* name, int dflt) {
  const char* e = std::getenv(name);
  return e && *e ? std::atoi(e) : dflt;
}

cudaError_t launch_node_slots(const NodeSlotArgs& a, cudaStream_t s) {
  if (a.T <= 0 || a.e < 2) return cudaSuccess;
  const int nb = int((a.T + 1023) / 1024);
  k_node_count<<<nb, 1024, 0, s>>>(a);
  k_node_slots<<<nb, 1024, 0, s>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_stage_ag(const StageAgArgs& a, int64_t max_rows, cudaStream_t s) {
  if (a.nsend <= 0 || max_rows <= 0) return cudaSuccess;
  if (a.row_bytes % 16 || a.col_lo % 16 || a.col_hi % 16) return cudaErrorNotSupported;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t pieces = ((a.col_hi - a.col_lo) / 16 + 127) / 128;
  const int64_t items = max_rows * pieces;
  const int gx = int(std::max<int64_t>(1, std::min<int64_t>((items + 7) / 8, int64_t(sms) * 4 / a.nsend + 1)));
  k_stage_ag<<<gx * a.nsend, 256, 0, s>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_node_fanout(const FanoutArgs& a, int64_t max_rows, int vec, cudaStream_t s) {
  if (a.nsend <= 0 || max_rows <= 0) return cudaSuccess;
  if (vec != 16 || a.row_bytes % 16) return cudaErrorNotSupported;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t pieces = (a.row_bytes / 16 + 127) / 128;
  const int64_t items = max_rows * pieces;
  const int gx = int(std::max<int64_t>(1, std::min<int64_t>((items + 7) / 8, int64_t(sms) * 4 / a.nsend + 1)));
  k_node_fanout<<<dim3(gx, a.nsend), 256, 0, s>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_aa_token(const TokArgs& a, int vec, int grid, cudaStream_t s) {
  if (a.k > kTokMaxK) return cudaErrorNotSupported;
  static const int bulk = env_int("MONTA_AA_BULK", 1);
  const uint32_t sb = uint32_t((a.row_bytes + 127) & ~int64_t(127));
  // the ring pays when each CTA streams many tokens (the full-batch launch;
  // a pipelined chunk of a few hundred tokens stays on the register path) and
  // each row fans out to many slots: DeepSeek k = 6 107.5 -> 103 us, while at
  // k = 2 / k = 1 the register path is faster (Mixtral 19.6 vs 26.5 us, 2x70B
  // 44.9 vs 51.0 us)
  const int64_t ntok = a.tok_end - a.tok_begin;
  if (bulk && ntok >= 2048 && a.k >= 4 && a.local_dst && !a.fp8 && !a.pace_list && vec == 16 && a.row_bytes % 16 == 0 &&
      a.dst_stride % 16 == 0 && reinterpret_cast<uintptr_t>(a.x) % 16 == 0 && sb <= 64 * 1024) {
    static const int want_stages = env_int("MONTA_AA_STAGES", 8);
    static const int depth_env = env_int("MONTA_AA_DEPTH", 4);
    static const int cps_env = env_int("MONTA_AA_CPS", 2);
    int dev = 0, sms = 148, smem_max = 227 * 1024;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&smem_max, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    const int cps = std::max(1, cps_env);
    const int per_cta = std::min(smem_max, 228 * 1024 / cps - 1024);
    const int stages = std::max(2, std::min(want_stages, int((per_cta - 256) / int(sb))));
    const int depth = std::min(depth_env == 1 || depth_env == 2 || depth_env == 4 ? depth_env : 0, stages - 1);
    const size_t smem = size_t(stages) * sb + size_t(stages) * 8;
    static bool attr = false;
    if (!attr) {
      cudaFuncSetAttribute(k_aa_bulk, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_max);
      attr = true;
    }
    const int64_t toks = a.tok_end - a.tok_begin;
    const int g = int(std::max<int64_t>(1, std::min<int64_t>(toks, int64_t(sms) * cps)));
    apply_carveout(k_aa_bulk);
    k_aa_bulk<<<g, 32, smem, s>>>(a, stages, depth);
    return cudaGetLastError();
  }
  if (a.nslot) {  // node dedup (16-byte rows only)
    if (vec != 16) return cudaErrorNotSupported;
    k_aa_token<16, true><<<grid, kTokThreads, 0, s>>>(a);
    return cudaGetLastError();
  }
  if (a.fp8) {  // the fp8 wire needs 16-byte bf16 rows (moe_ctx_set_wire checks the shape)
    if (vec != 16) return cudaErrorNotSupported;
    k_aa_token<16, false, true><<<grid, kTokThreads, 0, s>>>(a);
    return cudaGetLastError();
  }
  switch (vec) {
    case 16: k_aa_token<16><<<grid, kTokThreads, 0, s>>>(a); break;
    case 8: k_aa_token<8><<<grid, kTokThreads, 0, s>>>(a); break;
    case 4: k_aa_token<4><<<grid, kTokThreads, 0, s>>>(a); break;
    case 2: k_aa_token<2><<<grid, kTokThreads, 0, s>>>(a); break;
    default: k_aa_token<1><<<grid, kTokThreads, 0, s>>>(a); break;
  }
  return cudaGetLastError();
}

}  // namespace monta

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
#include "copy.cuh"

namespace monta {
namespace {

constexpr int kTokThreads = 256;
constexpr int kTokMaxK = 16;

template <int V>
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
  for (int64_t it = int64_t(blockIdx.x) * (kTokThreads / 32) + (threadIdx.x >> 5); it < n_items; it += warps) {
    const int64_t i = a.tok_begin + it / pieces;
    const int64_t v0 = (it % pieces) * kPieceVec;
    // lane s < k: destination of slot s (row pointer, byte window [off, end))
    char* dp = nullptr;
    int off = 0, end = 0;
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
        dp = a.dst[card] + row * a.dst_stride;
        if (v0 == 0 && a.dst_tags[card])
          *reinterpret_cast<int4*>(a.dst_tags[card] + 4 * row) = make_int4(__ldg(a.token_ids + i), a.source_card,
                                                                             int(i), x);
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
      Vec* dv = reinterpret_cast<Vec*>(d);
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t v = v0 + u * 32 + lane;
        const int64_t byte = v * V;
        if (v < nvec && byte >= o && byte < e) st_vec(dv + v, r[u]);
      }
    }
  }
  cta_signal(a.sig);
}

}  // namespace

cudaError_t launch_aa_token(const TokArgs& a, int vec, int grid, cudaStream_t s) {
  if (a.k > kTokMaxK) return cudaErrorNotSupported;
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

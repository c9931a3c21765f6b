// Token-side fused permute + AllToAll (reference dispatch_monolithic /
// dispatch_chunked data movement, dataplane.hpp:145-283).
//
// The permute-side form gathers each of the R = T*k destination rows from
// its source row (x is read k times).  Here one warp owns a TOKEN: it reads
// the token's row once, 4 KiB piece by piece (all loads of a piece in flight
// before any store), and stores each piece to every destination of the
// token — the final (or staged) row of each selected expert on its card,
// full width on own-node legs, this rank's 1/t column slice on cross-node
// legs under TP dedup (hidden_shard, dataplane.hpp:166-176).  The row index
// is base[expert] + slot_pos: the plan's per-expert table turns the permuted
// position into the receiver's offset.  Tags {token_id, source_card,
// source_position, expert} are written once per destination row.
#include "copy.cuh"

namespace monta {
namespace {

constexpr int kTokThreads = 256;
constexpr int kTokMaxK = 16;

template <int V>
__global__ void __launch_bounds__(kTokThreads) k_aa_token(const __grid_constant__ TokArgs a) {
  using Vec = typename VecT<V>::type;
  constexpr int U = CopyUnroll<V>::value;
  constexpr int kPiece = 32 * V * U;
  __shared__ char* s_dst[kTokThreads / 32][kTokMaxK];
  __shared__ int s_off[kTokThreads / 32][kTokMaxK];
  __shared__ int s_end[kTokThreads / 32][kTokMaxK];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t warps = int64_t(gridDim.x) * (blockDim.x / 32);
  const int E = a.E, k = a.k;
  for (int64_t i = a.tok_begin + int64_t(blockIdx.x) * (blockDim.x / 32) + w; i < a.tok_end; i += warps) {
    if (lane < k) {
      const int64_t q = i * k + lane;
      const int x = __ldg(a.experts + q);
      char* dp = nullptr;
      int off = 0, end = 0;
      if (x >= 0 && x < E) {
        const int p = __ldg(a.slot_pos + q);
        const int card = __ldg(a.table + x);
        const int base = a.staged ? __ldg(a.table + (4 + a.j) * E + x) : __ldg(a.table + E + x);
        const int64_t row = int64_t(base) + p;
        off = __ldg(a.table + 2 * E + x);
        end = off + __ldg(a.table + 3 * E + x);
        dp = a.dst[card] + row * a.dst_stride;
        if (a.dst_tags[card])
          *reinterpret_cast<int4*>(a.dst_tags[card] + 4 * row) =
              make_int4(__ldg(a.token_ids + i), a.source_card, int(i), x);
      }
      s_dst[w][lane] = dp;
      s_off[w][lane] = off;
      s_end[w][lane] = end;
    }
    __syncwarp();
    const Vec* src = reinterpret_cast<const Vec*>(a.x + i * a.row_bytes);
    const int64_t nvec = a.row_bytes / V;
    for (int64_t v0 = 0; v0 < nvec; v0 += 32 * U) {
      Vec r[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t v = v0 + u * 32 + lane;
        if (v < nvec) r[u] = ld_stream(src + v);
      }
      const int64_t piece_lo = v0 * V, piece_hi = piece_lo + kPiece;
      for (int s = 0; s < k; ++s) {
        char* dp = s_dst[w][s];
        const int off = s_off[w][s], end = s_end[w][s];
        if (!dp || end <= piece_lo || off >= piece_hi) continue;  // warp-uniform
        Vec* dv = reinterpret_cast<Vec*>(dp);
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int64_t v = v0 + u * 32 + lane;
          const int64_t byte = v * V;
          if (v < nvec && byte >= off && byte < end) st_vec(dv + v, r[u]);
        }
      }
    }
    __syncwarp();
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

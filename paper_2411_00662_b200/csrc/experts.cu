// Expert compute between dispatch and combine: a
// grouped bf16 GEMM over the expert-major rows the dispatch lands
// (dataplane.hpp:151-160's monolithic order: for local expert l, rows
// [offs[l], offs[l+1]) of recv), and the SwiGLU expert FFN built from two of
// them.  The reference schedules one expert task per chunk terminal
// (pipesim.hpp:102) but computes nothing; this is the compute it stands for.
//
//   Y[offs[l] + i, :] = X[offs[l] + i, :] . W_l^T      (W_l: [N, K], nn.Linear)
//   SwiGLU epilogue:  H = silu(X.Wg^T) * (X.Wu^T)     (W13 tile-interleaved)
//
// sm_100a design: one persistent CTA per SM, warp-specialised —
//   warp 0      TMA producer: A (128 x 64) and B (BN x 64) bf16 boxes,
//               128-byte swizzle, into a STAGES-deep shared-memory ring
//               (mbarrier full/empty pairs, expect_tx byte counts);
//   warp 1      MMA issuer: one elected lane issues tcgen05.mma.kind::f16
//               (M=128, N=BN, K=16, fp32 accumulate in TMEM), commits each
//               stage back to the producer and each finished tile to the
//               epilogue; two TMEM accumulators (2 x BN columns) so tile i+1
//               accumulates while tile i drains;
//   warps 2..5  epilogue: tcgen05.ld 32x32b (warp w owns TMEM lanes
//               32*(w%4)..+31 = tile rows), fp32 -> bf16 (SwiGLU fused), 16-byte
//               stores of the valid rows only (a tile may overhang its expert).
// Tiles are ordered (expert, n-block, m-block) with m fastest, so the CTAs
// working at one time share one weight tile through L2 and each expert's
// activations stay L2-resident across its n-blocks.
#include <cuda.h>

#include <algorithm>
#include <mutex>

#include "common.cuh"

namespace monta {
namespace {

constexpr int kBM = 128;                  // UMMA M (rows per tile, one per TMEM lane)
constexpr int kBK = 64;                   // 64 bf16 = 128 B: one swizzle row
constexpr int kUK = 16;                   // UMMA K for kind::f16
constexpr int kThreads = 192;             // 6 warps: producer, MMA, 4 epilogue
constexpr int kMaxExperts = 1024;
constexpr uint32_t kABytes = kBM * kBK * 2;
constexpr int kStgRow = 144;  // staged row pitch (128 B of data + 16 B against bank conflicts)

template <int BN> struct Cfg {
  static constexpr int kStages = BN == 256 ? 4 : 6;
  static constexpr uint32_t kBBytes = uint32_t(BN) * kBK * 2;
  static constexpr uint32_t kStageBytes = kABytes + kBBytes;
  static constexpr uint32_t kTmemCols = 2 * BN;  // two accumulators
  // ring | barriers (2*stages + 4) x 8 B | tmem slot | tile prefix [kMaxExperts+1]
  // ... | fused-store staging: 4 epilogue warps x 32 rows x (128 + 16) B
  static constexpr size_t kSmem = 1024 + size_t(kStages) * kStageBytes + (2 * kStages + 4) * 8 + 16 +
                                  (kMaxExperts + 1) * 4 + 4 * (kMaxExperts + 1) + 16 + 4 * 32 * kStgRow;
};

// ---------------------------------------------------------------------------
// PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  uint32_t done;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(smem_u32(b)), "r"(parity)
        : "memory");
  } while (!done);
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1,
                                            uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%3, %4}], [%2], %5;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "l"(policy)
      : "memory");
}
__device__ __forceinline__ void prefetch_tmap(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_normal() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// K-major operand tile in shared memory written by TMA with 128-byte swizzle:
// rows of 128 B, 8-row core groups 1024 B apart (SBO), LBO unused (1).
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
  return uint64_t((saddr >> 4) & 0x3FFFu) | (uint64_t(1) << 16) | (uint64_t(1024 >> 4) << 32) |
         (uint64_t(1) << 46) | (uint64_t(2) << 61);
}
// kind::f16 instruction descriptor: D fp32, A/B bf16, both K-major, M x N.
template <int N>
__device__ __forceinline__ constexpr uint32_t idesc_bf16() {
  return (1u << 4) | (1u << 7) | (1u << 10) | (uint32_t(N >> 3) << 17) | (uint32_t(kBM >> 4) << 24);
}
__device__ __forceinline__ void umma_bf16(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
// 32 lanes x 32 columns of 32-bit: thread i gets row (lane base + i), 32 consecutive columns.
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
        "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
        "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
        "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

__device__ __forceinline__ uint32_t pack_bf16(float a, float b) {
  const __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<const uint32_t*>(&h);
}
__device__ __forceinline__ float silu(float g) { return g / (1.0f + __expf(-g)); }

struct GemmArgs {
  const int32_t* offs;  // [L + 1] expert row offsets into X / Y
  int32_t L;
  int32_t N;            // output columns per expert of the MMA (2F for SwiGLU)
  int32_t K;
  __nv_bfloat16* y;
  int64_t ldy;          // elements
  int32_t swiglu;       // epilogue: columns [0, BN/2) gate, [BN/2, BN) up of the tile
  // fused reverse AllToAll (plain epilogue only): row r's bytes [col_lo, col_hi)
  // also go to rowdst[r] when it is non-null (a peer's landing row over NVLink)
  char* const* rowdst;
  int32_t col_lo, col_hi;
  // plain epilogue: compute output columns [n_off, n_off + N) of each expert
  // whose weight has n_stride rows (N == n_stride, n_off == 0: all of them)
  int32_t n_stride, n_off;
};

// Tile t -> (expert, n-block, m-block); tiles of one expert are n-major,
// m fastest.  prefix[l] = first tile of expert l, mtiles[l] = m-blocks.
__device__ __forceinline__ void decode_tile(int t, const int* prefix, const int* mtiles, int L, int nblocks, int& l,
                                            int& nb, int& mb) {
  int lo = 0, hi = L - 1;  // last l with prefix[l] <= t (non-empty experts are unique)
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (prefix[mid] <= t) lo = mid;
    else hi = mid - 1;
  }
  l = lo;
  const int r = t - prefix[l];
  nb = r / mtiles[l];
  mb = r - nb * mtiles[l];
  (void)nblocks;
}

template <int BN>
__global__ void __launch_bounds__(kThreads, 1)
    k_grouped_gemm(const __grid_constant__ CUtensorMap tma_a, const __grid_constant__ CUtensorMap tma_b,
                   const GemmArgs p) {
  using C = Cfg<BN>;
  constexpr int S = C::kStages;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* ring = smem;
  uint64_t* full = reinterpret_cast<uint64_t*>(ring + size_t(S) * C::kStageBytes);
  uint64_t* empty = full + S;
  uint64_t* tfull = empty + S;   // [2]
  uint64_t* tempty = tfull + 2;  // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  int* prefix = reinterpret_cast<int*>(tmem_slot + 4);
  int* mtiles = prefix + kMaxExperts + 1;
  uint8_t* stage_rows = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(mtiles + kMaxExperts + 1) + 15) &
                                                   ~uintptr_t(15));

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int L = p.L;
  const int nblocks = p.N / BN;
  const int kblocks = p.K / kBK;

  if (warp == 0 && lane == 0) {
    prefetch_tmap(&tma_a);
    prefetch_tmap(&tma_b);
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 4);  // one arrive per epilogue warp
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(C::kTmemCols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  // tile prefix over experts (m-blocks per expert from the device offsets)
  for (int l = threadIdx.x; l < L; l += blockDim.x) {
    const int rows = __ldg(p.offs + l + 1) - __ldg(p.offs + l);
    mtiles[l] = rows > 0 ? (rows + kBM - 1) / kBM : 0;
  }
  __syncthreads();
  if (warp == 2) {  // warp scan of mtiles * nblocks
    int carry = 0;
    for (int l0 = 0; l0 < L; l0 += 32) {
      const int l = l0 + lane;
      const int v = l < L ? mtiles[l] * nblocks : 0;
      int x = v;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
      }
      if (l < L) prefix[l] = carry + x - v;
      carry += __shfl_sync(0xffffffffu, x, 31);
    }
    if (lane == 0) prefix[L] = carry;
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const int total = prefix[L];

  if (warp == 0) {
    // ---------------- TMA producer
    if (lane == 0) {
      const uint64_t pol_a = policy_evict_normal();
      const uint64_t pol_b = policy_evict_normal();
      int stage = 0;
      uint32_t phase = 0;
      for (int t = blockIdx.x; t < total; t += gridDim.x) {
        int l, nb, mb;
        decode_tile(t, prefix, mtiles, L, nblocks, l, nb, mb);
        const int arow = __ldg(p.offs + l) + mb * kBM;
        const int brow = l * p.n_stride + p.n_off + nb * BN;
        for (int kb = 0; kb < kblocks; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* sa = ring + size_t(stage) * C::kStageBytes;
          mbar_expect_tx(&full[stage], C::kStageBytes);
          tma_load_2d(sa, &tma_a, &full[stage], kb * kBK, arow, pol_a);
          tma_load_2d(sa + kABytes, &tma_b, &full[stage], kb * kBK, brow, pol_b);
          if (++stage == S) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer
    if (lane == 0) {
      constexpr uint32_t idesc = idesc_bf16<BN>();
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int t = blockIdx.x; t < total; t += gridDim.x) {
        mbar_wait(&tempty[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d = tmem_base + uint32_t(acc * BN);
        for (int kb = 0; kb < kblocks; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint32_t sa = smem_u32(ring + size_t(stage) * C::kStageBytes);
          const uint64_t da = sw128_desc(sa), db = sw128_desc(sa + kABytes);
#pragma unroll
          for (int k = 0; k < kBK / kUK; ++k)  // +32 B along K inside the swizzle row = +2 in the address field
            umma_bf16(d, da + uint64_t(2 * k), db + uint64_t(2 * k), idesc, (kb | k) != 0);
          umma_commit(&empty[stage]);
          if (++stage == S) {
            stage = 0;
            phase ^= 1;
          }
        }
        umma_commit(&tfull[acc]);
        acc ^= 1;
        if (acc == 0) acc_phase ^= 1;
      }
    }
  } else {
    // ---------------- epilogue: TMEM -> registers -> bf16 -> global
    const int q = warp & 3;  // TMEM lane quarter this warp may access
    const int row_in_tile = q * 32 + lane;
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int t = blockIdx.x; t < total; t += gridDim.x) {
      int l, nb, mb;
      decode_tile(t, prefix, mtiles, L, nblocks, l, nb, mb);
      const int r0 = __ldg(p.offs + l) + mb * kBM;
      const int rend = __ldg(p.offs + l + 1);
      const bool valid = r0 + row_in_tile < rend;
      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
      const uint32_t tbase = tmem_base + uint32_t(acc * BN) + (uint32_t(q * 32) << 16);
      __nv_bfloat16* yrow = p.y + int64_t(r0 + row_in_tile) * p.ldy;
      if (p.swiglu) {
#pragma unroll 1
        for (int c = 0; c < BN / 2; c += 32) {
          uint32_t g[32], u[32];
          tmem_ld32(tbase + uint32_t(c), g);
          tmem_ld32(tbase + uint32_t(c + BN / 2), u);
          tmem_wait_ld();
          if (valid) {
            uint4* dst = reinterpret_cast<uint4*>(yrow + int64_t(nb) * (BN / 2) + c);
#pragma unroll
            for (int v = 0; v < 4; ++v) {
              uint32_t w[4];
#pragma unroll
              for (int j = 0; j < 4; ++j) {
                const int i = v * 8 + 2 * j;
                w[j] = pack_bf16(silu(__uint_as_float(g[i])) * __uint_as_float(u[i]),
                                 silu(__uint_as_float(g[i + 1])) * __uint_as_float(u[i + 1]));
              }
              dst[v] = make_uint4(w[0], w[1], w[2], w[3]);
            }
          }
        }
      } else {
        // fused reverse AllToAll: this row's peer landing row (null: stays on
        // this node).  The remote copy goes through a per-warp staging block
        // of 32 rows x 128 B so each store instruction writes four whole
        // 128-byte row segments over NVLink (a thread-per-row store would
        // send 32 scattered 16-byte pieces per instruction).
        const char* rrow = (valid && p.rowdst) ? p.rowdst[r0 + row_in_tile] : nullptr;
        const bool any_remote = __any_sync(0xffffffffu, rrow != nullptr);
        uint8_t* stg = stage_rows + size_t(q) * 32 * kStgRow;
#pragma unroll 1
        for (int c = 0; c < BN; c += 32) {
          uint32_t a[32];
          tmem_ld32(tbase + uint32_t(c), a);
          tmem_wait_ld();
          uint4 o[4];
#pragma unroll
          for (int v = 0; v < 4; ++v) {
            uint32_t w[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              const int i = v * 8 + 2 * j;
              w[j] = pack_bf16(__uint_as_float(a[i]), __uint_as_float(a[i + 1]));
            }
            o[v] = make_uint4(w[0], w[1], w[2], w[3]);
          }
          if (valid) {
            uint4* dst = reinterpret_cast<uint4*>(yrow + p.n_off + int64_t(nb) * BN + c);
#pragma unroll
            for (int v = 0; v < 4; ++v) dst[v] = o[v];
          }
          if (any_remote) {
            const int half = (c >> 5) & 1;  // 64 B of the 128-B staged segment
            uint4* srow = reinterpret_cast<uint4*>(stg + lane * kStgRow + half * 64);
#pragma unroll
            for (int v = 0; v < 4; ++v) srow[v] = o[v];
            if (half == 1 || c + 32 >= BN) {  // a 128-B segment (or the tile's last 64 B) is staged
              __syncwarp();
              const int64_t seg_b = (p.n_off + int64_t(nb) * BN + (c & ~63)) * 2;  // byte column of the segment
              const int nchunk = half == 1 ? 8 : 4;
#pragma unroll
              for (int i = 0; i < 8; ++i) {
                const int r = i * 4 + (lane >> 3), ch = lane & 7;
                const char* rr = reinterpret_cast<const char*>(
                    __shfl_sync(0xffffffffu, reinterpret_cast<unsigned long long>(rrow), r));
                const int64_t bc = seg_b + ch * 16;
                if (rr && ch < nchunk && bc >= p.col_lo && bc < p.col_hi)
                  *reinterpret_cast<uint4*>(const_cast<char*>(rr) + bc) =
                      *reinterpret_cast<const uint4*>(stg + r * kStgRow + ch * 16);
              }
              __syncwarp();
            }
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[acc]);
      acc ^= 1;
      if (acc == 0) acc_phase ^= 1;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(C::kTmemCols)
                 : "memory");
  }
}

// ---------------------------------------------------------------------------
// Host: tensor maps through the driver entry point (no libcuda link needed).
using EncodeTiled = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                 const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                 CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiled encode_fn() {
  static EncodeTiled fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q{};
    if (cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &p, 12000, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiled>(p);
  });
  return fn;
}

// 2-D bf16 K-major map: dims {K, rows}, box {64, box_rows}, 128-byte swizzle.
moe_status make_map(CUtensorMap* m, const void* base, int64_t rows, int64_t K, int64_t ld_elems, int box_rows) {
  EncodeTiled enc = encode_fn();
  if (!enc) return fail(MOE_ERR_CUDA, "grouped_gemm: cuTensorMapEncodeTiled unavailable");
  const cuuint64_t dims[2] = {cuuint64_t(K), cuuint64_t(rows)};
  const cuuint64_t strides[1] = {cuuint64_t(ld_elems) * 2};
  const cuuint32_t box[2] = {cuuint32_t(kBK), cuuint32_t(box_rows)};
  const cuuint32_t estr[2] = {1, 1};
  const CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
                         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                         CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(MOE_ERR_CUDA, "grouped_gemm: cuTensorMapEncodeTiled failed (%d)", int(r));
  return MOE_OK;
}

bool g_configured[16] = {false};
}  // namespace
moe_status configure_grouped_gemm();
namespace {

template <int BN>
moe_status launch_gemm(const CUtensorMap& ta, const CUtensorMap& tb, const GemmArgs& a, int grid, cudaStream_t s) {
  int dev = 0;
  cudaGetDevice(&dev);
  if (!g_configured[dev & 15])
    if (moe_status st = configure_grouped_gemm()) return st;
  k_grouped_gemm<BN><<<grid, kThreads, Cfg<BN>::kSmem, s>>>(ta, tb, a);
  MONTA_CHECK_LAUNCH("grouped_gemm launch");
  return MOE_OK;
}

// w13[l][256 b + j] = gate[l][128 b + j], w13[l][256 b + 128 + j] = up[l][128 b + j]
__global__ void k_interleave_w13(const uint4* __restrict__ gate, const uint4* __restrict__ up, int64_t L,
                                 int64_t ffn, int64_t row_vecs, uint4* __restrict__ w13) {
  const int64_t total = L * 2 * ffn * row_vecs;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < total; i += int64_t(gridDim.x) * blockDim.x) {
    const int64_t v = i % row_vecs, r = i / row_vecs;  // r: row of w13 (l, 2 ffn)
    const int64_t l = r / (2 * ffn), rr = r % (2 * ffn);
    const int64_t b = rr / (2 * MOE_W13_BLOCK), j = rr % (2 * MOE_W13_BLOCK);
    const int64_t f = b * MOE_W13_BLOCK + (j % MOE_W13_BLOCK);
    const uint4* src = j < MOE_W13_BLOCK ? gate : up;
    w13[i] = src[(l * ffn + f) * row_vecs + v];
  }
}

int sm_count_of_current() {
  int dev = 0, n = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  return n;
}

}  // namespace

// Kernel attributes (227 KB dynamic shared memory) of the current device; the
// context calls this when experts are bound, outside any graph capture.
moe_status configure_grouped_gemm() {
  int dev = 0;
  MONTA_CUDA(cudaGetDevice(&dev));
  MONTA_CUDA(cudaFuncSetAttribute(k_grouped_gemm<256>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  int(Cfg<256>::kSmem)));
  MONTA_CUDA(cudaFuncSetAttribute(k_grouped_gemm<128>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  int(Cfg<128>::kSmem)));
  if (!encode_fn()) return fail(MOE_ERR_CUDA, "grouped_gemm: cuTensorMapEncodeTiled unavailable");
  g_configured[dev & 15] = true;
  return MOE_OK;
}

moe_status grouped_gemm(const void* x, int64_t ldx, int64_t x_rows, const void* w, const int32_t* offs, int L,
                        int64_t N, int64_t K, void* y, int64_t ldy, int act, int grid, cudaStream_t s,
                        char* const* rowdst = nullptr, int32_t col_lo = 0, int32_t col_hi = 0, int64_t n_stride = 0,
                        int64_t n_off = 0) {
  if (L < 1 || L > kMaxExperts) return fail(MOE_ERR_INVALID_ARGUMENT, "grouped_gemm: need 1 <= L <= %d", kMaxExperts);
  if (!x || !w || !offs || !y) return fail(MOE_ERR_INVALID_ARGUMENT, "grouped_gemm: null pointer");
  if (K < kBK || K % kBK) return fail(MOE_ERR_INVALID_ARGUMENT, "grouped_gemm: K must be a positive multiple of 64");
  if (act != MOE_ACT_NONE && act != MOE_ACT_SWIGLU)
    return fail(MOE_ERR_INVALID_ARGUMENT, "grouped_gemm: unknown activation %d", act);
  const int bn = (N % 256 == 0) ? 256 : (N % 128 == 0 ? 128 : 0);
  if (!bn) return fail(MOE_ERR_INVALID_ARGUMENT, "grouped_gemm: N must be a multiple of 128");
  if (act == MOE_ACT_SWIGLU && bn != 2 * MOE_W13_BLOCK)
    return fail(MOE_ERR_INVALID_ARGUMENT, "grouped_gemm: SwiGLU needs N = 2*ffn with ffn %% %d == 0", MOE_W13_BLOCK);
  if (ldx < K || ldx % 8 || ldy % 8 || (reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(w) |
                                        reinterpret_cast<uintptr_t>(y)) % 16)
    return fail(MOE_ERR_INVALID_ARGUMENT, "grouped_gemm: rows must be 16-byte aligned");
  if (ldy < (act == MOE_ACT_SWIGLU ? N / 2 : N)) return fail(MOE_ERR_INVALID_ARGUMENT, "grouped_gemm: ldy too small");
  if (x_rows <= 0) return MOE_OK;
  if (x_rows > INT32_MAX || int64_t(L) * N > INT32_MAX)
    return fail(MOE_ERR_INVALID_ARGUMENT, "grouped_gemm: too many rows for 32-bit TMA coordinates");
  if (n_stride == 0) n_stride = N;
  if (n_off < 0 || n_off + N > n_stride || (act != MOE_ACT_NONE && n_stride != N) || n_off % 8)
    return fail(MOE_ERR_INVALID_ARGUMENT, "grouped_gemm: bad output column window");
  CUtensorMap ta, tb;
  if (moe_status st = make_map(&ta, x, x_rows, K, ldx, kBM)) return st;
  if (moe_status st = make_map(&tb, w, int64_t(L) * n_stride, K, K, bn)) return st;
  if (rowdst && act != MOE_ACT_NONE) return fail(MOE_ERR_INVALID_ARGUMENT, "grouped_gemm: fused stores need act NONE");
  GemmArgs a{offs, L, int32_t(N), int32_t(K), static_cast<__nv_bfloat16*>(y), ldy, act == MOE_ACT_SWIGLU,
             rowdst, col_lo, col_hi, int32_t(n_stride), int32_t(n_off)};
  if (grid <= 0) grid = sm_count_of_current();
  return bn == 256 ? launch_gemm<256>(ta, tb, a, grid, s) : launch_gemm<128>(ta, tb, a, grid, s);
}

moe_status expert_ffn_fused(const void* x, int64_t ldx, int64_t x_rows, const void* w13, const void* w2,
                            const int32_t* offs, int L, int64_t hidden, int64_t ffn, void* workspace, void* y,
                            int64_t ldy, char* const* rowdst, int32_t col_lo, int32_t col_hi, int64_t out_col0,
                            int64_t out_cols, cudaStream_t s) {
  if (!workspace) return fail(MOE_ERR_INVALID_ARGUMENT, "expert_ffn: null workspace");
  if (moe_status st = grouped_gemm(x, ldx, x_rows, w13, offs, L, 2 * ffn, hidden, workspace, ffn, MOE_ACT_SWIGLU, 0, s))
    return st;
  return grouped_gemm(workspace, ffn, x_rows, w2, offs, L, out_cols, ffn, y, ldy, MOE_ACT_NONE, 0, s, rowdst, col_lo,
                      col_hi, hidden, out_col0);
}

}  // namespace monta

using namespace monta;

extern "C" moe_status moe_grouped_gemm(const void* x, int64_t ldx, int64_t x_rows, const void* w,
                                       const int32_t* expert_offsets, int32_t num_experts, int64_t n, int64_t k,
                                       void* y, int64_t ldy, int act, void* stream) {
  return grouped_gemm(x, ldx, x_rows, w, expert_offsets, num_experts, n, k, y, ldy, act, 0,
                      static_cast<cudaStream_t>(stream));
}

extern "C" moe_status moe_interleave_w13(const void* w_gate, const void* w_up, int32_t num_experts, int64_t ffn,
                                         int64_t hidden, void* w13, void* stream) {
  if (!w_gate || !w_up || !w13) return fail(MOE_ERR_INVALID_ARGUMENT, "interleave_w13: null pointer");
  if (num_experts < 1 || ffn < 1 || ffn % MOE_W13_BLOCK || hidden % 8)
    return fail(MOE_ERR_INVALID_ARGUMENT, "interleave_w13: need ffn %% %d == 0 and hidden %% 8 == 0", MOE_W13_BLOCK);
  if ((reinterpret_cast<uintptr_t>(w_gate) | reinterpret_cast<uintptr_t>(w_up) | reinterpret_cast<uintptr_t>(w13)) % 16)
    return fail(MOE_ERR_INVALID_ARGUMENT, "interleave_w13: pointers must be 16-byte aligned");
  const int64_t row_vecs = hidden / 8;
  const int64_t total = int64_t(num_experts) * 2 * ffn * row_vecs;
  const int grid = int(std::min<int64_t>((total + 255) / 256, int64_t(sm_count_of_current()) * 16));
  k_interleave_w13<<<grid, 256, 0, static_cast<cudaStream_t>(stream)>>>(
      static_cast<const uint4*>(w_gate), static_cast<const uint4*>(w_up), num_experts, ffn, row_vecs,
      static_cast<uint4*>(w13));
  MONTA_CHECK_LAUNCH("interleave_w13 launch");
  return MOE_OK;
}

extern "C" moe_status moe_expert_ffn(const void* x, int64_t ldx, int64_t x_rows, const void* w13, const void* w2,
                                     const int32_t* expert_offsets, int32_t num_experts, int64_t hidden,
                                     int64_t ffn, void* workspace, void* y, int64_t ldy, void* stream) {
  if (!workspace) return fail(MOE_ERR_INVALID_ARGUMENT, "expert_ffn: null workspace");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (moe_status st = grouped_gemm(x, ldx, x_rows, w13, expert_offsets, num_experts, 2 * ffn, hidden, workspace,
                                   ffn, MOE_ACT_SWIGLU, 0, s))
    return st;
  return grouped_gemm(workspace, ffn, x_rows, w2, expert_offsets, num_experts, hidden, ffn, y, ldy, MOE_ACT_NONE, 0,
                      s);
}

// Row movement kernels: gather-permute, and the segment-list copy that
// implements every leg of the exchange (reference dataplane.hpp:145-283):
//   AA  — permute fused with the inter-node AllToAll: rows are gathered from
//         the node batch through perm_src and stored straight into the
//         destination card (an NVLink peer address) at its final (or staged)
//         offset; TP-deduplicated legs move only this rank's 1/t column slice
//         (hidden_shard, dataplane.hpp:166-176);
//   AG  — the intra-node AllGather: forward this rank's slice of the rows
//         that arrived from other nodes to every TP peer, same row offsets;
//   D2D — the reorder copy from the chunk-major staging to the final layout;
//   CAA — the combine's reverse AllToAll into the source's permuted order.
// One warp per row, 16-byte vectors, all loads of a row batch issued before
// the stores (HBM/NVLink latency hiding); grids are persistent (a multiple of
// the SM count) and stride over the rows the plan produced on the device.
#include "engine.cuh"

namespace monta {
namespace {

constexpr int kCopyThreads = 256;
constexpr int kSegSmem = 1024;  // segment starts cached in shared memory

template <int V> struct CopyUnroll { static constexpr int value = V >= 8 ? 8 : 4; };

// One batch per warp: up to U vectors per lane, every load issued before any
// store (predicated, so short rows and tails keep all loads in flight).
template <int V>
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
      if (i < nvec) r[u] = ld_stream(sv + i);
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
// warps, so latency per row does not serialise small transfers.
template <int V>
__global__ void __launch_bounds__(kCopyThreads) k_seg_copy(const CopyArgs a) {
  if (!cta_wait(a.wait, a.err)) {
    return;
  }
  constexpr int kItemBytes = 32 * V * CopyUnroll<V>::value;
  __shared__ int64_t sbeg[kSegSmem];
  const bool second = a.list2 != nullptr && int(blockIdx.x) >= a.split;
  const SegList* L = second ? a.list2 : a.list;
  const int64_t cta = second ? int64_t(blockIdx.x) - a.split : int64_t(blockIdx.x);
  const int64_t ctas = a.list2 ? (second ? int64_t(gridDim.x) - a.split : int64_t(a.split)) : int64_t(gridDim.x);
  const int nseg = L->nseg;
  const int64_t cpr = a.chunks_per_row > 0 ? a.chunks_per_row : 1;
  const int64_t total = L->total_rows * cpr;
  const bool cached = nseg <= kSegSmem;
  if (cached)
    for (int i = threadIdx.x; i < nseg; i += blockDim.x) sbeg[i] = L->segs[i].row_begin;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int64_t wpc = blockDim.x / 32;
  for (int64_t item = cta * wpc + (threadIdx.x >> 5); item < total; item += ctas * wpc) {
    const int64_t r = item / cpr;
    const int64_t chunk = item - r * cpr;
    int lo = 0, hi = nseg - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      const int64_t b = cached ? sbeg[mid] : L->segs[mid].row_begin;
      if (b <= r) lo = mid; else hi = mid - 1;
    }
    const Seg sg = L->segs[lo];
    const int64_t off = chunk * kItemBytes;
    if (off >= sg.width) continue;
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
    copy_bytes<V>(sp, dps, nd, bytes, lane);
    // tags ride along with the row: {token_id, source_card, source_position, expert}
    if (chunk == 0 && lane == 0) {
      int4 tag;
      bool have = true;
      if (a.synth_tags) {
        tag = make_int4(__ldg(a.token_ids + src_row), a.source_card, int(src_row), sg.expert);
      } else if (a.src_tags) {
        tag = *reinterpret_cast<const int4*>(a.src_tags + 4 * (sg.src_row + i));
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
  cta_signal(a.sig);
}

template <int V>
__global__ void __launch_bounds__(kCopyThreads)
    k_gather_rows(const char* __restrict__ src, int64_t src_stride, int64_t col_off, int64_t width,
                  const int32_t* __restrict__ perm, int64_t R, char* __restrict__ out,
                  int64_t out_stride) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = int64_t(gridDim.x) * (blockDim.x / 32);
  for (int64_t r = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) / 32; r < R; r += warps) {
    const int64_t s = __ldg(perm + r);
    char* d = out + r * out_stride;
    copy_bytes<V>(src + s * src_stride + col_off, &d, 1, width, lane);
  }
}

__global__ void k_wait(const WaitList w, int32_t* err) { cta_wait(w, err); }

__global__ void k_signal(const SignalList s) {
  if (threadIdx.x == 0) {
    __threadfence_system();
    const uint64_t epoch = s.epoch_ptr ? *s.epoch_ptr : s.epoch;
    for (int i = 0; i < s.n; ++i) st_release_sys(s.flags[i], epoch);
  }
}

}  // namespace

int copy_item_bytes(int vec) { return 32 * vec * (vec >= 8 ? 8 : 4); }

cudaError_t launch_seg_copy(const CopyArgs& a, int vec, int grid, cudaStream_t s) {
  switch (vec) {
    case 16: k_seg_copy<16><<<grid, kCopyThreads, 0, s>>>(a); break;
    case 8: k_seg_copy<8><<<grid, kCopyThreads, 0, s>>>(a); break;
    case 4: k_seg_copy<4><<<grid, kCopyThreads, 0, s>>>(a); break;
    case 2: k_seg_copy<2><<<grid, kCopyThreads, 0, s>>>(a); break;
    default: k_seg_copy<1><<<grid, kCopyThreads, 0, s>>>(a); break;
  }
  return cudaGetLastError();
}

cudaError_t launch_gather_rows(const void* src, int64_t src_stride, int64_t col_off, int64_t width,
                               const int32_t* perm, int64_t R, void* out, int64_t out_stride,
                               cudaStream_t s) {
  if (R == 0 || width == 0) return cudaSuccess;
  const int vec = vec_bytes(src_stride, col_off, width, out_stride,
                            int64_t(reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(out)));
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t warps_needed = R;
  const int per_cta = kCopyThreads / 32;
  int grid = int(std::min<int64_t>((warps_needed + per_cta - 1) / per_cta, int64_t(sms) * 8));
  const char* sp = static_cast<const char*>(src);
  char* op = static_cast<char*>(out);
  switch (vec) {
    case 16: k_gather_rows<16><<<grid, kCopyThreads, 0, s>>>(sp, src_stride, col_off, width, perm, R, op, out_stride); break;
    case 8: k_gather_rows<8><<<grid, kCopyThreads, 0, s>>>(sp, src_stride, col_off, width, perm, R, op, out_stride); break;
    case 4: k_gather_rows<4><<<grid, kCopyThreads, 0, s>>>(sp, src_stride, col_off, width, perm, R, op, out_stride); break;
    case 2: k_gather_rows<2><<<grid, kCopyThreads, 0, s>>>(sp, src_stride, col_off, width, perm, R, op, out_stride); break;
    default: k_gather_rows<1><<<grid, kCopyThreads, 0, s>>>(sp, src_stride, col_off, width, perm, R, op, out_stride); break;
  }
  return cudaGetLastError();
}

cudaError_t launch_wait(const WaitList& w, int32_t* err, cudaStream_t s) {
  if (w.n == 0) return cudaSuccess;
  k_wait<<<1, 32, 0, s>>>(w, err);
  return cudaGetLastError();
}

cudaError_t launch_signal(const SignalList& sg, cudaStream_t s) {
  if (sg.n == 0) return cudaSuccess;
  k_signal<<<1, 32, 0, s>>>(sg);
  return cudaGetLastError();
}

}  // namespace monta

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
#include "copy.cuh"

namespace monta {
namespace {

template <int V>
__global__ void __launch_bounds__(kCopyThreads) k_seg_copy(const __grid_constant__ CopyArgs a) {
  if (!cta_wait(a.wait, a.err)) return;
  const bool second = a.list2 != nullptr && int(blockIdx.x) >= a.split;
  const SegList* L = second ? a.list2 : a.list;
  const int64_t cta = second ? int64_t(blockIdx.x) - a.split : int64_t(blockIdx.x);
  const int64_t ctas = a.list2 ? (second ? int64_t(gridDim.x) - a.split : int64_t(a.split)) : int64_t(gridDim.x);
  const unsigned long long t0 = globaltimer();
  copy_items<V>(view_of(a), L, a.chunks_per_row, cta, ctas);
  if (!second) pace_list(L, t0, a.pace_bpus);  // `list` carries the cross-node legs (list2: own-node)
  cta_signal(a.sig);
}

template <int V>
__device__ __forceinline__ void store_zero(char* p) {
  if constexpr (V == 16) *reinterpret_cast<uint4*>(p) = make_uint4(0, 0, 0, 0);
  else if constexpr (V == 8) *reinterpret_cast<uint2*>(p) = make_uint2(0, 0);
  else if constexpr (V == 4) *reinterpret_cast<uint32_t*>(p) = 0u;
  else if constexpr (V == 2) *reinterpret_cast<uint16_t*>(p) = 0;
  else *p = 0;
}

// out[r] = x[perm[r]] (column slice); perm[r] < 0 -> a zero row.
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
    if (s < 0) {  // no source row (the index's tail past expert_offsets[E]): zero-fill
      for (int64_t c = int64_t(lane) * V; c < width; c += 32 * V) store_zero<V>(d + c);
      continue;
    }
    copy_bytes<V>(src + s * src_stride + col_off, &d, 1, width, lane);
  }
}

// rowdst: block per (chunk list, segment), threads over the segment's rows.
__global__ void __launch_bounds__(256) k_rowdst(const char* __restrict__ lists, size_t list_stride, int nseg_cap,
                                                const PeerRows comb, int64_t row_bytes, char** __restrict__ rowdst) {
  const int j = blockIdx.x / nseg_cap, q = blockIdx.x % nseg_cap;
  const SegList* L = reinterpret_cast<const SegList*>(lists + size_t(j) * list_stride);
  if (q >= L->nseg) return;
  const Seg sg = L->segs[q];
  if (sg.dst < 0) return;
  char* base = comb.base[sg.dst];
  for (int i = threadIdx.x; i < sg.rows; i += blockDim.x)
    rowdst[sg.src_row + i] = base + (sg.dst_row + i) * row_bytes;
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

cudaError_t launch_rowdst(const SegList* lists, size_t list_stride, int n, int nseg_cap, const PeerRows& comb,
                          int64_t row_bytes, char** rowdst, int64_t cap, cudaStream_t s) {
  cudaError_t e = cudaMemsetAsync(rowdst, 0, size_t(cap) * sizeof(char*), s);
  if (e != cudaSuccess || n <= 0) return e;
  k_rowdst<<<n * nseg_cap, 256, 0, s>>>(reinterpret_cast<const char*>(lists), list_stride, nseg_cap, comb, row_bytes,
                                        rowdst);
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

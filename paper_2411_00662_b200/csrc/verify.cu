// Device-side routing check (monta.h moe_ctx_enable_checks): after a
// dispatch, every landed row's tags are checked against the layout the
// reference defines for the receiving node (dataplane.hpp:151-160: for each
// local expert, for each source node ascending, that source's rows in its
// permuted — token-ascending — order).  The receive tags are poisoned (-1)
// before the dispatch, so a lost, duplicated or misplaced row fails the
// check; failures raise MOE_ERR_CORRUPT_ROUTING (the reference's
// CorruptRoutingError) at the next moe_ctx_sync.
#include "engine.cuh"

namespace monta {
namespace {

__global__ void k_verify_recv(const int32_t* __restrict__ tags, const int64_t* __restrict__ recv_rows,
                              const int32_t* __restrict__ offs, int L, int node, int e, int t, int64_t T,
                              int32_t* err) {
  const int64_t rows = *recv_rows;
  if (offs[0] != 0 || int64_t(offs[L]) != rows) {
    if (blockIdx.x == 0 && threadIdx.x == 0) atomicExch(err, int32_t(MOE_ERR_CORRUPT_ROUTING));
    return;
  }
  for (int64_t r = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; r < rows; r += int64_t(gridDim.x) * blockDim.x) {
    int lo = 0, hi = L - 1;  // segment l with offs[l] <= r < offs[l+1]
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (offs[mid] <= r) lo = mid;
      else hi = mid - 1;
    }
    const int4 tg = reinterpret_cast<const int4*>(tags)[r];  // {token_id, source_card, source_position, expert}
    bool ok = tg.w == node * L + lo && tg.y >= 0 && tg.y % t == 0 && tg.y / t < e && tg.z >= 0 && tg.z < T;
    if (ok && r + 1 < offs[lo + 1]) {  // strictly ascending (source, position) inside the expert's block
      const int4 nx = reinterpret_cast<const int4*>(tags)[r + 1];
      ok = nx.y > tg.y || (nx.y == tg.y && nx.z > tg.z);
    }
    if (!ok) atomicExch(err, int32_t(MOE_ERR_CORRUPT_ROUTING));
  }
}

}  // namespace

cudaError_t launch_verify_recv(const int32_t* tags, const int64_t* recv_rows, const int32_t* offs, int L, int node,
                               int e, int t, int64_t T, int64_t cap, int32_t* err, cudaStream_t s) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t want = (cap + 255) / 256;
  const int grid = int(want < 1 ? 1 : (want > sms * 4 ? sms * 4 : want));
  k_verify_recv<<<grid, 256, 0, s>>>(tags, recv_rows, offs, L, node, e, t, T, err);
  return cudaGetLastError();
}

}  // namespace monta

// Stable expert-major index build: the index form of dataplane::permute
// (reference dataplane.hpp:118-140) plus the per-chunk segment counts that
// dispatch_chunked derives on the fly (dataplane.hpp:224-240).
//
// The (token, slot) pairs are flattened to p = i*k + s.  Within an expert the
// reference orders records by token, and a token selects an expert at most
// once, so the permuted position of pair p is
//     expert_offset[x] + #{p' < p : experts[p'] == x}
// — a stable counting sort.  One CTA (index_block in front.cuh):
//   pass 1: each warp owns a contiguous pair range; per 32-pair step,
//           __match_any_sync groups lanes by expert and the group leader adds
//           the group size to the warp's histogram row (no atomics in the
//           ordering; a second match on (chunk, expert) feeds the counts);
//   scan  : warp-major exclusive scan per expert, then across experts;
//   pass 2: same walk; rank = popc(peers & lanemask_lt) + running base.
// Nothing in the ordering depends on atomics or scheduling, so the result is
// bit-identical run to run and to the CPU oracle.
#include <vector>

#include "front.cuh"

namespace monta {
namespace {

constexpr int kIndexThreads = 1024;

__global__ void __launch_bounds__(kIndexThreads)
    k_build_index(const int32_t* __restrict__ experts, int64_t T, int k, int E, int n_chunks,
                  int32_t* __restrict__ perm_src, int32_t* __restrict__ expert_of, int32_t* __restrict__ slot_pos,
                  int32_t* __restrict__ counts, int32_t* __restrict__ expert_offsets, int32_t* __restrict__ err,
                  int count_in_smem) {
  extern __shared__ int smem[];
  index_block(experts, T, k, E, n_chunks, perm_src, expert_of, slot_pos, counts, expert_offsets, err, smem,
              count_in_smem != 0);
}

constexpr size_t kSmemBudget = 200 * 1024;

int32_t* scratch_error() {
  static std::vector<int32_t*> per_dev(64, nullptr);
  int dev = 0;
  cudaGetDevice(&dev);
  if (!per_dev[dev]) cudaMalloc(&per_dev[dev], 16);
  return per_dev[dev];
}

}  // namespace

moe_status build_index(const int32_t* experts, int64_t T, int k, int E, int n_chunks, int32_t* perm_src,
                       int32_t* expert_of, int32_t* slot_pos, int32_t* counts, int32_t* expert_offsets,
                       int32_t* dev_error, cudaStream_t stream) {
  if (k < 1 || E < 1) return fail(MOE_ERR_INVALID_ARGUMENT, "build_index: k and E must be >= 1");
  if (n_chunks < 1) return fail(MOE_ERR_INVALID_ARGUMENT, "build_index: n must be >= 1");
  if (T < 0) return fail(MOE_ERR_INVALID_ARGUMENT, "build_index: negative token count");
  if (T % n_chunks != 0) return fail(MOE_ERR_INVALID_ARGUMENT, "build_index: n does not divide the sequence");
  if (T * k > INT32_MAX) return fail(MOE_ERR_UNSUPPORTED, "build_index: more than 2^31 rows");
  const int nw = kIndexThreads / 32;
  bool in_smem = index_smem_ints(nw, E, n_chunks, true) * 4 <= kSmemBudget;
  const size_t smem = index_smem_ints(nw, E, n_chunks, in_smem) * 4;
  if (smem > kSmemBudget) return fail(MOE_ERR_UNSUPPORTED, "build_index: too many experts (%d)", E);
  MONTA_CUDA(cudaFuncSetAttribute(k_build_index, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kSmemBudget)));
  if (!dev_error) dev_error = scratch_error();
  k_build_index<<<1, kIndexThreads, smem, stream>>>(experts, T, k, E, n_chunks, perm_src, expert_of, slot_pos, counts,
                                                    expert_offsets, dev_error, in_smem ? 1 : 0);
  MONTA_CHECK_LAUNCH("build_index launch");
  return MOE_OK;
}

}  // namespace monta

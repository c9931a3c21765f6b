// Plan kernel: turns the exchanged per-chunk counts into every offset of the
// exchange, on the device, so the data movement never waits on the host.
//
// Count table CT[g][j][x]: rows node g sends for expert x in chunk j (the
// reference's seg_len, dataplane.hpp:224-240, generalised to L = E/e local
// experts per node).  Layouts, for destination node xg with local experts
// l = 0..L-1 (expert x = xg*L + l):
//   final  : for l, for source node g ascending, rows token-ascending — the
//            reference's monolithic order (dataplane.hpp:151-160) and
//            expert-major for a grouped GEMM;
//   staged : chunk-major, for j, for g, for l — the reference's pre_copy
//            (dataplane.hpp:245-261) when L == 1.
// The arithmetic is plan_block (front.cuh), shared with the fused front
// kernel; this standalone launch serves virtual mode, where every card's
// counts must be pushed before any card plans.
#include "front.cuh"

namespace monta {
namespace {

constexpr int kPlanSmemMax = 200 * 1024;

__global__ void __launch_bounds__(1024) k_plan(const PlanArgs a, int32_t* scratch, int use_smem) {
  extern __shared__ int smem[];
  if (!cta_wait(a.wait, a.err)) return;
  plan_block(a, plan_tables(use_smem ? smem : scratch, a.e, a.E, a.n));
}

}  // namespace

size_t plan_scratch_ints(int e, int E, int max_chunks) { return plan_smem_ints(e, E, max_chunks); }

bool plan_fits_smem(int e, int E, int n) { return plan_smem_ints(e, E, n) * 4 <= size_t(kPlanSmemMax); }

moe_status configure_plan() {
  MONTA_CUDA(cudaFuncSetAttribute(k_plan, cudaFuncAttributeMaxDynamicSharedMemorySize, kPlanSmemMax));
  return MOE_OK;
}

cudaError_t launch_plan_with_scratch(const PlanArgs& a, int32_t* scratch, cudaStream_t s) {
  const bool in_smem = plan_fits_smem(a.e, a.E, a.n);
  const size_t smem = in_smem ? plan_smem_ints(a.e, a.E, a.n) * 4 : 0;
  k_plan<<<1, 1024, smem, s>>>(a, scratch, in_smem ? 1 : 0);
  return cudaGetLastError();
}

}  // namespace monta

// Device-side pieces of the multi-card layer backward (moe_ctx_backward*,
// SURVEY.md §8(f) item 2).  The reference has no backward; these are the
// adjoints of its combine_unpermute (dataplane.hpp:293-347) routed through
// the forward's own exchanges:
//   row_meta     for every landed gradient row (expert card): the weight p
//                and slot s of the (source, position, expert) it came from,
//                read from the source card's routing over NVLink (any TP card
//                of the source node holds the same routing: the same-rho one);
//   scatter      the partial <g, y> over this card's column slice into slot
//                [(pos*k + s)*t + rho] of every TP card of the source node;
//   sum_parts    grad_probs[i, s] = sum over rho of those partials, in rho
//                order (deterministic; 0 for empty slots).
#include "engine.cuh"

namespace monta {
namespace {

template <class PT>
__global__ void k_row_meta(const int32_t* __restrict__ tags, const int64_t* __restrict__ recv_rows, int64_t cap,
                           int t, int rho, int k, const BwdPeers pe, PT* __restrict__ prow,
                           int32_t* __restrict__ rowpos, int32_t* __restrict__ rowslot, int32_t* err) {
  const int64_t rows = *recv_rows;
  for (int64_t r = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; r < cap; r += int64_t(gridDim.x) * blockDim.x) {
    if (r >= rows) {
      rowpos[r] = -1;  // no row: skipped by the combine-backward kernel
      continue;
    }
    const int4 tg = reinterpret_cast<const int4*>(tags)[r];  // {token_id, source_card, source_position, expert}
    const int q = tg.y + rho;                                 // same-rho card of the source node
    const int32_t* ex = pe.experts[q] + int64_t(tg.z) * k;
    int s = 0;
    while (s < k && ex[s] != tg.w) ++s;
    if (s == k) {
      atomicExch(err, int32_t(MOE_ERR_CORRUPT_ROUTING));
      rowpos[r] = -1;
      continue;
    }
    prow[r] = static_cast<const PT*>(pe.probs[q])[int64_t(tg.z) * k + s];
    rowpos[r] = int32_t(r);
    rowslot[r] = s;
  }
}

template <class PT>
__global__ void k_scatter_parts(const int32_t* __restrict__ tags, const int64_t* __restrict__ recv_rows, int t,
                                int rho, int k, const int32_t* __restrict__ rowslot, const PT* __restrict__ dot,
                                const BwdPeers pe) {
  const int64_t rows = *recv_rows;
  for (int64_t r = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; r < rows; r += int64_t(gridDim.x) * blockDim.x) {
    const int4 tg = reinterpret_cast<const int4*>(tags)[r];
    const int64_t at = (int64_t(tg.z) * k + rowslot[r]) * t + rho;
    const PT v = dot[r];
    for (int p = 0; p < t; ++p) static_cast<PT*>(pe.parts[tg.y + p])[at] = v;  // every TP card of the source node
  }
}

template <class PT>
__global__ void k_sum_parts(const PT* __restrict__ parts, const int32_t* __restrict__ experts, int64_t Tk, int t,
                            PT* __restrict__ gprobs) {
  for (int64_t q = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; q < Tk; q += int64_t(gridDim.x) * blockDim.x) {
    PT s = PT(0);
    if (experts[q] >= 0)
      for (int p = 0; p < t; ++p) s += parts[q * t + p];
    gprobs[q] = s;
  }
}

template <class PT>
__global__ void k_fill(PT* __restrict__ p, int64_t n, PT v) {
  for (int64_t q = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; q < n; q += int64_t(gridDim.x) * blockDim.x) p[q] = v;
}

int grid_of(int64_t n) {
  const int64_t g = (n + 255) / 256;
  return int(g < 1 ? 1 : (g > 4096 ? 4096 : g));
}

}  // namespace

cudaError_t launch_row_meta(int logit_dtype, const int32_t* tags, const int64_t* recv_rows, int64_t cap, int t,
                            int rho, int k, const BwdPeers& pe, void* prow, int32_t* rowpos, int32_t* rowslot,
                            int32_t* err, cudaStream_t s) {
  if (logit_dtype == MOE_F64)
    k_row_meta<double><<<grid_of(cap), 256, 0, s>>>(tags, recv_rows, cap, t, rho, k, pe, static_cast<double*>(prow),
                                                    rowpos, rowslot, err);
  else
    k_row_meta<float><<<grid_of(cap), 256, 0, s>>>(tags, recv_rows, cap, t, rho, k, pe, static_cast<float*>(prow),
                                                   rowpos, rowslot, err);
  return cudaGetLastError();
}

cudaError_t launch_scatter_parts(int logit_dtype, const int32_t* tags, const int64_t* recv_rows, int64_t cap, int t,
                                 int rho, int k, const int32_t* rowslot, const void* dot, const BwdPeers& pe,
                                 cudaStream_t s) {
  if (logit_dtype == MOE_F64)
    k_scatter_parts<double><<<grid_of(cap), 256, 0, s>>>(tags, recv_rows, t, rho, k, rowslot,
                                                         static_cast<const double*>(dot), pe);
  else
    k_scatter_parts<float><<<grid_of(cap), 256, 0, s>>>(tags, recv_rows, t, rho, k, rowslot,
                                                        static_cast<const float*>(dot), pe);
  return cudaGetLastError();
}

cudaError_t launch_sum_parts(int logit_dtype, const void* parts, const int32_t* experts, int64_t Tk, int t,
                             void* gprobs, cudaStream_t s) {
  if (logit_dtype == MOE_F64)
    k_sum_parts<double><<<grid_of(Tk), 256, 0, s>>>(static_cast<const double*>(parts), experts, Tk, t,
                                                    static_cast<double*>(gprobs));
  else
    k_sum_parts<float><<<grid_of(Tk), 256, 0, s>>>(static_cast<const float*>(parts), experts, Tk, t,
                                                   static_cast<float*>(gprobs));
  return cudaGetLastError();
}

cudaError_t launch_fill_ones(int logit_dtype, void* p, int64_t n, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  if (logit_dtype == MOE_F64)
    k_fill<double><<<grid_of(n), 256, 0, s>>>(static_cast<double*>(p), n, 1.0);
  else
    k_fill<float><<<grid_of(n), 256, 0, s>>>(static_cast<float*>(p), n, 1.0f);
  return cudaGetLastError();
}

}  // namespace monta

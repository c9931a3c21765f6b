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
// Outputs: one segment list per (phase, chunk) for this card, the local
// permuted->final row delta for the un-permute, and the received row count.
#include "engine.cuh"

namespace monta {
namespace {

struct Tables {
  int32_t* tot;       // [e][E]
  int32_t* eo;        // [e][E+1]     sender-permuted expert offsets
  int32_t* cum;       // [e][n+1][E]  rows of (g, x) in chunks < j
  int32_t* fin;       // [xg][l][g]   final segment base
  int32_t* pre;       // [xg][j][g][l] staged segment base
};

__device__ __forceinline__ SegList* list_at(const PlanArgs& a, int phase, int j) {
  char* base = reinterpret_cast<char*>(a.lists);
  return reinterpret_cast<SegList*>(base + (size_t(phase) * a.max_chunks + j) *
                                               seglist_bytes(a.seg_cap));
}

__global__ void __launch_bounds__(1024) k_plan(const PlanArgs a, Tables tb) {
  if (!cta_wait(a.wait, a.err)) return;
  const int e = a.e, E = a.E, L = a.L, n = a.n, t = a.t;
  const int tid = threadIdx.x, nth = blockDim.x;
  auto CT = [&](int g, int j, int x) {
    return a.count_table[(int64_t(g) * a.max_chunks + j) * E + x];
  };
  // 1. totals and chunk prefixes per (g, x)
  for (int q = tid; q < e * E; q += nth) {
    const int g = q / E, x = q % E;
    int run = 0;
    for (int j = 0; j < n; ++j) {
      tb.cum[(int64_t(g) * (n + 1) + j) * E + x] = run;
      run += CT(g, j, x);
    }
    tb.cum[(int64_t(g) * (n + 1) + n) * E + x] = run;
    tb.tot[g * E + x] = run;
  }
  __syncthreads();
  // 2. sender-permuted expert offsets per node
  for (int g = tid; g < e; g += nth) {
    int run = 0;
    for (int x = 0; x < E; ++x) {
      tb.eo[g * (E + 1) + x] = run;
      run += tb.tot[g * E + x];
    }
    tb.eo[g * (E + 1) + E] = run;
  }
  // 3. final layout bases per destination node: (l, g) order
  for (int xg = tid; xg < e; xg += nth) {
    int run = 0;
    for (int l = 0; l < L; ++l)
      for (int g = 0; g < e; ++g) {
        tb.fin[(xg * L + l) * e + g] = run;
        run += tb.tot[g * E + xg * L + l];
      }
    if (xg == a.node) *a.recv_rows = run;
  }
  // 4. staged bases: within-chunk prefix over (g, l), then across chunks.
  for (int q = tid; q < e * n; q += nth) {
    const int xg = q / n, j = q % n;
    int run = 0;
    for (int g = 0; g < e; ++g)
      for (int l = 0; l < L; ++l) {
        tb.pre[((int64_t(xg) * n + j) * e + g) * L + l] = run;
        run += CT(g, j, xg * L + l);
      }
    // stash chunk size in the slot past the end of this (xg, j) block? no —
    // recompute below.
  }
  __syncthreads();
  for (int xg = tid; xg < e; xg += nth) {
    int run = 0;
    for (int j = 0; j < n; ++j) {
      int chunk_rows = 0;
      for (int g = 0; g < e; ++g)
        for (int l = 0; l < L; ++l) chunk_rows += CT(g, j, xg * L + l);
      for (int q = 0; q < e * L; ++q) tb.pre[(int64_t(xg) * n + j) * e * L + q] += run;
      run += chunk_rows;
    }
  }
  __syncthreads();
  // 5. local delta for the un-permute (own node's experts)
  for (int l = tid; l < L; l += nth) {
    const int x = a.node * L + l;
    a.local_delta[x] = tb.fin[(a.node * L + l) * e + a.node] - tb.eo[a.node * (E + 1) + x];
  }
  // 6. segment lists, one thread per (phase, chunk)
  const bool dedup = a.level != MOE_BASELINE && t > 1;
  const int full = int(a.row_bytes);
  const int slice = int(a.row_bytes / t);
  const int slice_off = a.rho * slice;
  const int me = a.node * t + a.rho;
  for (int q = tid; q < kNumPhases * n; q += nth) {
    const int phase = q / n, j = q % n;
    SegList* lst = list_at(a, phase, j);
    int ns = 0;
    int64_t rowsum = 0;
    auto push = [&](int64_t src, int64_t dst_row, int rows, int dst, int off, int width, int x) {
      if (rows <= 0) return;
      Seg s;
      s.row_begin = rowsum;
      s.src_row = src;
      s.dst_row = dst_row;
      s.rows = rows;
      s.dst = dst;
      s.col_off = off;
      s.width = width;
      s.expert = x;
      s.pad = 0;
      lst->segs[ns++] = s;
      rowsum += rows;
    };
    const int g0 = a.node;
    if (phase == kPhaseAA) {
      for (int x = 0; x < E; ++x) {
        const int xg = x / L, l = x % L;
        const int rows = CT(g0, j, x);
        const int64_t src = tb.eo[g0 * (E + 1) + x] + tb.cum[(int64_t(g0) * (n + 1) + j) * E + x];
        const int64_t dst_row =
            a.landing == MOE_LAND_STAGED
                ? int64_t(tb.pre[((int64_t(xg) * n + j) * e + g0) * L + l])
                : int64_t(tb.fin[(xg * L + l) * e + g0]) + tb.cum[(int64_t(g0) * (n + 1) + j) * E + x];
        const bool remote_slice = dedup && xg != g0;
        push(src, dst_row, rows, xg * t + a.rho, remote_slice ? slice_off : 0,
             remote_slice ? slice : full, x);
      }
    } else if (phase == kPhaseAG) {
      if (dedup) {
        for (int g = 0; g < e; ++g) {
          if (g == g0) continue;
          for (int l = 0; l < L; ++l) {
            const int x = g0 * L + l;
            const int rows = CT(g, j, x);
            const int64_t row =
                a.landing == MOE_LAND_STAGED
                    ? int64_t(tb.pre[((int64_t(g0) * n + j) * e + g) * L + l])
                    : int64_t(tb.fin[(g0 * L + l) * e + g]) + tb.cum[(int64_t(g) * (n + 1) + j) * E + x];
            push(row, row, rows, -1, slice_off, slice, x);
          }
        }
      }
    } else if (phase == kPhaseD2D) {
      if (a.landing == MOE_LAND_STAGED) {
        for (int g = 0; g < e; ++g)
          for (int l = 0; l < L; ++l) {
            const int x = g0 * L + l;
            const int rows = CT(g, j, x);
            push(tb.pre[((int64_t(g0) * n + j) * e + g) * L + l],
                 int64_t(tb.fin[(g0 * L + l) * e + g]) + tb.cum[(int64_t(g) * (n + 1) + j) * E + x],
                 rows, me, 0, full, x);
          }
      }
    } else {  // kPhaseCAA: reverse exchange of the expert outputs of this node
      for (int g = 0; g < e; ++g) {
        if (g == g0) continue;
        for (int l = 0; l < L; ++l) {
          const int x = g0 * L + l;
          const int rows = CT(g, j, x);
          const int64_t c = tb.cum[(int64_t(g) * (n + 1) + j) * E + x];
          push(int64_t(tb.fin[(g0 * L + l) * e + g]) + c, int64_t(tb.eo[g * (E + 1) + x]) + c, rows,
               g * t + a.rho, dedup ? slice_off : 0, dedup ? slice : full, x);
        }
      }
    }
    lst->nseg = ns;
    lst->total_rows = rowsum;
  }
}

}  // namespace

size_t plan_scratch_ints(int e, int E, int max_chunks) {
  const int L = E / e;
  return size_t(e) * E + size_t(e) * (E + 1) + size_t(e) * (max_chunks + 1) * E +
         size_t(e) * L * e + size_t(e) * max_chunks * e * L;
}

cudaError_t launch_plan_with_scratch(const PlanArgs& a, int32_t* scratch, cudaStream_t s) {
  Tables tb;
  const int e = a.e, E = a.E, L = a.L;
  tb.tot = scratch;
  tb.eo = tb.tot + size_t(e) * E;
  tb.cum = tb.eo + size_t(e) * (E + 1);
  tb.fin = tb.cum + size_t(e) * (a.max_chunks + 1) * E;
  tb.pre = tb.fin + size_t(e) * L * e;
  k_plan<<<1, 1024, 0, s>>>(a, tb);
  return cudaGetLastError();
}

}  // namespace monta

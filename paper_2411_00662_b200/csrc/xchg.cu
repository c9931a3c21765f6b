// Persistent, role-specialised chunked dispatch — MoNTA's O1/O2/O3 pipeline
// (dataplane.hpp:187-283; schedule of pipesim.hpp:58-83) in ONE cooperative
// launch per card.
//
// CTA roles (disjoint CTA ranges, all co-resident):
//   AA   the fused permute + cross-node AllToAll (this rank's 1/t slice under
//        dedup, straight into the peer's final/staged rows), chunk after
//        chunk without waiting for anything; the last CTA of chunk s releases
//        AA[s] at every EP peer;
//   AG   (chunked runs, r_ag > 0) for each chunk j: wait for every remote
//        AA[j], forward this rank's slice of those rows to the t-1 TP peers
//        (AllGather; releases AG[j]); under O2 with staged landing the
//        reorder of chunk j follows (the reference simulator queues the D2D
//        on the AllGather stream, pipesim.hpp:77-79).  The AllGather of chunk
//        j overlaps the AllToAll of chunks > j, which is MoNTA's pipeline.
//        With one chunk (r_ag == 0) there is nothing to overlap and the AA
//        CTAs run the AllGather themselves after the AllToAll, so every leg
//        gets every NVLink CTA;
//   LOC  own-node rows, full width, local HBM copy; releases a local chunk
//        flag (read by the reorder);
//   D2D  (O3, staged) for j: wait AA[j] remote, AG[j] from TP peers and the
//        local chunk flag, then reorder chunk j staged -> final.
// A chunk therefore costs a flag round trip (~µs), not kernel launches.
// Before exiting, CTA 0 waits until every peer contribution to this card
// has landed, so kernel completion == dispatch completion.
#include "copy.cuh"

namespace monta {
namespace {

constexpr int kXchgThreads = 256;

__device__ __forceinline__ int sig_of(const XchgArgs& a, int ps, int j) {
  return kSigChunkBase + ps * a.max_chunks + j;
}
__device__ __forceinline__ uint64_t* flag(const XchgArgs& a, int owner, int sig, int sender) {
  return a.flags[owner] + size_t(sig) * kMaxCards + sender;
}
__device__ __forceinline__ SegList* list_at(const XchgArgs& a, int phase, int j) {
  char* base = reinterpret_cast<char*>(a.lists);
  return reinterpret_cast<SegList*>(base + (size_t(phase) * a.max_chunks + j) * seglist_bytes(a.seg_cap));
}

// Reorder (staged -> final) on this card: source pre, destination slot of
// this card in the d2d tables.
__device__ __forceinline__ CopyView d2d_view(const XchgArgs& a) {
  CopyView d = view_of(a.cp);
  d.gather = nullptr;
  d.synth_tags = 0;
  d.src = a.pre_local;
  d.src_tags = a.pre_tags_local;
  d.dst = a.d2d_dst;
  d.dst_tags = a.d2d_dst_tags;
  return d;
}

template <int V>
__global__ void __launch_bounds__(kXchgThreads, 2) k_xchg(const __grid_constant__ XchgArgs a) {
  __shared__ int s_ok;
  __shared__ unsigned long long s_epoch;
  if (threadIdx.x == 0) {
    s_epoch = *a.epoch_ptr;
    if (a.dbg && blockIdx.x == 0) a.dbg[0] = globaltimer();
  }
  __syncthreads();
  const uint64_t epoch = s_epoch;
  const int b = blockIdx.x;
  const int n = a.n;
  // roles: AA = [0, r_aa); AG = [r_aa, r_aa + r_ag); LOC; D2D after
  const int ag0 = a.r_aa, loc0 = a.r_aa + a.r_ag, d2d0 = loc0 + a.r_aal;
  CopyView g = view_of(a.cp);  // AllGather view: this card's landed rows -> TP peers
  g.gather = nullptr;
  g.synth_tags = 0;
  g.src = a.staged ? a.pre_local : a.recv_local;
  g.src_tags = a.staged ? a.pre_tags_local : a.recv_tags_local;
  g.dst_mask = a.ag_mask;
  g.dst = a.ag_dst;
  g.dst_tags = a.ag_dst_tags;
  // AllGather of chunk j by `ctas` CTAs (c = this CTA's index among them)
  auto gather = [&](int j, int c, int ctas) -> bool {
    if (threadIdx.x == 0) {
      s_ok = 1;
      for (int x = 0; x < a.e && s_ok; ++x)
        if (x != a.node) s_ok = wait_flag(flag(a, a.me, sig_of(a, kPsAA, j), x * a.t + a.rho), epoch, a.err);
    }
    __syncthreads();
    if (!s_ok) return false;
    trace_start(a.trace, 2, a.max_chunks, j);
    copy_items<V, true, false>(g, list_at(a, kPhaseAG, j), a.cpr_slice, c, ctas);
    chunk_done(a.counters + (2 * a.max_chunks + j) * 17, ctas, c, [&] {
      trace_end(a.trace, 2, a.max_chunks, j);
      for (int r = 0; r < a.t; ++r)
        if (r != a.rho) st_release_sys(flag(a, a.node * a.t + r, sig_of(a, kPsAG, j), a.me), epoch);
    });
    if (a.d2d_in_ag) {  // O2 staged: the reorder queued behind the gather
      if (threadIdx.x == 0) {
        s_ok = wait_flag(a.local_flags + j, epoch, a.err);
        for (int r = 0; r < a.t && s_ok; ++r)
          if (r != a.rho) s_ok = wait_flag(flag(a, a.me, sig_of(a, kPsAG, j), a.node * a.t + r), epoch, a.err);
      }
      __syncthreads();
      if (!s_ok) return false;
      copy_items<V, true, false>(d2d_view(a), list_at(a, kPhaseD2D, j), a.cpr_full, c, ctas);
    }
    return true;
  };

  if (b < loc0) {  // ---------------- AA and AG roles (one loop, one gather site)
    const bool is_aa = b < ag0;
    const int c = is_aa ? b : b - ag0;
    const int ctas = is_aa ? a.r_aa : a.r_ag;
    // the AA CTAs gather too when there is no AG role (chunk s-1 after AA(s))
    const bool do_gather = a.dedup && (is_aa ? a.r_ag == 0 : true);
    const CopyView aa = view_of(a.cp);
    for (int s = 0; s <= n; ++s) {
      if (is_aa && s < n && a.e > 1) {
        trace_start(a.trace, 0, a.max_chunks, s);
        const unsigned long long t0 = globaltimer();
        copy_items<V, false, false>(aa, list_at(a, kPhaseAA, s), a.cpr_full, c, a.r_aa);
        pace_list(list_at(a, kPhaseAA, s), t0, a.cp.pace_bpus);
        chunk_done(a.counters + (0 * a.max_chunks + s) * 17, a.r_aa, c, [&] {
          trace_end(a.trace, 0, a.max_chunks, s);
          for (int x = 0; x < a.e; ++x)
            if (x != a.node) st_release_sys(flag(a, x * a.t + a.rho, sig_of(a, kPsAA, s), a.me), epoch);
        });
      }
      const int j = is_aa ? s - 1 : s;
      if (do_gather && j >= 0 && j < n && !gather(j, c, ctas)) return;
    }
  } else if (b < d2d0) {  // ---------------- LOC: own-node legs
    const int c = b - loc0;
    for (int j = 0; j < n; ++j) {
      trace_start(a.trace, 1, a.max_chunks, j);
      copy_items<V, false, false>(view_of(a.cp), list_at(a, kPhaseAAL, j), a.cpr_full, c, a.r_aal);
      chunk_done(a.counters + (1 * a.max_chunks + j) * 17, a.r_aal, c, [&] {
        trace_end(a.trace, 1, a.max_chunks, j);
        st_release_sys(a.local_flags + j, epoch);
      });
    }
  } else {  // ---------------- D2D (O3, staged)
    const int c = b - d2d0;
    const CopyView d = d2d_view(a);
    for (int j = 0; j < n; ++j) {
      if (threadIdx.x == 0) {
        s_ok = wait_flag(a.local_flags + j, epoch, a.err);
        for (int x = 0; x < a.e && s_ok; ++x)
          if (x != a.node) s_ok = wait_flag(flag(a, a.me, sig_of(a, kPsAA, j), x * a.t + a.rho), epoch, a.err);
        if (a.dedup)
          for (int r = 0; r < a.t && s_ok; ++r)
            if (r != a.rho) s_ok = wait_flag(flag(a, a.me, sig_of(a, kPsAG, j), a.node * a.t + r), epoch, a.err);
      }
      __syncthreads();
      if (!s_ok) return;
      trace_start(a.trace, 3, a.max_chunks, j);
      copy_items<V, true, false>(d, list_at(a, kPhaseD2D, j), a.cpr_full, c, a.r_d2d);
      chunk_done(a.counters + (3 * a.max_chunks + j) * 17, a.r_d2d, c, [&] { trace_end(a.trace, 3, a.max_chunks, j); });
    }
  }
  // ---------------- tail: CTA 0 waits for every contribution to this card
  if (b == 0 && threadIdx.x == 0 && !a.staged) {
    bool ok = true;
    for (int j = 0; j < n && ok; ++j) {
      if (a.dedup) {
        for (int r = 0; r < a.t && ok; ++r)
          if (r != a.rho) ok = wait_flag(flag(a, a.me, sig_of(a, kPsAG, j), a.node * a.t + r), epoch, a.err);
      } else {
        for (int x = 0; x < a.e && ok; ++x)
          if (x != a.node) ok = wait_flag(flag(a, a.me, sig_of(a, kPsAA, j), x * a.t + a.rho), epoch, a.err);
      }
    }
    if (a.dbg) a.dbg[1] = globaltimer();
  }
}

}  // namespace

int xchg_max_ctas(int vec) {
  int dev = 0, sms = 0, per_sm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  switch (vec) {
    case 16: cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_xchg<16>, kXchgThreads, 0); break;
    case 8: cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_xchg<8>, kXchgThreads, 0); break;
    case 4: cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_xchg<4>, kXchgThreads, 0); break;
    default: return 0;
  }
  return per_sm * sms;
}

cudaError_t launch_xchg(const XchgArgs& a, int vec, cudaStream_t s) {
  const int grid = a.r_aa + a.r_ag + a.r_aal + a.r_d2d;
  void* args[] = {const_cast<XchgArgs*>(&a)};
  switch (vec) {
    case 16: return cudaLaunchCooperativeKernel((const void*)k_xchg<16>, dim3(grid), dim3(kXchgThreads), args, 0, s);
    case 8: return cudaLaunchCooperativeKernel((const void*)k_xchg<8>, dim3(grid), dim3(kXchgThreads), args, 0, s);
    case 4: return cudaLaunchCooperativeKernel((const void*)k_xchg<4>, dim3(grid), dim3(kXchgThreads), args, 0, s);
  }
  return cudaErrorInvalidValue;
}

}  // namespace monta

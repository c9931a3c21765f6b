// Device-side building blocks of the dispatch front end, shared by the
// standalone kernels (router.cu, index.cu, plan.cu) and the fused front
// kernel (front.cu):
//   route_tokens  — top-k gating of the tokens owned by this CTA
//                   (dataplane::route_topk, dataplane.hpp:72-106);
//   index_block   — one CTA's stable counting sort of the (token, slot)
//                   pairs (dataplane::permute, dataplane.hpp:118-140) plus
//                   per-chunk counts (dataplane.hpp:224-240);
//   plan_block    — counts -> every offset / segment list of the exchange.
#pragma once

#include "engine.cuh"

namespace monta {

template <class T> __device__ __forceinline__ T dev_exp(T x);
template <> __device__ __forceinline__ float dev_exp<float>(float x) { return expf(x); }
template <> __device__ __forceinline__ double dev_exp<double>(double x) { return exp(x); }

template <class T> __device__ __forceinline__ T neg_inf();
template <> __device__ __forceinline__ float neg_inf<float>() { return -INFINITY; }
template <> __device__ __forceinline__ double neg_inf<double>() { return -(double)INFINITY; }

// ---------------------------------------------------------------------------
// Router: G lanes per token (G = next pow2 >= E, <= 32), PER elements per
// lane.  Token index = global sub-warp group id.  Softmax in T precision;
// k rounds of group argmax over RAW scores, ties -> lower index; experts
// written ascending, probs = softmax values of the selected experts.
template <class T, int G, int PER>
__device__ __forceinline__ void route_tokens(const T* __restrict__ logits, int64_t T_tokens, int E, int k,
                                             int32_t* __restrict__ experts, T* __restrict__ probs,
                                             int64_t token, int* s_exp = nullptr, int64_t s_base = 0) {
  const int lane = threadIdx.x & (kWarp - 1);
  const int sub = lane % G;
  const bool active = token < T_tokens;
  const unsigned gmask = (G == 32) ? 0xffffffffu : (((1u << G) - 1u) << ((lane / G) * G));
  constexpr unsigned kNone = 0x7fffffff;
  T v[PER];
  const T* row = logits + (active ? token : 0) * int64_t(E);
#pragma unroll
  for (int m = 0; m < PER; ++m) {
    const int x = sub + m * G;
    v[m] = (active && x < E) ? row[x] : neg_inf<T>();
  }
  if constexpr (sizeof(T) == 4 && G == 32) {
    // fp32 scores, whole-warp groups (E > 16).  Each entry's order-preserving
    // 32-bit key is computed once (-0.0 canonicalised to +0.0 first: the
    // reference compares values, scores[l] > scores[r] at dataplane.hpp:97-98,
    // for which the two zeros tie and the lower index wins; entries past E get
    // key 0, below every real score).  The row max is one redux.sync over the
    // keys (it differs from a float max only in the sign of a zero maximum,
    // which leaves every exp(v - max) unchanged).  Round s: the lane's best
    // key (strict > keeps its lower index on ties), the warp's max key, the
    // lowest expert index holding it (redux.sync max/min), the owner zeroes
    // that entry and lane s keeps {winner, exp}; the k winners then leave in
    // ascending expert order (rank by k shuffles) with probs = exp / sum.
    unsigned u[PER];
    unsigned lmax = 0u;
#pragma unroll
    for (int m = 0; m < PER; ++m) {
      const int x = sub + m * G;
      unsigned b = __float_as_uint(float(v[m]));
      b = (b == 0x80000000u) ? 0u : b;
      u[m] = x < E ? ((b & 0x80000000u) ? ~b : (b | 0x80000000u)) : 0u;
      lmax = u[m] > lmax ? u[m] : lmax;
    }
    const unsigned mkey = __reduce_max_sync(0xffffffffu, lmax);
    const T mx = T(__uint_as_float((mkey & 0x80000000u) ? (mkey & 0x7fffffffu) : ~mkey));
    T ex[PER];
    T sum = T(0);
#pragma unroll
    for (int m = 0; m < PER; ++m) {
      ex[m] = dev_exp<T>(v[m] - mx);  // entries past E: v = -inf, exp = 0 (as the masked form)
      sum += ex[m];
    }
#pragma unroll
    for (int off = G / 2; off > 0; off >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, off, G);
    int my_w = -1;
    T my_e = T(0);
    for (int s = 0; s < k; ++s) {
      unsigned key = 0u, bm = 0u;
#pragma unroll
      for (int m = 0; m < PER; ++m)
        if (u[m] > key) {
          key = u[m];
          bm = unsigned(m);
        }
      const unsigned bi = key ? unsigned(sub) + bm * G : 0xffffffffu;
      const unsigned mk = __reduce_max_sync(0xffffffffu, key);
      const unsigned wi = __reduce_min_sync(0xffffffffu, key == mk ? bi : 0xffffffffu);  // k <= E: exists
      const unsigned mw = wi / G, owner = wi % G;
      T e = T(0);
#pragma unroll
      for (int m = 0; m < PER; ++m)
        if (unsigned(m) == mw) {
          e = ex[m];
          if (owner == unsigned(sub)) u[m] = 0u;
        }
      e = __shfl_sync(0xffffffffu, e, int(owner));
      if (lane == s) {
        my_w = int(wi);
        my_e = e;
      }
    }
    int slot = 0;
    for (int s = 0; s < k; ++s) slot += __shfl_sync(0xffffffffu, my_w, s) < my_w ? 1 : 0;
    if (active && lane < k) {
      experts[token * k + slot] = my_w;
      probs[token * k + slot] = my_e / sum;
      if (s_exp) s_exp[(token - s_base) * k + slot] = my_w;  // the tile's mirror in shared memory
    }
    return;
  }
  T mx = v[0];
#pragma unroll
  for (int m = 1; m < PER; ++m) mx = v[m] > mx ? v[m] : mx;
#pragma unroll
  for (int off = G / 2; off > 0; off >>= 1) {
    const T o = __shfl_xor_sync(gmask, mx, off, G);
    mx = o > mx ? o : mx;
  }
  T ex[PER];
  T sum = T(0);
#pragma unroll
  for (int m = 0; m < PER; ++m) {
    const int x = sub + m * G;
    ex[m] = (x < E) ? dev_exp<T>(v[m] - mx) : T(0);
    sum += ex[m];
  }
#pragma unroll
  for (int off = G / 2; off > 0; off >>= 1) sum += __shfl_xor_sync(gmask, sum, off, G);
  if constexpr (sizeof(T) == 4) {
    // fp32 scores: each entry's order-preserving 32-bit key is computed once
    // (-0.0 canonicalised to +0.0 first: the reference compares values,
    // scores[l] > scores[r] at dataplane.hpp:97-98, for which the two zeros
    // tie and the lower index wins); a taken entry's key drops to 0 (every
    // real score maps above it).  Per round: the lane's best key (strict >
    // keeps its lower index on ties), then the group argmax — one redux.sync
    // max/min pair for whole warps, a packed 64-bit {key, ~index} shuffle tree
    // for sub-warp groups; ties go to the lower expert index in both.
    unsigned u[PER];
#pragma unroll
    for (int m = 0; m < PER; ++m) {
      const int x = sub + m * G;
      unsigned b = __float_as_uint(float(v[m]));
      b = (b == 0x80000000u) ? 0u : b;
      u[m] = x < E ? ((b & 0x80000000u) ? ~b : (b | 0x80000000u)) : 0u;
    }
    unsigned sel = 0;  // bit m: entry m (expert sub + m*G) selected
    for (int s = 0; s < k; ++s) {
      unsigned key = 0u, bm = 0u;
#pragma unroll
      for (int m = 0; m < PER; ++m)
        if (u[m] > key) {
          key = u[m];
          bm = unsigned(m);
        }
      const unsigned bi = key ? unsigned(sub) + bm * G : 0xffffffffu;
      unsigned wi;
      if constexpr (G == 32) {
        const unsigned mk = __reduce_max_sync(0xffffffffu, key);
        wi = __reduce_min_sync(0xffffffffu, key == mk ? bi : 0xffffffffu);
      } else {
        unsigned long long pk = (static_cast<unsigned long long>(key) << 32) | (0xffffffffu - bi);
#pragma unroll
        for (int off = G / 2; off > 0; off >>= 1) {
          const unsigned long long o = __shfl_xor_sync(gmask, pk, off, G);
          pk = o > pk ? o : pk;
        }
        wi = 0xffffffffu - unsigned(pk & 0xffffffffull);
      }
      if (wi != 0xffffffffu && int(wi % G) == sub) {
        const unsigned mw = wi / G;
#pragma unroll
        for (int m = 0; m < PER; ++m)
          if (unsigned(m) == mw) u[m] = 0u;
        sel |= 1u << mw;
      }
    }
    // experts leave in ascending order: entry (lane, m)'s slot is the number
    // of selected entries of the group with a smaller index (ballots by m)
    const int gshift = (lane / G) * G;
    const unsigned lt = (1u << sub) - 1u;
    int before = 0;
#pragma unroll
    for (int m = 0; m < PER; ++m) {
      const unsigned bal = __ballot_sync(0xffffffffu, (sel >> m) & 1u);
      const unsigned gb = G == 32 ? bal : ((bal >> gshift) & ((1u << G) - 1u));
      if (active && ((sel >> m) & 1u)) {
        const int slot = before + __popc(gb & lt);
        const int x = sub + m * G;
        experts[token * k + slot] = x;
        probs[token * k + slot] = ex[m] / sum;
        if (s_exp) s_exp[(token - s_base) * k + slot] = x;  // the tile's mirror in shared memory
      }
      before += __popc(gb);
    }
  } else {
    unsigned taken = 0;
    int my_sel = -1;
    T my_soft = T(0);
    for (int s = 0; s < k; ++s) {
      T bv = neg_inf<T>();
      int bi = int(kNone);
      T bs = T(0);
#pragma unroll
      for (int m = 0; m < PER; ++m) {
        const int x = sub + m * G;
        if (x < E && !((taken >> m) & 1u)) {
          if (bi == int(kNone) || v[m] > bv || (v[m] == bv && x < bi)) {
            bv = v[m];
            bi = x;
            bs = ex[m];
          }
        }
      }
#pragma unroll
      for (int off = G / 2; off > 0; off >>= 1) {
        const T ov = __shfl_xor_sync(gmask, bv, off, G);
        const int oi = __shfl_xor_sync(gmask, bi, off, G);
        const T os = __shfl_xor_sync(gmask, bs, off, G);
        const bool take = (oi != int(kNone)) && (bi == int(kNone) || ov > bv || (ov == bv && oi < bi));
        if (take) {
          bv = ov;
          bi = oi;
          bs = os;
        }
      }
      if (bi != int(kNone) && (bi % G) == sub) taken |= 1u << (bi / G);
      if (sub == s) {
        my_sel = bi;
        my_soft = bs / sum;
      }
    }
    int rank = 0;
    for (int s = 0; s < k; ++s) {
      const int other = __shfl_sync(gmask, my_sel, (lane / G) * G + s, kWarp);
      if (other < my_sel) ++rank;
    }
    if (active && sub < k) {
      experts[token * k + rank] = my_sel;
      probs[token * k + rank] = my_soft;
      if (s_exp) s_exp[(token - s_base) * k + rank] = my_sel;  // the tile's mirror in shared memory
    }
  }
}

// Two tokens per warp (fp32 scores, whole-warp groups): the arithmetic of
// route_tokens for token a and token b, interleaved so the dependent
// reduction chains of the two overlap (the router is issue-latency bound:
// ~65 % issue slots busy with one token per warp).  Bit-identical per token.
template <int PER>
__device__ __forceinline__ void route_tokens_w32x2(const float* __restrict__ logits, int64_t T_tokens, int E, int k,
                                                   int32_t* __restrict__ experts, float* __restrict__ probs,
                                                   int64_t tok_a, int64_t tok_b, int* s_exp, int64_t s_base) {
  constexpr int G = 32;
  const int lane = threadIdx.x & (kWarp - 1);
  const int64_t tok[2] = {tok_a, tok_b};
  bool active[2];
  unsigned u[2][PER];
  float ex[2][PER];
  float sum[2];
  float vv[2][PER];
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    active[q] = tok[q] < T_tokens;
    const float* row = logits + (active[q] ? tok[q] : 0) * int64_t(E);
#pragma unroll
    for (int m = 0; m < PER; ++m) {
      const int x = lane + m * G;
      vv[q][m] = (active[q] && x < E) ? row[x] : -INFINITY;
    }
  }
  unsigned lmax[2] = {0u, 0u};
#pragma unroll
  for (int q = 0; q < 2; ++q)
#pragma unroll
    for (int m = 0; m < PER; ++m) {
      const int x = lane + m * G;
      unsigned b = __float_as_uint(vv[q][m]);
      b = (b == 0x80000000u) ? 0u : b;
      u[q][m] = x < E ? ((b & 0x80000000u) ? ~b : (b | 0x80000000u)) : 0u;
      lmax[q] = u[q][m] > lmax[q] ? u[q][m] : lmax[q];
    }
  float mx[2];
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    const unsigned mkey = __reduce_max_sync(0xffffffffu, lmax[q]);
    mx[q] = __uint_as_float((mkey & 0x80000000u) ? (mkey & 0x7fffffffu) : ~mkey);
  }
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    sum[q] = 0.f;
#pragma unroll
    for (int m = 0; m < PER; ++m) {
      ex[q][m] = dev_exp<float>(vv[q][m] - mx[q]);
      sum[q] += ex[q][m];
    }
  }
#pragma unroll
  for (int off = G / 2; off > 0; off >>= 1) {
    sum[0] += __shfl_xor_sync(0xffffffffu, sum[0], off, G);
    sum[1] += __shfl_xor_sync(0xffffffffu, sum[1], off, G);
  }
  int my_w[2] = {-1, -1};
  float my_e[2] = {0.f, 0.f};
  for (int s = 0; s < k; ++s) {
    unsigned key[2], bm[2];
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      key[q] = 0u;
      bm[q] = 0u;
#pragma unroll
      for (int m = 0; m < PER; ++m)
        if (u[q][m] > key[q]) {
          key[q] = u[q][m];
          bm[q] = unsigned(m);
        }
    }
    unsigned wi[2];
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const unsigned bi = key[q] ? unsigned(lane) + bm[q] * G : 0xffffffffu;
      const unsigned mk = __reduce_max_sync(0xffffffffu, key[q]);
      wi[q] = __reduce_min_sync(0xffffffffu, key[q] == mk ? bi : 0xffffffffu);
    }
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const unsigned mw = wi[q] / G, owner = wi[q] % G;
      float e = 0.f;
#pragma unroll
      for (int m = 0; m < PER; ++m)
        if (unsigned(m) == mw) {
          e = ex[q][m];
          if (owner == unsigned(lane)) u[q][m] = 0u;
        }
      e = __shfl_sync(0xffffffffu, e, int(owner));
      if (lane == s) {
        my_w[q] = int(wi[q]);
        my_e[q] = e;
      }
    }
  }
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    int slot = 0;
    for (int s = 0; s < k; ++s) slot += __shfl_sync(0xffffffffu, my_w[q], s) < my_w[q] ? 1 : 0;
    if (active[q] && lane < k) {
      experts[tok[q] * k + slot] = my_w[q];
      probs[tok[q] * k + slot] = my_e[q] / sum[q];
      if (s_exp) s_exp[(tok[q] - s_base) * k + slot] = my_w[q];
    }
  }
}

// ---------------------------------------------------------------------------
// Index build by one CTA (any warp count).  smem layout (ints):
//   hist [nw][E] | offs [E+1] | ccount [n][E] (when count_in_smem)
// Loads of `experts` use the L2-coherent path (.cg): in the fused kernel the
// router CTAs of the same launch wrote them.
__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}


__device__ __forceinline__ void index_block(const int32_t* experts, int64_t T, int k, int E, int n,
                                            int32_t* __restrict__ perm_src, int32_t* __restrict__ expert_of,
                                            int32_t* __restrict__ slot_pos, int32_t* __restrict__ counts,
                                            int32_t* __restrict__ expert_offsets, int32_t* __restrict__ err,
                                            int* smem, bool count_in_smem) {
  constexpr int kUnroll = 8;
  const int nw = blockDim.x >> 5;
  int* hist = smem;
  int* offs = smem + nw * E;
  int* ccount = count_in_smem ? offs + E + 1 : counts;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int64_t R = T * k;
  const int64_t ct = T / n;
  const int64_t per_warp = ((R + nw - 1) / nw + 31) / 32 * 32;
  const int64_t begin = int64_t(w) * per_warp;
  const int64_t end = begin + per_warp < R ? begin + per_warp : R;
  for (int i = tid; i < nw * E + E + 1; i += blockDim.x) smem[i] = 0;
  for (int i = tid; i < n * E; i += blockDim.x) ccount[i] = 0;
  __syncthreads();
  int* my_hist = hist + w * E;
  for (int64_t base = begin; base < end; base += 32 * kUnroll) {
    int key[kUnroll];
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      const int64_t p = base + u * 32 + lane;
      key[u] = p < end ? __ldcg(experts + p) : -1;
    }
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      if (base + u * 32 >= end) break;  // warp-uniform
      const int64_t p = base + u * 32 + lane;
      int x = key[u];
      if (p < end && x >= E) {
        atomicExch(err, (int)MOE_ERR_INVALID_ARGUMENT);
        x = -1;
      }
      if (x < 0) x = -1;  // negative id: an empty slot (the reference's permute never matches it)
      const unsigned peers = __match_any_sync(0xffffffffu, x);
      if (x >= 0 && lane == __ffs(peers) - 1) my_hist[x] += __popc(peers);
      // per-(chunk, expert) counts: aggregate lanes with the same key
      const int ck = x >= 0 ? int((p / k) / ct) * E + x : -1;
      const unsigned cpeers = __match_any_sync(0xffffffffu, ck);
      if (ck >= 0 && lane == __ffs(cpeers) - 1) atomicAdd(ccount + ck, __popc(cpeers));
    }
  }
  __syncthreads();
  for (int x = tid; x < E; x += blockDim.x) {
    int run = 0;
    for (int ww = 0; ww < nw; ++ww) {
      const int c = hist[ww * E + x];
      hist[ww * E + x] = run;
      run += c;
    }
    offs[x] = run;
  }
  __syncthreads();
  if (w == 0) {
    int carry = 0;
    for (int x0 = 0; x0 < E; x0 += 32) {
      const int x = x0 + lane;
      const int v = x < E ? offs[x] : 0;
      int inc = v;
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const int o = __shfl_up_sync(0xffffffffu, inc, off);
        if (lane >= off) inc += o;
      }
      if (x < E) offs[x] = carry + inc - v;
      carry += __shfl_sync(0xffffffffu, inc, 31);
    }
    if (lane == 0) offs[E] = carry;
  }
  __syncthreads();
  for (int i = tid; i < nw * E; i += blockDim.x) hist[i] += offs[i % E];
  __syncthreads();
  for (int64_t base = begin; base < end; base += 32 * kUnroll) {
    int key[kUnroll];
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      const int64_t p = base + u * 32 + lane;
      key[u] = p < end ? __ldcg(experts + p) : -1;
    }
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      if (base + u * 32 >= end) break;
      const int64_t p = base + u * 32 + lane;
      int x = key[u];
      if (x >= E || x < 0) x = -1;
      const unsigned peers = __match_any_sync(0xffffffffu, x);
      int pos = 0;
      if (x >= 0) pos = my_hist[x] + __popc(peers & lanemask_lt());
      __syncwarp();
      if (x >= 0 && lane == __ffs(peers) - 1) my_hist[x] += __popc(peers);
      __syncwarp();
      if (x >= 0 && p < end) {
        expert_of[pos] = x;
        perm_src[pos] = int32_t(p / k);
        slot_pos[p] = pos;
      } else if (p < end) {
        slot_pos[p] = -1;
      }
    }
  }
  __syncthreads();
  if (count_in_smem)
    for (int i = tid; i < n * E; i += blockDim.x) counts[i] = ccount[i];
  for (int x = tid; x <= E; x += blockDim.x) expert_offsets[x] = offs[x];
}

// ---------------------------------------------------------------------------
// Plan: counts -> every offset / segment list of the exchange, one CTA.
//
// Tables (ints), in shared memory when they fit (plan_smem_ints), else in the
// card's global scratch — same code, different pointers:
//   ct   [e][n][E]    the exchanged counts (copied once, coalesced)
//   cum  [e][n+1][E]  rows of (g, x) in chunks < j   (cum[g][n][x] = total)
//   eo   [e][E+1]     sender-permuted expert offsets per node
//   fin  [xg][L][e]   final-layout segment base (l-major, then source g)
//   pre  [xg][n][e*L] staged-layout segment base (chunk-major, g, l)
//   cb   [xg][n+1]    staged chunk bases
// Every scan is a warp-level scan (shuffles) so the critical path is a few
// hundred cycles per table instead of a serial global-memory chain.
struct PlanTables {
  int32_t* ct;
  int32_t* cum;
  int32_t* eo;
  int32_t* fin;
  int32_t* pre;
  int32_t* cb;
};

__host__ __device__ inline size_t plan_smem_ints(int e, int E, int n) {
  return size_t(e) * n * E + size_t(e) * (n + 1) * E + size_t(e) * (E + 1) + size_t(e) * E + size_t(e) * n * E +
         size_t(e) * (n + 1);
}

__host__ __device__ inline PlanTables plan_tables(int32_t* base, int e, int E, int n) {
  PlanTables tb;
  tb.ct = base;
  tb.cum = tb.ct + size_t(e) * n * E;
  tb.eo = tb.cum + size_t(e) * (n + 1) * E;
  tb.fin = tb.eo + size_t(e) * (E + 1);
  tb.pre = tb.fin + size_t(e) * E;
  tb.cb = tb.pre + size_t(e) * n * E;
  return tb;
}

__device__ __forceinline__ SegList* plan_list_at(const PlanArgs& a, int phase, int j) {
  char* base = reinterpret_cast<char*>(a.lists);
  return reinterpret_cast<SegList*>(base + (size_t(phase) * a.max_chunks + j) * seglist_bytes(a.seg_cap));
}

// Warp-wide exclusive scan of v; returns the exclusive prefix, *total = sum.
__device__ __forceinline__ int warp_exscan(int v, int lane, int* total) {
  int inc = v;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const int o = __shfl_up_sync(0xffffffffu, inc, off);
    if (lane >= off) inc += o;
  }
  *total = __shfl_sync(0xffffffffu, inc, 31);
  return inc - v;
}
__device__ __forceinline__ int64_t warp_exscan64(int64_t v, int lane, int64_t* total) {
  int64_t inc = v;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const int64_t o = __shfl_up_sync(0xffffffffu, inc, off);
    if (lane >= off) inc += o;
  }
  *total = __shfl_sync(0xffffffffu, inc, 31);
  return inc - v;
}

__device__ __forceinline__ void plan_block(const PlanArgs& a, const PlanTables& tb) {
  const int e = a.e, E = a.E, L = a.L, n = a.n, t = a.t;
  const int tid = threadIdx.x, nth = blockDim.x;
  const int lane = tid & 31, wid = tid >> 5, nw = nth >> 5;
  // 1. counts (peers wrote them over NVLink: L2-coherent loads)
  #pragma unroll 1
  for (int i = tid; i < e * n * E; i += nth) {
    const int g = i / (n * E), r = i % (n * E);
    tb.ct[i] = int(uint32_t(__ldcg(reinterpret_cast<const unsigned long long*>(a.count_table) +
                                   int64_t(g) * a.max_chunks * E + r)));
  }
  __syncthreads();
  if (a.dbg && tid == 0) a.dbg[8] = globaltimer();
  auto CT = [&](int g, int j, int x) { return tb.ct[(g * n + j) * E + x]; };
  auto CUM = [&](int g, int j, int x) -> int& { return tb.cum[(g * (n + 1) + j) * E + x]; };
  // 2. per-(g, x) chunk prefixes
  #pragma unroll 1
  for (int q = tid; q < e * E; q += nth) {
    const int g = q / E, x = q % E;
    int run = 0;
    #pragma unroll 1
    for (int j = 0; j < n; ++j) {
      CUM(g, j, x) = run;
      run += CT(g, j, x);
    }
    CUM(g, n, x) = run;
  }
  __syncthreads();
  if (a.dbg && tid == 0) a.dbg[9] = globaltimer();
  // 3. eo[g][x]: scan over x of totals; 4. fin[xg][l][g]: scan over (l, g)
  #pragma unroll 1
  for (int task = wid; task < 2 * e; task += nw) {
    const int g = task % e;
    int carry = 0;
    if (task < e) {
      #pragma unroll 1
      for (int x0 = 0; x0 < E; x0 += 32) {
        const int x = x0 + lane;
        int tot;
        const int ex = warp_exscan(x < E ? CUM(g, n, x) : 0, lane, &tot);
        if (x < E) tb.eo[g * (E + 1) + x] = carry + ex;
        carry += tot;
      }
      if (lane == 0) tb.eo[g * (E + 1) + E] = carry;
    } else {
      const int xg = g;
      #pragma unroll 1
      for (int u0 = 0; u0 < E; u0 += 32) {  // u = l*e + src, L*e == E
        const int u = u0 + lane;
        const int l = u / e, src = u % e;
        int tot;
        const int ex = warp_exscan(u < E ? CUM(src, n, xg * L + l) : 0, lane, &tot);
        if (u < E) tb.fin[(xg * L + l) * e + src] = carry + ex;
        carry += tot;
      }
      if (lane == 0 && xg == a.node) *a.recv_rows = carry;
    }
  }
  // 5. staged bases: within-chunk scan over (g, l) per (xg, j)
  #pragma unroll 1
  for (int task = wid; task < e * n; task += nw) {
    const int xg = task / n, j = task % n;
    int carry = 0;
    #pragma unroll 1
    for (int u0 = 0; u0 < E; u0 += 32) {  // u = src*L + l, e*L == E
      const int u = u0 + lane;
      int tot;
      const int ex = warp_exscan(u < E ? CT(u / L, j, xg * L + u % L) : 0, lane, &tot);
      if (u < E) tb.pre[(xg * n + j) * E + u] = carry + ex;
      carry += tot;
    }
    if (lane == 0) tb.cb[xg * (n + 1) + j] = carry;
  }
  __syncthreads();
  if (a.dbg && tid == 0) a.dbg[10] = globaltimer();
  #pragma unroll 1
  for (int xg = tid; xg < e; xg += nth) {
    int run = 0;
    #pragma unroll 1
    for (int j = 0; j < n; ++j) {
      const int c = tb.cb[xg * (n + 1) + j];
      tb.cb[xg * (n + 1) + j] = run;
      run += c;
    }
    tb.cb[xg * (n + 1) + n] = run;
  }
  __syncthreads();
  if (a.dbg && tid == 0) a.dbg[11] = globaltimer();
  #pragma unroll 1
  for (int i = tid; i < e * n * E; i += nth) tb.pre[i] += tb.cb[(i / (n * E)) * (n + 1) + (i / E) % n];
  // 6. local permuted->final delta of this node's experts
  #pragma unroll 1
  for (int l = tid; l < L; l += nth) {
    const int x = a.node * L + l;
    a.local_delta[x] = tb.fin[(a.node * L + l) * e + a.node] - tb.eo[a.node * (E + 1) + x];
  }
  // 6a. this node's local-expert row offsets in recv (final layout: for l,
  //     for source g) — the grouped GEMM's segments (experts.cu)
  if (a.recv_offs) {
    #pragma unroll 1
    for (int l = tid; l <= L; l += nth) {
      if (l < L) a.recv_offs[l] = tb.fin[(a.node * L + l) * e];
      else a.recv_offs[L] = tb.fin[(a.node * L + L - 1) * e + e - 1] + CUM(e - 1, n, a.node * L + L - 1);
    }
  }
  // 6b. per-expert destination table of this sender for the token-side AA:
  //     dst row of permuted position p = base[x] + p on card[x], columns
  //     [off, off + width) (this rank's slice on cross-node legs under dedup)
  if (a.aa_table) {
    const bool dd = a.level != MOE_BASELINE && t > 1;
    const int g = a.node;
    #pragma unroll 1
    for (int x = tid; x < E; x += nth) {
      const int xg = x / L, l = x % L;
      const int eo = tb.eo[g * (E + 1) + x];
      const bool slice = dd && xg != g;
      a.aa_table[x] = xg * t + a.rho;
      a.aa_table[E + x] = tb.fin[(xg * L + l) * e + g] - eo;
      a.aa_table[2 * E + x] = slice ? a.rho * int(a.row_bytes / t) : 0;
      a.aa_table[3 * E + x] = slice ? int(a.row_bytes / t) : int(a.row_bytes);
      #pragma unroll 1
      for (int j = 0; j < n; ++j)
        a.aa_table[(4 + j) * E + x] = tb.pre[(xg * n + j) * E + g * L + l] - eo - CUM(g, j, x);
    }
  }
  __syncthreads();
  if (a.dbg && tid == 0) a.dbg[12] = globaltimer();
  // 7. segment lists: one warp per (phase, chunk); candidates u in [0, E)
  const bool dedup = a.level != MOE_BASELINE && t > 1;
  const bool staged = a.landing == MOE_LAND_STAGED;
  const int full = int(a.row_bytes);
  const int slice = int(a.row_bytes / t);
  const int slice_off = a.rho * slice;
  const int g0 = a.node;
  const int me = g0 * t + a.rho;
  #pragma unroll 1
  for (int task = wid; task < kNumPhases * n; task += nw) {
    const int phase = task / n, j = task % n;
    SegList* lst = plan_list_at(a, phase, j);
    int pos = 0;
    int64_t rowsum = 0;
    #pragma unroll 1
    for (int u0 = 0; u0 < E; u0 += 32) {
      const int u = u0 + lane;
      Seg sg;
      sg.rows = 0;
      sg.pad = 0;
      if (u < E) {
        if (phase == kPhaseAA || phase == kPhaseAAL) {
          const bool local_list = phase == kPhaseAAL;
          const int x = local_list ? g0 * L + u : u;
          const int xg = x / L, l = x % L;
          if ((local_list && u < L) || (!local_list && xg != g0)) {
            sg.rows = CT(g0, j, x);
            sg.src_row = tb.eo[g0 * (E + 1) + x] + CUM(g0, j, x);
            sg.dst_row = staged ? int64_t(tb.pre[(xg * n + j) * E + g0 * L + l])
                                : int64_t(tb.fin[(xg * L + l) * e + g0]) + CUM(g0, j, x);
            const bool rs = dedup && !local_list;
            sg.dst = xg * t + a.rho;
            sg.col_off = rs ? slice_off : 0;
            sg.width = rs ? slice : full;
            sg.expert = x;
          }
        } else {
          const int src = u / L, l = u % L, x = g0 * L + l;
          const int rows = CT(src, j, x);
          const int64_t fin_row = int64_t(tb.fin[(g0 * L + l) * e + src]) + CUM(src, j, x);
          const int64_t pre_row = tb.pre[(g0 * n + j) * E + src * L + l];
          if (phase == kPhaseAG) {
            if (dedup && src != g0) {
              sg.rows = rows;
              sg.src_row = sg.dst_row = staged ? pre_row : fin_row;
              sg.dst = -1;
              sg.col_off = slice_off;
              sg.width = slice;
              sg.expert = x;
            }
          } else if (phase == kPhaseD2D) {
            if (staged) {
              sg.rows = rows;
              sg.src_row = pre_row;
              sg.dst_row = fin_row;
              sg.dst = me;
              sg.col_off = 0;
              sg.width = full;
              sg.expert = x;
            }
          } else {  // kPhaseCAA: expert outputs back to the sender's permuted order
            if (src != g0) {
              sg.rows = rows;
              sg.src_row = fin_row;
              sg.dst_row = int64_t(tb.eo[src * (E + 1) + x]) + CUM(src, j, x);
              sg.dst = src * t + a.rho;
              sg.col_off = dedup ? slice_off : 0;
              sg.width = dedup ? slice : full;
              sg.expert = x;
            }
          }
        }
      }
      const bool keep = sg.rows > 0;
      const unsigned ball = __ballot_sync(0xffffffffu, keep);
      int64_t rtot;
      const int64_t rex = warp_exscan64(keep ? sg.rows : 0, lane, &rtot);
      if (keep) {
        sg.row_begin = rowsum + rex;
        lst->segs[pos + __popc(ball & ((1u << lane) - 1u))] = sg;
      }
      pos += __popc(ball);
      rowsum += rtot;
    }
    if (lane == 0) {
      lst->nseg = pos;
      lst->total_rows = rowsum;
    }
  }
}

}  // namespace monta

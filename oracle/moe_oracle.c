/*
 * moe_oracle.c — CPU restatement of the reference data plane.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library, and
 * only as the checker or the timed CPU baseline — never on the product path.
 *
 * Each function restates /root/reference/proj/include/moeplan/dataplane.hpp
 * over flat arrays (the reference's AoS TokenRecord / std::vector buffers
 * become SoA: payload bytes + int32 tags {token_id, source_card,
 * source_position, expert}).  Pinned against the reference itself
 * (oracle/_ref, built by oracle/Makefile from the reference headers) at E == e
 * and against the reference's known-answer tests (tests/golden).
 *
 * Generalisation to E > e (SURVEY.md §7 decision 1): node x hosts experts
 * [x*L, (x+1)*L), L = E/e.  Final layout on node x: for local expert l, for
 * source node g, records in the sender's permuted order; staged (pre-copy)
 * layout: for chunk j, for source g, for l.  Both reduce to the reference's
 * layouts when L == 1.
 *
 * Status codes match include/monta.h: 0 ok, 1 invalid argument, 2 corrupt
 * routing, 6 out of memory.
 *
 * Host threads (OpenMP, OMP_NUM_THREADS): the router, permute, monolithic
 * dispatch and combine split their independent work (tokens, experts,
 * records) across threads; every output position is computed exactly as the
 * serial loops define it, so results do not depend on the thread count.
 */
#include <math.h>
#include <omp.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

enum { OK = 0, INVALID = 1, CORRUPT = 2, OOM = 6 };
enum { BASELINE = 0, O1 = 1, O2 = 2, O3 = 3 };
enum { F32 = 0, BF16 = 1, F16 = 2, F64 = 3, I64 = 4 };

static char g_msg[512];
const char* oracle_last_error(void) { return g_msg; }
static int err(int code, const char* m) {
  strncpy(g_msg, m, sizeof(g_msg) - 1);
  return code;
}

/* route_topk — dataplane.hpp:72-106.  Softmax in double (max-subtract, exp,
 * sum in index order, divide); the k largest raw scores win with the lower
 * index first on ties (stable sort by score); experts ascending; probs are
 * the softmax values of the selected experts. */
int oracle_route_topk(const double* scores, int64_t T, int E, int k, int32_t* experts, double* probs) {
  if (k < 1) return err(INVALID, "route_topk: k must be >= 1");
  if (T == 0) return OK;
  if (E < 1) return err(INVALID, "route_topk: empty gate score row");
  if (k > E) return err(INVALID, "route_topk: k exceeds the expert count");
  int oom = 0;
#pragma omp parallel
  {
  double* soft = (double*)malloc(sizeof(double) * E);
  int* order = (int*)malloc(sizeof(int) * E);
  if (!soft || !order) {
#pragma omp atomic write
    oom = 1;
  }
#pragma omp for schedule(static)
  for (int64_t i = 0; i < T; ++i) {
    if (!soft || !order) continue;
    const double* s = scores + i * E;
    double peak = s[0];
    for (int x = 0; x < E; ++x) peak = s[x] > peak ? s[x] : peak;
    double denom = 0.0;
    for (int x = 0; x < E; ++x) {
      soft[x] = exp(s[x] - peak);
      denom += soft[x];
    }
    for (int x = 0; x < E; ++x) soft[x] /= denom;
    /* stable insertion sort of indices by score, descending */
    for (int x = 0; x < E; ++x) {
      int y = x;
      while (y > 0 && s[order[y - 1]] < s[x]) {
        order[y] = order[y - 1];
        --y;
      }
      order[y] = x;
    }
    int32_t* ex = experts + i * k;
    for (int q = 0; q < k; ++q) ex[q] = order[q];
    /* ascending expert ids */
    for (int a = 1; a < k; ++a) {
      int32_t v = ex[a];
      int b = a;
      while (b > 0 && ex[b - 1] > v) {
        ex[b] = ex[b - 1];
        --b;
      }
      ex[b] = v;
    }
    for (int q = 0; q < k; ++q) probs[i * k + q] = soft[ex[q]];
  }
  free(soft);
  free(order);
  }
  if (oom) return err(OOM, "route_topk: oom");
  return OK;
}

/* permute — dataplane.hpp:118-140.  For x = 0..max_expert, for token i, for
 * each selected expert equal to x: append (token i).  inverse_map[i] lists
 * the record indices of token i in ascending expert order; it is returned as
 * inv[i*k + s] (s-th smallest record index), with inv_len[i] entries. */
int oracle_permute(const int32_t* experts, int64_t T, int k, int32_t* perm_src, int32_t* expert_of,
                   int32_t* inv, int32_t* inv_len) {
  int max_expert = -1;
  for (int64_t q = 0; q < T * k; ++q) max_expert = experts[q] > max_expert ? experts[q] : max_expert;
  /* the serial definition: for x ascending, for token i, for slot s with
   * experts[i,s] == x, append record (i); token i's inverse map lists its
   * records in that order.  Record index = start[x] + rank among x's
   * records; inverse slot = number of token i's entries appended before it
   * (smaller expert, or equal expert at an earlier slot) — each computed
   * independently, so experts split across threads. */
  const int nx = max_expert + 1;
  int64_t* start = (int64_t*)calloc((size_t)(nx > 0 ? nx : 1) + 1, sizeof(int64_t));
  if (!start) return err(OOM, "permute: oom");
  for (int64_t q = 0; q < T * k; ++q)
    if (experts[q] >= 0) ++start[experts[q] + 1];
  for (int x = 0; x < nx; ++x) start[x + 1] += start[x];
  for (int64_t i = 0; i < T; ++i) {
    int n = 0;
    for (int s = 0; s < k; ++s) n += experts[i * k + s] >= 0 && experts[i * k + s] <= max_expert;
    inv_len[i] = n;
  }
#pragma omp parallel for schedule(dynamic, 1)
  for (int x = 0; x < nx; ++x) {
    int64_t r = start[x];
    for (int64_t i = 0; i < T; ++i)
      for (int s = 0; s < k; ++s) {
        if (experts[i * k + s] != x) continue;
        int slot = 0;
        for (int s2 = 0; s2 < k; ++s2) {
          const int32_t y = experts[i * k + s2];
          if (y >= 0 && (y < x || (y == x && s2 < s))) ++slot;
        }
        inv[i * k + slot] = (int32_t)r;
        perm_src[r] = (int32_t)i;
        expert_of[r] = x;
        ++r;
      }
  }
  free(start);
  return OK;
}

/* Per-node inputs for the exchange, flattened over nodes g = 0..e-1. */
typedef struct {
  int e, t, E;
  int64_t T, k, row_bytes;
  const uint8_t* x;          /* [e][T][row_bytes] node batches */
  const int32_t* token_ids;  /* [e][T] */
  const int32_t* perm_src;   /* [e][T*k] permuted record -> source position */
  const int32_t* expert_of;  /* [e][T*k] */
  const int32_t* n_records;  /* [e] permuted records per node (T*k normally) */
} oracle_batches;

static void emit(uint8_t* rows, int32_t* tags, int64_t at, const oracle_batches* b, int g, int64_t r,
                 int64_t col_off, int64_t width) {
  const int64_t R = b->T * b->k;
  const int32_t pos = b->perm_src[g * R + r];
  memcpy(rows + at * b->row_bytes + col_off, b->x + ((int64_t)g * b->T + pos) * b->row_bytes + col_off,
         (size_t)width);
  if (tags) {
    tags[at * 4 + 0] = b->token_ids[(int64_t)g * b->T + pos];
    tags[at * 4 + 1] = g * b->t; /* canonical card of the source node */
    tags[at * 4 + 2] = pos;
    tags[at * 4 + 3] = b->expert_of[g * R + r];
  }
}

/* dispatch_monolithic — dataplane.hpp:145-162 (generalised).  Output per
 * NODE (every card of node x holds the same buffer): rows [e][cap][row_bytes],
 * tags [e][cap][4], counts [e]. */
int oracle_dispatch_monolithic(const oracle_batches* b, uint8_t* rows, int32_t* tags, int64_t* count,
                               int64_t cap) {
  const int L = b->E / b->e;
  const int64_t R = b->T * b->k;
  /* destination of record (g, r) with expert x*L + l on node x:
   * base(x, l, g) + its rank among g's records of that expert (the serial
   * order: for l, for g, for r); ranks from one pass per node g */
  const int64_t nb = (int64_t)b->e * b->E;
  int64_t* base = (int64_t*)calloc((size_t)(nb > 0 ? nb : 1), sizeof(int64_t)); /* [g][expert] */
  int64_t* rank = (int64_t*)malloc(sizeof(int64_t) * (size_t)(b->e * R > 0 ? b->e * R : 1));
  if (!base || !rank) {
    free(base);
    free(rank);
    return err(OOM, "dispatch_monolithic: oom");
  }
  int64_t* seen = (int64_t*)calloc((size_t)(b->E > 0 ? b->E : 1), sizeof(int64_t));
  for (int g = 0; g < b->e; ++g) {
    for (int xe = 0; xe < b->E; ++xe) seen[xe] = 0;
    for (int64_t r = 0; r < b->n_records[g]; ++r) {
      const int32_t xe = b->expert_of[g * R + r];
      rank[g * R + r] = (xe >= 0 && xe < b->E) ? seen[xe]++ : -1;
    }
    for (int xe = 0; xe < b->E; ++xe) base[(int64_t)g * b->E + xe] = seen[xe]; /* counts for now */
  }
  free(seen);
  for (int x = 0; x < b->e; ++x) {
    int64_t at = 0;
    for (int l = 0; l < L; ++l)
      for (int g = 0; g < b->e; ++g) {
        const int64_t c = base[(int64_t)g * b->E + x * L + l];
        base[(int64_t)g * b->E + x * L + l] = at;
        at += c;
      }
    if (at > cap) {
      free(base);
      free(rank);
      return err(INVALID, "dispatch_monolithic: capacity exceeded");
    }
    count[x] = at;
  }
  for (int g = 0; g < b->e; ++g) {
#pragma omp parallel for schedule(static)
    for (int64_t r = 0; r < b->n_records[g]; ++r) {
      const int32_t xe = b->expert_of[g * R + r];
      if (xe < 0 || xe >= L * b->e) continue; /* experts no node hosts are dropped */
      const int x = xe / L;
      emit(rows + (int64_t)x * cap * b->row_bytes, tags + (int64_t)x * cap * 4,
           base[(int64_t)g * b->E + xe] + rank[g * R + r], b, g, r, 0, b->row_bytes);
    }
  }
  free(base);
  free(rank);
  return OK;
}

/* dispatch_chunked — dataplane.hpp:187-283 (generalised).  Validation in the
 * reference's order; per expert node x and chunk j every tensor rank rho
 * receives hidden shard rho of each (src, chunk j) record (hidden_shard,
 * dataplane.hpp:166-176), the node gathers the shards back into full rows,
 * the chunk blocks are concatenated chunk-major (pre_copy), and the reorder
 * copy moves each (chunk, source[, local expert]) segment to its final
 * offset.  elem_bytes: bytes per payload element (width % t is checked in
 * elements, like the reference). */
int oracle_dispatch_chunked(const oracle_batches* b, int level, int n, int64_t elem_bytes, uint8_t* rows,
                            int32_t* tags, int64_t* count, uint8_t* pre_rows, int32_t* pre_tags, int64_t cap) {
  if (level != O1 && level != O2 && level != O3) return err(INVALID, "dispatch_chunked: level must be O1, O2 or O3");
  if (n < 1) return err(INVALID, "dispatch_chunked: n must be >= 1");
  if (level == O1 && n != 1) return err(INVALID, "dispatch_chunked: O1 is unchunked (n = 1)");
  if (b->T % n != 0) return err(INVALID, "dispatch_chunked: n does not divide the sequence");
  const int64_t width = b->row_bytes / elem_bytes;
  if (width % b->t != 0) return err(INVALID, "dispatch_chunked: tensor group must evenly split the payload");
  const int L = b->E / b->e;
  const int64_t R = b->T * b->k;
  const int64_t chunk_tokens = b->T / n;
  const int64_t shard = b->row_bytes / b->t;
  int64_t* seg = (int64_t*)calloc((size_t)n * b->e * L, sizeof(int64_t)); /* seg_len[j][g][l] */
  if (!seg) return err(OOM, "dispatch_chunked: oom");
  for (int x = 0; x < b->e; ++x) {
    uint8_t* pr = pre_rows + (int64_t)x * cap * b->row_bytes;
    int32_t* pt = pre_tags + (int64_t)x * cap * 4;
    int64_t at = 0;
    memset(seg, 0, sizeof(int64_t) * (size_t)n * b->e * L);
    for (int j = 0; j < n; ++j) {
      const int64_t block = at;
      /* rank rho receives shard rho of every record of chunk j; the gather
       * concatenates the shards: both land in the same full row. */
      for (int rho = 0; rho < b->t; ++rho) {
        int64_t q = block;
        for (int g = 0; g < b->e; ++g)
          for (int l = 0; l < L; ++l)
            for (int64_t r = 0; r < b->n_records[g]; ++r) {
              if (b->expert_of[g * R + r] != x * L + l) continue;
              if (b->perm_src[g * R + r] / chunk_tokens != j) continue;
              if (q >= cap) {
                free(seg);
                return err(INVALID, "dispatch_chunked: capacity exceeded");
              }
              emit(pr, rho == 0 ? pt : NULL, q, b, g, r, rho * shard, shard);
              if (rho == 0) ++seg[((int64_t)j * b->e + g) * L + l];
              ++q;
            }
        if (rho == b->t - 1) at = q;
      }
      if (b->t == 0) at = block;
    }
    /* reorder copy: final order l, g, j */
    uint8_t* fr = rows + (int64_t)x * cap * b->row_bytes;
    int32_t* ft = tags + (int64_t)x * cap * 4;
    int64_t out = 0;
    for (int l = 0; l < L; ++l)
      for (int g = 0; g < b->e; ++g)
        for (int j = 0; j < n; ++j) {
          /* offset of segment (j, g, l) inside the chunk-major layout */
          int64_t off = 0;
          for (int jj = 0; jj < j; ++jj)
            for (int gg = 0; gg < b->e; ++gg)
              for (int ll = 0; ll < L; ++ll) off += seg[((int64_t)jj * b->e + gg) * L + ll];
          for (int gg = 0; gg < g; ++gg)
            for (int ll = 0; ll < L; ++ll) off += seg[((int64_t)j * b->e + gg) * L + ll];
          for (int ll = 0; ll < l; ++ll) off += seg[((int64_t)j * b->e + g) * L + ll];
          const int64_t len = seg[((int64_t)j * b->e + g) * L + l];
          memcpy(fr + out * b->row_bytes, pr + off * b->row_bytes, (size_t)(len * b->row_bytes));
          memcpy(ft + out * 4, pt + off * 4, (size_t)(len * 16));
          out += len;
        }
    count[x] = out;
  }
  free(seg);
  return OK;
}

static double decode(const uint8_t* p, int dtype) {
  switch (dtype) {
    case F32: { float v; memcpy(&v, p, 4); return v; }
    case F64: { double v; memcpy(&v, p, 8); return v; }
    case I64: { int64_t v; memcpy(&v, p, 8); return (double)v; }
    case BF16: {
      uint16_t h; memcpy(&h, p, 2);
      uint32_t u = (uint32_t)h << 16; float v; memcpy(&v, &u, 4); return v;
    }
    case F16: {
      uint16_t h; memcpy(&h, p, 2);
      const int sgn = h >> 15, ex = (h >> 10) & 31, man = h & 1023;
      double v;
      if (ex == 0) v = ldexp((double)man, -24);
      else if (ex == 31) v = man ? NAN : INFINITY;
      else v = ldexp((double)(man | 1024), ex - 25);
      return sgn ? -v : v;
    }
  }
  return 0.0;
}

/* combine_unpermute — dataplane.hpp:293-347 (generalised).  Expert outputs
 * per node (the canonical card's buffer): rows [e][cap][row_bytes] with tags
 * [e][cap][4] and counts [e].  For node g, token i, slot s: the output row of
 * expert x = experts[i,s] is located by its tags (source card g*t, position
 * i, expert x) on node x/L; out[i] += probs[i,s] * double(payload) starting
 * from 0 in ascending slot order.  inv_len[i] must equal k (the reference's
 * inverse-map check).  Output out [e][T][width] doubles, token ids [e][T]. */
int oracle_combine(const oracle_batches* b, int dtype, const uint8_t* y, const int32_t* y_tags,
                   const int64_t* y_count, int64_t cap, const int32_t* experts, const double* probs,
                   const int32_t* inv, const int32_t* inv_len, double* out, int32_t* out_token) {
  const int L = b->E / b->e;
  const int64_t R = b->T * b->k;
  const int64_t esz = (dtype == BF16 || dtype == F16) ? 2 : (dtype == F32 ? 4 : 8);
  const int64_t width = b->row_bytes / esz;
  /* where[x][(g, pos, l)] -> row */
  const int64_t keys = (int64_t)b->e * b->T * L;
  int64_t* where = (int64_t*)malloc(sizeof(int64_t) * (size_t)(keys > 0 ? keys : 1));
  if (!where) return err(OOM, "combine: oom");
  for (int64_t q = 0; q < (int64_t)b->e * b->T * width; ++q) out[q] = 0.0;
  /* every token is independent (its slots accumulate in ascending order, as
   * in the serial loops): tokens split across threads; the first failing
   * token in (x, g, i) order reports, as the serial scan would */
  int status = OK;
  int64_t bad_at = -1;
  int bad_code = OK;
  for (int x = 0; x < b->e && status == OK; ++x) {
    for (int64_t q = 0; q < keys; ++q) where[q] = -1;
    for (int64_t r = 0; r < y_count[x]; ++r) {
      const int32_t* tg = y_tags + ((int64_t)x * cap + r) * 4;
      const int g = tg[1] / b->t, pos = tg[2], xe = tg[3];
      if (g < 0 || g >= b->e || pos < 0 || pos >= b->T || xe / L != x) continue;
      where[((int64_t)g * b->T + pos) * L + (xe - x * L)] = r;
    }
    const int64_t n_tok = (int64_t)b->e * b->T;
#pragma omp parallel for schedule(static)
    for (int64_t gi = 0; gi < n_tok; ++gi) {
      const int64_t g = gi / b->T;
      int code = OK;
      if (inv_len[gi] == 0 || inv_len[gi] != b->k) code = CORRUPT + 100; /* inverse map */
      if (code == OK) {
        out_token[gi] = b->token_ids[gi - (gi % b->T) + b->perm_src[g * R + inv[gi * b->k]]];
        for (int64_t s = 0; s < b->k; ++s) {
          const int xe = experts[gi * b->k + s];
          if (xe / L != x) continue; /* handled when node xe/L is scanned */
          const int64_t r = where[gi * L + (xe - x * L)];
          if (r < 0) {
            code = CORRUPT;
            break;
          }
          const uint8_t* row = y + ((int64_t)x * cap + r) * b->row_bytes;
          const double p = probs[gi * b->k + s];
          double* o = out + gi * width;
          if (dtype == BF16) { /* the common payload, decoded inline (same value as decode()) */
            for (int64_t q = 0; q < width; ++q) {
              uint16_t hb;
              memcpy(&hb, row + q * 2, 2);
              const uint32_t u = (uint32_t)hb << 16;
              float v;
              memcpy(&v, &u, 4);
              o[q] += p * (double)v;
            }
          } else {
            for (int64_t q = 0; q < width; ++q) o[q] += p * decode(row + q * esz, dtype);
          }
        }
      }
      if (code != OK) {
#pragma omp critical
        if (bad_at < 0 || gi < bad_at) {
          bad_at = gi;
          bad_code = code;
        }
      }
    }
    if (bad_at >= 0)
      status = err(CORRUPT, bad_code == CORRUPT + 100 ? "combine_unpermute: inverse map does not match routing"
                                                      : "combine_unpermute: missing expert output");
  }
  free(where);
  return status;
}

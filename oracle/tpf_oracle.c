/*
 * TEST INFRASTRUCTURE ONLY — the CPU oracle. Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline leg may load this (as the checker, never as the
 * thing measured or shipped). The product library never links it.
 *
 * A plain-C restatement of the reference's algorithm for the fused
 * AG-GEMM / GEMM-RS path (reference = /root/reference/proj, `tpfuse`):
 *
 *   pairwise_partner      collectives.cpp:37-43
 *   ring_indices_ag/rs    collectives.cpp:47-55 (arg check :25-33)
 *   build_schedule        collectives.cpp:57-107
 *   check_schedule        collectives.cpp:118-235 (counts, own-last, pairwise
 *                         symmetry, exactly-once symbolic delivery)
 *   matmul                tensor.cpp:68-85   (fp64, loop order b,s,c,k)
 *   split_seq/concat_seq  tensor.cpp:145-189 (batch-strided sequence slices)
 *   fuse_all_gather       collectives.cpp:237-279 (+ column_parallel_forward layers.cpp:120-127)
 *   rs_pipelined          collectives.cpp:285-311 (Ring, CircularSlices: partial += inbox)
 *   rs_direct             collectives.cpp:317-358 (Pairwise: fold one round late, own last)
 *   fuse_reduce_scatter   collectives.cpp:362-405 (+ row_parallel_forward layers.cpp:129-138)
 *   tpsp_mlp_forward      layers.cpp:140-147 (activation = square, experiment.cpp:172)
 *   randint_fill          tensor.cpp:234-250 (std::mt19937_64 restated below)
 *   mix_seed              experiment.cpp:163-168 (splitmix64)
 *
 * Parity of this restatement is pinned in tests/test_oracle.py against the
 * compiled reference (oracle/_ref/libtpfuse_ref.so) and against the golden
 * fixtures the reference's own tests hold (tests/golden/).
 *
 * The fused RS restatement reproduces the reference's *reduction order*
 * exactly, so it is bit-exact with the reference even on
 * non-integer fp64 data.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

enum { OR_RING = 0, OR_PAIRWISE = 1, OR_CIRCULAR = 2 };

/* ------------------------------------------------------------------ rng */
/* std::mt19937_64 (ISO C++ [rand.predef]: 312, 156, 31, 0xb5026f5aa96619e9, 29,
 * 0x5555555555555555, 17, 0x71d67fffeda60000, 37, 0xfff7eee000000000, 43,
 * 6364136223846793005). */
typedef struct { uint64_t mt[312]; int idx; } or_mt64;

static void mt64_seed(or_mt64* g, uint64_t seed) {
  g->mt[0] = seed;
  for (int i = 1; i < 312; ++i)
    g->mt[i] = 6364136223846793005ULL * (g->mt[i - 1] ^ (g->mt[i - 1] >> 62)) + (uint64_t)i;
  g->idx = 312;
}

static uint64_t mt64_next(or_mt64* g) {
  const uint64_t UM = 0xFFFFFFFF80000000ULL, LM = 0x7FFFFFFFULL;
  if (g->idx >= 312) {
    for (int i = 0; i < 312; ++i) {
      uint64_t x = (g->mt[i] & UM) | (g->mt[(i + 1) % 312] & LM);
      uint64_t xa = x >> 1;
      if (x & 1ULL) xa ^= 0xB5026F5AA96619E9ULL;
      g->mt[i] = g->mt[(i + 156) % 312] ^ xa;
    }
    g->idx = 0;
  }
  uint64_t x = g->mt[g->idx++];
  x ^= (x >> 29) & 0x5555555555555555ULL;
  x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
  x ^= (x << 37) & 0xFFF7EEE000000000ULL;
  x ^= (x >> 43);
  return x;
}

/* tensor.cpp:234-250: v = lo + (engine() % span), row-major fill. */
int or_randint_fill(int64_t n, int lo, int hi, uint64_t seed, double* out) {
  if (lo >= hi) return -1;
  or_mt64* g = (or_mt64*)malloc(sizeof(or_mt64));
  if (!g) return -1;
  mt64_seed(g, seed);
  const uint64_t span = (uint64_t)((int64_t)hi - (int64_t)lo);
  for (int64_t i = 0; i < n; ++i) out[i] = (double)(lo + (int64_t)(mt64_next(g) % span));
  free(g);
  return 0;
}

/* experiment.cpp:163-168 */
uint64_t or_mix_seed(uint64_t seed, uint64_t salt) {
  uint64_t z = seed + 0x9e3779b97f4a7c15ULL * (salt + 1);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

/* ------------------------------------------------------------ schedules */
static int pairwise_partner(int r, int round, int n) {
  const int u = n - 2 - round;
  if (r == n - 1) return u;
  if (r == u) return n - 1;
  const int m = n - 1;
  return ((2 * u - r) % m + m) % m;
}

int or_pairwise_partner(int r, int round, int n) { return pairwise_partner(r, round, n); }

/* rs != 0: ring_indices_rs, else ring_indices_ag. -1 on bad args. */
int or_ring_indices(int rs, int r, int i, int n, int32_t* out) {
  if (n < 1 || r < 0 || r >= n || i < 0 || i >= n) return -1;
  out[0] = (r + 1) % n;
  out[1] = (r - 1 + n) % n;
  out[2] = rs ? ((r - i - 1) % n + n) % n : (r - i + n) % n;
  return 0;
}

/* Symbolic exactly-once delivery replay (collectives.cpp:118-178).
 * Tags are (source, slice) pairs encoded as source*n+slice, counted per rank. */
static int check_delivery(int kind, int n, const int32_t* t) {
  int* final_acc = (int*)calloc((size_t)n * n * n, sizeof(int)); /* [rank][tag] */
  int* cur = (int*)calloc((size_t)n * n * n, sizeof(int));
  int* nxt = (int*)calloc((size_t)n * n * n, sizeof(int));
  int ok = final_acc && cur && nxt;
#define ST(r, i, f) t[((r) * n + (i)) * 3 + (f)]
  if (ok && kind == OR_PAIRWISE) {
    for (int i = 0; i < n; ++i) {
      memset(nxt, 0, sizeof(int) * (size_t)n * n * n); /* outbox[dst][tag] */
      for (int r = 0; r < n; ++r) {
        const int tag = r * n + ST(r, i, 2);
        if (ST(r, i, 0) >= 0) nxt[ST(r, i, 0) * n * n + tag] += 1;
        else final_acc[r * n * n + tag] += 1;
      }
      for (int r = 0; r < n; ++r)
        if (ST(r, i, 0) >= 0)
          for (int k = 0; k < n * n; ++k) final_acc[r * n * n + k] += nxt[r * n * n + k];
    }
  } else if (ok) {
    for (int i = 0; i < n; ++i) {
      memset(nxt, 0, sizeof(int) * (size_t)n * n * n);
      for (int r = 0; r < n; ++r) {
        int* part = (int*)calloc((size_t)n * n, sizeof(int));
        part[r * n + ST(r, i, 2)] += 1;
        if (i > 0)
          for (int k = 0; k < n * n; ++k) part[k] += cur[r * n * n + k];
        if (ST(r, i, 0) >= 0) memcpy(nxt + ST(r, i, 0) * n * n, part, sizeof(int) * (size_t)n * n);
        else memcpy(final_acc + r * n * n, part, sizeof(int) * (size_t)n * n);
        free(part);
      }
      int* tmp = cur; cur = nxt; nxt = tmp;
    }
  }
  int rc = ok ? 0 : -1;
  for (int r = 0; ok && r < n && rc == 0; ++r) {
    int total = 0;
    for (int k = 0; k < n * n; ++k) total += final_acc[r * n * n + k];
    if (total != n) rc = -1;
    for (int q = 0; q < n; ++q)
      if (final_acc[r * n * n + q * n + r] != 1) rc = -1;
  }
#undef ST
  free(final_acc); free(cur); free(nxt);
  return rc;
}

/* collectives.cpp:180-235. 0 = valid, -1 = violated. */
int or_check_schedule(int kind, int n, const int32_t* t) {
  if (n < 1) return -1;
  if (n == 1) return 0;
  for (int r = 0; r < n; ++r) {
    int sends = 0, recvs = 0;
    for (int i = 0; i < n; ++i) {
      const int32_t* st = t + (r * n + i) * 3;
      if (st[0] >= 0) ++sends;
      if (st[1] >= 0) ++recvs;
      if (st[2] < 0 || st[2] >= n) return -1;
    }
    if (sends != n - 1 || recvs != n - 1) return -1;
    if (t[(r * n + n - 1) * 3 + 2] != r) return -1;
  }
  if (kind == OR_PAIRWISE) {
    for (int i = 0; i < n - 1; ++i) {
      int busy = 0;
      for (int r = 0; r < n; ++r) {
        const int32_t* st = t + (r * n + i) * 3;
        if (st[0] != st[1]) return -1;
        if (st[0] < 0 || st[0] >= n) return -1;
        if (t[(st[0] * n + i) * 3 + 0] != r) return -1;
        ++busy;
      }
      if (busy != n) return -1;
    }
  }
  return check_delivery(kind, n, t);
}

/* collectives.cpp:57-107. out: n*n*3 (nothing for n == 1). -1 on rejection. */
int or_build_schedule(int kind, int n, int32_t* out) {
  if (n < 1) return -1;
  if (kind == OR_PAIRWISE && n % 2 != 0 && n != 1) return -1;
  if (kind < 0 || kind > 2) return -1;
  if (n == 1) return 0;
  for (int r = 0; r < n; ++r)
    for (int i = 0; i < n; ++i) {
      const int comm = i < n - 1;
      int32_t* st = out + (r * n + i) * 3;
      if (kind == OR_RING) {
        int32_t idx[3];
        or_ring_indices(1, r, i, n, idx);
        st[0] = comm ? idx[0] : -1;
        st[1] = comm ? idx[1] : -1;
        st[2] = idx[2];
      } else if (kind == OR_CIRCULAR) {
        st[0] = comm ? (r - 1 + n) % n : -1;
        st[1] = comm ? (r + 1) % n : -1;
        st[2] = (r + i + 1) % n;
      } else {
        if (comm) {
          const int p = pairwise_partner(r, i, n);
          st[0] = p; st[1] = p; st[2] = p;
        } else {
          st[0] = -1; st[1] = -1; st[2] = r;
        }
      }
    }
  return or_check_schedule(kind, n, out);
}

/* ---------------------------------------------------------- dense math */
/* tensor.cpp:68-85: out[b,s,c] = sum_k x[b,s,k] * w[k,c], k innermost. */
void or_matmul(int64_t bs, int64_t k, int64_t n, const double* x, const double* w,
               double* out) {
  for (int64_t r = 0; r < bs; ++r)
    for (int64_t c = 0; c < n; ++c) {
      double acc = 0.0;
      for (int64_t kk = 0; kk < k; ++kk) acc += x[r * k + kk] * w[kk * n + c];
      out[r * n + c] = acc;
    }
}

/* split_seq(x, nchunks)[c] -> dst (B, S/nchunks, D); tensor.cpp:145-165 */
static void chunk_of(const double* x, int64_t b, int64_t s, int64_t d, int nchunks, int c,
                     double* dst) {
  const int64_t piece = s / nchunks;
  for (int64_t bb = 0; bb < b; ++bb)
    memcpy(dst + bb * piece * d, x + (bb * s + (int64_t)c * piece) * d,
           sizeof(double) * (size_t)(piece * d));
}

/* place chunk c of (B, S_total, D) from src (B, piece, D); concat_seq inverse */
static void place_chunk(double* out, int64_t b, int64_t s_total, int64_t d, int64_t piece,
                        int c, const double* src) {
  for (int64_t bb = 0; bb < b; ++bb)
    memcpy(out + (bb * s_total + (int64_t)c * piece) * d, src + bb * piece * d,
           sizeof(double) * (size_t)(piece * d));
}

/* Rank-local weight shards (ShardedLinear::split_rows / split_columns,
 * layers.cpp:10-48). */
static void col_shard(const double* w, int64_t k, int64_t n, int t, int r, double* dst) {
  const int64_t nl = n / t;
  for (int64_t i = 0; i < k; ++i) memcpy(dst + i * nl, w + i * n + r * nl, sizeof(double) * (size_t)nl);
}

/* ----------------------------------------------------- fused collectives */
/* column_parallel_forward = fuse_all_gather with f = matmul(., W_col[r]).
 * x_full (B,S,K) is sliced by rank (rank r owns sequence slice r);
 * out: T consecutive (B,S,N/T). The restatement follows Alg. 1 literally:
 * pass p carries sub-chunk p; iteration i computes slice l = (r-i) mod T into
 * out_chunks[l*m+p]. */
int or_column_parallel(int t, int m, int64_t b, int64_t s, int64_t k, int64_t n,
                       const double* x_full, const double* w_full, double* out) {
  if (t < 1 || m < 1 || s % t != 0 || n % t != 0) return -1;
  const int64_t sl = s / t;
  if (sl % m != 0) return -1;
  const int64_t piece = sl / m, nl = n / t;
  double* wr = (double*)malloc(sizeof(double) * (size_t)(k * nl));
  double* x_l = (double*)malloc(sizeof(double) * (size_t)(b * sl * k));
  double* trav = (double*)malloc(sizeof(double) * (size_t)(b * piece * k));
  double* part = (double*)malloc(sizeof(double) * (size_t)(b * piece * nl));
  for (int r = 0; r < t; ++r) {
    col_shard(w_full, k, n, t, r, wr);
    double* out_r = out + (int64_t)r * b * s * nl;
    for (int p = 0; p < m; ++p)
      for (int i = 0; i < t; ++i) {
        int32_t idx[3];
        or_ring_indices(0, r, i, t, idx);
        const int l = idx[2];
        chunk_of(x_full, b, s, k, t, l, x_l);           /* rank l's slice  */
        chunk_of(x_l, b, sl, k, m, p, trav);             /* its sub-chunk p */
        or_matmul(b * piece, k, nl, trav, wr, part);
        place_chunk(out_r, b, s, nl, piece, l * m + p, part);
      }
  }
  free(wr); free(x_l); free(trav); free(part);
  return 0;
}

/* Generic FuseRS driver over precomputed partials.
 * partial(q, c) = rank q's f applied to its sequence chunk c (of t*m chunks),
 * shape (B, S/(t*m), N), provided by the callback buffer layout
 * parts[((q * t*m) + c) * chunk_elems]. out: T consecutive (B, S/T, N). */
static int fuse_rs_from_partials(int t, int kind, int m, int64_t b, int64_t s, int64_t n,
                                 const int32_t* sched, const double* parts, double* out) {
  const int nch = t * m;
  const int64_t piece = s / nch;
  const int64_t ce = b * piece * n;
  double* inbox = (double*)calloc((size_t)(t * ce), sizeof(double));
  double* next = (double*)calloc((size_t)(t * ce), sizeof(double));
  double* acc = (double*)calloc((size_t)(t * ce), sizeof(double));
  int* has_acc = (int*)calloc((size_t)t, sizeof(int));
  double* cur = (double*)malloc(sizeof(double) * (size_t)ce);
  for (int p = 0; p < m; ++p) {
    memset(has_acc, 0, sizeof(int) * (size_t)t);
    for (int i = 0; i < t; ++i) {
      for (int q = 0; q < t; ++q) {
        const int32_t* st = sched + (q * t + i) * 3;
        const int owner = st[2];
        memcpy(cur, parts + ((int64_t)q * nch + owner * m + p) * ce, sizeof(double) * (size_t)ce);
        double* a = acc + q * ce;
        if (kind == OR_PAIRWISE) {
          /* rs_direct: fold the previous round's contribution first. */
          if (i > 0) {
            const double* in = inbox + q * ce;
            if (!has_acc[q]) { memcpy(a, in, sizeof(double) * (size_t)ce); has_acc[q] = 1; }
            else for (int64_t e = 0; e < ce; ++e) a[e] += in[e];
          }
          if (st[0] >= 0) memcpy(next + st[0] * ce, cur, sizeof(double) * (size_t)ce);
          else {
            if (!has_acc[q]) { memcpy(a, cur, sizeof(double) * (size_t)ce); has_acc[q] = 1; }
            else for (int64_t e = 0; e < ce; ++e) a[e] += cur[e];
          }
        } else {
          /* rs_pipelined: partial = f(slice); partial += inbox; forward. */
          if (i > 0) {
            const double* in = inbox + q * ce;
            for (int64_t e = 0; e < ce; ++e) cur[e] += in[e];
          }
          if (st[0] >= 0) memcpy(next + st[0] * ce, cur, sizeof(double) * (size_t)ce);
          else memcpy(a, cur, sizeof(double) * (size_t)ce);
        }
      }
      double* tmp = inbox; inbox = next; next = tmp;
    }
    for (int q = 0; q < t; ++q)
      place_chunk(out + (int64_t)q * b * (s / t) * n, b, s / t, n, piece, p, acc + q * ce);
  }
  free(inbox); free(next); free(acc); free(has_acc); free(cur);
  return 0;
}

static int rs_checks(int t, int kind, int m, int64_t s) {
  if (t < 1 || m < 1 || kind < 0 || kind > 2) return -1;
  if (m > 1 && kind != OR_RING) return -1;
  if (kind == OR_PAIRWISE && t % 2 != 0 && t != 1) return -1;
  if (t > 1 && s % ((int64_t)t * m) != 0) return -1;
  return 0;
}

/* row_parallel_forward = fuse_reduce_scatter with f = matmul(., W_row[r]).
 * x_full (B,S,K) feature-sharded (rank r: columns [r*K/T,(r+1)*K/T));
 * w_full (K,N). out: T consecutive (B,S/T,N). */
int or_row_parallel(int t, int kind, int m, int64_t b, int64_t s, int64_t k, int64_t n,
                    const double* x_full, const double* w_full, double* out) {
  if (rs_checks(t, kind, m, s) || k % t != 0) return -1;
  const int64_t kl = k / t;
  if (t == 1) { or_matmul(b * s, k, n, x_full, w_full, out); return 0; }
  int32_t* sched = (int32_t*)malloc(sizeof(int32_t) * (size_t)(t * t * 3));
  if (or_build_schedule(kind, t, sched)) { free(sched); return -1; }
  const int nch = t * m;
  const int64_t piece = s / nch, ce = b * piece * n;
  double* parts = (double*)malloc(sizeof(double) * (size_t)(t * nch * ce));
  double* xr = (double*)malloc(sizeof(double) * (size_t)(b * s * kl));
  double* xc = (double*)malloc(sizeof(double) * (size_t)(b * piece * kl));
  for (int q = 0; q < t; ++q) {
    for (int64_t row = 0; row < b * s; ++row)
      memcpy(xr + row * kl, x_full + row * k + q * kl, sizeof(double) * (size_t)kl);
    const double* wq = w_full + (int64_t)q * kl * n; /* row shard q */
    for (int c = 0; c < nch; ++c) {
      chunk_of(xr, b, s, kl, nch, c, xc);
      or_matmul(b * piece, kl, n, xc, wq, parts + ((int64_t)q * nch + c) * ce);
    }
  }
  int rc = fuse_rs_from_partials(t, kind, m, b, s, n, sched, parts, out);
  free(sched); free(parts); free(xr); free(xc);
  return rc;
}

/* fuse_reduce_scatter with identity f on per-rank inputs (T x (B,S,D)). */
int or_fuse_rs_identity(int t, int kind, int m, int64_t b, int64_t s, int64_t d,
                        const double* inputs, double* out) {
  if (rs_checks(t, kind, m, s)) return -1;
  if (t == 1) { memcpy(out, inputs, sizeof(double) * (size_t)(b * s * d)); return 0; }
  int32_t* sched = (int32_t*)malloc(sizeof(int32_t) * (size_t)(t * t * 3));
  if (or_build_schedule(kind, t, sched)) { free(sched); return -1; }
  const int nch = t * m;
  const int64_t piece = s / nch, ce = b * piece * d;
  double* parts = (double*)malloc(sizeof(double) * (size_t)(t * nch * ce));
  for (int q = 0; q < t; ++q)
    for (int c = 0; c < nch; ++c)
      chunk_of(inputs + (int64_t)q * b * s * d, b, s, d, nch, c, parts + ((int64_t)q * nch + c) * ce);
  int rc = fuse_rs_from_partials(t, kind, m, b, s, d, sched, parts, out);
  free(sched); free(parts);
  return rc;
}

/* tpsp_mlp_forward with the square activation. x_full (B,S,D), up (D,H),
 * down (H,D). out: T consecutive (B,S/T,D). */
int or_mlp_square(int t, int kind, int m, int64_t b, int64_t s, int64_t d, int64_t h,
                  const double* x_full, const double* up, const double* down, double* out) {
  if (t < 1 || h % t != 0 || s % t != 0) return -1;
  const int64_t hl = h / t;
  double* hid = (double*)malloc(sizeof(double) * (size_t)(t * b * s * hl));
  if (or_column_parallel(t, m, b, s, d, h, x_full, up, hid)) { free(hid); return -1; }
  for (int64_t e = 0; e < t * b * s * hl; ++e) hid[e] = hid[e] * hid[e];
  /* Row-parallel with each rank's own (B,S,H/T) activation as x_r. Build the
   * equivalent feature-concatenated full input so or_row_parallel slices it. */
  double* act_full = (double*)malloc(sizeof(double) * (size_t)(b * s * h));
  for (int r = 0; r < t; ++r)
    for (int64_t row = 0; row < b * s; ++row)
      memcpy(act_full + row * h + r * hl, hid + ((int64_t)r * b * s + row) * hl,
             sizeof(double) * (size_t)hl);
  int rc = or_row_parallel(t, kind, m, b, s, h, d, act_full, down, out);
  free(hid); free(act_full);
  return rc;
}

/* ------------------------------------------------ UP: fused all-to-all attention */
#include <math.h>
/* attention_context (layers.cpp:107-118): softmax(q k^T * scale) v for one folded head,
 * q (sq, dh), k/v (sk, dh) -> o (sq, dh). softmax_rows: max-subtracted (tensor.cpp:123-143). */
static void attention_head(int64_t sq, int64_t sk, int64_t dh, int scale, const double* q,
                           const double* k, const double* v, double* o, double* scores) {
  const double sc = scale ? 1.0 / sqrt((double)dh) : 1.0;
  for (int64_t i = 0; i < sq; ++i) {
    double* row = scores + i * sk;
    for (int64_t j = 0; j < sk; ++j) {
      double acc = 0.0;
      for (int64_t d = 0; d < dh; ++d) acc += q[i * dh + d] * k[j * dh + d];
      row[j] = acc * sc;
    }
    double mx = row[0];
    for (int64_t j = 1; j < sk; ++j) mx = row[j] > mx ? row[j] : mx;
    double den = 0.0;
    for (int64_t j = 0; j < sk; ++j) { row[j] = exp(row[j] - mx); den += row[j]; }
    for (int64_t j = 0; j < sk; ++j) row[j] /= den;
    for (int64_t d = 0; d < dh; ++d) {
      double acc = 0.0;
      for (int64_t j = 0; j < sk; ++j) acc += row[j] * v[j * dh + d];
      o[i * dh + d] = acc;
    }
  }
}

/* fuse_all_to_all_attention (Alg. 5, layers.cpp:174-218). Per rank r: q/k/v
 * (batch*heads, S, dh) for its head group over the full sequence. Iteration i sends
 * slice l = (r+i+1)%T's context to rank l (keeps its own at i = T-1); rank l assembles
 * concat_feat over SOURCE rank of merge_heads(part): out[l] (batch, S/T, T*heads*dh),
 * feature index (src*heads + hh)*dh + d. q/k/v: T stacked ranks; out: T stacked. */
int or_attention_a2a(int t, int batch, int heads, int64_t s, int64_t dh, int scale,
                     const double* q, const double* k, const double* v, double* out) {
  if (t < 1 || batch < 1 || heads < 1 || s % t != 0) return -1;
  const int64_t sl = s / t, bh = (int64_t)batch * heads, per = bh * s * dh;
  const int64_t fw = (int64_t)t * heads * dh;
  double* scores = (double*)malloc(sizeof(double) * (size_t)(sl * s));
  double* o = (double*)malloc(sizeof(double) * (size_t)(sl * dh));
  for (int r = 0; r < t; ++r)
    for (int i = 0; i < t; ++i) {
      const int l = (r + i + 1) % t;  /* send_to == slice */
      for (int64_t g = 0; g < bh; ++g) {
        const int64_t b = g / heads, hh = g % heads;
        const double* qg = q + r * per + g * s * dh + (int64_t)l * sl * dh;
        attention_head(sl, s, dh, scale, qg, k + r * per + g * s * dh, v + r * per + g * s * dh, o,
                       scores);
        double* dst = out + (int64_t)l * batch * sl * fw;
        for (int64_t row = 0; row < sl; ++row)
          for (int64_t d = 0; d < dh; ++d)
            dst[(b * sl + row) * fw + ((int64_t)r * heads + hh) * dh + d] = o[row * dh + d];
      }
    }
  free(scores); free(o);
  return 0;
}

/* query_split_attention (Alg. 4, layers.cpp:149-172): fuse_reduce_scatter over the query
 * sequence with f(q_slice) = matmul(merge_heads(attention_context(q_slice, k, v)), W_o[r]).
 * q/k/v: T stacked ranks of (batch*heads, S, dh); w_o: (T*heads*dh, d) row-sharded by rank
 * (row block r = this rank's head group). out: T stacked (batch, S/T, d). */
int or_query_split_attention(int t, int kind, int batch, int heads, int64_t s, int64_t dh, int64_t d,
                             int scale, const double* q, const double* k, const double* v,
                             const double* w_o, double* out) {
  if (rs_checks(t, kind, 1, s)) return -1;
  const int64_t bh = (int64_t)batch * heads, per = bh * s * dh, hd = (int64_t)heads * dh;
  const int64_t piece = s / t, ce = (int64_t)batch * piece * d;
  int32_t* sched = NULL;
  if (t > 1) {
    sched = (int32_t*)malloc(sizeof(int32_t) * (size_t)(t * t * 3));
    if (or_build_schedule(kind, t, sched)) { free(sched); return -1; }
  }
  double* parts = (double*)malloc(sizeof(double) * (size_t)(t * t * ce));
  double* scores = (double*)malloc(sizeof(double) * (size_t)(piece * s));
  double* o = (double*)malloc(sizeof(double) * (size_t)(piece * dh));
  double* ctx = (double*)malloc(sizeof(double) * (size_t)(batch * piece * hd));
  for (int r = 0; r < t; ++r) {
    const double* wr = w_o + (int64_t)r * hd * d;
    for (int c = 0; c < t; ++c) {
      for (int64_t g = 0; g < bh; ++g) {
        const int64_t b = g / heads, hh = g % heads;
        attention_head(piece, s, dh, scale, q + r * per + g * s * dh + (int64_t)c * piece * dh,
                       k + r * per + g * s * dh, v + r * per + g * s * dh, o, scores);
        for (int64_t row = 0; row < piece; ++row)
          for (int64_t e = 0; e < dh; ++e) ctx[(b * piece + row) * hd + hh * dh + e] = o[row * dh + e];
      }
      or_matmul(batch * piece, hd, d, ctx, wr, parts + ((int64_t)r * t + c) * ce);
    }
  }
  int rc = 0;
  if (t == 1) memcpy(out, parts, sizeof(double) * (size_t)ce);
  else rc = fuse_rs_from_partials(t, kind, 1, batch, s, d, sched, parts, out);
  free(sched); free(parts); free(scores); free(o); free(ctx);
  return rc;
}

/* Ulysses first all-to-all. Restates layers_test.cpp:347-397's
 * to_head_sharded: rank r splits its sequence slice (batch*heads, S/T, dh) into T head-group
 * parts p_g(b*hl + h, s, d) = slice(b*heads + g*hl + h, s, d) (hl = heads/T), trades them with
 * ref_all_to_all (fabric.cpp:183-207: out[k] on rank r = parts[r] of rank k), then concat_seq
 * (tensor.cpp) stacks the received parts in source-rank order along the sequence.
 * in: T stacked (batch*heads, S/T, dh); out: T stacked (batch*hl, S, dh). */
int or_ulysses_a2a(int t, int batch, int heads, int64_t s, int64_t dh, const double* in, double* out) {
  if (t < 1 || batch < 1 || heads < 1 || s % t != 0 || heads % t != 0) return -1;
  const int64_t sl = s / t, hl = heads / t;
  const int64_t in_per = (int64_t)batch * heads * sl * dh, out_per = (int64_t)batch * hl * s * dh;
  for (int g = 0; g < t; ++g)            /* receiving rank = head group */
    for (int src = 0; src < t; ++src)    /* sending rank = sequence slice */
      for (int64_t b = 0; b < batch; ++b)
        for (int64_t h = 0; h < hl; ++h)
          for (int64_t i = 0; i < sl; ++i)
            for (int64_t d = 0; d < dh; ++d)
              out[g * out_per + ((b * hl + h) * s + src * sl + i) * dh + d] =
                  in[src * in_per + ((b * heads + g * hl + h) * sl + i) * dh + d];
  return 0;
}

/*
 * Plain-C restatement of the reference algorithms on the verification path.
 * TEST INFRASTRUCTURE ONLY (see spin_oracle.h). Each function cites the
 * reference file:line (under /root/reference/proj/core) it follows.
 */
#include <math.h>
#include <stdlib.h>
#include <string.h>

#include "spin_oracle.h"

/* ------------------------------------------------------------ rng.hpp:11-25 */
uint64_t so_splitmix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}

uint64_t so_mix_seed(uint64_t seed, uint64_t a, uint64_t b, uint64_t c) {
  uint64_t h = so_splitmix64(seed);
  h = so_splitmix64(h ^ a);
  h = so_splitmix64(h ^ b);
  return so_splitmix64(h ^ c);
}

/* rng.hpp:40-68: std::mt19937_64 (parameters fixed by the C++ standard) with
 * hand-written unit / uniform / uniform_int. */
enum { MT_N = 312, MT_M = 156 };

void so_rng_init(so_rng* r, uint64_t seed) {
  r->mt[0] = seed;
  for (int i = 1; i < MT_N; ++i) r->mt[i] = 6364136223846793005ULL * (r->mt[i - 1] ^ (r->mt[i - 1] >> 62)) + (uint64_t)i;
  r->idx = MT_N;
}

static void mt_twist(so_rng* r) {
  static const uint64_t kMatrix = 0xB5026F5AA96619E9ULL, kUpper = 0xFFFFFFFF80000000ULL, kLower = 0x7FFFFFFFULL;
  for (int i = 0; i < MT_N; ++i) {
    const uint64_t x = (r->mt[i] & kUpper) | (r->mt[(i + 1) % MT_N] & kLower);
    uint64_t y = x >> 1;
    if (x & 1ULL) y ^= kMatrix;
    r->mt[i] = r->mt[(i + MT_M) % MT_N] ^ y;
  }
  r->idx = 0;
}

uint64_t so_rng_next(so_rng* r) {
  if (r->idx >= MT_N) mt_twist(r);
  uint64_t x = r->mt[r->idx++];
  x ^= (x >> 29) & 0x5555555555555555ULL;
  x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
  x ^= (x << 37) & 0xFFF7EEE000000000ULL;
  x ^= x >> 43;
  return x;
}

double so_rng_unit(so_rng* r) { return (double)(so_rng_next(r) >> 11) * 0x1.0p-53; }

double so_rng_uniform(so_rng* r, double lo, double hi) { return lo + (hi - lo) * so_rng_unit(r); }

long long so_rng_uniform_int(so_rng* r, long long lo, long long hi) {
  if (hi <= lo) return lo;
  const uint64_t span = (uint64_t)(hi - lo) + 1;
  const uint64_t limit = UINT64_MAX - UINT64_MAX % span;
  uint64_t draw;
  do {
    draw = so_rng_next(r);
  } while (draw >= limit);
  return lo + (long long)(draw % span);
}

/* ------------------------------------------------------ attention.cpp:164-175 */
void so_make_toy_input(uint64_t seed, int queries, int kv_len, int dim, double* q, double* k, double* v) {
  so_rng r;
  so_rng_init(&r, so_mix_seed(seed, 0x04 /* kStreamToyAttention */, 0, 0));
  for (long i = 0; i < (long)queries * dim; ++i) q[i] = so_rng_uniform(&r, -1.0, 1.0);
  for (long i = 0; i < (long)kv_len * dim; ++i) k[i] = so_rng_uniform(&r, -1.0, 1.0);
  for (long i = 0; i < (long)kv_len * dim; ++i) v[i] = so_rng_uniform(&r, -1.0, 1.0);
}

/* ------------------------------------------------------- packing.cpp:16-103 */
static int try_place(const int* len, int n, int rows, int L, const int* order, int* segs, int seg_cap, int* n_segs,
                     int* used) {
  int ns = 0;
  for (int r = 0; r < rows; ++r) used[r] = 0;
  for (int oi = 0; oi < n; ++oi) {
    const int id = order[oi], need = len[id];
    int home = -1;
    for (int r = 0; r < rows; ++r)
      if (L - used[r] >= need) {
        home = r;
        break;
      }
    if (home >= 0) {
      if (ns >= seg_cap) return -1;
      int* s = segs + 5 * ns++;
      s[0] = id, s[1] = home, s[2] = used[home], s[3] = used[home] + need, s[4] = 0;
      used[home] += need;
      continue;
    }
    int left = need;
    for (int r = 0; r < rows && left > 0; ++r) {
      const int room = L - used[r];
      if (room <= 0) continue;
      const int take = room < left ? room : left;
      if (ns >= seg_cap) return -1;
      int* s = segs + 5 * ns++;
      s[0] = id, s[1] = r, s[2] = used[r], s[3] = used[r] + take, s[4] = need - left;
      used[r] += take;
      left -= take;
    }
    if (left > 0) return 0;
  }
  *n_segs = ns;
  return 1;
}

int so_pack(const int* kv_lens, int n, int width, int* length, int* rows_out, int* segs, int seg_cap, int* n_segs,
            long long* padding, int* q_replica_rows) {
  if (width < 1) return 1;
  for (int i = 0; i < n; ++i)
    if (kv_lens[i] < 1) return 1;
  *length = 0, *rows_out = 0, *n_segs = 0, *padding = 0;
  if (n == 0) return 0;
  const int rows = width < n ? width : n;
  long long total = 0;
  int longest = 0;
  for (int i = 0; i < n; ++i) {
    total += kv_lens[i];
    if (kv_lens[i] > longest) longest = kv_lens[i];
  }
  /* stable order by decreasing length (insertion sort keeps ties in index order) */
  int* order = (int*)malloc(sizeof(int) * n);
  int* used = (int*)malloc(sizeof(int) * rows);
  for (int i = 0; i < n; ++i) {
    int j = i;
    while (j > 0 && kv_lens[order[j - 1]] < kv_lens[i]) {
      order[j] = order[j - 1];
      --j;
    }
    order[j] = i;
  }
  const long long lo = (total + rows - 1) / rows;
  long long hi = longest > total ? longest : total;
  if (hi < lo) hi = lo;
  int status = 5;
  for (long long L = lo; L <= hi; ++L) {
    const int ok = try_place(kv_lens, n, rows, (int)L, order, segs, seg_cap, n_segs, used);
    if (ok < 0) {
      status = 4;
      break;
    }
    if (ok == 1) {
      long long filled = 0;
      for (int r = 0; r < rows; ++r) filled += used[r];
      *length = (int)L;
      *rows_out = rows;
      *padding = (long long)rows * L - filled;
      for (int i = 0; i < n; ++i) q_replica_rows[i] = 0;
      for (int s = 0; s < *n_segs; ++s) {
        /* count distinct rows per request (packing.cpp:63-68) */
        const int id = segs[5 * s], row = segs[5 * s + 1];
        int seen = 0;
        for (int p = 0; p < s; ++p)
          if (segs[5 * p] == id && segs[5 * p + 1] == row) seen = 1;
        if (!seen) ++q_replica_rows[id];
      }
      status = 0;
      break;
    }
  }
  free(order);
  free(used);
  return status;
}

/* packing.cpp:105-113 */
int so_naive_padding(const int* kv_lens, int n, long long* padding) {
  if (n <= 0) return 3;
  int longest = kv_lens[0];
  for (int i = 1; i < n; ++i)
    if (kv_lens[i] > longest) longest = kv_lens[i];
  long long pad = 0;
  for (int i = 0; i < n; ++i) pad += longest - kv_lens[i];
  *padding = pad;
  return 0;
}

/* packing.cpp:115-136 */
int so_build_indicator(int width, int length, const int* segs, int n_segs, int* cells) {
  for (long i = 0; i < (long)width * length; ++i) cells[i] = -1;
  for (int s = 0; s < n_segs; ++s) {
    const int* g = segs + 5 * s;
    if (g[1] < 0 || g[1] >= width || g[2] < 0 || g[3] > length || g[2] >= g[3]) return 5;
    for (int c = g[2]; c < g[3]; ++c) {
      if (cells[(long)g[1] * length + c] != -1) return 5;
      cells[(long)g[1] * length + c] = g[0];
    }
  }
  return 0;
}

/* slot_engine.cpp:24-45 */
int so_verify_batch_cost(const int* kv_lens, int n, int window, int packing, int pack_width, long long* tokens,
                         long long* padding) {
  *tokens = 0, *padding = 0;
  if (n <= 0) return 0;
  if (packing) {
    const int cap = 2 * n + 2;
    int* segs = (int*)malloc(sizeof(int) * 5 * cap);
    int* reps = (int*)malloc(sizeof(int) * n);
    int L, rows, ns;
    long long pad;
    const int st = so_pack(kv_lens, n, pack_width > 0 ? pack_width : n, &L, &rows, segs, cap, &ns, &pad, reps);
    if (st == 0) {
      *padding = pad;
      *tokens = (long long)rows * L;
      for (int i = 0; i < n; ++i) *tokens += (long long)reps[i] * window;
    }
    free(segs);
    free(reps);
    return st;
  }
  const int st = so_naive_padding(kv_lens, n, padding);
  if (st) return st;
  long long kv = 0;
  for (int i = 0; i < n; ++i) kv += kv_lens[i];
  *tokens = kv + *padding + (long long)n * window;
  return 0;
}

/* ------------------------------------------------------- attention.cpp:67-96 */
static double dotd(const double* a, const double* b, int dim) {
  double s = 0.0;
  for (int c = 0; c < dim; ++c) s += a[c] * b[c];
  return s;
}

int so_reference_attention(int q_rows, int kv_rows, int dim, const double* q, const double* k, const double* v,
                           double* out) {
  if (kv_rows == 0) return 3;
  double* sc = (double*)malloc(sizeof(double) * kv_rows);
  for (int i = 0; i < q_rows; ++i) {
    double mx = -INFINITY;
    for (int j = 0; j < kv_rows; ++j) {
      sc[j] = dotd(q + (long)i * dim, k + (long)j * dim, dim);
      if (sc[j] > mx) mx = sc[j];
    }
    double den = 0.0;
    for (int j = 0; j < kv_rows; ++j) {
      sc[j] = exp(sc[j] - mx);
      den += sc[j];
    }
    for (int c = 0; c < dim; ++c) {
      double num = 0.0;
      for (int j = 0; j < kv_rows; ++j) num += sc[j] * v[(long)j * dim + c];
      out[(long)i * dim + c] = num / den;
    }
  }
  free(sc);
  return 0;
}

/* ------------------------------------------------------ attention.cpp:98-162
 * Layout consistency (attention.cpp:23-63), packed K/V scatter (:106-121), then
 * per request and query one shared max over all of its cells (:134-141) and an
 * indicator-gated numerator / denominator sum over the whole grid (:142-157). */
int so_decomposed_attention(int n, int dim, const int* q_rows, const int* kv_rows, const double* q,
                            const double* k, const double* v, const int* segs, int n_segs, int width, int length,
                            const int* mask, double* out) {
  const long cells = (long)width * length;
  int* rebuilt = (int*)malloc(sizeof(int) * (cells > 0 ? cells : 1));
  int st = so_build_indicator(width, length, segs, n_segs, rebuilt);
  if (st == 0 && mask != NULL && memcmp(rebuilt, mask, sizeof(int) * cells) != 0) st = 5;
  long* kofs = (long*)calloc(n + 1, sizeof(long));
  long* qofs = (long*)calloc(n + 1, sizeof(long));
  for (int i = 0; i < n; ++i) kofs[i + 1] = kofs[i] + kv_rows[i], qofs[i + 1] = qofs[i] + q_rows[i];
  char* covered = (char*)calloc(kofs[n] + 1, 1);
  for (int s = 0; st == 0 && s < n_segs; ++s) {
    const int* g = segs + 5 * s;
    if (g[0] < 0 || g[0] >= n) {
      st = 5;
      break;
    }
    for (int t = 0; t < g[3] - g[2]; ++t) {
      const int tok = g[4] + t;
      if (tok >= kv_rows[g[0]] || covered[kofs[g[0]] + tok]) {
        st = 5;
        break;
      }
      covered[kofs[g[0]] + tok] = 1;
    }
  }
  for (long i = 0; st == 0 && i < kofs[n]; ++i)
    if (!covered[i]) st = 5;
  double* pk = NULL;
  double* pv = NULL;
  if (st == 0) {
    pk = (double*)calloc(cells * dim + 1, sizeof(double));
    pv = (double*)calloc(cells * dim + 1, sizeof(double));
    for (int s = 0; s < n_segs; ++s) {
      const int* g = segs + 5 * s;
      for (int t = 0; t < g[3] - g[2]; ++t) {
        const long cell = (long)g[1] * length + g[2] + t;
        memcpy(pk + cell * dim, k + (kofs[g[0]] + g[4] + t) * dim, sizeof(double) * dim);
        memcpy(pv + cell * dim, v + (kofs[g[0]] + g[4] + t) * dim, sizeof(double) * dim);
      }
    }
    double* num = (double*)malloc(sizeof(double) * dim);
    for (int i = 0; i < n; ++i) {
      for (int qi = 0; qi < q_rows[i]; ++qi) {
        const double* qq = q + (qofs[i] + qi) * dim;
        double mx = -INFINITY;
        for (int s = 0; s < n_segs; ++s) {
          const int* g = segs + 5 * s;
          if (g[0] != i) continue;
          for (int c = g[2]; c < g[3]; ++c) {
            const double d = dotd(qq, pk + ((long)g[1] * length + c) * dim, dim);
            if (d > mx) mx = d;
          }
        }
        double den = 0.0;
        for (int c = 0; c < dim; ++c) num[c] = 0.0;
        for (long cell = 0; cell < cells; ++cell) {
          if (rebuilt[cell] != i) continue;
          const double f = exp(dotd(qq, pk + cell * dim, dim) - mx);
          den += f;
          for (int c = 0; c < dim; ++c) num[c] += f * pv[cell * dim + c];
        }
        for (int c = 0; c < dim; ++c) out[(qofs[i] + qi) * dim + c] = num[c] / den;
      }
    }
    free(num);
  }
  free(pk);
  free(pv);
  free(covered);
  free(kofs);
  free(qofs);
  free(rebuilt);
  return st;
}

/* ------------------------------------------------------- model.cpp:110-141 */
int so_sample_accepted_prefix(double p, int window, so_rng* rng) {
  int accepted = 0, alive = 1;
  for (int k = 0; k < window; ++k) {
    const int ok = so_rng_unit(rng) < p;
    if (alive && ok)
      ++accepted;
    else
      alive = 0;
  }
  return accepted;
}

double so_expected_accepted_prefix(double p, int window) {
  if (p >= 1.0) return (double)window;
  if (p <= 0.0) return 0.0;
  return (p - pow(p, window + 1)) / (1.0 - p);
}

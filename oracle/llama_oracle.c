/*
 * fp32 LLaMA-style oracle for the Spin verification path (draft loop, verify
 * forward, greedy accept with KV rollback). TEST INFRASTRUCTURE ONLY (see
 * spin_oracle.h). The reference has no network; this restates the reference's
 * *semantics* on real computation:
 *   - kv_len = prompt + generated + window             model.hpp:26-28
 *   - leading-run acceptance, + bonus token            model.cpp:110-134, slot_engine.cpp:139-141
 *   - generated_len update / commit                    slot_engine.cpp:151-156
 *   - softmax attention, max-subtracted                attention.cpp:67-96
 * Rounding points mirror the GPU exactly (bf16 storage of weights, normalised
 * activations, attention output, SwiGLU output and KV -- the tensor-core GEMM
 * inputs and HBM-resident state; fp32 everywhere else, including q),
 * so argmax tokens agree bit-for-bit and logits to ~1e-6 relative.
 */
#include <math.h>
#include <omp.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

#include "spin_oracle.h"

/* ------------------------------------------------------------------ bf16 */
static inline float bf2f(uint16_t b) {
  uint32_t u = (uint32_t)b << 16;
  float f;
  memcpy(&f, &u, 4);
  return f;
}
static inline uint16_t f2bf(float f) { /* round to nearest even, like __float2bfloat16_rn */
  uint32_t u;
  memcpy(&u, &f, 4);
  if ((u & 0x7fffffffu) > 0x7f800000u) return 0x7fc0;
  u += 0x7fffu + ((u >> 16) & 1u);
  return (uint16_t)(u >> 16);
}
static inline float rbf(float f) { return bf2f(f2bf(f)); }

/* --------------------------------------------------------- synthetic weights
 * Spec (identical in paper_2503_15921_b200/csrc/kernels.cu init_weights_kernel, engine.cu init_model):
 *   stream = mix_seed(seed, 0x5350494E, tag, layer)
 *   r      = float(splitmix64(stream + row*cols + col) >> 40) * 2^-23 - 1   in [-1, 1), exact
 *   w      = bf16_rne(r * scale)                           (one fp32 multiply)
 * lm_head row v additionally carries the planted next-token map (if v's domain is planted):
 *   w      = bf16_rne(r * scale + (planted_gain / d) * E[pi^-1(v)][col])
 */
enum { TAG_EMBED = 1, TAG_LM_HEAD = 2, TAG_QKV = 3, TAG_O = 4, TAG_GATE_UP = 5, TAG_DOWN = 6 };

static float tag_scale(const so_model_desc* m, int tag) {
  const double d = m->d_model, f = m->ffn;
  switch (tag) {
    case TAG_EMBED: return (float)(sqrt(3.0) * m->embed_scale);
    case TAG_LM_HEAD: return (float)sqrt(3.0 / d);
    case TAG_QKV:
    case TAG_GATE_UP: return (float)(sqrt(3.0 / d) * m->init_scale);
    case TAG_O: return (float)(sqrt(3.0 / d) * m->resid_scale);
    case TAG_DOWN: return (float)(sqrt(3.0 / f) * m->resid_scale);
  }
  return 0.f;
}

static int64_t tag_cols(const so_model_desc* m, int tag) { return tag == TAG_DOWN ? m->ffn : m->d_model; }

static inline float uniform_pm1(uint64_t stream, uint64_t idx) {
  return (float)(so_splitmix64(stream + idx) >> 40) * 0x1.0p-23f - 1.0f;
}

static uint64_t weight_stream(const so_model_desc* m, int tag, int layer) {
  return so_mix_seed(m->seed, 0x5350494EULL, (uint64_t)tag, (uint64_t)layer);
}

static int64_t mod_inverse(int64_t a, int64_t n) {
  int64_t t = 0, nt = 1, r = n, nr = a % n;
  while (nr != 0) {
    const int64_t q = r / nr, tt = t - q * nt, rr = r - q * nr;
    t = nt, nt = tt, r = nr, nr = rr;
  }
  return t < 0 ? t + n : t;
}

static int64_t gcd64(int64_t a, int64_t b) {
  while (b) {
    const int64_t t = a % b;
    a = b, b = t;
  }
  return a;
}

/* Domains of the planted map: nd = max(planted_domains, 1) contiguous ranges of
 * S = vocab / nd ids; inside each, pi(t) = base + (A (t - base) + C) mod S with A the
 * first value >= 7919 coprime to S (nd = 1: pi(t) = (A t + C) mod V). Row v of the
 * lm_head is planted iff bit (v / S) of planted_mask is set (mask 0 = all). */
typedef struct {
  int64_t S, A, Cc, Ainv;
  uint32_t mask;
} planted_t;

static planted_t planted_params(const so_model_desc* m) {
  planted_t p;
  const int64_t nd = m->planted_domains > 1 ? m->planted_domains : 1;
  p.S = m->vocab / nd;
  int64_t a = 7919 % p.S;
  if (a == 0) a = 1;
  while (gcd64(a, p.S) != 1) a = (a + 1) % p.S;
  p.A = a;
  p.Cc = 12345 % p.S;
  p.Ainv = mod_inverse(a, p.S);
  p.mask = m->planted_mask ? m->planted_mask : 0xffffffffu;
  return p;
}

/* pi^-1(v) if row v is planted, else -1 */
static int64_t planted_src(const planted_t* p, int64_t v) {
  const int64_t dom = v / p->S, base = dom * p->S;
  if (dom >= 32 || !((p->mask >> dom) & 1u)) return -1;
  return base + (p->Ainv * (((v - base - p->Cc) % p->S) + p->S)) % p->S;
}

int so_planted_next(const so_model_desc* m, int token) {
  const planted_t p = planted_params(m);
  const int64_t base = token / p.S * p.S;
  return (int)(base + (p.A * (token - base) + p.Cc) % p.S);
}

uint16_t so_weight_bits(const so_model_desc* m, int tag, int layer, int64_t row, int64_t col) {
  const int64_t cols = tag_cols(m, tag);
  const float s = tag_scale(m, tag);
  const float r = uniform_pm1(weight_stream(m, tag, layer), (uint64_t)(row * cols + col));
  if (tag != TAG_LM_HEAD || m->planted_gain == 0.0f) return f2bf(r * s);
  const planted_t p = planted_params(m);
  const int64_t src = planted_src(&p, row);
  if (src < 0) return f2bf(r * s);
  const float e = bf2f(so_weight_bits(m, TAG_EMBED, 0, src, col));
  const float g = (float)((double)m->planted_gain / (double)m->d_model);
  const float a = r * s;
  const float b = g * e;
  return f2bf(a + b);
}

static uint16_t* make_weight(const so_model_desc* m, int tag, int layer, int64_t rows, const uint16_t* emb) {
  const int64_t cols = tag_cols(m, tag);
  const float s = tag_scale(m, tag);
  const uint64_t stream = weight_stream(m, tag, layer);
  const int planted = tag == TAG_LM_HEAD && m->planted_gain != 0.0f;
  const planted_t p = planted_params(m);
  const float g = (float)((double)m->planted_gain / (double)m->d_model);
  uint16_t* w = (uint16_t*)malloc(sizeof(uint16_t) * rows * cols);
#pragma omp parallel for schedule(static)
  for (int64_t r = 0; r < rows; ++r) {
    const int64_t src = planted ? planted_src(&p, r) : -1;
    for (int64_t c = 0; c < cols; ++c) {
      const float a = uniform_pm1(stream, (uint64_t)(r * cols + c)) * s;
      if (src < 0) {
        w[r * cols + c] = f2bf(a);
      } else {
        const float b = g * bf2f(emb[src * cols + c]);
        w[r * cols + c] = f2bf(a + b);
      }
    }
  }
  return w;
}

/* -------------------------------------------------------------------- model */
typedef struct layer_w {
  uint16_t *qkv, *o, *gu, *dn;
} layer_w;

typedef struct model {
  so_model_desc d;
  int slots, ctx;
  uint16_t *emb, *head;
  layer_w* L;
  uint16_t *kc, *vc; /* [layer][slot][head][ctx][hd] bf16 */
  float *rcos, *rsin;  /* [ctx][hd/2] */
} model;

static size_t kv_index(const model* m, int l, int slot, int h, int pos) {
  const so_model_desc* d = &m->d;
  return ((((size_t)l * m->slots + slot) * d->n_heads + h) * m->ctx + pos) * d->head_dim;
}

static model* model_create(const so_model_desc* d, int slots, int ctx) {
  model* m = (model*)calloc(1, sizeof(model));
  m->d = *d;
  m->slots = slots;
  m->ctx = ctx;
  m->emb = make_weight(d, TAG_EMBED, 0, d->vocab, NULL);
  m->head = make_weight(d, TAG_LM_HEAD, 0, d->vocab, m->emb);
  m->L = (layer_w*)calloc(d->n_layers, sizeof(layer_w));
  for (int l = 0; l < d->n_layers; ++l) {
    m->L[l].qkv = make_weight(d, TAG_QKV, l, 3 * (int64_t)d->d_model, NULL);
    m->L[l].o = make_weight(d, TAG_O, l, d->d_model, NULL);
    m->L[l].gu = make_weight(d, TAG_GATE_UP, l, 2 * (int64_t)d->ffn, NULL);
    m->L[l].dn = make_weight(d, TAG_DOWN, l, d->d_model, NULL);
  }
  const size_t kv = (size_t)d->n_layers * slots * d->n_heads * ctx * d->head_dim;
  m->kc = (uint16_t*)calloc(kv, sizeof(uint16_t));
  m->vc = (uint16_t*)calloc(kv, sizeof(uint16_t));
  const int half = d->head_dim / 2;
  m->rcos = (float*)malloc(sizeof(float) * (size_t)ctx * half);
  m->rsin = (float*)malloc(sizeof(float) * (size_t)ctx * half);
  for (int p = 0; p < ctx; ++p)
    for (int i = 0; i < half; ++i) {
      const double inv = pow((double)d->rope_theta, -2.0 * i / (double)d->head_dim);
      const double ang = (double)p * inv;
      m->rcos[(size_t)p * half + i] = (float)cos(ang);
      m->rsin[(size_t)p * half + i] = (float)sin(ang);
    }
  return m;
}

static void model_destroy(model* m) {
  if (!m) return;
  for (int l = 0; l < m->d.n_layers; ++l) {
    free(m->L[l].qkv), free(m->L[l].o), free(m->L[l].gu), free(m->L[l].dn);
  }
  free(m->L), free(m->emb), free(m->head), free(m->kc), free(m->vc), free(m->rcos), free(m->rsin);
  free(m);
}

/* Tie-aware argmax state (so_engine_set_hints). */
static float g_tau = 0.0f;
static long g_forced = 0;
static float g_forced_deficit = 0.0f; /* largest (own max - adopted logit) over forced decisions */

/* Debug knob (sensitivity experiments only): number of partial sums. */
static int g_lanes = 16;
void so_set_gemm_lanes(int lanes) { g_lanes = lanes == 8 ? 8 : 16; }

/* Y[t][n] = sum_k X[t][k] W[n][k]; fp32, each output accumulated in 16 fixed
 * partial sums (k mod 16) reduced by a fixed tree. Four weight rows share each
 * pass over an activation row; the per-output order is independent of that. */
static float reduce16(float* acc) {
  for (int s = 8; s > 0; s >>= 1)
    for (int j = 0; j < s; ++j) acc[j] += acc[j + s];
  return acc[0];
}

static void gemm(const float* X, int T, int K, const uint16_t* W, int N, float* Y) {
  const int nblk = (N + 3) / 4;
#pragma omp parallel
  {
    float* wr = (float*)malloc(sizeof(float) * 4 * (K + 16));
#pragma omp for schedule(dynamic, 4)
    for (int nb = 0; nb < nblk; ++nb) {
      const int n0 = nb * 4, nn = N - n0 < 4 ? N - n0 : 4;
      for (int r = 0; r < nn; ++r)
        for (int k = 0; k < K; ++k) wr[r * (K + 16) + k] = bf2f(W[(size_t)(n0 + r) * K + k]);
      for (int t = 0; t < T; ++t) {
        const float* x = X + (size_t)t * K;
        if (g_lanes == 16 && nn == 4) {
          float a0[16] = {0}, a1[16] = {0}, a2[16] = {0}, a3[16] = {0};
          const float *w0 = wr, *w1 = wr + (K + 16), *w2 = wr + 2 * (K + 16), *w3 = wr + 3 * (K + 16);
          int k = 0;
          for (; k + 16 <= K; k += 16)
            for (int j = 0; j < 16; ++j) {
              const float xv = x[k + j];
              a0[j] += xv * w0[k + j];
              a1[j] += xv * w1[k + j];
              a2[j] += xv * w2[k + j];
              a3[j] += xv * w3[k + j];
            }
          for (int j = 0; k < K; ++k, ++j) {
            a0[j] += x[k] * w0[k];
            a1[j] += x[k] * w1[k];
            a2[j] += x[k] * w2[k];
            a3[j] += x[k] * w3[k];
          }
          Y[(size_t)t * N + n0] = reduce16(a0);
          Y[(size_t)t * N + n0 + 1] = reduce16(a1);
          Y[(size_t)t * N + n0 + 2] = reduce16(a2);
          Y[(size_t)t * N + n0 + 3] = reduce16(a3);
          continue;
        }
        for (int r = 0; r < nn; ++r) {
          const float* w = wr + r * (K + 16);
          float acc[16] = {0};
          int k = 0;
          if (g_lanes == 16) {
            for (; k + 16 <= K; k += 16)
              for (int j = 0; j < 16; ++j) acc[j] += x[k + j] * w[k + j];
            for (int j = 0; k < K; ++k, ++j) acc[j] += x[k] * w[k];
          } else {
            for (; k < K; ++k) acc[k & 7] += x[k] * w[k];
          }
          Y[(size_t)t * N + n0 + r] = reduce16(acc);
        }
      }
    }
    free(wr);
  }
}

static void rmsnorm_bf16(const float* h, int T, int d, float eps, float* x) {
  for (int t = 0; t < T; ++t) {
    const float* r = h + (size_t)t * d;
    float ss = 0.f;
    for (int i = 0; i < d; ++i) ss += r[i] * r[i];
    const float inv = 1.0f / sqrtf(ss / (float)d + eps);
    for (int i = 0; i < d; ++i) x[(size_t)t * d + i] = rbf(r[i] * inv);
  }
}

/* Forward of T tokens (slot, pos) through the model; writes KV at (slot, pos)
 * and attends causally over keys [0, pos] of the slot. */
/* Debug capture (sensitivity experiments): residual stream after each layer of
 * the last forward, up to 64 layers x 4096 floats. */
static float g_dbg[64][4096];
static float g_dbg2[8][4][4096]; /* layer<8: attn-out, o-proj, act, down */
static int g_dbg_n = 0;
void so_debug_inner(int layer, int which, float* out, int n) {
  memcpy(out, g_dbg2[layer][which], sizeof(float) * (n < 4096 ? n : 4096));
}
void so_debug_layer(int layer, float* out, int n) {
  memcpy(out, g_dbg[layer], sizeof(float) * (n < 4096 ? n : 4096));
}

static double now_s(void) {
  struct timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return (double)ts.tv_sec + 1e-9 * (double)ts.tv_nsec;
}
static double g_t_blocks = 0.0, g_t_head = 0.0; /* seconds spent in the last forward */

static void model_forward_gap(model* m, int T, const int* tok, const int* slot, const int* pos, int* amax,
                              float* logits, float* gap, const int* hint);
static void model_forward(model* m, int T, const int* tok, const int* slot, const int* pos, int* amax,
                          float* logits) {
  model_forward_gap(m, T, tok, slot, pos, amax, logits, NULL, NULL);
}

/* gap[t] (optional) = top-1 minus top-2 logit: the decision margin of row t.
 * hint[t] >= 0 (optional): a tie-aware argmax -- the hinted token is taken when
 * its logit is within g_tau of the maximum (a near-tie at the bf16 noise floor);
 * every such override is counted in g_forced. */
static void model_forward_gap(model* m, int T, const int* tok, const int* slot, const int* pos, int* amax,
                              float* logits, float* gap, const int* hint) {
  const double t0 = now_s();
  const so_model_desc* d = &m->d;
  const int D = d->d_model, H = d->n_heads, hd = d->head_dim, F = d->ffn, V = d->vocab, half = hd / 2;
  const float scale = (float)(1.0 / sqrt((double)hd));
  float* h = (float*)malloc(sizeof(float) * (size_t)T * D);
  float* x = (float*)malloc(sizeof(float) * (size_t)T * (F > D ? F : D));
  float* y = (float*)malloc(sizeof(float) * (size_t)T * (2 * F > 3 * D ? 2 * F : 3 * D));
  float* q = (float*)malloc(sizeof(float) * (size_t)T * D);
  for (int t = 0; t < T; ++t)
    for (int i = 0; i < D; ++i) h[(size_t)t * D + i] = bf2f(m->emb[(size_t)tok[t] * D + i]);
  for (int l = 0; l < d->n_layers; ++l) {
    rmsnorm_bf16(h, T, D, d->rms_eps, x);
    gemm(x, T, D, m->L[l].qkv, 3 * D, y);
    for (int t = 0; t < T; ++t) {
      const float* c = m->rcos + (size_t)pos[t] * half;
      const float* s = m->rsin + (size_t)pos[t] * half;
      float* row = y + (size_t)t * 3 * D;
      for (int hh = 0; hh < H; ++hh) {
        float* qh = row + hh * hd;
        float* kh = row + D + hh * hd;
        const float* vh = row + 2 * D + hh * hd;
        uint16_t* kd = m->kc + kv_index(m, l, slot[t], hh, pos[t]);
        uint16_t* vd = m->vc + kv_index(m, l, slot[t], hh, pos[t]);
        for (int i = 0; i < half; ++i) {
          const float q0 = qh[i], q1 = qh[i + half], k0 = kh[i], k1 = kh[i + half];
          const float a = q0 * c[i], b = q1 * s[i], e = q1 * c[i], f = q0 * s[i];
          q[(size_t)t * D + hh * hd + i] = a - b;
          q[(size_t)t * D + hh * hd + i + half] = e + f;
          const float ka = k0 * c[i], kb = k1 * s[i], ke = k1 * c[i], kf = k0 * s[i];
          kd[i] = f2bf(ka - kb);
          kd[i + half] = f2bf(ke + kf);
        }
        for (int i = 0; i < hd; ++i) vd[i] = f2bf(vh[i]);
      }
    }
    /* attention: softmax(q k^T * scale) v over keys [0, pos] */
#pragma omp parallel for collapse(2) schedule(dynamic)
    for (int t = 0; t < T; ++t)
      for (int hh = 0; hh < H; ++hh) {
        const int nk = pos[t] + 1;
        float* sc = (float*)malloc(sizeof(float) * nk);
        const float* qq = q + (size_t)t * D + hh * hd;
        float mx = -INFINITY;
        for (int j = 0; j < nk; ++j) {
          const uint16_t* kr = m->kc + kv_index(m, l, slot[t], hh, j);
          float acc = 0.f;
          for (int i = 0; i < hd; ++i) acc += qq[i] * bf2f(kr[i]);
          sc[j] = acc * scale;
          if (sc[j] > mx) mx = sc[j];
        }
        float den = 0.f;
        float o[256];
        for (int i = 0; i < hd; ++i) o[i] = 0.f;
        for (int j = 0; j < nk; ++j) {
          const float p = expf(sc[j] - mx);
          den += p;
          const uint16_t* vr = m->vc + kv_index(m, l, slot[t], hh, j);
          for (int i = 0; i < hd; ++i) o[i] += p * bf2f(vr[i]);
        }
        for (int i = 0; i < hd; ++i) x[(size_t)t * D + hh * hd + i] = rbf(o[i] / den);
        free(sc);
      }
#define DBG(w, src, cnt) if (l < 8) memcpy(g_dbg2[l][w], src, sizeof(float) * ((size_t)(cnt) < 4096 ? (size_t)(cnt) : 4096))
    DBG(0, x, (size_t)T * D);
    gemm(x, T, D, m->L[l].o, D, y);
    DBG(1, y, (size_t)T * D);
    for (size_t i = 0; i < (size_t)T * D; ++i) h[i] += y[i];
    rmsnorm_bf16(h, T, D, d->rms_eps, x);
    gemm(x, T, D, m->L[l].gu, 2 * F, y);
    for (int t = 0; t < T; ++t)
      for (int i = 0; i < F; ++i) {
        const float g = y[(size_t)t * 2 * F + i], u = y[(size_t)t * 2 * F + F + i];
        const float sg = g / (1.0f + expf(-g));
        x[(size_t)t * F + i] = rbf(sg * u);
      }
    DBG(2, x, (size_t)T * F);
    gemm(x, T, F, m->L[l].dn, D, y);
    DBG(3, y, (size_t)T * D);
    for (size_t i = 0; i < (size_t)T * D; ++i) h[i] += y[i];
    if (l < 64) memcpy(g_dbg[l], h, sizeof(float) * ((size_t)T * D < 4096 ? (size_t)T * D : 4096));
  }
  g_dbg_n = d->n_layers;
  const double t1 = now_s();
  rmsnorm_bf16(h, T, D, d->rms_eps, x);
  float* lg = logits ? logits : (float*)malloc(sizeof(float) * (size_t)T * V);
  gemm(x, T, D, m->head, V, lg);
  for (int t = 0; t < T; ++t) {
    const float* r = lg + (size_t)t * V;
    int best = 0;
    for (int v = 1; v < V; ++v)
      if (r[v] > r[best]) best = v;
    amax[t] = best;
    if (hint && hint[t] >= 0 && hint[t] < V && hint[t] != best && r[hint[t]] >= r[best] - g_tau) {
      amax[t] = hint[t];
      ++g_forced;
      if (r[best] - r[hint[t]] > g_forced_deficit) g_forced_deficit = r[best] - r[hint[t]];
    }
    if (gap) {
      float second = -INFINITY;
      for (int v = 0; v < V; ++v)
        if (v != best && r[v] > second) second = r[v];
      gap[t] = r[best] - second;
    }
  }
  if (!logits) free(lg);
  free(h), free(x), free(y), free(q);
  g_t_blocks = t1 - t0;
  g_t_head = now_s() - t1;
}

/* ------------------------------------------------------------------- engine */
struct so_engine {
  model* target;
  model** ssm;
  int n_ssm, slots, ctx, window;
  int* tokens;    /* [slot][ctx] committed token history */
  int* committed; /* [slot] */
  int* ssm_len;   /* [ssm][slot] KV positions valid in the SSM cache */
};

so_engine* so_engine_create(const so_model_desc* target, const so_model_desc* ssms, int n_ssm, int max_slots,
                            int max_ctx, int window, int n_threads) {
  if (n_threads > 0) omp_set_num_threads(n_threads);
  so_engine* e = (so_engine*)calloc(1, sizeof(so_engine));
  e->target = model_create(target, max_slots, max_ctx);
  e->ssm = (model**)calloc(n_ssm > 0 ? n_ssm : 1, sizeof(model*));
  for (int j = 0; j < n_ssm; ++j) e->ssm[j] = model_create(&ssms[j], max_slots, max_ctx);
  e->n_ssm = n_ssm;
  e->slots = max_slots;
  e->ctx = max_ctx;
  e->window = window;
  e->tokens = (int*)calloc((size_t)max_slots * max_ctx, sizeof(int));
  e->committed = (int*)calloc(max_slots, sizeof(int));
  e->ssm_len = (int*)calloc((size_t)(n_ssm > 0 ? n_ssm : 1) * max_slots, sizeof(int));
  return e;
}

void so_engine_destroy(so_engine* e) {
  if (!e) return;
  model_destroy(e->target);
  for (int j = 0; j < e->n_ssm; ++j) model_destroy(e->ssm[j]);
  free(e->ssm), free(e->tokens), free(e->committed), free(e->ssm_len), free(e);
}

/* Runs `m` over positions [from, to) of each listed slot (ragged extend). */
static void extend(so_engine* e, model* m, int n, const int* slots, const int* from, const int* to) {
  int T = 0;
  for (int i = 0; i < n; ++i) T += to[i] > from[i] ? to[i] - from[i] : 0;
  if (T == 0) return;
  int *tok = (int*)malloc(sizeof(int) * T), *sl = (int*)malloc(sizeof(int) * T), *ps = (int*)malloc(sizeof(int) * T);
  int *am = (int*)malloc(sizeof(int) * T), k = 0;
  for (int i = 0; i < n; ++i)
    for (int p = from[i]; p < to[i]; ++p) tok[k] = e->tokens[(size_t)slots[i] * e->ctx + p], sl[k] = slots[i], ps[k++] = p;
  model_forward(m, T, tok, sl, ps, am, NULL);
  free(tok), free(sl), free(ps), free(am);
}

int so_engine_prefill(so_engine* e, int n, const int* slots, const int* prompt_lens, const int* prompts) {
  int* from = (int*)calloc(n, sizeof(int));
  int* to = (int*)calloc(n, sizeof(int));
  int off = 0;
  for (int i = 0; i < n; ++i) {
    if (prompt_lens[i] < 2 || prompt_lens[i] > e->ctx) return 3;
    memcpy(e->tokens + (size_t)slots[i] * e->ctx, prompts + off, sizeof(int) * prompt_lens[i]);
    off += prompt_lens[i];
    e->committed[slots[i]] = prompt_lens[i];
    to[i] = prompt_lens[i] - 1;
  }
  extend(e, e->target, n, slots, from, to);
  for (int j = 0; j < e->n_ssm; ++j) {
    extend(e, e->ssm[j], n, slots, from, to);
    for (int i = 0; i < n; ++i) e->ssm_len[(size_t)j * e->slots + slots[i]] = to[i];
  }
  free(from), free(to);
  return 0;
}

/* Recomputes SSM KV up to committed-2 for requests whose cache lags
 * (switching_cost, slot_engine.cpp:12-22). */
int so_engine_switch(so_engine* e, int n, const int* slots, const int* ssm_of) {
  for (int j = 0; j < e->n_ssm; ++j) {
    int *sl = (int*)malloc(sizeof(int) * n), *fr = (int*)malloc(sizeof(int) * n), *to = (int*)malloc(sizeof(int) * n), c = 0;
    for (int i = 0; i < n; ++i) {
      if (ssm_of[i] != j) continue;
      const int s = slots[i], need = e->committed[s] - 2;
      int* len = &e->ssm_len[(size_t)j * e->slots + s];
      if (*len < need) {
        sl[c] = s, fr[c] = *len, to[c] = need, ++c;
        *len = need;
      }
    }
    extend(e, e->ssm[j], c, sl, fr, to);
    free(sl), free(fr), free(to);
  }
  return 0;
}

static double g_round_draft = 0.0, g_round_vblocks = 0.0, g_round_vhead = 0.0;
static const int* g_draft_hint = NULL;  /* [n][window] GPU draft tokens for the next round */
static const int* g_target_hint = NULL; /* [rows] GPU target argmax for the next round */
void so_engine_set_hints(const int* draft_hint, const int* target_hint, float tau) {
  g_draft_hint = draft_hint;
  g_target_hint = target_hint;
  g_tau = tau;
}
long so_engine_forced_count(void) { return g_forced; }
float so_engine_forced_deficit(void) { return g_forced_deficit; }
void so_engine_reset_forced(void) {
  g_forced = 0;
  g_forced_deficit = 0.0f;
}
static float* g_draft_gap = NULL;  /* [n][window] per next so_engine_round, optional */
static float* g_target_gap = NULL; /* [rows] */
void so_engine_set_gap_outputs(float* draft_gap, float* target_gap) {
  g_draft_gap = draft_gap;
  g_target_gap = target_gap;
}
void so_engine_last_timing(double* draft_s, double* verify_blocks_s, double* verify_head_s) {
  *draft_s = g_round_draft, *verify_blocks_s = g_round_vblocks, *verify_head_s = g_round_vhead;
}

int so_engine_round(so_engine* e, int n, const int* slots, const int* ssm_of, int* accepted, int* bonus,
                    int* committed, int* drafts, int* target_tokens, float* logits) {
  const int g = e->window;
  const double r0 = now_s();
  for (int i = 0; i < n; ++i) {
    if (ssm_of[i] < -1 || ssm_of[i] >= e->n_ssm) return 3;
    if (ssm_of[i] >= 0 && e->committed[slots[i]] + g + 1 > e->ctx) return 2;
  }
  so_engine_switch(e, n, slots, ssm_of);
  int* dr = (int*)calloc((size_t)n * g + 1, sizeof(int));
  /* ---- draft: every SSM batch, gamma greedy steps (step 0 re-feeds the last two committed tokens) */
  for (int j = 0; j < e->n_ssm; ++j) {
    int cnt = 0;
    for (int i = 0; i < n; ++i) cnt += ssm_of[i] == j;
    if (!cnt) continue;
    int *idx = (int*)malloc(sizeof(int) * cnt), *tok = (int*)malloc(sizeof(int) * 2 * cnt),
        *sl = (int*)malloc(sizeof(int) * 2 * cnt), *ps = (int*)malloc(sizeof(int) * 2 * cnt),
        *am = (int*)malloc(sizeof(int) * 2 * cnt);
    int k = 0;
    for (int i = 0; i < n; ++i) {
      if (ssm_of[i] != j) continue;
      const int s = slots[i], c = e->committed[s];
      idx[k / 2] = i;
      for (int r = 0; r < 2; ++r) {
        tok[k] = e->tokens[(size_t)s * e->ctx + c - 2 + r], sl[k] = s, ps[k] = c - 2 + r;
        ++k;
      }
    }
    float* gp = (float*)malloc(sizeof(float) * 2 * cnt);
    int* hn = (int*)malloc(sizeof(int) * 2 * cnt);
    for (int b = 0; b < cnt; ++b) {
      hn[2 * b] = -1;
      hn[2 * b + 1] = g_draft_hint ? g_draft_hint[(size_t)idx[b] * g] : -1;
    }
    model_forward_gap(e->ssm[j], 2 * cnt, tok, sl, ps, am, NULL, gp, hn);
    for (int b = 0; b < cnt; ++b) {
      dr[(size_t)idx[b] * g] = am[2 * b + 1];
      if (g_draft_gap) g_draft_gap[(size_t)idx[b] * g] = gp[2 * b + 1];
    }
    for (int step = 1; step < g; ++step) {
      for (int b = 0; b < cnt; ++b) {
        const int s = slots[idx[b]];
        tok[b] = dr[(size_t)idx[b] * g + step - 1], sl[b] = s, ps[b] = e->committed[s] - 1 + step;
      }
      for (int b = 0; b < cnt; ++b) hn[b] = g_draft_hint ? g_draft_hint[(size_t)idx[b] * g + step] : -1;
      model_forward_gap(e->ssm[j], cnt, tok, sl, ps, am, NULL, gp, hn);
      for (int b = 0; b < cnt; ++b) {
        dr[(size_t)idx[b] * g + step] = am[b];
        if (g_draft_gap) g_draft_gap[(size_t)idx[b] * g + step] = gp[b];
      }
    }
    free(gp);
    free(hn);
    for (int b = 0; b < cnt; ++b) {
      const int s = slots[idx[b]];
      e->ssm_len[(size_t)j * e->slots + s] = e->committed[s] + g - 1;
    }
    free(idx), free(tok), free(sl), free(ps), free(am);
  }
  g_round_draft = now_s() - r0;
  g_round_vblocks = g_round_vhead = 0.0;
  /* ---- verify: rows (pending, d_1..d_g) at positions c-1 .. c+g-1 */
  int act = 0;
  for (int i = 0; i < n; ++i) act += ssm_of[i] >= 0;
  const int T = act * (g + 1);
  int *tok = (int*)malloc(sizeof(int) * (T + 1)), *sl = (int*)malloc(sizeof(int) * (T + 1)),
      *ps = (int*)malloc(sizeof(int) * (T + 1)), *am = (int*)malloc(sizeof(int) * (T + 1));
  int k = 0;
  for (int i = 0; i < n; ++i) {
    if (ssm_of[i] < 0) continue;
    const int s = slots[i], c = e->committed[s];
    for (int r = 0; r <= g; ++r) {
      tok[k] = r == 0 ? e->tokens[(size_t)s * e->ctx + c - 1] : dr[(size_t)i * g + r - 1];
      sl[k] = s, ps[k] = c - 1 + r;
      ++k;
    }
  }
  if (T > 0) {
    model_forward_gap(e->target, T, tok, sl, ps, am, logits, g_target_gap, g_target_hint);
    g_round_vblocks = g_t_blocks;
    g_round_vhead = g_t_head;
  }
  /* ---- accept: leading run of drafts equal to the target argmax, plus bonus */
  k = 0;
  for (int i = 0; i < n; ++i) {
    const int s = slots[i];
    if (ssm_of[i] < 0) {
      if (accepted) accepted[i] = 0;
      if (bonus) bonus[i] = -1;
      if (committed) committed[i] = e->committed[s];
      continue;
    }
    const int* y = am + k;
    const int* dd = dr + (size_t)i * g;
    int a = 0;
    while (a < g && dd[a] == y[a]) ++a;
    const int c = e->committed[s];
    for (int r = 0; r < a; ++r) e->tokens[(size_t)s * e->ctx + c + r] = dd[r];
    e->tokens[(size_t)s * e->ctx + c + a] = y[a];
    e->committed[s] = c + a + 1;
    int* len = &e->ssm_len[(size_t)ssm_of[i] * e->slots + s];
    if (*len > c + a) *len = c + a;
    if (accepted) accepted[i] = a;
    if (bonus) bonus[i] = y[a];
    if (committed) committed[i] = e->committed[s];
    if (drafts) memcpy(drafts + (size_t)i * g, dd, sizeof(int) * g);
    if (target_tokens) memcpy(target_tokens + (size_t)i * (g + 1), y, sizeof(int) * (g + 1));
    k += g + 1;
  }
  free(tok), free(sl), free(ps), free(am), free(dr);
  return 0;
}

int so_engine_read_tokens(so_engine* e, int slot, int* tokens, int cap, int* len) {
  if (slot < 0 || slot >= e->slots) return 3;
  const int c = e->committed[slot];
  *len = c;
  memcpy(tokens, e->tokens + (size_t)slot * e->ctx, sizeof(int) * (c < cap ? c : cap));
  return 0;
}

double so_engine_verify_seconds(so_engine* e, int n, const int* slots) {
  const int g = e->window, T = n * (g + 1);
  int *tok = (int*)malloc(sizeof(int) * T), *sl = (int*)malloc(sizeof(int) * T), *ps = (int*)malloc(sizeof(int) * T),
      *am = (int*)malloc(sizeof(int) * T);
  int k = 0;
  for (int i = 0; i < n; ++i) {
    const int s = slots[i], c = e->committed[s];
    for (int r = 0; r <= g; ++r) {
      const int prev = r == 0 ? e->tokens[(size_t)s * e->ctx + c - 1] : tok[k - 1];
      tok[k] = r == 0 ? prev : so_planted_next(&e->target->d, prev);
      sl[k] = s, ps[k] = c - 1 + r;
      ++k;
    }
  }
  struct timespec a, b;
  clock_gettime(CLOCK_MONOTONIC, &a);
  model_forward(e->target, T, tok, sl, ps, am, NULL);
  clock_gettime(CLOCK_MONOTONIC, &b);
  free(tok), free(sl), free(ps), free(am);
  return (double)(b.tv_sec - a.tv_sec) + 1e-9 * (double)(b.tv_nsec - a.tv_nsec);
}

/* Ragged verification without commit (BASELINE config 3): request i verifies
 * draft_lens[i] drafts -- rows (pending, d_1..d_len) at positions c-1 .. c-1+len --
 * through the target; target_out gets the argmax of every row (request-major,
 * sum(len+1) entries). KV rows at those positions are (re)written, nothing is
 * committed (the GPU's spin_verify_bench contract). hint: GPU argmax per row or
 * NULL (tie-aware, see so_engine_set_hints); logits: [rows][vocab] or NULL. */
int so_engine_verify_ragged(so_engine* e, int n, const int* slots, const int* draft_lens, const int* drafts,
                            const int* hint, int* target_out, float* logits) {
  int T = 0;
  for (int i = 0; i < n; ++i) {
    if (slots[i] < 0 || slots[i] >= e->slots || draft_lens[i] < 0) return 3;
    if (e->committed[slots[i]] + draft_lens[i] > e->ctx) return 2;
    T += draft_lens[i] + 1;
  }
  int *tok = (int*)malloc(sizeof(int) * (T + 1)), *sl = (int*)malloc(sizeof(int) * (T + 1)),
      *ps = (int*)malloc(sizeof(int) * (T + 1));
  int k = 0, d = 0;
  for (int i = 0; i < n; ++i) {
    const int s = slots[i], c = e->committed[s];
    for (int r = 0; r <= draft_lens[i]; ++r) {
      tok[k] = r == 0 ? e->tokens[(size_t)s * e->ctx + c - 1] : drafts[d + r - 1];
      sl[k] = s, ps[k] = c - 1 + r;
      ++k;
    }
    d += draft_lens[i];
  }
  if (T > 0) model_forward_gap(e->target, T, tok, sl, ps, target_out, logits, NULL, hint);
  free(tok), free(sl), free(ps);
  return 0;
}

/* CPU-baseline setup (bench.py): admits slots with a committed history of lens[i]
 * seeded tokens and fills every model's KV cache rows [0, lens[i]-1) with seeded
 * bf16 values in [-1, 1) instead of running the prefill forward. The timed
 * verify / draft work on such a context costs exactly what it costs after a real
 * prefill of the same length; the outcomes are not comparable with the GPU. */
static void fill_kv(model* m, int slot, int upto, uint64_t seed) {
  const so_model_desc* d = &m->d;
  const int64_t per = (int64_t)upto * d->head_dim;
#pragma omp parallel for collapse(2) schedule(static)
  for (int l = 0; l < d->n_layers; ++l)
    for (int h = 0; h < d->n_heads; ++h) {
      uint16_t* kd = m->kc + kv_index(m, l, slot, h, 0);
      uint16_t* vd = m->vc + kv_index(m, l, slot, h, 0);
      const uint64_t st = so_mix_seed(seed, (uint64_t)slot, (uint64_t)l, (uint64_t)h);
      for (int64_t i = 0; i < per; ++i) {
        kd[i] = f2bf(uniform_pm1(st, (uint64_t)(2 * i)));
        vd[i] = f2bf(uniform_pm1(st, (uint64_t)(2 * i + 1)));
      }
    }
}

int so_engine_fake_context(so_engine* e, int n, const int* slots, const int* lens, uint64_t seed) {
  for (int i = 0; i < n; ++i) {
    const int s = slots[i], L = lens[i];
    if (s < 0 || s >= e->slots || L < 2 || L > e->ctx) return 3;
    for (int p = 0; p < L; ++p)
      e->tokens[(size_t)s * e->ctx + p] = (int)(so_splitmix64(so_mix_seed(seed, 7, (uint64_t)s, (uint64_t)p)) %
                                                (uint64_t)e->target->d.vocab);
    e->committed[s] = L;
    fill_kv(e->target, s, L - 1, so_mix_seed(seed, 1, 0, 0));
    for (int j = 0; j < e->n_ssm; ++j) {
      fill_kv(e->ssm[j], s, L - 1, so_mix_seed(seed, 2, (uint64_t)j, 0));
      e->ssm_len[(size_t)j * e->slots + s] = L - 1;
    }
  }
  return 0;
}

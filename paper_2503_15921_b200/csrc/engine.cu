// Engine: synthetic models on the device, forward orchestration, the
// speculate -> verify -> accept round (SlotEngine::run_slot, slot_engine.cpp:70-167)
// captured as one CUDA graph per assignment shape, SSM drafts on their own
// streams joined before verification.
#include "engine.hpp"

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>

#include "status.hpp"

namespace spin {

namespace {

constexpr int kExtendRows = 512;  // rows per prefill / catch-up chunk
constexpr int kExtendQ = 8;       // queries per virtual request in a chunk

uint64_t host_splitmix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}
uint64_t host_mix_seed(uint64_t seed, uint64_t a, uint64_t b, uint64_t c) {
  uint64_t h = host_splitmix64(seed);
  h = host_splitmix64(h ^ a);
  h = host_splitmix64(h ^ b);
  return host_splitmix64(h ^ c);
}

enum { kTagEmbed = 1, kTagHead = 2, kTagQkv = 3, kTagO = 4, kTagGateUp = 5, kTagDown = 6 };

int64_t gcd64(int64_t a, int64_t b) {
  while (b) {
    const int64_t t = a % b;
    a = b;
    b = t;
  }
  return a;
}
int64_t mod_inverse(int64_t a, int64_t n) {
  int64_t t = 0, nt = 1, r = n, nr = a % n;
  while (nr != 0) {
    const int64_t q = r / nr, tt = t - q * nt, rr = r - q * nr;
    t = nt, nt = tt, r = nr, nr = rr;
  }
  return t < 0 ? t + n : t;
}

template <typename T>
T* dalloc(std::vector<void*>& list, size_t count) {
  void* p = nullptr;
  check_cuda(cudaMalloc(&p, std::max<size_t>(count, 1) * sizeof(T)), "cudaMalloc");
  list.push_back(p);
  return static_cast<T*>(p);
}

void validate_desc(const spin_model_desc& d, const char* who) {
  const std::string w(who);
  if (d.d_model < 64 || d.n_layers < 1 || d.n_heads < 1 || d.vocab < 2 || d.ffn < 8)
    fail(SPIN_CONFIG_ERROR, w + ": model dimensions out of range");
  if (d.head_dim != 64 && d.head_dim != 128) fail(SPIN_CONFIG_ERROR, w + ": head_dim must be 64 or 128");
  if (d.n_heads * d.head_dim != d.d_model) fail(SPIN_CONFIG_ERROR, w + ": n_heads * head_dim must equal d_model");
  if (d.d_model % 64 != 0 || d.ffn % 8 != 0) fail(SPIN_CONFIG_ERROR, w + ": d_model % 64 and ffn % 8 required");
  if (d.d_model > 8192) fail(SPIN_CONFIG_ERROR, w + ": d_model above 8192 unsupported");
  if (!(d.rope_theta > 0.f) || !(d.rms_eps > 0.f)) fail(SPIN_CONFIG_ERROR, w + ": rope_theta / rms_eps must be > 0");
  if (d.planted_domains < 0 || d.planted_domains > 32 ||
      (d.planted_domains > 1 && d.vocab % d.planted_domains != 0))
    fail(SPIN_CONFIG_ERROR, w + ": planted_domains must be 0..32 and divide the vocabulary");
}

}  // namespace

struct Engine::RoundPlan {
  std::vector<int> key;  // [n_act, n_0 .. n_{M-1}]
  int n_act = 0;
  std::vector<int> n_ssm;
  int off_list = 0, off_ssm_of = 0;
  std::vector<int> off_ssm_list;
  int in_ints = 0, out_ints = 0;
  int64_t launches = 0;  // kernels per round
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
};

// ------------------------------------------------------------------ models
void Engine::init_model(ModelDev& m, const spin_model_desc& d, bool draft) {
  m.d = d;
  m.D = d.d_model, m.H = d.n_heads, m.hd = d.head_dim, m.F = d.ffn, m.V = d.vocab, m.L = d.n_layers;
  const size_t D = m.D, F = m.F, V = m.V;
  // GEMM weights in the tiled layout (gemm.cuh); the embedding stays row-major (gathered)
  const size_t n_qkv = tiled_weight_elems(3 * D, D), n_o = tiled_weight_elems(D, D);
  const size_t n_gu = tiled_weight_elems(2 * F, D), n_dn = tiled_weight_elems(D, F);
  const size_t per_layer = n_qkv + n_o + n_gu + n_dn;
  const size_t total = V * D + tiled_weight_elems(V, D) + per_layer * m.L;
  m.weight_bytes = total * 2;
  check_cuda(cudaMalloc(&m.wbuf, m.weight_bytes), "weights");
  m.emb = m.wbuf;
  m.head = m.wbuf + V * D;
  bf16* p = m.head + tiled_weight_elems(V, D);
  m.layers.resize(m.L);
  for (int l = 0; l < m.L; ++l) {
    LayerW& w = m.layers[l];
    w.qkv = p, p += n_qkv;
    w.o = p, p += n_o;
    w.gu = p, p += n_gu;
    w.dn = p, p += n_dn;
  }
  // Synthetic weights, same spec as oracle/llama_oracle.c.
  auto stream_of = [&](int tag, int layer) { return host_mix_seed(d.seed, 0x5350494EULL, tag, layer); };
  const float s_emb = static_cast<float>(std::sqrt(3.0) * d.embed_scale);
  const float s_head = static_cast<float>(std::sqrt(3.0 / D));
  const float s_in = static_cast<float>(std::sqrt(3.0 / D) * d.init_scale);
  const float s_o = static_cast<float>(std::sqrt(3.0 / D) * d.resid_scale);
  const float s_dn = static_cast<float>(std::sqrt(3.0 / F) * d.resid_scale);
  launch_init_weights(m.emb, V, D, stream_of(kTagEmbed, 0), s_emb, nullptr, 0.f, V, 1, 0, 0u, 0, sv_);
  // planted map: pi maps each of nd domains of S ids onto itself (spin_c.h planted_domains)
  const int64_t nd = d.planted_domains > 1 ? d.planted_domains : 1, S = V / nd;
  int64_t a = 7919 % S;
  if (a == 0) a = 1;
  while (gcd64(a, S) != 1) a = (a + 1) % S;
  const int64_t cc = 12345 % S;
  const uint32_t mask = d.planted_mask ? d.planted_mask : 0xffffffffu;
  const float g = static_cast<float>(static_cast<double>(d.planted_gain) / static_cast<double>(D));
  launch_init_weights(m.head, V, D, stream_of(kTagHead, 0), s_head, d.planted_gain != 0.f ? m.emb : nullptr, g, S,
                      mod_inverse(a, S), cc, mask, 1, sv_);
  for (int l = 0; l < m.L; ++l) {
    launch_init_weights(const_cast<bf16*>(m.layers[l].qkv), 3 * D, D, stream_of(kTagQkv, l), s_in, nullptr, 0.f, V, 1,
                        0, 0u, 1, sv_);
    launch_init_weights(const_cast<bf16*>(m.layers[l].o), D, D, stream_of(kTagO, l), s_o, nullptr, 0.f, V, 1, 0, 0u, 1,
                        sv_);
    launch_init_weights(const_cast<bf16*>(m.layers[l].gu), 2 * F, D, stream_of(kTagGateUp, l), s_in, nullptr, 0.f, V,
                        1, 0, 0u, 1, sv_);
    launch_init_weights(const_cast<bf16*>(m.layers[l].dn), D, F, stream_of(kTagDown, l), s_dn, nullptr, 0.f, V, 1, 0,
                        0u, 1, sv_);
  }
  check_cuda(cudaGetLastError(), "init weights");
  // SSMs on the fused draft path also keep unit-contiguous slab copies (draft.cu)
  if (draft && draft_fused_ && draft_fused_supported(m.D, m.H, m.hd, m.F, 1)) {
    const size_t sq = draft_slab_elems(3 * D, D), so = draft_slab_elems(D, D);
    const size_t sg = draft_slab_elems(2 * F, D), sd = draft_slab_elems(D, F);
    check_cuda(cudaMalloc(&m.sbuf, (sq + so + sg + sd) * m.L * 2), "draft slabs");
    m.weight_bytes += (sq + so + sg + sd) * m.L * 2;
    bf16* q = m.sbuf;
    for (int l = 0; l < m.L; ++l) {
      LayerW& w = m.layers[l];
      launch_slab_weights(w.qkv, q, kDpQkv, 3 * D, D, m.hd, sv_), w.sqkv = q, q += sq;
      launch_slab_weights(w.o, q, kDpResid, D, D, m.hd, sv_), w.so = q, q += so;
      launch_slab_weights(w.gu, q, kDpGateUp, 2 * F, D, m.hd, sv_), w.sgu = q, q += sg;
      launch_slab_weights(w.dn, q, kDpResid, D, F, m.hd, sv_), w.sdn = q, q += sd;
    }
    check_cuda(cudaGetLastError(), "draft slabs");
  }
  // KV cache [layer][slot][head][ctx][hd], zero-filled.
  const size_t kv = static_cast<size_t>(m.L) * opts_.max_requests * m.H * opts_.max_ctx * m.hd;
  // + 16 padding rows: a 16-key tile starting near the end of the last context stays in bounds
  const size_t kv_alloc = kv + static_cast<size_t>(16) * m.hd;
  m.kv_bytes = 2 * kv_alloc * 2;
  check_cuda(cudaMalloc(&m.kc, kv_alloc * 2), "k cache");
  check_cuda(cudaMalloc(&m.vc, kv_alloc * 2), "v cache");
  check_cuda(cudaMemsetAsync(m.kc, 0, kv_alloc * 2, sv_), "memset");
  check_cuda(cudaMemsetAsync(m.vc, 0, kv_alloc * 2, sv_), "memset");
  const uint64_t rows = static_cast<uint64_t>(m.L) * opts_.max_requests * m.H * opts_.max_ctx;
  if (!encode_tmap_bf16(&m.tm_k, m.kc, rows, m.hd, 16, 64, true) ||
      !encode_tmap_bf16(&m.tm_v, m.vc, rows, m.hd, 16, 64, true))
    fail(SPIN_CUDA_ERROR, "KV tensor map encode failed");
  // RoPE tables in double, rounded once (matches the oracle bit for bit).
  const int half = m.hd / 2;
  std::vector<float> c(static_cast<size_t>(opts_.max_ctx) * half), s(c.size());
  for (int pos = 0; pos < opts_.max_ctx; ++pos)
    for (int i = 0; i < half; ++i) {
      const double inv = std::pow(static_cast<double>(d.rope_theta), -2.0 * i / static_cast<double>(m.hd));
      const double ang = static_cast<double>(pos) * inv;
      c[static_cast<size_t>(pos) * half + i] = static_cast<float>(std::cos(ang));
      s[static_cast<size_t>(pos) * half + i] = static_cast<float>(std::sin(ang));
    }
  check_cuda(cudaMalloc(&m.rcos, c.size() * 4), "rope");
  check_cuda(cudaMalloc(&m.rsin, s.size() * 4), "rope");
  check_cuda(upload_sync(m.rcos, c.data(), c.size() * 4), "rope");
  check_cuda(upload_sync(m.rsin, s.data(), s.size() * 4), "rope");
}

const GemmPlan& Engine::plan(int n_out, int k, int t, int mode, int sms) {
  std::lock_guard<std::mutex> lock(plan_mu_);  // std::map references stay valid across inserts
  if (sms <= 0 || sms > num_sms_) sms = num_sms_;
  const auto key = std::make_tuple(n_out, k, t, mode, sms);
  auto it = plans_.find(key);
  if (it == plans_.end()) {
    GemmPlan p = gemm_plan(n_out, k, t, mode, sms);
    if (!p.tile_pieces.empty()) {  // device copy of the stream-K piece table (consumer kernels)
      void* d = nullptr;
      check_cuda(cudaMalloc(&d, p.tile_pieces.size()), "piece table");
      check_cuda(upload_sync(d, p.tile_pieces.data(), p.tile_pieces.size()), "piece table");
      p.map.tbl = static_cast<const uint8_t*>(d);
      plan_tables_.push_back(d);
    }
    it = plans_.emplace(key, std::move(p)).first;
  }
  return it->second;
}

void Engine::init_lane(Lane& ln, const ModelDev& m, int T_cap, int R_cap, bool logits) {
  ln.T_cap = T_cap;
  ln.R_cap = R_cap;
  ln.rows_cap = R_cap;
  ln.seg_cap = R_cap + ln.rows_cap;
  auto& A = ln.allocs;
  ln.meta.row_tok = dalloc<int32_t>(A, T_cap);
  ln.meta.row_slot = dalloc<int32_t>(A, T_cap);
  ln.meta.row_pos = dalloc<int32_t>(A, T_cap);
  ln.meta.req_slot = dalloc<int32_t>(A, R_cap);
  ln.meta.req_qstart = dalloc<int32_t>(A, R_cap);
  ln.meta.req_qlen = dalloc<int32_t>(A, R_cap);
  ln.meta.req_kvlen = dalloc<int32_t>(A, R_cap);
  ln.meta.seg = dalloc<int32_t>(A, static_cast<size_t>(ln.seg_cap) * 5);
  ln.meta.row_ptr = dalloc<int32_t>(A, ln.rows_cap + 1);
  ln.meta.row_seg = dalloc<int32_t>(A, ln.seg_cap);
  ln.meta.req_seg0 = dalloc<int32_t>(A, R_cap);
  ln.meta.req_nseg = dalloc<int32_t>(A, R_cap);
  ln.meta.n_seg = dalloc<int32_t>(A, 2);
  ln.meta.err = d_err_;
  ln.h = dalloc<float>(A, static_cast<size_t>(T_cap) * m.D);
  ln.xn = dalloc<bf16>(A, static_cast<size_t>(T_cap) * m.D);
  ln.q = dalloc<float>(A, static_cast<size_t>(T_cap) * m.D);
  ln.attn = dalloc<bf16>(A, static_cast<size_t>(T_cap) * m.D);
  ln.act = dalloc<bf16>(A, static_cast<size_t>(T_cap) * m.F);
  ln.ssp = dalloc<float>(A, static_cast<size_t>(m.D / 16 + 1) * std::min(T_cap, kDraftMaxT));
  ln.hb = dalloc<bf16>(A, static_cast<size_t>(std::min(T_cap, kDraftMaxT)) * m.D);
  // split-K partials of the largest plan over EVERY row count this lane can run (pieces per tile
  // vary irregularly with T, and the GEMM writes them with TMA stores bounded only by the plan's
  // tensor map, not by this allocation); gemm_plan directly, so no plan is cached for each T
  size_t part = 0;
  const int shapes[4][2] = {{3 * m.D, m.D}, {m.D, m.D}, {2 * m.F, m.D}, {m.D, m.F}};
  for (auto& sh : shapes)
    for (int t = 1; t <= T_cap; ++t) {
      const GemmPlan p = gemm_plan(sh[0], sh[1], t, kGemmPartial, num_sms_);
      part = std::max(part, static_cast<size_t>(p.max_pieces) * t * sh[0]);
    }
  ln.part = dalloc<float>(A, part);
  // attention work list + split-KV partials: pieces <= segments + rows x (chunks - 1), and
  // rows x chunks x heads ~ 8 x SMs bounds the chunk splits (attn_chunks); partial slots
  // are 8 queries wide (extends) or 8 * ceil((window + 1) / 8) (verify)
  ln.piece_cap = ln.seg_cap + 8 * num_sms_ / m.H + 64;
  ln.meta.piece_cap = ln.piece_cap;
  ln.meta.item_ptr = dalloc<int32_t>(A, static_cast<size_t>(ln.rows_cap) * 16 + 1);
  ln.meta.pieces = dalloc<int32_t>(A, static_cast<size_t>(ln.piece_cap) * 16);
  ln.meta.req_pptr = dalloc<int32_t>(A, R_cap + 1);
  ln.meta.req_plist = dalloc<int32_t>(A, ln.piece_cap);
  ln.meta.n_pieces = dalloc<int32_t>(A, 1);
  ln.meta.row_len = dalloc<int32_t>(A, ln.rows_cap);
  const size_t np = static_cast<size_t>(ln.piece_cap) * m.H * (8 * ((opts_.window + 8) / 8));
  ln.aw.part_m = dalloc<float>(A, np);
  ln.aw.part_l = dalloc<float>(A, np);
  ln.aw.part_o = dalloc<float>(A, np * m.hd);
  ln.aw.counter = dalloc<int32_t>(A, static_cast<size_t>(R_cap) * m.H);
  check_cuda(zero_sync(ln.aw.counter, static_cast<size_t>(R_cap) * m.H * 4), "memset");
  const int tiles = (m.V + 127) / 128;
  ln.amax_val = dalloc<float>(A, static_cast<size_t>(tiles) * T_cap);
  ln.amax_idx = dalloc<int32_t>(A, static_cast<size_t>(tiles) * T_cap);
  if (logits) ln.logits = dalloc<float>(A, static_cast<size_t>(T_cap) * m.V);
}

// ------------------------------------------------------------------ forward
// Per-launch accounting: launch count (gpu_launches in bench.py) and, in a
// profiling round, CUDA events around each launch grouped by kernel class.
void Engine::prof_begin(int cat, cudaStream_t s) {
  ++launches_;
  if (!prof_ || capturing_) return;
  ProfRec r{cat, nullptr, nullptr, 0.0};
  check_cuda(cudaEventCreate(&r.a), "event");
  check_cuda(cudaEventCreate(&r.b), "event");
  check_cuda(cudaEventRecord(r.a, s), "event");
  prof_recs_.push_back(r);
}
void Engine::prof_end(cudaStream_t s, double bytes) {
  if (!prof_ || capturing_) return;
  check_cuda(cudaEventRecord(prof_recs_.back().b, s), "event");
  prof_recs_.back().bytes = bytes;
}

// head_mode: 0 no lm_head (prefill), 1 argmax, 2 argmax + fp32 logits.
void Engine::forward(ModelDev& m, Lane& ln, const FwdShape& sh, cudaStream_t s, int head_mode) {
  const int T = sh.T, D = m.D, F = m.F;
  const bool pdl = opts_.use_pdl != 0;
  const float eps = m.d.rms_eps;
  const int base = (&m == &target_) ? kProfTargetGemm : kProfSsmGemm;  // + {0 gemm, 1 head, 2 attn, 3 epi}
  auto gemm_bytes = [&](int n_out, int k) { return 2.0 * n_out * k + 2.0 * T * k + 2.0 * T * n_out; };
  AttnGeom g{m.H, m.hd, opts_.max_requests, opts_.max_ctx, 0, static_cast<float>(1.0 / std::sqrt(double(m.hd))),
             m.kc, m.vc};
  // Draft steps and extends of <= 32 rows (switch catch-ups, prewarm chunks) take the fused
  // draft kernels; SPIN_DRAFT_NO_FUSED_EXTEND sends the extends to the generic ones (timing).
  static const bool fused_extends = std::getenv("SPIN_DRAFT_NO_FUSED_EXTEND") == nullptr;
  if (m.sbuf != nullptr && head_mode != 2 && (sh.early || fused_extends) && draft_fused_supported(D, m.H, m.hd, F, T)) {
    forward_draft(m, ln, sh, g, s, head_mode);
    return;
  }
  prof_begin(base + 3, s);
  launch_embed_norm(m.emb, ln.meta, T, D, eps, ln.h, ln.xn, s);
  prof_end(s, 0);
  GemmEpilogue ep;
  ep.mode = kGemmPartial;
  ep.part = ln.part;
  AttnWork aw = ln.aw;
  aw.qmax = sh.qmax;
  aw.chunks = attn_chunks(sh.rows, m.H, num_sms_, sh.qmax);
  aw.early = sh.early;
  static const int vskip = [] {  // timing experiments only: skip target kernels (results invalid)
    const char* e = std::getenv("SPIN_VERIFY_SKIP");
    return e ? std::atoi(e) : 0;
  }();
  const int skip = &m == &target_ ? vskip : 0;
  for (int l = 0; l < m.L; ++l) {
    const LayerW& w = m.layers[l];
    g.layer = l;
    const GemmPlan& pq = plan(3 * D, D, T, kGemmPartial);
    prof_begin(base, s);
    const bool stamp_layer = &m == &target_ && l == 1;
    ep.st = stamp_layer ? stamp_slot(10, 2 * pq.grid) : nullptr;
    check_cuda(gemm_launch(pq, w.qkv, ln.xn, ep, s, pdl), "gemm qkv");
    prof_end(s, gemm_bytes(3 * D, D));
    if (!(skip & 1)) {
      prof_begin(base + 3, s);
      launch_qkv_epilogue(ln.part, pq.map, ln.meta, T, g, m.rcos, m.rsin, ln.q, s,
                          stamp_layer ? stamp_slot(16, qkv_epilogue_blocks(T, m.H * m.hd)) : nullptr);
      prof_end(s, 0);
    }
    prof_begin(base + 2, s);
    aw.st = stamp_layer ? stamp_slot(14, 2 * attn_ctas(sh.rows, aw.chunks, m.H, sh.qmax)) : nullptr;
    if (!(skip & 8)) launch_attention(m.tm_k, m.tm_v, ln.meta, sh.rows, sh.R, g, ln.q, aw, ln.attn, s);
    aw.st = nullptr;
    prof_end(s, 0);
    const GemmPlan& po = plan(D, D, T, kGemmPartial);
    prof_begin(base, s);
    ep.st = stamp_layer ? stamp_slot(11, 2 * po.grid) : nullptr;
    check_cuda(gemm_launch(po, w.o, ln.attn, ep, s, pdl), "gemm o");
    prof_end(s, gemm_bytes(D, D));
    if (!(skip & 2)) {
      prof_begin(base + 3, s);
      launch_resid_norm(ln.part, po.map, T, D, eps, ln.h, ln.xn, s, stamp_layer ? stamp_slot(17, T) : nullptr);
      prof_end(s, 0);
    }
    const GemmPlan& pg = plan(2 * F, D, T, kGemmPartial);
    prof_begin(base, s);
    ep.st = stamp_layer ? stamp_slot(12, 2 * pg.grid) : nullptr;
    check_cuda(gemm_launch(pg, w.gu, ln.xn, ep, s, pdl), "gemm gate_up");
    prof_end(s, gemm_bytes(2 * F, D));
    if (!(skip & 4)) {
      prof_begin(base + 3, s);
      launch_swiglu(ln.part, pg.map, T, F, ln.act, s, stamp_layer ? stamp_slot(18, swiglu_blocks(T, F)) : nullptr);
      prof_end(s, 0);
    }
    const GemmPlan& pd = plan(D, F, T, kGemmPartial);
    prof_begin(base, s);
    ep.st = stamp_layer ? stamp_slot(13, 2 * pd.grid) : nullptr;
    check_cuda(gemm_launch(pd, w.dn, ln.act, ep, s, pdl), "gemm down");
    ep.st = nullptr;
    prof_end(s, gemm_bytes(D, F));
    if (!(skip & 2)) {
      prof_begin(base + 3, s);
      launch_resid_norm(ln.part, pd.map, T, D, eps, ln.h, ln.xn, s, stamp_layer ? stamp_slot(19, T) : nullptr);
      prof_end(s, 0);
    }
  }
  if (head_mode > 0) {
    GemmEpilogue eh;
    eh.mode = kGemmArgmax;
    eh.amax_val = ln.amax_val;
    eh.amax_idx = ln.amax_idx;
    eh.logits = head_mode == 2 ? ln.logits : nullptr;
    prof_begin(base + 1, s);
    check_cuda(gemm_launch(plan(m.V, D, T, kGemmArgmax), m.head, ln.xn, eh, s, pdl), "gemm lm_head");
    prof_end(s, gemm_bytes(m.V, D));
  }
  check_cuda(cudaGetLastError(), "forward launch");
}

// Draft-step forward of an SSM over few rows (draft.cu): five launches per layer,
// epilogues inside the projections, RMSNorm folded into the consumers.
void Engine::forward_draft(ModelDev& m, Lane& ln, const FwdShape& sh, AttnGeom g, cudaStream_t s, int head_mode) {
  const int T = sh.T, D = m.D, F = m.F;
  const float eps = m.d.rms_eps;
  const int base = kProfSsmGemm;
  auto wbytes = [&](int n_out, int k) { return 2.0 * n_out * k + 2.0 * T * k + 2.0 * T * n_out; };
  prof_begin(base + 3, s);
  launch_embed_ss(m.emb, ln.meta, T, D, ln.h, ln.hb, ln.ssp, s);
  prof_end(s, 0);
  int n_ssp = 1;
  AttnWork aw = ln.aw;
  aw.qmax = sh.qmax;
  aw.chunks = attn_chunks(sh.rows, m.H, num_sms_, sh.qmax);
  aw.early = sh.early;
  DraftProj a{};
  a.T = T;
  a.eps = eps;
  a.row_slot = ln.meta.row_slot;
  a.row_pos = ln.meta.row_pos;
  a.rcos = m.rcos;
  a.rsin = m.rsin;
  a.h = ln.h;
  a.hb = ln.hb;
  a.q = ln.q;
  a.act = ln.act;
  static const int skip = [] {  // timing experiments only: skip kernels (results invalid)
    const char* e = std::getenv("SPIN_DRAFT_SKIP");
    return e ? std::atoi(e) : 0;
  }();
  for (int l = 0; l < m.L; ++l) {
    const LayerW& w = m.layers[l];
    g.layer = l;
    a.g = g;
    a.mode = kDpQkv, a.w = w.sqkv, a.n_out = 3 * D, a.K = D, a.x = ln.hb, a.ssp = ln.ssp, a.n_ssp = n_ssp;
    if (!(skip & 2)) {
      prof_begin(base, s);
      a.st = stamp_slot(0, draft_proj_units(a));
      check_cuda(launch_draft_proj(a, s), "draft qkv");
      prof_end(s, wbytes(3 * D, D));
    }
    if (!(skip & 1)) {
      prof_begin(base + 2, s);
      aw.st = stamp_slot(1, 2 * attn_ctas(sh.rows, aw.chunks, m.H, sh.qmax));  // 8 stamps per CTA
      launch_attention(m.tm_k, m.tm_v, ln.meta, sh.rows, sh.R, g, ln.q, aw, ln.attn, s);
      prof_end(s, 0);
    }
    a.mode = kDpResid, a.w = w.so, a.n_out = D, a.K = D, a.x = ln.attn, a.ssp_out = ln.ssp;
    if (!(skip & 4)) {
      prof_begin(base, s);
      a.st = stamp_slot(2, draft_proj_units(a));
      check_cuda(launch_draft_proj(a, s), "draft o");
      prof_end(s, wbytes(D, D));
    }
    n_ssp = D / 16;
    a.mode = kDpGateUp, a.w = w.sgu, a.n_out = 2 * F, a.K = D, a.x = ln.hb, a.ssp = ln.ssp, a.n_ssp = n_ssp;
    if (!(skip & 8)) {
      prof_begin(base, s);
      a.st = stamp_slot(3, draft_proj_units(a));
      check_cuda(launch_draft_proj(a, s), "draft gate_up");
      prof_end(s, wbytes(2 * F, D));
    }
    a.mode = kDpResid, a.w = w.sdn, a.n_out = D, a.K = F, a.x = ln.act, a.ssp_out = ln.ssp;
    if (!(skip & 16)) {
      prof_begin(base, s);
      a.st = stamp_slot(4, draft_proj_units(a));
      check_cuda(launch_draft_proj(a, s), "draft down");
      prof_end(s, wbytes(D, F));
    }
  }
  if (head_mode > 0) {
    prof_begin(base + 3, s);
    launch_norm_ss(ln.h, ln.ssp, n_ssp, T, D, eps, ln.xn, s);
    prof_end(s, 0);
    GemmEpilogue eh;
    eh.mode = kGemmArgmax;
    eh.amax_val = ln.amax_val;
    eh.amax_idx = ln.amax_idx;
    prof_begin(base + 1, s);
    const GemmPlan& ph = plan(m.V, D, T, kGemmArgmax, ln.head_sms);
    eh.st = stamp_slot(15, 2 * ph.grid);
    check_cuda(gemm_launch(ph, m.head, ln.xn, eh, s, opts_.use_pdl != 0), "gemm lm_head");
    prof_end(s, wbytes(m.V, D));
  }
  check_cuda(cudaGetLastError(), "draft forward launch");
}

unsigned long long* Engine::stamp_slot(int kind, int ctas) {
  if (!stamps_ || stamp_used_ + size_t(4) * ctas > stamp_cap_) return nullptr;
  stamp_tab_.push_back({kind, ctas, static_cast<int>(stamp_used_)});
  unsigned long long* p = stamps_ + stamp_used_;
  stamp_used_ += size_t(4) * ctas;
  return p;
}

void Engine::dump_stamps() {
  if (!stamps_ || stamp_tab_.empty()) return;
  std::vector<unsigned long long> h(stamp_used_);
  check_cuda(cudaMemcpy(h.data(), stamps_, stamp_used_ * 8, cudaMemcpyDeviceToHost), "stamps");
  FILE* f = std::fopen(stamp_path_.c_str(), "w");
  if (!f) return;
  std::fprintf(f, "launch,kind,cta,t0,t1,t2,t3\n");
  for (size_t l = 0; l < stamp_tab_.size(); ++l) {
    const auto& e = stamp_tab_[l];
    for (int c = 0; c < e[1]; ++c) {
      const unsigned long long* t = h.data() + e[2] + 4 * c;
      std::fprintf(f, "%zu,%d,%d,%llu,%llu,%llu,%llu\n", l, e[0], c, t[0], t[1], t[2], t[3]);
    }
  }
  std::fclose(f);
}

// ------------------------------------------------------------------ engine
Engine::Engine(const spin_model_desc& target, const spin_model_desc* ssms, int n_ssm, const spin_engine_opts& opts)
    : opts_(opts) {
  if (n_ssm < 1 || n_ssm > kMaxSsm) fail(SPIN_CONFIG_ERROR, "engine: need 1..8 SSMs");
  if (opts.max_requests < 1 || opts.max_requests > 1024) fail(SPIN_CONFIG_ERROR, "engine: max_requests in 1..1024");
  if (opts.window < 1 || opts.window > 16) fail(SPIN_CONFIG_ERROR, "engine: window must be in 1..16");
  if (opts.max_ctx < opts.window + 4) fail(SPIN_CONFIG_ERROR, "engine: max_ctx too small");
  validate_desc(target, "target");
  for (int j = 0; j < n_ssm; ++j) {
    validate_desc(ssms[j], "ssm");
    if (ssms[j].vocab != target.vocab) fail(SPIN_CONFIG_ERROR, "ssm vocabulary must match the target's");
    if (std::max(ssms[j].planted_domains, 1) != std::max(target.planted_domains, 1))
      fail(SPIN_CONFIG_ERROR, "ssm planted_domains must match the target's (one planted map)");
  }
  check_cuda(cudaSetDevice(opts.device), "cudaSetDevice");
  (void)cudaGetLastError();  // drop a stale non-sticky error left by an earlier caller
  cudaDeviceGetAttribute(&num_sms_, cudaDevAttrMultiProcessorCount, opts.device);
  if (const char* e = std::getenv("SPIN_DRAFT_FUSED")) draft_fused_ = std::atoi(e) != 0;  // A/B switch
  if (const char* e = std::getenv("SPIN_STAMPS")) {
    stamp_path_ = e;
    stamp_cap_ = size_t(8) << 20;
    check_cuda(cudaMalloc(&stamps_, stamp_cap_ * 8), "stamps");
    check_cuda(zero_sync(stamps_, stamp_cap_ * 8), "stamps");
  }
  check_cuda(cudaStreamCreateWithFlags(&sv_, cudaStreamNonBlocking), "stream");
  ss_.resize(n_ssm);
  for (auto& s : ss_) check_cuda(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking), "stream");
  // sticky device status word (FwdMeta::err), host-mapped: read after every synchronisation
  void* err_host = nullptr;
  check_cuda(cudaHostAlloc(&err_host, 8 * 4, cudaHostAllocMapped), "pinned status");  // [status, detail x 7]
  h_err_ = static_cast<volatile int32_t*>(err_host);
  for (int i = 0; i < 8; ++i) h_err_[i] = 0;
  void* err_dev = nullptr;
  check_cuda(cudaHostGetDevicePointer(&err_dev, err_host, 0), "mapped status");
  d_err_ = static_cast<int32_t*>(err_dev);
  init_model(target_, target, false);
  ssm_.resize(n_ssm);
  for (int j = 0; j < n_ssm; ++j) init_model(ssm_[j], ssms[j], true);
  const int R = opts.max_requests, W = opts.window;
  init_lane(tlane_, target_, std::max(R * (W + 1), kExtendRows), std::max(R, kExtendRows), opts.debug_logits != 0);
  slane_.resize(n_ssm);
  for (int j = 0; j < n_ssm; ++j)
    init_lane(slane_[j], ssm_[j], std::max(2 * R, kExtendRows), std::max(R, kExtendRows), false);
  st_.slots = R;
  st_.ctx = opts.max_ctx;
  st_.window = W;
  st_.n_ssm = n_ssm;
  check_cuda(cudaMalloc(&st_.tokens, static_cast<size_t>(R) * opts.max_ctx * 4), "tokens");
  check_cuda(cudaMalloc(&st_.committed, R * 4), "committed");
  check_cuda(cudaMalloc(&st_.ssm_len, static_cast<size_t>(n_ssm) * R * 4), "ssm_len");
  check_cuda(cudaMalloc(&st_.drafts, static_cast<size_t>(R) * W * 4), "drafts");
  check_cuda(zero_sync(st_.tokens, static_cast<size_t>(R) * opts.max_ctx * 4), "memset");
  check_cuda(zero_sync(st_.committed, R * 4), "memset");
  check_cuda(zero_sync(st_.ssm_len, static_cast<size_t>(n_ssm) * R * 4), "memset");
  check_cuda(zero_sync(st_.drafts, static_cast<size_t>(R) * W * 4), "memset");
  h_tokens_.assign(static_cast<size_t>(R) * opts.max_ctx, 0);
  h_committed_.assign(R, 0);
  h_ssm_len_.assign(static_cast<size_t>(n_ssm) * R, 0);
  in_cap_ = static_cast<size_t>(3) * R + 16;
  out_cap_ = static_cast<size_t>(R) * (3 + 2 * W + 1) + 16;
  check_cuda(cudaMallocHost(&pin_in_, in_cap_ * 4), "pinned");
  check_cuda(cudaMallocHost(&pin_out_, out_cap_ * 4), "pinned");
  check_cuda(cudaMalloc(&d_in_, in_cap_ * 4), "in");
  check_cuda(cudaMalloc(&d_out_, out_cap_ * 4), "out");
  check_cuda(cudaMalloc(&d_emitted_, 8), "emitted");
  check_cuda(zero_sync(d_emitted_, 8), "memset");
  check_cuda(cudaEventCreateWithFlags(&ev_fork_, cudaEventDisableTiming), "event");
  check_cuda(cudaEventCreate(&ev_start_), "event");
  check_cuda(cudaEventCreate(&ev_draft_), "event");
  check_cuda(cudaEventCreate(&ev_end_), "event");
  check_cuda(cudaEventCreate(&ev_r0_), "event");
  check_cuda(cudaEventCreate(&ev_r1_), "event");
  ps_.resize(n_ssm);
  for (auto& st : ps_) check_cuda(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking), "stream");
  ev_pw_.resize(n_ssm);
  for (auto& e : ev_pw_) check_cuda(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
  pw_pending_.assign(n_ssm, 0);
  ev_join_.resize(n_ssm);
  for (auto& e : ev_join_) check_cuda(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
  ev_spec_end_.resize(n_ssm);  // per-SSM draft end (timing; the event trace)
  for (auto& e : ev_spec_end_) check_cuda(cudaEventCreate(&e), "event");
  last_spec_ms_.assign(n_ssm, -1.f);
  mb_.assign(n_ssm, 1);
  sync_sv("init sync");
}

Engine::~Engine() {
  if (pw_thread_.joinable()) pw_thread_.join();
  cudaDeviceSynchronize();
  for (auto& kv : pipes_)
    for (PipeUnit& u : kv.second->units) {
      if (u.draft) cudaGraphExecDestroy(u.draft);
      if (u.verify) cudaGraphExecDestroy(u.verify);
      if (u.gd) cudaGraphDestroy(u.gd);
      if (u.gv) cudaGraphDestroy(u.gv);
      for (cudaEvent_t e : {u.ev_d, u.ev_v, u.t_d, u.t_v0, u.t_v1}) cudaEventDestroy(e);
    }
  for (auto& kv : rounds_) {
    if (kv.second->exec) cudaGraphExecDestroy(kv.second->exec);
    if (kv.second->graph) cudaGraphDestroy(kv.second->graph);
  }
  auto free_model = [](ModelDev& m) {
    cudaFree(m.wbuf), cudaFree(m.sbuf), cudaFree(m.kc), cudaFree(m.vc), cudaFree(m.rcos), cudaFree(m.rsin);
  };
  free_model(target_);
  for (auto& m : ssm_) free_model(m);
  for (void* p : tlane_.allocs) cudaFree(p);
  for (auto& l : slane_)
    for (void* p : l.allocs) cudaFree(p);
  cudaFree(st_.tokens), cudaFree(st_.committed), cudaFree(st_.ssm_len), cudaFree(st_.drafts);
  for (void* p : plan_tables_) cudaFree(p);
  if (stamps_) cudaFree(stamps_);
  cudaFreeHost(const_cast<int32_t*>(h_err_));
  cudaFreeHost(pin_in_), cudaFreeHost(pin_out_), cudaFree(d_in_), cudaFree(d_out_), cudaFree(d_emitted_);
  cudaEventDestroy(ev_fork_), cudaEventDestroy(ev_start_), cudaEventDestroy(ev_draft_), cudaEventDestroy(ev_end_);
  cudaEventDestroy(ev_r0_), cudaEventDestroy(ev_r1_);
  for (auto& e : ev_pw_) cudaEventDestroy(e);
  for (auto& e : ev_pw_stage_) cudaEventDestroy(e);
  for (auto& st : ps_) cudaStreamDestroy(st);
  for (auto& l : pwlane_)
    for (void* p : l.allocs) cudaFree(p);
  for (int32_t* p : pw_pin_) cudaFreeHost(p);
  for (int32_t* p : pw_len_pin_) cudaFreeHost(p);
  for (auto& e : ev_join_) cudaEventDestroy(e);
  for (auto& e : ev_spec_end_) cudaEventDestroy(e);
  for (auto& s : ss_) cudaStreamDestroy(s);
  cudaStreamDestroy(sv_);
}

void Engine::sync_sv(const char* what) {
  check_cuda(cudaStreamSynchronize(sv_), what);
  if (*h_err_ != 0) {
    const int e = *h_err_;
    *h_err_ = 0;
    if (e == 3 || e == 4) {  // non-finite logits: the slot's host-side state for the report
      const int slot = h_err_[1], j = h_err_[2];
      std::string st = "slot " + std::to_string(slot) + (e == 3 ? " ssm " + std::to_string(j) : " target") +
                       " step/k " + std::to_string(h_err_[3]) + " row " + std::to_string(h_err_[4]);
      if (slot >= 0 && slot < opts_.max_requests) {
        st += " committed " + std::to_string(h_committed_[slot]) + " ssm_len";
        for (size_t m = 0; m < ssm_.size(); ++m)
          st += " " + std::to_string(h_ssm_len_[m * opts_.max_requests + slot]);
      }
      // diagnostics: non-finite K/V entries of the slot in that model's cache, per layer
      if (slot >= 0 && slot < opts_.max_requests && cudaDeviceSynchronize() == cudaSuccess) {
        ModelDev& md = (e == 3 && j >= 0 && j < static_cast<int>(ssm_.size())) ? ssm_[j] : target_;
        const int c = h_committed_[slot];
        const size_t rowel = static_cast<size_t>(md.hd);
        std::vector<uint16_t> buf(static_cast<size_t>(c) * rowel);
        for (int l = 0; l < md.L; ++l) {
          int bad_k = 0, bad_v = 0, first = -1;
          for (int h = 0; h < md.H; ++h) {
            const size_t off = (((static_cast<size_t>(l) * opts_.max_requests + slot) * md.H + h) * opts_.max_ctx) * rowel;
            for (int kv = 0; kv < 2; ++kv) {
              cudaMemcpy(buf.data(), (kv ? md.vc : md.kc) + off, buf.size() * 2, cudaMemcpyDeviceToHost);
              for (size_t i = 0; i < buf.size(); ++i)
                if ((buf[i] & 0x7f80) == 0x7f80) {
                  (kv ? bad_v : bad_k)++;
                  const int pos = static_cast<int>(i / rowel);
                  if (first < 0 || pos < first) first = pos;
                }
            }
          }
          if (bad_k || bad_v)
            st += " | layer " + std::to_string(l) + ": non-finite K " + std::to_string(bad_k) + " V " +
                  std::to_string(bad_v) + " first pos " + std::to_string(first);
        }
      }
      fail(SPIN_CUDA_ERROR, std::string(what) + ": non-finite logits (argmax undefined): " + st);
    }
    fail(SPIN_CAPACITY_ERROR, std::string(what) + (e == 2 ? ": a round would commit past max_ctx"
                                                           : ": attention work list exceeds its buffers") +
                                  " (device status " + std::to_string(e) + ")");
  }
}

void Engine::sync_state_from_device() {
  if (!mirror_stale_) return;
  sync_sv("sync");
  check_cuda(cudaMemcpy(h_tokens_.data(), st_.tokens, h_tokens_.size() * 4, cudaMemcpyDeviceToHost), "d2h");
  check_cuda(cudaMemcpy(h_committed_.data(), st_.committed, h_committed_.size() * 4, cudaMemcpyDeviceToHost), "d2h");
  check_cuda(cudaMemcpy(h_ssm_len_.data(), st_.ssm_len, h_ssm_len_.size() * 4, cudaMemcpyDeviceToHost), "d2h");
  mirror_stale_ = false;
}

// Ragged extend of one model over positions [from, to) of each slot: the
// prompt prefill, and the KV recompute of an SSM switch (switching_cost,
// slot_engine.cpp:12-22). Rows are cut into virtual requests of <= 8 queries.
// Synchronous on sv_ (lane = the model's own lane) unless `pinned` is given: then
// the chunks are staged in that pinned buffer and enqueued on `s` without any host
// wait (the prewarm path; the caller owns the ordering).
void Engine::extend(int model, const std::vector<std::tuple<int, int, int>>& ranges, cudaStream_t s, Lane* lane,
                    int32_t* pinned, size_t pinned_cap) {
  ModelDev& m = model < 0 ? target_ : ssm_[model];
  Lane& ln = lane ? *lane : (model < 0 ? tlane_ : slane_[model]);
  if (!s) s = sv_;
  std::vector<int32_t> rt, rs, rp, qs_, ql, kv, sl;
  size_t pin_used = 0;
  auto flush = [&]() {
    if (rt.empty()) return;
    const int T = static_cast<int>(rt.size()), R = static_cast<int>(sl.size());
    const int32_t* src[7] = {rt.data(), rs.data(), rp.data(), sl.data(), qs_.data(), ql.data(), kv.data()};
    int32_t* dst[7] = {ln.meta.row_tok, ln.meta.row_slot, ln.meta.row_pos, ln.meta.req_slot, ln.meta.req_qstart,
                       ln.meta.req_qlen, ln.meta.req_kvlen};
    const int cnt[7] = {T, T, T, R, R, R, R};
    for (int k = 0; k < 7; ++k) {
      const int32_t* from = src[k];
      if (pinned) {  // stage in pinned memory: the copy is truly asynchronous
        if (pin_used + cnt[k] > pinned_cap) fail(SPIN_CAPACITY_ERROR, "extend: prewarm staging buffer exhausted");
        std::memcpy(pinned + pin_used, src[k], cnt[k] * 4);
        from = pinned + pin_used;
        pin_used += cnt[k];
      }
      check_cuda(cudaMemcpyAsync(dst[k], from, cnt[k] * 4, cudaMemcpyHostToDevice, s), "h2d");
    }
    MetaArgs a{};
    a.mode = kMetaExtend;
    a.n_req = R;
    a.width = R;
    a.chunks = attn_chunks(R, m.H, num_sms_);
    launch_meta(a, st_, ln.meta, s);
    forward(m, ln, FwdShape{T, R, R, kExtendQ}, s, 0);
    if (!pinned) sync_sv("extend");  // host vectors are reused
    rt.clear(), rs.clear(), rp.clear(), qs_.clear(), ql.clear(), kv.clear(), sl.clear();
  };
  for (const auto& [slot, from, to] : ranges) {
    for (int p0 = from; p0 < to; p0 += kExtendQ) {
      const int p1 = std::min(to, p0 + kExtendQ);
      if (static_cast<int>(rt.size()) + (p1 - p0) > kExtendRows) flush();
      qs_.push_back(static_cast<int32_t>(rt.size()));
      ql.push_back(p1 - p0);
      kv.push_back(p1);
      sl.push_back(slot);
      for (int p = p0; p < p1; ++p) {
        rt.push_back(h_tokens_[static_cast<size_t>(slot) * opts_.max_ctx + p]);
        rs.push_back(slot);
        rp.push_back(p);
      }
    }
  }
  flush();
}

// Device-side ordering: work on sv_ after this waits for every enqueued prewarm.
void Engine::join_prewarm() {
  if (pw_thread_.joinable()) pw_thread_.join();
  if (pw_error_) {
    pw_error_ = false;
    fail(SPIN_CUDA_ERROR, "prewarm: " + pw_error_msg_);
  }
  for (size_t j = 0; j < pw_pending_.size(); ++j) {
    if (!pw_pending_[j]) continue;
    check_cuda(cudaStreamWaitEvent(sv_, ev_pw_[j], 0), "join prewarm");
    pw_pending_[j] = 0;
  }
}

// KV catch-up of SSM j for the listed requests on j's prewarm stream, concurrently
// with whatever the device runs next (the destination of a future switch is warmed
// in idle time: prewarm_destination, bandit.cpp:122-139; switching_cost = 0 when
// prewarmed, slot_engine.cpp:12-22). Positions up to committed - 2 of the host
// mirror; the round that later uses SSM j only catches up its own commits.
void Engine::enqueue_prewarm(int n, const int32_t* slots, const int32_t* prewarm, const int32_t* ssm_of) {
  const int M = static_cast<int>(ssm_.size()), R = opts_.max_requests;
  if (pw_thread_.joinable()) pw_thread_.join();
  std::vector<std::vector<std::tuple<int, int, int>>> jobs(M);
  bool any = false;
  for (int j = 0; j < M; ++j) {
    for (int i = 0; i < n; ++i) {
      if (prewarm[i] != j || (ssm_of && ssm_of[i] == j)) continue;
      const int s = slots[i];
      const int need = h_committed_[s] - 2;
      int32_t& len = h_ssm_len_[static_cast<size_t>(j) * R + s];
      if (len < need) {
        jobs[j].emplace_back(s, len, need);
        pw_tokens_ += need - len;
        len = need;  // the host mirror; the device copy is written by the prewarm stream
        any = true;
      }
    }
  }
  if (!any) return;
  if (pwlane_.empty()) init_prewarm();
  for (int j = 0; j < M; ++j)
    if (!jobs[j].empty()) pw_pending_[j] = 1;
  // The enqueue (staging + ~100 launches per 512-row chunk) runs on a worker thread
  // while this thread waits for the round. It reads h_tokens_ positions < committed - 2
  // of the prewarmed slots, which the round's host update (positions >= committed)
  // never touches; join_prewarm() joins it before anything else is enqueued.
  int dev = 0;
  check_cuda(cudaGetDevice(&dev), "device");
  const bool pipe_drafts = pipelined();  // the slot just launched ran micro-batched units
  pw_thread_ = std::thread([this, dev, pipe_drafts, jobs = std::move(jobs)]() {
    try {
      check_cuda(cudaSetDevice(dev), "cudaSetDevice");
      for (size_t j = 0; j < jobs.size(); ++j) {
        if (jobs[j].empty()) continue;
        cudaStream_t ps = ps_[j];
        const size_t hb = 2 * j + static_cast<size_t>(pw_half_[j]);  // this job's staging half
        pw_half_[j] ^= 1;
        check_cuda(cudaEventSynchronize(ev_pw_stage_[hb]), "prewarm staging");  // the job before last
        static const bool after_drafts = std::getenv("SPIN_PREWARM_AFTER_DRAFTS") != nullptr;
        if (after_drafts) {  // overlap the verification only (timing experiments)
          if (pipe_drafts)  // micro-batched slot: every SSM stream's last unit draft (launch_pipe_slot)
            for (size_t jj = 0; jj < ev_join_.size(); ++jj)
              check_cuda(cudaStreamWaitEvent(ps, ev_join_[jj], 0), "prewarm after drafts");
          else
            check_cuda(cudaStreamWaitEvent(ps, ev_draft_, 0), "prewarm after drafts");
        }
        extend(static_cast<int>(j), jobs[j], ps, &pwlane_[j], pw_pin_[hb], pw_pin_cap_);
        for (const auto& r : jobs[j]) {
          const size_t idx = j * opts_.max_requests + std::get<0>(r);
          pw_len_pin_[hb][std::get<0>(r)] = std::get<2>(r);
          check_cuda(cudaMemcpyAsync(st_.ssm_len + idx, pw_len_pin_[hb] + std::get<0>(r), 4, cudaMemcpyHostToDevice,
                                     ps),
                     "h2d");
        }
        check_cuda(cudaEventRecord(ev_pw_[j], ps), "prewarm event");
        check_cuda(cudaEventRecord(ev_pw_stage_[hb], ps), "prewarm event");
      }
    } catch (const std::exception& e) {
      pw_error_msg_ = e.what();
      pw_error_ = true;
    }
  });
}

void Engine::init_prewarm() {
  const int M = static_cast<int>(ssm_.size()), R = opts_.max_requests;
  pwlane_.resize(M);
  pw_pin_.assign(2 * M, nullptr);
  pw_pin_cap_ = static_cast<size_t>(8) * (static_cast<size_t>(R) * opts_.max_ctx + kExtendRows);
  pw_len_pin_.assign(2 * M, nullptr);
  ev_pw_stage_.assign(2 * M, nullptr);
  pw_half_.assign(M, 0);
  for (int j = 0; j < M; ++j) init_lane(pwlane_[j], ssm_[j], kExtendRows, kExtendRows, false);
  for (int h = 0; h < 2 * M; ++h) {
    check_cuda(cudaMallocHost(&pw_pin_[h], pw_pin_cap_ * 4), "prewarm staging");
    check_cuda(cudaMallocHost(&pw_len_pin_[h], static_cast<size_t>(R) * 4), "prewarm staging");
    check_cuda(cudaEventCreateWithFlags(&ev_pw_stage_[h], cudaEventDisableTiming), "event");
  }
}

void Engine::prefill(int n, const int32_t* slots, const int32_t* lens, const int32_t* prompts) {
  sync_state_from_device();
  join_prewarm();
  std::vector<std::tuple<int, int, int>> ranges;
  std::vector<char> seen(opts_.max_requests, 0);
  size_t off = 0;
  for (int i = 0; i < n; ++i) {
    const int s = slots[i], L = lens[i];
    if (s < 0 || s >= opts_.max_requests) fail(SPIN_INPUT_ERROR, "prefill: slot out of range");
    if (seen[s]) fail(SPIN_INPUT_ERROR, "prefill: duplicate slot");
    seen[s] = 1;
    if (L < 2) fail(SPIN_INPUT_ERROR, "prefill: prompts need at least 2 tokens");
    if (L + opts_.window + 1 > opts_.max_ctx) fail(SPIN_CAPACITY_ERROR, "prefill: prompt exceeds max_ctx");
    for (int p = 0; p < L; ++p) {
      const int32_t tok = prompts[off + p];
      if (tok < 0 || tok >= target_.V) fail(SPIN_INPUT_ERROR, "prefill: token id out of range");
      h_tokens_[static_cast<size_t>(s) * opts_.max_ctx + p] = tok;
    }
    off += L;
    h_committed_[s] = L;
    ranges.emplace_back(s, 0, L - 1);
  }
  for (int i = 0; i < n; ++i) {
    const int s = slots[i];
    check_cuda(cudaMemcpyAsync(st_.tokens + static_cast<size_t>(s) * opts_.max_ctx,
                               h_tokens_.data() + static_cast<size_t>(s) * opts_.max_ctx, lens[i] * 4,
                               cudaMemcpyHostToDevice, sv_),
               "h2d");
    check_cuda(cudaMemcpyAsync(st_.committed + s, h_committed_.data() + s, 4, cudaMemcpyHostToDevice, sv_), "h2d");
  }
  extend(-1, ranges);
  for (int j = 0; j < static_cast<int>(ssm_.size()); ++j) {
    extend(j, ranges);
    for (int i = 0; i < n; ++i) {
      const int s = slots[i];
      h_ssm_len_[static_cast<size_t>(j) * opts_.max_requests + s] = lens[i] - 1;
      check_cuda(cudaMemcpyAsync(st_.ssm_len + static_cast<size_t>(j) * opts_.max_requests + s,
                                 h_ssm_len_.data() + static_cast<size_t>(j) * opts_.max_requests + s, 4,
                                 cudaMemcpyHostToDevice, sv_),
                 "h2d");
    }
  }
  sync_sv("prefill");
}

// Synchronous KV catch-up of requests whose SSM cache lags (a switch, or the
// commits since a prewarm): recomputed on sv_ before the round. Returns the
// positions recomputed per request in `per_req` (optional, [n]).
int64_t Engine::switch_ssm(int n, const int32_t* slots, const int32_t* ssm_of, int32_t* per_req) {
  sync_state_from_device();
  join_prewarm();
  int64_t total = 0;
  for (int j = 0; j < static_cast<int>(ssm_.size()); ++j) {
    std::vector<std::tuple<int, int, int>> ranges;
    for (int i = 0; i < n; ++i) {
      if (per_req && j == 0) per_req[i] = 0;
      if (ssm_of[i] != j) continue;
      const int s = slots[i];
      const int need = h_committed_[s] - 2;
      int32_t& len = h_ssm_len_[static_cast<size_t>(j) * opts_.max_requests + s];
      if (len < need) {
        ranges.emplace_back(s, len, need);
        if (per_req) per_req[i] = need - len;
        total += need - len;
        len = need;
      }
    }
    if (ranges.empty()) continue;
    extend(j, ranges);
    for (const auto& r : ranges) {
      const int s = std::get<0>(r);
      check_cuda(cudaMemcpyAsync(st_.ssm_len + static_cast<size_t>(j) * opts_.max_requests + s,
                                 h_ssm_len_.data() + static_cast<size_t>(j) * opts_.max_requests + s, 4,
                                 cudaMemcpyHostToDevice, sv_),
                 "h2d");
    }
    sync_sv("switch");
  }
  return total;
}

Engine::RoundPlan& Engine::plan_round(int n, const int32_t* slots, const int32_t* ssm_of) {
  const int M = static_cast<int>(ssm_.size());
  std::vector<int> key(1 + M, 0);
  for (int i = 0; i < n; ++i)
    if (ssm_of[i] >= 0) ++key[0], ++key[1 + ssm_of[i]];
  auto it = rounds_.find(key);
  if (it != rounds_.end()) return *it->second;
  auto p = std::make_unique<RoundPlan>();
  p->key = key;
  p->n_act = key[0];
  p->n_ssm.assign(key.begin() + 1, key.end());
  p->off_list = 0;
  p->off_ssm_of = p->n_act;
  int off = 2 * p->n_act;
  for (int j = 0; j < M; ++j) {
    p->off_ssm_list.push_back(off);
    off += p->n_ssm[j];
  }
  p->in_ints = off;
  p->out_ints = p->n_act * (3 + 2 * opts_.window + 1);
  RoundPlan& ref = *p;
  rounds_.emplace(key, std::move(p));
  return ref;
}

// Timing events: inside a graph capture they must be external record nodes.
void Engine::record_timing(cudaEvent_t ev, cudaStream_t s) {
  if (capturing_)
    check_cuda(cudaEventRecordWithFlags(ev, s, cudaEventRecordExternal), "event");
  else
    check_cuda(cudaEventRecord(ev, s), "event");
}

// The gamma-step draft loop of SSM j over nj requests (device list d_list) on stream sj.
void Engine::enqueue_draft(int j, const int32_t* d_list, int nj, cudaStream_t sj) {
  const int W = opts_.window;
  ModelDev& m = ssm_[j];
  Lane& ln = slane_[j];
  const int tiles = (m.V + 127) / 128;
  MetaArgs a{};
  a.mode = kMetaDraft0;
  a.n_req = nj;
  a.list = d_list;
  a.ssm = j;
  a.width = nj;
  a.chunks = attn_chunks(nj, m.H, num_sms_, 2);
  a.padded = 1;  // few-query steps: one row per request, whole requests per CTA (no merges)
  prof_begin(kProfMeta, sj);
  launch_meta(a, st_, ln.meta, sj);
  prof_end(sj, 0);
  forward(m, ln, FwdShape{2 * nj, nj, nj, 2, 1}, sj, 1);
  int prev_t = 2 * nj, prev_q = 2;
  for (int k = 1; k <= W; ++k) {
    MetaArgs b{};
    b.mode = k < W ? kMetaDraftK : kMetaCollect;
    b.n_req = nj;
    b.list = d_list;
    b.step = k;
    b.ssm = j;
    b.width = nj;
    b.chunks = attn_chunks(nj, m.H, num_sms_, 1);
    b.padded = 1;
    b.amax_val = ln.amax_val;
    b.amax_idx = ln.amax_idx;
    b.amax_tiles = tiles;
    b.prev_t = prev_t;
    b.prev_qlen = prev_q;
    prof_begin(kProfMeta, sj);
    launch_meta(b, st_, ln.meta, sj);
    prof_end(sj, 0);
    if (k < W) forward(m, ln, FwdShape{nj, nj, nj, 1, 1}, sj, 1);
    prev_t = nj, prev_q = 1;
  }
}

// Pack (device request decomposition), target verify forward and greedy accept of n
// requests (d_list slots, d_ssm_of their SSMs) on stream s; outcomes to d_out.
void Engine::enqueue_verify(const int32_t* d_list, const int32_t* d_ssm_of, int n, int32_t* d_out, cudaStream_t s) {
  const int W = opts_.window;
  const int T = n * (W + 1);
  const int width = opts_.pack_width > 0 ? std::min(opts_.pack_width, n) : n;
  MetaArgs a{};
  a.mode = kMetaVerify;
  a.n_req = n;
  a.list = d_list;
  a.width = width;
  a.padded = opts_.packing ? 0 : 1;
  a.chunks = attn_chunks(a.padded ? n : width, target_.H, num_sms_);
  prof_begin(kProfMeta, s);
  launch_meta(a, st_, tlane_.meta, s);
  prof_end(s, 0);
  forward(target_, tlane_, FwdShape{T, n, a.padded ? n : width, W + 1, 1}, s, opts_.debug_logits ? 2 : 1);
  int32_t* o = d_out;
  prof_begin(kProfMeta, s);
  launch_accept(tlane_.meta, n, W, d_list, d_ssm_of, tlane_.amax_val, tlane_.amax_idx, (target_.V + 127) / 128, T,
                st_, o, o + n, o + 2 * n, o + 3 * n, o + 3 * n + n * W, d_emitted_, s);
  prof_end(s, 0);
}

// Enqueues one round on sv_ (+ SSM streams); used for capture and direct runs.
void Engine::capture_round(RoundPlan& p) {
  const int M = static_cast<int>(ssm_.size());
  const int64_t launches_before = launches_;
  stamp_used_ = 0;
  stamp_tab_.clear();
  cudaStream_t s = sv_;
  record_timing(ev_start_, s);
  check_cuda(cudaMemcpyAsync(d_in_, pin_in_, p.in_ints * 4, cudaMemcpyHostToDevice, s), "h2d lists");
  check_cuda(cudaEventRecord(ev_fork_, s), "event");
  // The deepest active SSM's step chain bounds the draft phase; the others run beside it and
  // their lm_head (a 49-MB weight stream over every SM) stalls its latency-bound kernels, so
  // theirs may be held to fewer SMs (SPIN_MINOR_HEAD_SMS; 0 = all).
  static const int minor_head_sms = [] {
    const char* e = std::getenv("SPIN_MINOR_HEAD_SMS");
    return e ? std::atoi(e) : 0;
  }();
  int crit = -1;
  for (int j = 0; j < M; ++j)
    if (p.n_ssm[j] > 0 && (crit < 0 || ssm_[j].L > ssm_[crit].L)) crit = j;
  for (int j = 0; j < M; ++j) slane_[j].head_sms = (j == crit) ? 0 : minor_head_sms;
  for (int j = 0; j < M; ++j) {
    cudaStream_t sj = ss_[j];
    check_cuda(cudaStreamWaitEvent(sj, ev_fork_, 0), "fork");
    if (p.n_ssm[j] > 0) {
      enqueue_draft(j, d_in_ + p.off_ssm_list[j], p.n_ssm[j], sj);
      record_timing(ev_spec_end_[j], sj);
    }
    check_cuda(cudaEventRecord(ev_join_[j], sj), "join");
    check_cuda(cudaStreamWaitEvent(s, ev_join_[j], 0), "join");
  }
  record_timing(ev_draft_, s);
  const int n = p.n_act;
  if (n > 0) {
    enqueue_verify(d_in_ + p.off_list, d_in_ + p.off_ssm_of, n, d_out_, s);
    check_cuda(cudaMemcpyAsync(pin_out_, d_out_, p.out_ints * 4, cudaMemcpyDeviceToHost, s), "d2h outcome");
  }
  record_timing(ev_end_, s);
  check_cuda(cudaGetLastError(), "round launch");
  p.launches = launches_ - launches_before;
}

// ------------------------------------------------------------------ pipelining
void Engine::set_micro_batches(const int32_t* per_ssm, int m) {
  if (m != static_cast<int>(ssm_.size())) fail(SPIN_INPUT_ERROR, "micro_batches: one count per SSM");
  for (int j = 0; j < m; ++j)
    if (per_ssm[j] < 1 || per_ssm[j] > 16) fail(SPIN_INPUT_ERROR, "micro_batches: counts must be in 1..16");
  mb_.assign(per_ssm, per_ssm + m);
}

void Engine::get_micro_batches(int32_t* per_ssm, int m) const {
  for (int j = 0; j < m && j < static_cast<int>(mb_.size()); ++j) per_ssm[j] = mb_[j];
}

// Units of the current micro-batch plan for this assignment shape: SSM j's n_j active
// requests (batch order) split into min(b_j, n_j) near-equal groups, the remainder to
// the earlier groups (pipeline.cpp:176-189). Verify order: expected arrival, i.e.
// group g of SSM j done at (g + 1) / b_j of j's measured draft time (FIFO verifier,
// pipeline.cpp:265-282).
Engine::PipePlan& Engine::plan_pipe(int n, const int32_t* ssm_of) {
  const int M = static_cast<int>(ssm_.size()), W = opts_.window;
  std::vector<int> cnt(M, 0);
  for (int i = 0; i < n; ++i)
    if (ssm_of[i] >= 0) ++cnt[ssm_of[i]];
  std::vector<int> key = mb_;
  key.insert(key.end(), cnt.begin(), cnt.end());
  auto it = pipes_.find(key);
  if (it != pipes_.end()) return *it->second;
  auto pp = std::make_unique<PipePlan>();
  int off = 0, off_out = 0;
  for (int j = 0; j < M; ++j) {
    if (cnt[j] == 0) continue;
    const int b = std::max(1, std::min(mb_[j], cnt[j]));
    const int base = cnt[j] / b, extra = cnt[j] % b;
    const double t_j = last_spec_ms_[j] > 0.f ? last_spec_ms_[j] : 0.1 * ssm_[j].L;
    for (int g = 0; g < b; ++g) {
      PipeUnit u;
      u.ssm = j, u.g = g, u.n = base + (g < extra ? 1 : 0);
      u.off_list = off, u.off_ssm_of = off + u.n, off += 2 * u.n;
      u.off_out = off_out, off_out += u.n * (3 + 2 * W + 1);
      u.arrival = t_j * (g + 1) / b;
      check_cuda(cudaEventCreateWithFlags(&u.ev_d, cudaEventDisableTiming), "event");
      check_cuda(cudaEventCreateWithFlags(&u.ev_v, cudaEventDisableTiming), "event");
      check_cuda(cudaEventCreate(&u.t_d), "event");
      check_cuda(cudaEventCreate(&u.t_v0), "event");
      check_cuda(cudaEventCreate(&u.t_v1), "event");
      pp->units.push_back(u);
      pp->n_act += u.n;
    }
  }
  pp->in_ints = off;
  pp->out_ints = off_out;
  pp->vorder.resize(pp->units.size());
  for (size_t k = 0; k < pp->units.size(); ++k) pp->vorder[k] = static_cast<int>(k);
  std::stable_sort(pp->vorder.begin(), pp->vorder.end(),
                   [&](int a, int b) { return pp->units[a].arrival < pp->units[b].arrival; });
  PipePlan& ref = *pp;
  pipes_.emplace(key, std::move(pp));
  return ref;
}

// Host staging of the unit lists (pinned): unit (j, g) takes SSM j's requests of
// group g, in batch order.
void Engine::stage_pipe(PipePlan& pp, int n, const int32_t* slots, const int32_t* ssm_of) {
  std::vector<std::vector<int>> by_ssm(ssm_.size());
  for (int i = 0; i < n; ++i)
    if (ssm_of[i] >= 0) by_ssm[ssm_of[i]].push_back(i);
  std::vector<size_t> cursor(ssm_.size(), 0);
  for (PipeUnit& u : pp.units) {
    for (int k = 0; k < u.n; ++k) {
      const int i = by_ssm[u.ssm][cursor[u.ssm]++];
      pin_in_[u.off_list + k] = slots[i];
      pin_in_[u.off_ssm_of + k] = u.ssm;
    }
  }
}

// One pipelined slot: unit drafts on the SSM streams, unit verifies FIFO on sv_.
// first: order the SSM streams after sv_ (host-driven slots, the first slot of a
// device loop); later slots of a device loop only wait for their unit's previous
// verification, so the next slot's drafting overlaps this slot's verifications.
void Engine::launch_pipe_slot(PipePlan& pp, bool first, bool host_round) {
  const bool graphs = opts_.use_graphs != 0;
  if (first) {
    check_cuda(cudaEventRecord(ev_start_, sv_), "event");
    if (host_round)
      check_cuda(cudaMemcpyAsync(d_in_, pin_in_, pp.in_ints * 4, cudaMemcpyHostToDevice, sv_), "h2d lists");
    check_cuda(cudaEventRecord(ev_fork_, sv_), "event");
    for (size_t j = 0; j < ssm_.size(); ++j) check_cuda(cudaStreamWaitEvent(ss_[j], ev_fork_, 0), "fork");
  }
  const int64_t before = launches_;
  for (PipeUnit& u : pp.units) {
    cudaStream_t sj = ss_[u.ssm];
    if (!first) check_cuda(cudaStreamWaitEvent(sj, u.ev_v, 0), "unit causality");
    if (graphs) {
      if (!u.draft) {
        check_cuda(cudaStreamBeginCapture(sj, cudaStreamCaptureModeRelaxed), "capture");
        capturing_ = true;
        enqueue_draft(u.ssm, d_in_ + u.off_list, u.n, sj);
        capturing_ = false;
        check_cuda(cudaStreamEndCapture(sj, &u.gd), "capture");
        check_cuda(cudaGraphInstantiate(&u.draft, u.gd, 0), "instantiate");
      }
      check_cuda(cudaGraphLaunch(u.draft, sj), "graph launch");
    } else {
      enqueue_draft(u.ssm, d_in_ + u.off_list, u.n, sj);
    }
    check_cuda(cudaEventRecord(u.t_d, sj), "event");
    check_cuda(cudaEventRecord(u.ev_d, sj), "event");
  }
  // the slot's draft phase on every SSM stream (SPIN_PREWARM_AFTER_DRAFTS: a catch-up waits for it)
  for (size_t j = 0; j < ssm_.size(); ++j) check_cuda(cudaEventRecord(ev_join_[j], ss_[j]), "drafts done");
  for (int k : pp.vorder) {
    PipeUnit& u = pp.units[k];
    check_cuda(cudaStreamWaitEvent(sv_, u.ev_d, 0), "unit drafted");
    check_cuda(cudaEventRecord(u.t_v0, sv_), "event");
    if (graphs) {
      if (!u.verify) {
        check_cuda(cudaStreamBeginCapture(sv_, cudaStreamCaptureModeRelaxed), "capture");
        capturing_ = true;
        enqueue_verify(d_in_ + u.off_list, d_in_ + u.off_ssm_of, u.n, d_out_ + u.off_out, sv_);
        capturing_ = false;
        check_cuda(cudaStreamEndCapture(sv_, &u.gv), "capture");
        check_cuda(cudaGraphInstantiate(&u.verify, u.gv, 0), "instantiate");
      }
      check_cuda(cudaGraphLaunch(u.verify, sv_), "graph launch");
    } else {
      enqueue_verify(d_in_ + u.off_list, d_in_ + u.off_ssm_of, u.n, d_out_ + u.off_out, sv_);
    }
    check_cuda(cudaEventRecord(u.t_v1, sv_), "event");
    check_cuda(cudaEventRecord(u.ev_v, sv_), "event");
  }
  if (pp.launches == 0 && launches_ > before) pp.launches = launches_ - before;  // counted at capture
  if (host_round)
    check_cuda(cudaMemcpyAsync(pin_out_, d_out_, pp.out_ints * 4, cudaMemcpyDeviceToHost, sv_), "d2h outcome");
  check_cuda(cudaEventRecord(ev_end_, sv_), "event");
  check_cuda(cudaGetLastError(), "pipelined slot launch");
}

// tune_micro_batches (pipeline.cpp:345-380) on MEASURED throughput: uniform plans with
// b = 1 (the serial round) and b = 2 .. max_mb (capped by the largest SSM batch), each
// probed with `probe_rounds` device-resident rounds on the live requests; the search
// stops at the first plan more than `threshold` below the best so far and keeps the
// last non-degraded plan.
void Engine::tune_micro_batches(int n, const int32_t* slots, const int32_t* ssm_of, int max_mb, int probe_rounds,
                                double threshold, int32_t* chosen, double* curve, int curve_cap, int* n_curve) {
  const int M = static_cast<int>(ssm_.size());
  if (probe_rounds < 1 || max_mb < 1 || !(threshold >= 0.0)) fail(SPIN_INPUT_ERROR, "tune: bad arguments");
  std::vector<int> sizes(M, 0);
  int largest = 1;
  for (int i = 0; i < n; ++i)
    if (ssm_of[i] >= 0) largest = std::max(largest, ++sizes[ssm_of[i]]);
  std::vector<int> cand{1};
  for (int b = 2; b <= std::min(max_mb, largest); ++b) cand.push_back(b);
  auto uniform = [&](int b) {
    std::vector<int32_t> p(M);
    for (int j = 0; j < M; ++j) p[j] = std::max(1, std::min(b, sizes[j]));
    return p;
  };
  std::vector<int32_t> last_good = uniform(1);
  double best = -1.0;
  int k = 0;
  std::vector<int64_t> em(probe_rounds);
  for (int b : cand) {
    const std::vector<int32_t> plan = uniform(b);
    set_micro_batches(plan.data(), M);
    float ms = 0.f;
    run_rounds(n, slots, ssm_of, probe_rounds, em.data(), &ms);
    int64_t tok = 0;
    for (int64_t e : em) tok += e;
    const double tput = ms > 0.f ? tok / (ms * 1e-3) : 0.0;
    if (curve && k < curve_cap) curve[k] = tput;
    ++k;
    best = std::max(best, tput);
    if (tput >= (1.0 - threshold) * best) {
      last_good = plan;
    } else {
      break;  // first clear degradation ends the search
    }
  }
  set_micro_batches(last_good.data(), M);
  if (chosen) std::copy(last_good.begin(), last_good.end(), chosen);
  if (n_curve) *n_curve = k;
}

void Engine::round(int n, const int32_t* slots, const int32_t* ssm_of, const int32_t* prewarm, spin_round_out* out) {
  sync_state_from_device();
  const int M = static_cast<int>(ssm_.size()), W = opts_.window, R = opts_.max_requests;
  if (n < 0 || n > R) fail(SPIN_CAPACITY_ERROR, "round: batch exceeds max_requests");
  std::vector<char> seen(R, 0);
  for (int i = 0; i < n; ++i) {
    const int s = slots[i];
    if (s < 0 || s >= R) fail(SPIN_INPUT_ERROR, "round: slot out of range");
    if (seen[s]) fail(SPIN_INPUT_ERROR, "round: duplicate slot");
    seen[s] = 1;
    if (ssm_of[i] < -1 || ssm_of[i] >= M) fail(SPIN_INPUT_ERROR, "round: unknown ssm in assignment");
    if (prewarm && (prewarm[i] < -1 || prewarm[i] >= M)) fail(SPIN_INPUT_ERROR, "round: unknown ssm in prewarm");
    if (ssm_of[i] >= 0) {
      if (h_committed_[s] < 2) fail(SPIN_INPUT_ERROR, "round: slot was not prefilled");
      if (h_committed_[s] + W + 1 > opts_.max_ctx) fail(SPIN_CAPACITY_ERROR, "round: slot context is full");
    }
  }
  // The round's clock starts before the synchronous KV catch-up of switched
  // requests: switching costs real device time and is charged to the round.
  check_cuda(cudaEventRecord(ev_r0_, sv_), "event");
  std::vector<int32_t> sw_tok(n, 0);
  const int64_t sw_total = switch_ssm(n, slots, ssm_of, sw_tok.data());
  check_cuda(cudaEventRecord(ev_r1_, sv_), "event");
  // Outcome rows of request i: accepted, bonus, committed, drafts [W], target [W + 1].
  struct Rows {
    const int32_t *acc, *bon, *com, *dr, *tg;
    int a;
  };
  std::vector<Rows> rows_of(n, Rows{nullptr, nullptr, nullptr, nullptr, nullptr, -1});
  float draft_ms = 0.f, total_ms = 0.f, verify_ms = 0.f;
  if (pipelined()) {
    PipePlan& pp = plan_pipe(n, ssm_of);
    stage_pipe(pp, n, slots, ssm_of);
    launch_pipe_slot(pp, true, true);
    if (prewarm) enqueue_prewarm(n, slots, prewarm, ssm_of);
    sync_sv("round");
    check_cuda(cudaEventElapsedTime(&total_ms, ev_start_, ev_end_), "event timing");
    for (int j = 0; j < M; ++j) last_spec_ms_[j] = -1.f;
    for (const PipeUnit& u : pp.units) {
      float d = 0.f, v = 0.f;
      check_cuda(cudaEventElapsedTime(&d, ev_start_, u.t_d), "event timing");
      check_cuda(cudaEventElapsedTime(&v, u.t_v0, u.t_v1), "event timing");
      draft_ms = std::max(draft_ms, d);
      verify_ms += v;  // verifier busy time
      last_spec_ms_[u.ssm] = std::max(last_spec_ms_[u.ssm], d);
    }
    // unit rows back to the requests (stage_pipe order)
    std::vector<std::vector<int>> by_ssm(M);
    for (int i = 0; i < n; ++i)
      if (ssm_of[i] >= 0) by_ssm[ssm_of[i]].push_back(i);
    std::vector<size_t> cur(M, 0);
    for (const PipeUnit& u : pp.units) {
      const int32_t* o = pin_out_ + u.off_out;
      for (int k = 0; k < u.n; ++k) {
        const int i = by_ssm[u.ssm][cur[u.ssm]++];
        rows_of[i] = Rows{o, o + u.n, o + 2 * u.n, o + 3 * u.n, o + 3 * u.n + u.n * W, k};
      }
    }
    last_verify_rows_ = 0;  // the in-situ kernel replays expect a serial round's layout
  } else {
    RoundPlan& p = plan_round(n, slots, ssm_of);
    // stage the lists
    std::vector<int> act;
    for (int i = 0; i < n; ++i)
      if (ssm_of[i] >= 0) act.push_back(i);
    for (int a = 0; a < p.n_act; ++a) {
      pin_in_[p.off_list + a] = slots[act[a]];
      pin_in_[p.off_ssm_of + a] = ssm_of[act[a]];
    }
    std::vector<int> fill(M, 0);
    for (int i : act) pin_in_[p.off_ssm_list[ssm_of[i]] + fill[ssm_of[i]]++] = slots[i];
    if (opts_.use_graphs) {
      if (!p.exec) {
        check_cuda(cudaStreamBeginCapture(sv_, cudaStreamCaptureModeRelaxed), "capture");
        capturing_ = true;
        capture_round(p);
        capturing_ = false;
        check_cuda(cudaStreamEndCapture(sv_, &p.graph), "capture");
        check_cuda(cudaGraphInstantiate(&p.exec, p.graph, 0), "instantiate");
      }
      check_cuda(cudaGraphLaunch(p.exec, sv_), "graph launch");
    } else {
      capture_round(p);
    }
    // destinations of future switches recomputed on idle streams while this round runs
    if (prewarm) enqueue_prewarm(n, slots, prewarm, ssm_of);
    sync_sv("round");
    dump_stamps();
    check_cuda(cudaEventElapsedTime(&draft_ms, ev_start_, ev_draft_), "event timing");
    check_cuda(cudaEventElapsedTime(&total_ms, ev_start_, ev_end_), "event timing");
    verify_ms = total_ms - draft_ms;
    for (int j = 0; j < M; ++j) {
      last_spec_ms_[j] = -1.f;
      if (p.n_ssm[j] > 0)
        check_cuda(cudaEventElapsedTime(&last_spec_ms_[j], ev_start_, ev_spec_end_[j]), "event timing");
    }
    const int na = p.n_act;
    for (int a = 0; a < na; ++a)
      rows_of[act[a]] = Rows{pin_out_, pin_out_ + na, pin_out_ + 2 * na, pin_out_ + 3 * na,
                             pin_out_ + 3 * na + na * W, a};
    last_verify_rows_ = na * (W + 1);
  }
  for (int i = 0; i < n; ++i) {
    const int s = slots[i];
    if (ssm_of[i] < 0) {
      if (out && out->accepted) out->accepted[i] = 0;
      if (out && out->bonus_token) out->bonus_token[i] = -1;
      if (out && out->committed) out->committed[i] = h_committed_[s];
      continue;
    }
    const Rows& r = rows_of[i];
    const int a = r.a, acc = r.acc[a], bon = r.bon[a], com = r.com[a];
    const int32_t* dr = r.dr + static_cast<size_t>(a) * W;
    const int c = h_committed_[s];
    int32_t* hist = h_tokens_.data() + static_cast<size_t>(s) * opts_.max_ctx;
    for (int k = 0; k < acc; ++k) hist[c + k] = dr[k];
    hist[c + acc] = bon;
    h_committed_[s] = com;
    int32_t& len = h_ssm_len_[static_cast<size_t>(ssm_of[i]) * R + s];
    len = std::min(c + W - 1, c + acc);
    if (out) {
      if (out->accepted) out->accepted[i] = acc;
      if (out->bonus_token) out->bonus_token[i] = bon;
      if (out->committed) out->committed[i] = com;
      if (out->drafts) std::memcpy(out->drafts + static_cast<size_t>(i) * W, dr, W * 4);
      if (out->target_tokens)
        std::memcpy(out->target_tokens + static_cast<size_t>(i) * (W + 1), r.tg + static_cast<size_t>(a) * (W + 1),
                    (W + 1) * 4);
    }
  }
  float switch_ms = 0.f;
  if (sw_total > 0) check_cuda(cudaEventElapsedTime(&switch_ms, ev_r0_, ev_r1_), "event timing");
  last_switch_ms_ = switch_ms;
  if (out) {
    out->draft_ms = draft_ms;
    out->round_ms = total_ms + switch_ms;
    out->verify_ms = verify_ms;
    out->switch_ms = switch_ms;
    out->switch_tokens = static_cast<int32_t>(sw_total);
    for (int j = 0; j < SPIN_MAX_SSM; ++j) out->spec_end_ms[j] = j < M ? last_spec_ms_[j] : -1.f;
    if (out->switch_tokens_per_request) std::memcpy(out->switch_tokens_per_request, sw_tok.data(), n * 4);
  }
}

void Engine::run_rounds(int n, const int32_t* slots, const int32_t* ssm_of, int rounds, int64_t* emitted, float* ms) {
  if (rounds < 1) fail(SPIN_INPUT_ERROR, "run_rounds: rounds must be >= 1");
  sync_state_from_device();
  const int W = opts_.window;
  for (int i = 0; i < n; ++i) {
    // the host-driven warm-up round + `rounds` graph replays, each committing up to W + 1
    if (ssm_of[i] >= 0 && h_committed_[slots[i]] + static_cast<int64_t>(rounds + 1) * (W + 1) > opts_.max_ctx)
      fail(SPIN_CAPACITY_ERROR, "run_rounds: context would overflow max_ctx");
  }
  // one host-driven round first: validates, switches SSMs, captures the graph
  spin_round_out tmp{};
  round(n, slots, ssm_of, nullptr, &tmp);
  const bool pipe = pipelined();
  RoundPlan* p = pipe ? nullptr : &plan_round(n, slots, ssm_of);
  PipePlan* pp = pipe ? &plan_pipe(n, ssm_of) : nullptr;
  std::vector<unsigned long long> counts(rounds, 0);
  unsigned long long* d_counts = nullptr;
  check_cuda(cudaMalloc(&d_counts, rounds * 8), "counts");
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  check_cuda(cudaMemsetAsync(d_emitted_, 0, 8, sv_), "memset");
  check_cuda(cudaEventRecord(a, sv_), "event");
  for (int r = 0; r < rounds; ++r) {
    if (pipe)  // slots overlap: a unit's next draft waits only for that unit's verification
      launch_pipe_slot(*pp, r == 0, false);
    else if (opts_.use_graphs)
      check_cuda(cudaGraphLaunch(p->exec, sv_), "graph launch");
    else
      capture_round(*p);
    check_cuda(cudaMemcpyAsync(d_counts + r, d_emitted_, 8, cudaMemcpyDeviceToDevice, sv_), "count");
  }
  check_cuda(cudaEventRecord(b, sv_), "event");
  sync_sv("rounds");
  float t = 0.f;
  cudaEventElapsedTime(&t, a, b);
  check_cuda(cudaMemcpy(counts.data(), d_counts, rounds * 8, cudaMemcpyDeviceToHost), "d2h");
  cudaFree(d_counts);
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  unsigned long long prev = 0;
  for (int r = 0; r < rounds; ++r) {
    if (emitted) emitted[r] = static_cast<int64_t>(counts[r] - prev);
    prev = counts[r];
  }
  if (ms) *ms = t;
  mirror_stale_ = true;
}

void Engine::profile_round(int n, const int32_t* slots, const int32_t* ssm_of, double* ms, double* bytes,
                           int64_t* launches) {
  join_prewarm();
  const int saved = opts_.use_graphs;
  opts_.use_graphs = 0;
  prof_ = true;
  prof_recs_.clear();
  try {
    round(n, slots, ssm_of, nullptr, nullptr);
  } catch (...) {
    prof_ = false;
    opts_.use_graphs = saved;
    throw;
  }
  prof_ = false;
  opts_.use_graphs = saved;
  for (int c = 0; c < kProfCats; ++c) ms[c] = bytes[c] = 0.0, launches[c] = 0;
  for (auto& r : prof_recs_) {
    float t = 0.f;
    check_cuda(cudaEventElapsedTime(&t, r.a, r.b), "profile timing");
    ms[r.cat] += t;
    bytes[r.cat] += r.bytes;
    ++launches[r.cat];
    cudaEventDestroy(r.a);
    cudaEventDestroy(r.b);
  }
  prof_recs_.clear();
}

// In-situ kernel benchmark on the target's state of the last verify: kind 0
// replays the 4 projection GEMMs of every layer, kind 1 the attention (+combine)
// of every layer, as one CUDA graph launched `iters` times; per-launch device
// time and algorithmic bytes (weights + activations in/out, or KV read + q/out).
void Engine::kernel_bench(int kind, int iters, double* us_per_launch, double* bytes_per_launch) {
  sync_state_from_device();
  join_prewarm();
  const int T = last_verify_rows_;
  if (T <= 0) fail(SPIN_INPUT_ERROR, "kernel_bench: run a round first");
  if (iters < 1) fail(SPIN_INPUT_ERROR, "kernel_bench: iters must be >= 1");
  ModelDev& m = target_;
  Lane& ln = tlane_;
  const int D = m.D, F = m.F, n = T / (opts_.window + 1);
  const bool pdl = opts_.use_pdl != 0;
  double bytes = 0.0;
  int launches = 0;
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
  check_cuda(cudaStreamBeginCapture(sv_, cudaStreamCaptureModeRelaxed), "capture");
  capturing_ = true;
  GemmEpilogue ep;
  ep.mode = kGemmPartial;
  ep.part = ln.part;
  AttnGeom g{m.H, m.hd, opts_.max_requests, opts_.max_ctx, 0, static_cast<float>(1.0 / std::sqrt(double(m.hd))),
             m.kc, m.vc};
  AttnWork aw = ln.aw;
  aw.qmax = opts_.window + 1;
  const int bench_rows = opts_.packing ? (opts_.pack_width > 0 ? std::min(opts_.pack_width, n) : n) : n;
  aw.chunks = attn_chunks(bench_rows, m.H, num_sms_);
  double kv_tokens = 0.0;
  for (int l = 0; l < m.L; ++l) {
    const LayerW& w = m.layers[l];
    if (kind == 0) {
      const int shapes[4][2] = {{3 * D, D}, {D, D}, {2 * F, D}, {D, F}};
      const bf16* W[4] = {w.qkv, w.o, w.gu, w.dn};
      const bf16* X[4] = {ln.xn, ln.attn, ln.xn, ln.act};
      for (int k = 0; k < 4; ++k) {
        check_cuda(gemm_launch(plan(shapes[k][0], shapes[k][1], T, kGemmPartial), W[k], X[k], ep, sv_, pdl), "gemm");
        bytes += 2.0 * shapes[k][0] * shapes[k][1] + 2.0 * T * shapes[k][1] + 2.0 * T * shapes[k][0];
        ++launches;
      }
    } else {
      g.layer = l;
      launch_attention(m.tm_k, m.tm_v, ln.meta, bench_rows, n, g, ln.q,
                       aw, ln.attn, sv_);
      ++launches;
    }
  }
  capturing_ = false;
  check_cuda(cudaStreamEndCapture(sv_, &graph), "capture");
  check_cuda(cudaGraphInstantiate(&exec, graph, 0), "instantiate");
  if (kind == 1) {
    // KV bytes actually read: per request kv_len = committed + window at verify time
    std::vector<int32_t> kvl(n);
    check_cuda(cudaMemcpy(kvl.data(), ln.meta.req_kvlen, n * 4, cudaMemcpyDeviceToHost), "d2h");
    for (int i = 0; i < n; ++i) kv_tokens += kvl[i];
    bytes = static_cast<double>(m.L) * (kv_tokens * m.H * m.hd * 2.0 * 2.0 + T * D * 4.0 + T * D * 2.0);
  }
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  check_cuda(cudaGraphLaunch(exec, sv_), "warm");
  check_cuda(cudaEventRecord(a, sv_), "event");
  for (int i = 0; i < iters; ++i) check_cuda(cudaGraphLaunch(exec, sv_), "graph");
  check_cuda(cudaEventRecord(b, sv_), "event");
  sync_sv("sync");
  float ms = 0.f;
  cudaEventElapsedTime(&ms, a, b);
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  cudaGraphExecDestroy(exec);
  cudaGraphDestroy(graph);
  *us_per_launch = ms * 1e3 / (static_cast<double>(iters) * launches);
  *bytes_per_launch = bytes / launches;
}

// Ragged-window verification step (BASELINE config 3): request i verifies
// draft_lens[i] drafts (its pending token + drafts at positions c-1 .. c-1+len).
// packed: request decomposition of the true lengths (pack(), Sigma(len+1) query rows);
// padded: every request padded to the longest window (n x (max+1) query rows, KV
// padded to the longest request -- the reference's naive_padding baseline).
// The KV rows are (re)written idempotently and nothing is committed, so the step
// can be replayed; timing = `iters` replays of one CUDA graph (CUDA events).
void Engine::verify_bench(int n, const int32_t* slots, const int32_t* draft_lens, const int32_t* drafts, int packed,
                          int iters, spin_verify_stats* out) {
  sync_state_from_device();
  join_prewarm();
  const int W = opts_.window, R = opts_.max_requests;
  if (n < 1 || n > R) fail(SPIN_CAPACITY_ERROR, "verify_bench: batch exceeds max_requests");
  if (iters < 1) fail(SPIN_INPUT_ERROR, "verify_bench: iters must be >= 1");
  int gmax = 0;
  std::vector<char> seen(R, 0);
  for (int i = 0; i < n; ++i) {
    if (slots[i] < 0 || slots[i] >= R || seen[slots[i]]) fail(SPIN_INPUT_ERROR, "verify_bench: bad slot list");
    seen[slots[i]] = 1;
    if (draft_lens[i] < 1 || draft_lens[i] > W) fail(SPIN_INPUT_ERROR, "verify_bench: draft length outside 1..window");
    if (h_committed_[slots[i]] < 2) fail(SPIN_INPUT_ERROR, "verify_bench: slot was not prefilled");
    if (h_committed_[slots[i]] + W + 1 > opts_.max_ctx) fail(SPIN_CAPACITY_ERROR, "verify_bench: context is full");
    gmax = std::max(gmax, draft_lens[i]);
  }
  // rows and requests (host-built; the meta kernel only packs)
  std::vector<int32_t> rt, rs, rp, qs, ql, kv, sl;
  size_t doff = 0;
  for (int i = 0; i < n; ++i) {
    const int s = slots[i], c = h_committed_[s], len = draft_lens[i];
    const int q = packed ? len + 1 : gmax + 1;
    qs.push_back(static_cast<int32_t>(rt.size()));
    ql.push_back(q);
    kv.push_back(c - 1 + q);  // last query position + 1
    sl.push_back(s);
    for (int j = 0; j < q; ++j) {
      const bool real = j <= len;
      int32_t tok = h_tokens_[static_cast<size_t>(s) * opts_.max_ctx + c - 1];
      if (j > 0) tok = real && drafts ? drafts[doff + j - 1] : tok;
      rt.push_back(tok);
      rs.push_back(real ? s : -1);  // padding rows write no KV
      rp.push_back(c - 1 + j);
    }
    doff += len;
  }
  const int T = static_cast<int>(rt.size());
  Lane& ln = tlane_;
  if (T > ln.T_cap) fail(SPIN_CAPACITY_ERROR, "verify_bench: too many query rows for this engine (raise window)");
  check_cuda(upload_sync(ln.meta.row_tok, rt.data(), T * 4), "h2d");
  check_cuda(upload_sync(ln.meta.row_slot, rs.data(), T * 4), "h2d");
  check_cuda(upload_sync(ln.meta.row_pos, rp.data(), T * 4), "h2d");
  check_cuda(upload_sync(ln.meta.req_slot, sl.data(), n * 4), "h2d");
  check_cuda(upload_sync(ln.meta.req_qstart, qs.data(), n * 4), "h2d");
  check_cuda(upload_sync(ln.meta.req_qlen, ql.data(), n * 4), "h2d");
  check_cuda(upload_sync(ln.meta.req_kvlen, kv.data(), n * 4), "h2d");
  const int width = opts_.pack_width > 0 ? std::min(opts_.pack_width, n) : n;
  MetaArgs a{};
  a.mode = kMetaExtend;
  a.n_req = n;
  a.width = width;
  a.padded = packed ? 0 : 1;
  a.chunks = attn_chunks(packed ? width : n, target_.H, num_sms_);
  const int qmax = packed ? gmax + 1 : gmax + 1;
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
  check_cuda(cudaStreamBeginCapture(sv_, cudaStreamCaptureModeRelaxed), "capture");
  capturing_ = true;
  launch_meta(a, st_, ln.meta, sv_);
  forward(target_, ln, FwdShape{T, n, packed ? width : n, qmax, 1}, sv_, opts_.debug_logits ? 2 : 1);
  capturing_ = false;
  check_cuda(cudaStreamEndCapture(sv_, &graph), "capture");
  check_cuda(cudaGraphInstantiate(&exec, graph, 0), "instantiate");
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  check_cuda(cudaGraphLaunch(exec, sv_), "warm");
  check_cuda(cudaEventRecord(e0, sv_), "event");
  for (int i = 0; i < iters; ++i) check_cuda(cudaGraphLaunch(exec, sv_), "graph");
  check_cuda(cudaEventRecord(e1, sv_), "event");
  sync_sv("verify_bench");
  float ms = 0.f;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaEventDestroy(e0), cudaEventDestroy(e1);
  cudaGraphExecDestroy(exec), cudaGraphDestroy(graph);
  // target argmax per real query row (lowest index on ties over the 128-row lm_head tiles)
  const int tiles = (target_.V + 127) / 128;
  std::vector<float> av(static_cast<size_t>(tiles) * T);
  std::vector<int32_t> ai(static_cast<size_t>(tiles) * T);
  check_cuda(cudaMemcpy(av.data(), ln.amax_val, av.size() * 4, cudaMemcpyDeviceToHost), "d2h");
  check_cuda(cudaMemcpy(ai.data(), ln.amax_idx, ai.size() * 4, cudaMemcpyDeviceToHost), "d2h");
  int64_t kv_read = 0, real_rows = 0;
  size_t o = 0;
  for (int i = 0; i < n; ++i) {
    for (int j = 0; j <= draft_lens[i]; ++j) {
      const int row = qs[i] + j;
      float bv = -INFINITY;
      int bi = 0x7fffffff;
      for (int tl = 0; tl < tiles; ++tl) {
        const float v = av[static_cast<size_t>(tl) * T + row];
        const int id = ai[static_cast<size_t>(tl) * T + row];
        if (v > bv || (v == bv && id < bi)) bv = v, bi = id;
      }
      if (out && out->target_tokens) out->target_tokens[o] = bi;
      ++o;
    }
    real_rows += draft_lens[i] + 1;
  }
  if (packed) {
    for (int i = 0; i < n; ++i) kv_read += kv[i];
  } else {
    int longest = 0;
    for (int i = 0; i < n; ++i) longest = std::max(longest, kv[i]);
    kv_read = static_cast<int64_t>(longest) * n;
  }
  last_verify_rows_ = 0;  // the kernel_bench replays expect a round's layout
  if (out) {
    out->us = ms * 1e3 / iters;
    out->query_rows = T;
    out->real_rows = real_rows;
    out->kv_tokens = kv_read;
  }
}

void Engine::last_round_trace(float* spec_end_ms, int cap) const {
  for (int j = 0; j < cap && j < static_cast<int>(last_spec_ms_.size()); ++j) spec_end_ms[j] = last_spec_ms_[j];
}

int64_t Engine::launches_per_round(int n, const int32_t* slots, const int32_t* ssm_of) {
  if (pipelined()) return plan_pipe(n, ssm_of).launches;
  return plan_round(n, slots, ssm_of).launches;
}

void Engine::read_tokens(int slot, int32_t* tokens, int cap, int32_t* len) {
  sync_state_from_device();
  if (slot < 0 || slot >= opts_.max_requests) fail(SPIN_INPUT_ERROR, "read_tokens: slot out of range");
  const int c = h_committed_[slot];
  *len = c;
  std::memcpy(tokens, h_tokens_.data() + static_cast<size_t>(slot) * opts_.max_ctx, std::min(c, cap) * 4);
}

void Engine::read_logits(float* logits, int64_t cap, int32_t* rows) {
  if (!opts_.debug_logits) fail(SPIN_CONFIG_ERROR, "read_logits: engine created without debug_logits");
  const int64_t need = static_cast<int64_t>(last_verify_rows_) * target_.V;
  if (cap < need) fail(SPIN_SIZE_ERROR, "read_logits: buffer too small");
  check_cuda(cudaMemcpy(logits, tlane_.logits, need * 4, cudaMemcpyDeviceToHost), "d2h logits");
  *rows = last_verify_rows_;
}

}  // namespace spin

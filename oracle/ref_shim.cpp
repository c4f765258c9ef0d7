// extern "C" shim over the UNMODIFIED reference library functions on the
// verification path, compiled together with the reference's own sources
// (see oracle/Makefile, target `ref`). TEST INFRASTRUCTURE ONLY: used to pin
// the oracle and to generate tests/golden/ fixtures; never shipped or linked
// by libspin.so. Output goes to oracle/_ref/ (git-ignored).
#include <chrono>
#include <cstring>
#include <numeric>
#include <exception>
#include <vector>

#include "specsim/attention.hpp"
#include "specsim/bandit.hpp"
#include "specsim/errors.hpp"
#include "specsim/model.hpp"
#include "specsim/packing.hpp"
#include "specsim/rng.hpp"
#include "specsim/slot_engine.hpp"

using namespace specsim;

namespace {
int code_of(const std::exception& e) {
  if (dynamic_cast<const ConfigError*>(&e)) return 1;
  if (dynamic_cast<const CapacityError*>(&e)) return 2;
  if (dynamic_cast<const InputError*>(&e)) return 3;
  if (dynamic_cast<const SizeError*>(&e)) return 4;
  if (dynamic_cast<const ConsistencyError*>(&e)) return 5;
  if (dynamic_cast<const MetricError*>(&e)) return 6;
  if (dynamic_cast<const IoError*>(&e)) return 7;
  return 99;
}
template <typename F>
int run(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::exception& e) {
    return code_of(e);
  }
}
Matrix mat(const double* p, int r, int c) {
  Matrix m(r, c);
  std::memcpy(m.data.data(), p, sizeof(double) * r * c);
  return m;
}
}  // namespace

extern "C" {

unsigned long long ref_mix_seed(unsigned long long s, unsigned long long a, unsigned long long b,
                                unsigned long long c) {
  return mix_seed(s, a, b, c);
}

// Draws `count` values from Rng(seed): kind 0 next(), 1 unit(), 2 uniform_int(lo, hi).
void ref_rng_draws(unsigned long long seed, int kind, long long lo, long long hi, int count, double* out_d,
                   unsigned long long* out_u) {
  Rng r(seed);
  for (int i = 0; i < count; ++i) {
    if (kind == 0) out_u[i] = r.next();
    if (kind == 1) out_d[i] = r.unit();
    if (kind == 2) out_u[i] = static_cast<unsigned long long>(r.uniform_int(lo, hi));
  }
}

void ref_make_toy_input(unsigned long long seed, int queries, int kv_len, int dim, double* q, double* k,
                        double* v) {
  const ToyAttentionInput in = make_toy_input(seed, queries, kv_len, dim);
  std::memcpy(q, in.q.data.data(), sizeof(double) * queries * dim);
  std::memcpy(k, in.k.data.data(), sizeof(double) * kv_len * dim);
  std::memcpy(v, in.v.data.data(), sizeof(double) * kv_len * dim);
}

int ref_pack(const int* kv_lens, int n, int width, int* length, int* rows, int* segs, int seg_cap, int* n_segs,
             long long* padding, int* q_replica_rows) {
  return run([&] {
    const PackedLayout L = pack(std::vector<int>(kv_lens, kv_lens + n), width);
    *length = L.length;
    *rows = L.width;
    *padding = L.padding_tokens;
    *n_segs = static_cast<int>(L.segments.size());
    if (*n_segs > seg_cap) throw SizeError("segment buffer");
    for (int i = 0; i < *n_segs; ++i) {
      const Segment& s = L.segments[i];
      int* o = segs + 5 * i;
      o[0] = s.request_id, o[1] = s.row, o[2] = s.col_start, o[3] = s.col_end, o[4] = s.token_offset;
    }
    for (int i = 0; i < static_cast<int>(L.q_replica_rows.size()); ++i) q_replica_rows[i] = L.q_replica_rows[i];
  });
}

int ref_naive_padding(const int* kv_lens, int n, long long* padding) {
  return run([&] { *padding = naive_padding(std::vector<int>(kv_lens, kv_lens + n)); });
}

int ref_verify_batch_cost(const int* kv_lens, int n, int window, int packing, int pack_width, long long* tokens,
                          long long* padding) {
  return run([&] {
    const VerifyBatchCost c = verify_batch_cost(std::vector<int>(kv_lens, kv_lens + n), window, packing != 0,
                                                pack_width);
    *tokens = c.tokens;
    *padding = c.padding;
  });
}

int ref_reference_attention(int qr, int kr, int dim, const double* q, const double* k, const double* v,
                            double* out) {
  return run([&] {
    const Matrix o = reference_attention(mat(q, qr, dim), mat(k, kr, dim), mat(v, kr, dim));
    std::memcpy(out, o.data.data(), sizeof(double) * qr * dim);
  });
}

// Packs the requests' kv lengths itself (pack(kv_rows, width)) like the
// reference tests do, then runs decomposed_attention on that layout.
int ref_decomposed_attention(int n, int dim, const int* q_rows, const int* kv_rows, const double* q, const double* k,
                             const double* v, int width, double* out) {
  return run([&] {
    std::vector<ToyAttentionInput> in(n);
    std::vector<int> lens(n);
    long qo = 0, ko = 0;
    for (int i = 0; i < n; ++i) {
      in[i].q = mat(q + qo * dim, q_rows[i], dim);
      in[i].k = mat(k + ko * dim, kv_rows[i], dim);
      in[i].v = mat(v + ko * dim, kv_rows[i], dim);
      lens[i] = kv_rows[i];
      qo += q_rows[i];
      ko += kv_rows[i];
    }
    const PackedLayout L = pack(lens, width);
    const auto outs = decomposed_attention(in, L, build_indicator(L));
    long oo = 0;
    for (int i = 0; i < n; ++i) {
      std::memcpy(out + oo * dim, outs[i].data.data(), sizeof(double) * q_rows[i] * dim);
      oo += q_rows[i];
    }
  });
}

int ref_sample_accepted_prefix(double p, int window, unsigned long long seed, int draws, int* out) {
  return run([&] {
    Request r;
    r.accept_prob = {p};
    Rng rng(seed);
    for (int i = 0; i < draws; ++i) out[i] = sample_accepted_prefix(r, 0, window, rng);
  });
}

double ref_expected_accepted_prefix(double p, int window) { return expected_accepted_prefix(p, window); }

// Replays run_lbss's control flow (bandit.cpp:248-332) with the reference's own
// selector functions (draw_exploration_assignment, prewarm_destination,
// plan_exploitation, exploitation_duration) on a synthetic observation table:
// at slot t every served request i on ssm j observes
//   goodput = g[i*m + j] * (1 + 0.05 * ((i + 3*j + t) % 5)).
// Writes assignment / prewarm [slots][n] and the explore flag per slot.
int ref_lbss_trace(int n, int m, const int* caps, int alpha, int beta, unsigned long long seed, int slots,
                   const double* g, int* assign_out, int* prewarm_out, int* explore_out) {
  return run([&] {
    BanditConfig cfg;
    cfg.alpha = alpha;
    cfg.beta = beta;
    cfg.max_slots = slots;
    validate(cfg);
    std::vector<SsmProfile> ssms(m);
    for (int j = 0; j < m; ++j) ssms[j].id = j, ssms[j].batch_capacity = caps[j];
    std::vector<int> admitted(n);
    std::iota(admitted.begin(), admitted.end(), 0);
    BanditState st = BanditState::make(n, m);
    Rng rng(mix_seed(seed, kStreamPolicy));
    int t = 0;
    auto emit_observe = [&](const std::vector<int>& a, const std::vector<int>& pw, int explore) {
      std::memcpy(assign_out + static_cast<size_t>(t) * n, a.data(), sizeof(int) * n);
      std::memcpy(prewarm_out + static_cast<size_t>(t) * n, pw.data(), sizeof(int) * n);
      explore_out[t] = explore;
      for (int i = 0; i < n; ++i)
        if (a[i] >= 0) st.estimates[i][a[i]].add(g[i * m + a[i]] * (1.0 + 0.05 * ((i + 3 * a[i] + t) % 5)));
      ++t;
    };
    while (t < slots) {
      for (int chunk = 0; chunk < alpha / beta && t < slots; ++chunk) {
        std::vector<int> a = draw_exploration_assignment(admitted, ssms, n, rng);
        st.prewarmed = a;
        for (int s = 0; s < beta && t < slots; ++s) emit_observe(a, st.prewarmed, 1);
      }
      if (t >= slots) break;
      st.prewarmed = prewarm_destination(st, admitted);
      const std::vector<int> plan = plan_exploitation(st, admitted, ssms);
      const long long dur = exploitation_duration(st.epoch, slots - t);
      for (long long s = 0; s < dur; ++s) emit_observe(plan, st.prewarmed, 0);
      ++st.epoch;
    }
  });
}

// ---- single-threaded timings of the reference's own hot-path functions
// (BASELINE.md section 4 row 1), on the caller's config-2 shapes. Seconds per call.
namespace {
double now_s() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}
volatile long long g_sink = 0;
}  // namespace

double ref_time_pack(const int* kv_lens, int n, int width, int iters) {
  const std::vector<int> lens(kv_lens, kv_lens + n);
  const double t0 = now_s();
  for (int i = 0; i < iters; ++i) g_sink = g_sink + pack(lens, width).padding_tokens;
  return (now_s() - t0) / iters;
}

double ref_time_verify_batch_cost(const int* kv_lens, int n, int window, int packing, int width, int iters) {
  const std::vector<int> lens(kv_lens, kv_lens + n);
  const double t0 = now_s();
  for (int i = 0; i < iters; ++i) g_sink = g_sink + verify_batch_cost(lens, window, packing != 0, width).tokens;
  return (now_s() - t0) / iters;
}

// One head of the paper's decomposed attention (attention.cpp:98-162) over the
// batch: request i has q_rows queries against kv_lens[i] keys of width dim
// (make_toy_input data), packed by pack(kv_lens, width). Seconds per call.
double ref_time_decomposed_attention(const int* kv_lens, int n, int q_rows, int dim, int width, int iters) {
  std::vector<ToyAttentionInput> in;
  std::vector<int> lens(kv_lens, kv_lens + n);
  for (int i = 0; i < n; ++i) in.push_back(make_toy_input(1000 + i, q_rows, kv_lens[i], dim));
  const PackedLayout L = pack(lens, width);
  const IndicatorMask mask = build_indicator(L);
  const double t0 = now_s();
  for (int i = 0; i < iters; ++i) g_sink = g_sink + static_cast<long long>(decomposed_attention(in, L, mask).size());
  return (now_s() - t0) / iters;
}

// SlotEngine::run_slot (slot_engine.cpp:70-167) on a config-2-like spec: n requests
// with prompts U[lo, hi], 2 SSMs of capacity n, packing on; every request on ssm i%2.
// Seconds per slot over `slots` slots.
double ref_time_run_slot(int n, int prompt_lo, int prompt_hi, int window, int slots) {
  WorkloadSpec spec;
  spec.num_requests = n;
  spec.window = window;
  spec.seed = 2503;
  for (int j = 0; j < 2; ++j) {
    SsmProfile p;
    p.id = j;
    p.tokens_per_sec = j == 0 ? 400.0 : 150.0;
    p.batch_capacity = n;
    p.batch_slowdown = 0.01;
    spec.ssm_profiles.push_back(p);
  }
  spec.llm.fixed_overhead_sec = 0.02;
  spec.llm.per_token_sec = 1e-5;
  DifficultyClass c;
  c.name = "mix";
  c.accept_range = {{0.5, 0.8}, {0.6, 0.9}};
  c.prompt_len_lo = prompt_lo;
  c.prompt_len_hi = prompt_hi;
  c.target_len_lo = 1000000;
  c.target_len_hi = 1000000;
  spec.difficulty_mix.push_back(c);
  EngineOptions opt;
  opt.packing = true;
  SlotEngine eng(spec, generate_workload(spec), opt);
  std::vector<int> assign(n), prewarm(n, -1);
  for (int i = 0; i < n; ++i) assign[i] = i % 2;
  const double t0 = now_s();
  for (int t = 0; t < slots; ++t) g_sink = g_sink + eng.run_slot(assign, prewarm, false, nullptr).served;
  return (now_s() - t0) / slots;
}

}  // extern "C"

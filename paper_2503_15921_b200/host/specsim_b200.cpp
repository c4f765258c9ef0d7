// Host side of the drop-in API (include/specsim/*.hpp) over the C ABI of
// libspin.so. Reference semantics cited per function (paths under
// /root/reference/proj/core); compute goes to the B200 through spin_*.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <string>

#include "spin_c.h"
#include "specsim/attention.hpp"
#include "specsim/errors.hpp"
#include "specsim/model.hpp"
#include "specsim/packing.hpp"
#include "specsim/rng.hpp"
#include "specsim/slot_engine.hpp"

namespace specsim {

void throw_status(int status, const std::string& message) {
  switch (status) {
    case SPIN_OK: return;
    case SPIN_CONFIG_ERROR: throw ConfigError(message);
    case SPIN_CAPACITY_ERROR: throw CapacityError(message);
    case SPIN_INPUT_ERROR: throw InputError(message);
    case SPIN_SIZE_ERROR: throw SizeError(message);
    case SPIN_CONSISTENCY_ERROR: throw ConsistencyError(message);
    case SPIN_METRIC_ERROR: throw MetricError(message);
    case SPIN_IO_ERROR: throw IoError(message);
    default: throw CudaError(message);
  }
}

namespace {
void check(spin_status st) {
  if (st != SPIN_OK) throw_status(st, spin_last_error());
}
}  // namespace

// ------------------------------------------------------------------ rng.hpp:11-68
std::uint64_t splitmix64(std::uint64_t x) {
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}

std::uint64_t mix_seed(std::uint64_t seed, std::uint64_t a, std::uint64_t b, std::uint64_t c) {
  std::uint64_t h = splitmix64(seed);
  for (std::uint64_t tag : {a, b, c}) h = splitmix64(h ^ tag);
  return h;
}

double Rng::unit() { return static_cast<double>(engine_() >> 11) * 0x1.0p-53; }
double Rng::uniform(double lo, double hi) { return lo + (hi - lo) * unit(); }
long long Rng::uniform_int(long long lo, long long hi) {
  if (hi <= lo) return lo;
  const std::uint64_t span = static_cast<std::uint64_t>(hi - lo) + 1;
  const std::uint64_t limit = UINT64_MAX - UINT64_MAX % span;
  std::uint64_t v = engine_();
  while (v >= limit) v = engine_();
  return lo + static_cast<long long>(v % span);
}

// ------------------------------------------------------------------ model.cpp
int WorkloadSpec::total_capacity() const {
  int cap = 0;
  for (const SsmProfile& s : ssm_profiles) cap += s.batch_capacity;
  return cap;
}

// model.cpp:10-71
void validate(const WorkloadSpec& spec) {
  auto bad = [](const std::string& m) { throw ConfigError(m); };
  if (spec.ssm_profiles.empty()) bad("workload: ssm_profiles must not be empty");
  if (spec.num_requests < 0) bad("workload: num_requests must be non-negative");
  if (spec.window < 1) bad("workload: window must be at least 1");
  for (const SsmProfile& s : spec.ssm_profiles) {
    const std::string who = "ssm " + std::to_string(s.id);
    if (!(s.tokens_per_sec > 0.0)) bad(who + ": tokens_per_sec must be positive");
    if (s.batch_capacity < 1) bad(who + ": batch_capacity must be at least 1");
    if (s.batch_slowdown < 0.0) bad(who + ": batch_slowdown must be non-negative");
  }
  if (!(spec.llm.fixed_overhead_sec >= 0.0) || !std::isfinite(spec.llm.fixed_overhead_sec))
    bad("llm: fixed_overhead_sec must be finite and >= 0");
  if (!(spec.llm.per_token_sec >= 0.0) || !std::isfinite(spec.llm.per_token_sec))
    bad("llm: per_token_sec must be finite and >= 0");
  if (spec.difficulty_mix.empty()) bad("workload: difficulty_mix must not be empty");
  double weights = 0.0;
  for (const DifficultyClass& c : spec.difficulty_mix) {
    const std::string who = "class " + c.name;
    if (c.weight < 0.0) bad(who + ": weight must be non-negative");
    weights += c.weight;
    if (c.accept_range.size() != spec.ssm_profiles.size()) bad(who + ": accept_range needs one [lo, hi] entry per ssm");
    for (const auto& r : c.accept_range)
      if (!(0.0 <= r.first && r.first <= r.second && r.second <= 1.0))
        bad(who + ": acceptance ranges must satisfy 0 <= lo <= hi <= 1");
    if (c.prompt_len_lo < 1 || c.prompt_len_hi < c.prompt_len_lo) bad(who + ": invalid prompt length range");
    if (c.target_len_lo < 1 || c.target_len_hi < c.target_len_lo) bad(who + ": invalid target length range");
  }
  if (std::abs(weights - 1.0) > 1e-9) bad("workload: difficulty_mix weights must sum to 1");
}

// model.cpp:73-108: class by cumulative weight, lengths, then per-SSM
// acceptance -- the draw order is the determinism contract.
std::vector<Request> generate_workload(const WorkloadSpec& spec) {
  validate(spec);
  Rng rng(mix_seed(spec.seed, kStreamWorkload));
  std::vector<Request> out;
  out.reserve(spec.num_requests);
  for (int i = 0; i < spec.num_requests; ++i) {
    const double u = rng.unit();
    std::size_t cls = spec.difficulty_mix.size() - 1;
    double cum = 0.0;
    for (std::size_t c = 0; c < spec.difficulty_mix.size(); ++c) {
      cum += spec.difficulty_mix[c].weight;
      if (u < cum) {
        cls = c;
        break;
      }
    }
    const DifficultyClass& dc = spec.difficulty_mix[cls];
    Request r;
    r.id = i;
    r.prompt_len = static_cast<int>(rng.uniform_int(dc.prompt_len_lo, dc.prompt_len_hi));
    r.target_len = rng.uniform_int(dc.target_len_lo, dc.target_len_hi);
    for (const auto& range : dc.accept_range)
      r.accept_prob.push_back(range.first == range.second ? range.first : rng.uniform(range.first, range.second));
    out.push_back(std::move(r));
  }
  return out;
}

// model.cpp:110-134 (the Bernoulli stand-in of the reference simulator).
int sample_accepted_prefix(const Request& request, int ssm_id, int window, Rng& rng) {
  if (ssm_id < 0 || static_cast<std::size_t>(ssm_id) >= request.accept_prob.size())
    throw InputError("sample_accepted_prefix: unknown ssm id " + std::to_string(ssm_id));
  if (window < 1) throw InputError("sample_accepted_prefix: window must be at least 1");
  int run = 0;
  bool alive = true;
  for (int k = 0; k < window; ++k) {
    const bool hit = rng.bernoulli(request.accept_prob[ssm_id]);
    alive = alive && hit;
    run += alive ? 1 : 0;
  }
  return run;
}

double expected_accepted_prefix(double p, int window) {
  if (p >= 1.0) return window;
  if (p <= 0.0) return 0.0;
  return (p - std::pow(p, window + 1)) / (1.0 - p);
}

double speculation_time(const SsmProfile& ssm, int batch_size, int window) {
  if (batch_size < 1) throw CapacityError("speculation_time: batch_size must be at least 1");
  if (batch_size > ssm.batch_capacity)
    throw CapacityError("speculation_time: batch_size " + std::to_string(batch_size) + " exceeds capacity " +
                        std::to_string(ssm.batch_capacity) + " of ssm " + std::to_string(ssm.id));
  return window / ssm.tokens_per_sec * (1.0 + ssm.batch_slowdown * (batch_size - 1));
}

double verification_time(const LlmProfile& llm, long long total_tokens) {
  if (total_tokens < 0) throw InputError("verification_time: token count must be non-negative");
  return llm.fixed_overhead_sec + llm.per_token_sec * static_cast<double>(total_tokens);
}

double observed_goodput(const SpeculationOutcome& o) {
  if (!(o.wall_time_sec > 0.0)) throw InputError("observed_goodput: wall time must be positive");
  return (o.accepted + o.bonus) / o.wall_time_sec;
}

// ------------------------------------------------------------------ packing
PackedLayout pack(const std::vector<int>& kv_lens, int width) {
  const int n = static_cast<int>(kv_lens.size());
  const int rows_cap = std::max(1, std::min(width, n));
  std::vector<spin_segment> segs(n + rows_cap + 1);
  std::vector<int32_t> reps(std::max(n, 1));
  int32_t L = 0, rows = 0, ns = 0;
  int64_t pad = 0;
  check(spin_pack(kv_lens.data(), n, width, &L, &rows, segs.data(), static_cast<int32_t>(segs.size()), &ns, &pad,
                  reps.data()));
  PackedLayout out;
  out.length = L;
  out.width = rows;
  out.padding_tokens = pad;
  for (int s = 0; s < ns; ++s)
    out.segments.push_back({segs[s].request_id, segs[s].row, segs[s].col_start, segs[s].col_end, segs[s].token_offset});
  if (n > 0) out.q_replica_rows.assign(reps.begin(), reps.begin() + n);
  return out;
}

long long naive_padding(const std::vector<int>& kv_lens) {
  int64_t pad = 0;
  check(spin_naive_padding(kv_lens.data(), static_cast<int32_t>(kv_lens.size()), &pad));
  return pad;
}

// packing.cpp:115-136
IndicatorMask build_indicator(const PackedLayout& layout) {
  IndicatorMask mask;
  mask.width = layout.width;
  mask.length = layout.length;
  mask.cells.assign(static_cast<std::size_t>(layout.width) * layout.length, kEmptyCell);
  for (const Segment& s : layout.segments) {
    if (s.row < 0 || s.row >= layout.width || s.col_start < 0 || s.col_end > layout.length || s.col_start >= s.col_end)
      throw ConsistencyError("build_indicator: segment out of bounds");
    for (int c = s.col_start; c < s.col_end; ++c) {
      if (mask.at(s.row, c) != kEmptyCell)
        throw ConsistencyError("build_indicator: overlapping segments at row " + std::to_string(s.row) + " col " +
                               std::to_string(c));
      mask.at(s.row, c) = s.request_id;
    }
  }
  return mask;
}

// ------------------------------------------------------------------ attention
Matrix reference_attention(const Matrix& q, const Matrix& k, const Matrix& v) {
  if (k.rows != v.rows || q.cols != k.cols || v.cols != q.cols) throw InputError("reference_attention: shape mismatch");
  if (k.rows == 0) throw InputError("reference_attention: empty KV");
  Matrix out(q.rows, q.cols);
  check(spin_reference_attention(q.rows, k.rows, q.cols, q.data.data(), k.data.data(), v.data.data(), out.data.data()));
  return out;
}

std::vector<Matrix> decomposed_attention(const std::vector<ToyAttentionInput>& inputs, const PackedLayout& layout,
                                         const IndicatorMask& mask) {
  const int n = static_cast<int>(inputs.size());
  const int dim = n > 0 ? inputs[0].q.cols : 0;
  std::vector<int32_t> qr(n), kr(n);
  std::vector<double> q, k, v;
  for (int i = 0; i < n; ++i) {
    const ToyAttentionInput& in = inputs[i];
    if (in.k.rows != in.v.rows || in.k.cols != in.q.cols || in.v.cols != in.q.cols || in.q.cols != dim)
      throw InputError("decomposed_attention: inconsistent input shapes");
    qr[i] = in.q.rows;
    kr[i] = in.k.rows;
    q.insert(q.end(), in.q.data.begin(), in.q.data.end());
    k.insert(k.end(), in.k.data.begin(), in.k.data.end());
    v.insert(v.end(), in.v.data.begin(), in.v.data.end());
  }
  if (mask.width != layout.width || mask.length != layout.length)
    throw ConsistencyError("decomposed_attention: mask does not match layout");
  std::vector<spin_segment> segs;
  for (const Segment& s : layout.segments) segs.push_back({s.request_id, s.row, s.col_start, s.col_end, s.token_offset});
  std::vector<double> out(q.size());
  check(spin_decomposed_attention(n, std::max(dim, 1), qr.data(), kr.data(), q.data(), k.data(), v.data(), segs.data(),
                                  static_cast<int32_t>(segs.size()), layout.width, layout.length, mask.cells.data(),
                                  out.data()));
  std::vector<Matrix> res;
  std::size_t off = 0;
  for (int i = 0; i < n; ++i) {
    Matrix m(qr[i], dim);
    std::copy(out.begin() + off, out.begin() + off + m.data.size(), m.data.begin());
    off += m.data.size();
    res.push_back(std::move(m));
  }
  return res;
}

// attention.cpp:164-175
ToyAttentionInput make_toy_input(std::uint64_t seed, int queries, int kv_len, int dim) {
  Rng rng(mix_seed(seed, kStreamToyAttention));
  ToyAttentionInput in{Matrix(queries, dim), Matrix(kv_len, dim), Matrix(kv_len, dim)};
  for (Matrix* m : {&in.q, &in.k, &in.v})
    for (double& x : m->data) x = rng.uniform(-1.0, 1.0);
  return in;
}

// ------------------------------------------------------------------ slot engine
double switching_cost(const Request& request, int from_ssm, int to_ssm, int prewarmed_ssm,
                      const std::vector<SsmProfile>& ssms) {
  if (from_ssm == to_ssm || from_ssm < 0 || to_ssm < 0) return 0.0;
  if (static_cast<std::size_t>(to_ssm) >= ssms.size()) throw InputError("switching_cost: unknown destination ssm");
  if (prewarmed_ssm == to_ssm) return 0.0;
  return static_cast<double>(request.prompt_len + request.generated_len) / ssms[to_ssm].tokens_per_sec;
}

VerifyBatchCost verify_batch_cost(const std::vector<int>& kv_lens, int window, bool packing, int pack_width) {
  int64_t tokens = 0, padding = 0;
  check(spin_verify_batch_cost(kv_lens.data(), static_cast<int32_t>(kv_lens.size()), window, packing ? 1 : 0,
                               pack_width, &tokens, &padding));
  return {tokens, padding};
}

namespace {

// Tiny synthetic family (config 1) used when the caller does not supply models.
spin_model_desc tiny(int d, int layers, uint64_t seed, float gain, float resid) {
  spin_model_desc m{};
  m.d_model = d;
  m.n_layers = layers;
  m.n_heads = d / 64;
  m.head_dim = 64;
  m.ffn = d * 43 / 16;
  m.vocab = 4096;
  m.rope_theta = 10000.f;
  m.rms_eps = 1e-5f;
  m.seed = seed;
  m.embed_scale = 1.f;
  m.planted_gain = gain;
  m.resid_scale = resid;
  m.init_scale = 1.f;
  return m;
}

}  // namespace

// slot_engine.cpp:47-61: admit up to the total SSM capacity in id order.
SlotEngine::SlotEngine(const WorkloadSpec& spec, std::vector<Request> requests, EngineOptions options)
    : spec_(spec), requests_(std::move(requests)), options_(options) {
  last_ssm_.assign(requests_.size(), -1);
  kv_slot_.assign(requests_.size(), -1);
  const int capacity = spec_.total_capacity();
  for (std::size_t i = 0; i < requests_.size(); ++i) {
    if (static_cast<int>(admitted_.size()) < capacity && requests_[i].state != RequestState::Finished) {
      requests_[i].state = RequestState::Active;
      admitted_.push_back(static_cast<int>(i));
    }
    next_waiting_ = static_cast<int>(i) + 1;
    if (static_cast<int>(admitted_.size()) == capacity) break;
  }
  if (!spec_.bonus_token) throw ConfigError("SlotEngine (B200): greedy verification always emits the bonus token");
  // models
  const int M = static_cast<int>(spec_.ssm_profiles.size());
  spin_model_desc target = options_.target_model ? *options_.target_model
                                                 : tiny(256, 4, mix_seed(spec_.seed, 0x10), 9.f, 0.15f);
  std::vector<spin_model_desc> ssms(M);
  for (int j = 0; j < M; ++j)
    ssms[j] = options_.ssm_models ? options_.ssm_models[j]
                                  : tiny(j % 2 ? 256 : 128, 1 + j, mix_seed(spec_.seed, 0x11, j), 7.f + j, 1.2f / (1 + j));
  vocab_ = target.vocab;
  int longest = 2;
  for (const Request& r : requests_)
    longest = std::max<long long>(longest, std::max(2, r.prompt_len) + r.target_len);
  spin_engine_opts eo{};
  eo.device = options_.device;
  eo.max_requests = std::max(1, capacity);
  eo.window = spec_.window;
  eo.max_ctx = options_.max_ctx > 0 ? options_.max_ctx : ((longest + 2 * spec_.window + 8 + 63) / 64) * 64;
  eo.pack_width = options_.pack_width;
  eo.packing = options_.packing ? 1 : 0;
  eo.use_graphs = options_.use_graphs ? 1 : 0;
  eo.use_pdl = 1;
  check(spin_ctx_create(&target, ssms.data(), M, &eo, &ctx_));
  for (int s = eo.max_requests - 1; s >= 0; --s) free_slots_.push_back(s);
  admit_to_device(admitted_);
}

SlotEngine::~SlotEngine() {
  if (ctx_) spin_ctx_destroy(ctx_);
}

// Prompt tokens are synthetic: Rng(mix_seed(seed, kStreamPrompt, id)) draws
// U[0, vocab); a 1-token prompt gets a leading token 0 (the engine keeps the
// last committed token pending, so it needs two).
void SlotEngine::admit_to_device(const std::vector<int>& ids) {
  if (ids.empty()) return;
  std::vector<int32_t> slots, lens, toks;
  for (int id : ids) {
    if (free_slots_.empty()) throw CapacityError("SlotEngine: no free KV slot");
    const int s = free_slots_.back();
    free_slots_.pop_back();
    kv_slot_[id] = s;
    const Request& r = requests_[id];
    Rng rng(mix_seed(spec_.seed, kStreamPrompt, static_cast<std::uint64_t>(id)));
    if (r.prompt_len < 2) toks.push_back(0);
    for (int t = 0; t < r.prompt_len; ++t) toks.push_back(static_cast<int32_t>(rng.uniform_int(0, vocab_ - 1)));
    slots.push_back(s);
    lens.push_back(std::max(2, r.prompt_len));
  }
  check(spin_prefill(ctx_, static_cast<int32_t>(slots.size()), slots.data(), lens.data(), toks.data()));
}

bool SlotEngine::all_finished() const {
  return std::all_of(requests_.begin(), requests_.end(),
                     [](const Request& r) { return r.state == RequestState::Finished; });
}

std::vector<int> SlotEngine::tokens(int request_id) const {
  if (request_id < 0 || request_id >= static_cast<int>(requests_.size()) || kv_slot_[request_id] < 0)
    throw InputError("SlotEngine::tokens: request not resident");
  std::vector<int32_t> buf(8192);
  int32_t len = 0;
  check(spin_read_tokens(ctx_, kv_slot_[request_id], buf.data(), static_cast<int32_t>(buf.size()), &len));
  buf.resize(std::min<int32_t>(len, static_cast<int32_t>(buf.size())));
  return std::vector<int>(buf.begin(), buf.end());
}

// slot_engine.cpp:70-167 with real speculation / verification: one spin_round
// over the served requests; durations are measured device times.
SlotStats SlotEngine::run_slot(const std::vector<int>& assignment, const std::vector<int>& prewarm, bool explore,
                               std::vector<SlotRecord>* history) {
  const int num_ssms = static_cast<int>(spec_.ssm_profiles.size());
  std::vector<int> batch(num_ssms, 0);
  for (int id : admitted_) {
    const int j = assignment[id];
    if (j < 0) continue;
    if (j >= num_ssms) throw InputError("run_slot: unknown ssm in assignment");
    ++batch[j];
  }
  for (int j = 0; j < num_ssms; ++j)
    if (batch[j] > spec_.ssm_profiles[j].batch_capacity)
      throw CapacityError("run_slot: ssm " + std::to_string(j) + " batch exceeds capacity");

  SlotStats stats;
  const long long slot = options_.base_slot + next_slot_;
  std::vector<int32_t> slots, ssm_of;
  std::vector<int> kv_lens;
  for (int id : admitted_) {
    if (assignment[id] < 0) continue;
    slots.push_back(kv_slot_[id]);
    ssm_of.push_back(assignment[id]);
    kv_lens.push_back(static_cast<int>(requests_[id].kv_len(spec_.window)));
  }
  stats.served = static_cast<int>(slots.size());
  const int n = stats.served, W = spec_.window;
  std::vector<int32_t> acc(n), bonus(n), comm(n), sw_tok(n, 0), pw;
  for (int id : admitted_) {
    if (assignment[id] < 0) continue;
    pw.push_back(id < static_cast<int>(prewarm.size()) ? prewarm[id] : -1);
  }
  spin_round_out out{};
  out.accepted = acc.data();
  out.bonus_token = bonus.data();
  out.committed = comm.data();
  out.switch_tokens_per_request = sw_tok.data();
  if (n > 0) {
    // the caller's prewarm destinations are warmed on idle streams during this round
    check(spin_round_prewarm(ctx_, n, slots.data(), ssm_of.data(), pw.data(), &out));
    const VerifyBatchCost cost = verify_batch_cost(kv_lens, W, options_.packing, options_.pack_width);
    stats.verify_tokens = cost.tokens;
    stats.padding_tokens = cost.padding;
    stats.spec_max_sec = out.draft_ms * 1e-3;
    stats.verify_sec = out.verify_ms * 1e-3;
    stats.duration_sec = out.round_ms * 1e-3;
  }
  int k = 0;
  for (int id : admitted_) {
    Request& r = requests_[id];
    const int j = assignment[id];
    SlotRecord rec;
    rec.slot = slot;
    rec.request_id = id;
    rec.ssm_id = j;
    rec.explore = explore;
    if (j >= 0) {
      const int prev = last_ssm_[id];
      rec.switched = prev >= 0 && prev != j;
      // measured switching cost: this request's share (by recomputed KV positions) of
      // the round's synchronous catch-up; 0 when the destination was prewarmed
      if (rec.switched && out.switch_tokens > 0)
        rec.switch_cost_sec = out.switch_ms * 1e-3 * sw_tok[k] / static_cast<double>(out.switch_tokens);
      r.active_ssm = j;
      rec.proposed = W;
      rec.accepted = acc[k];
      rec.bonus = 1;
      // slot_engine.cpp:145: the request's own SSM's speculation time + the verify time
      rec.wall_time_sec = (out.spec_end_ms[j] + out.verify_ms) * 1e-3;
      stats.outcomes.push_back({id, j, W, acc[k], 1, rec.wall_time_sec});
      const long long emitted = acc[k] + 1;
      r.generated_len = std::min(r.target_len, r.generated_len + emitted);
      if (r.generated_len >= r.target_len) r.state = RequestState::Finished;
      total_accepted += static_cast<double>(emitted);
      last_ssm_[id] = j;
      ++k;
    }
    if (history != nullptr) history->push_back(rec);
  }
  total_time_sec += stats.duration_sec;
  total_padding += stats.padding_tokens;
  total_verify_sec += stats.verify_sec;
  ++next_slot_;
  return stats;
}

// slot_engine.cpp:169-193, plus KV slot recycling and prefill of newcomers.
std::vector<std::pair<int, int>> SlotEngine::refill_admitted() {
  std::vector<std::pair<int, int>> transfers;
  std::vector<int> kept, fresh;
  for (int id : admitted_) {
    if (requests_[id].state != RequestState::Finished) {
      kept.push_back(id);
      continue;
    }
    free_slots_.push_back(kv_slot_[id]);
    int replacement = -1;
    while (next_waiting_ < static_cast<int>(requests_.size())) {
      Request& cand = requests_[next_waiting_++];
      if (cand.state == RequestState::Waiting) {
        cand.state = RequestState::Active;
        replacement = cand.id;
        break;
      }
    }
    transfers.emplace_back(id, replacement);
    if (replacement >= 0) {
      kept.push_back(replacement);
      fresh.push_back(replacement);
    }
  }
  std::sort(kept.begin(), kept.end());
  admitted_ = std::move(kept);
  admit_to_device(fresh);
  return transfers;
}

}  // namespace specsim

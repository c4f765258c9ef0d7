// Tests of the C++ drop-in API (include/specsim) in the style of the
// reference's own suites (tests/test_packing.cpp, test_attention.cpp,
// test_model.cpp, slot engine behaviour). Usage: test_specsim_api host|gpu
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <functional>
#include <string>

#include "specsim/attention.hpp"
#include "specsim/errors.hpp"
#include "specsim/model.hpp"
#include "specsim/packing.hpp"
#include "specsim/slot_engine.hpp"

using namespace specsim;

static int g_fail = 0, g_checks = 0;
#define CHECK(cond)                                                     \
  do {                                                                  \
    ++g_checks;                                                         \
    if (!(cond)) {                                                      \
      ++g_fail;                                                         \
      std::fprintf(stderr, "FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond); \
    }                                                                   \
  } while (0)
template <typename E, typename F>
static bool throws(F&& f) {
  try {
    f();
  } catch (const E&) {
    return true;
  } catch (...) {
    return false;
  }
  return false;
}

static void host_tests() {
  // test_packing.cpp:38-87 known answers
  {
    const PackedLayout l = pack({4, 4, 4}, 3);
    CHECK(l.length == 4 && l.width == 3 && l.padding_tokens == 0 && l.segments.size() == 3);
    const PackedLayout m = pack({8, 5, 3}, 2);
    CHECK(m.length == 8 && m.padding_tokens == 0);
    const IndicatorMask mask = build_indicator(m);
    for (int c = 0; c < 8; ++c) CHECK(mask.at(0, c) == 0);
    for (int c = 0; c < 5; ++c) CHECK(mask.at(1, c) == 1);
    for (int c = 5; c < 8; ++c) CHECK(mask.at(1, c) == 2);
    const PackedLayout w = pack({10, 2}, 2);
    CHECK(w.length == 6 && w.padding_tokens == 0 && w.q_replica_rows[0] == 2 && w.q_replica_rows[1] == 1);
    CHECK(naive_padding({7, 5, 5}) == 4 && naive_padding({8, 5, 3}) == 8);
    CHECK(pack({7, 5, 5}, 3).padding_tokens < 4);
    CHECK(throws<ConfigError>([] { pack({1, 2}, 0); }));
    CHECK(throws<ConfigError>([] { pack({0}, 2); }));
    CHECK(throws<InputError>([] { naive_padding({}); }));
    CHECK(pack({}, 3).segments.empty());
    PackedLayout corrupt = pack({5}, 1);
    corrupt.segments.push_back({1, 0, 2, 4, 0});
    CHECK(throws<ConsistencyError>([&] { build_indicator(corrupt); }));
  }
  // token conservation (test_packing.cpp:128-142)
  {
    Rng rng(313);
    for (int trial = 0; trial < 300; ++trial) {
      const int n = static_cast<int>(rng.uniform_int(1, 10));
      std::vector<int> lens(n);
      long long total = 0;
      for (int& len : lens) total += (len = static_cast<int>(rng.uniform_int(1, 30)));
      const PackedLayout l = pack(lens, static_cast<int>(rng.uniform_int(1, 6)));
      long long covered = 0;
      for (const Segment& s : l.segments) covered += s.length();
      CHECK(covered == total && l.total_cells() == total + l.padding_tokens);
    }
  }
  // verify_batch_cost (slot_engine.cpp:24-45)
  {
    const VerifyBatchCost p = verify_batch_cost({8, 5, 3}, 4, true, 2);
    CHECK(p.tokens == 16 + 4 * 3 && p.padding == 0);  // 2 x 8 cells + q rows: req0 1 row, req1 1, req2 1
    const VerifyBatchCost d = verify_batch_cost({8, 5, 3}, 4, false, 0);
    CHECK(d.tokens == 16 + 8 + 12 && d.padding == 8);
  }
  // model.cpp semantics (test_model.cpp:112-189)
  {
    CHECK(std::abs(expected_accepted_prefix(0.8, 4) - 2.3616) < 1e-12);
    Request r;
    r.accept_prob = {1.0, 0.0};
    Rng rng(5);
    CHECK(sample_accepted_prefix(r, 0, 4, rng) == 4 && sample_accepted_prefix(r, 1, 4, rng) == 0);
    CHECK(throws<InputError>([&] { sample_accepted_prefix(r, 2, 4, rng); }));
    const SsmProfile s{0, 100.0, 4, 0.1};
    CHECK(std::abs(speculation_time(s, 1, 5) - 0.05) < 1e-15);
    CHECK(std::abs(speculation_time(s, 2, 5) - 0.055) < 1e-15);
    CHECK(throws<CapacityError>([&] { speculation_time(s, 5, 5); }));
    CHECK(std::abs(verification_time({0.01, 0.0}, 1000) - 0.01) < 1e-15);
    CHECK(std::abs(observed_goodput({0, 0, 4, 4, 1, 0.1}) - 50.0) < 1e-12);
  }
}

static WorkloadSpec small_spec() {
  WorkloadSpec spec;
  spec.num_requests = 10;
  spec.window = 4;
  spec.seed = 77;
  for (int j = 0; j < 2; ++j) spec.ssm_profiles.push_back({j, 100.0 + 50 * j, 3, 0.0});
  DifficultyClass c;
  c.name = "all";
  c.accept_range = {{0.5, 0.5}, {0.7, 0.7}};
  c.prompt_len_lo = 8;
  c.prompt_len_hi = 40;
  c.target_len_lo = 10;
  c.target_len_hi = 30;
  spec.difficulty_mix = {c};
  return spec;
}

static void gpu_tests() {
  // decomposed == reference attention (test_attention.cpp:94-161)
  {
    Rng rng(424242);
    double worst = 0.0;
    for (int trial = 0; trial < 50; ++trial) {
      const int n = static_cast<int>(rng.uniform_int(1, 6));
      std::vector<ToyAttentionInput> inputs;
      std::vector<int> lens;
      for (int i = 0; i < n; ++i) {
        inputs.push_back(make_toy_input(rng.next(), static_cast<int>(rng.uniform_int(1, 4)),
                                        static_cast<int>(rng.uniform_int(1, 12)), 4));
        lens.push_back(inputs.back().k.rows);
      }
      const PackedLayout layout = pack(lens, static_cast<int>(rng.uniform_int(1, n)));
      const auto outs = decomposed_attention(inputs, layout, build_indicator(layout));
      for (int i = 0; i < n; ++i) {
        const Matrix ref = reference_attention(inputs[i].q, inputs[i].k, inputs[i].v);
        for (std::size_t e = 0; e < ref.data.size(); ++e) worst = std::max(worst, std::abs(ref.data[e] - outs[i].data[e]));
      }
    }
    CHECK(worst <= 1e-9);
    std::vector<ToyAttentionInput> one{make_toy_input(51, 2, 5, 4)};
    const PackedLayout short_layout = pack({4}, 1);
    CHECK(throws<ConsistencyError>([&] { decomposed_attention(one, short_layout, build_indicator(short_layout)); }));
  }
  // SlotEngine: admission, capacity errors, outcomes, continuous batching
  {
    const WorkloadSpec spec = small_spec();
    SlotEngine engine(spec, generate_workload(spec), EngineOptions{true, 0, 0});
    CHECK(engine.admitted().size() == 6);  // total capacity 3 + 3
    std::vector<int> assign(spec.num_requests, -1), prewarm(spec.num_requests, -1);
    for (int id : engine.admitted()) assign[id] = id % 2;
    std::vector<int> over(spec.num_requests, 0);  // 6 on ssm 0 > capacity 3
    CHECK(throws<CapacityError>([&] { engine.run_slot(over, prewarm, false, nullptr); }));
    std::vector<int> bad(spec.num_requests, 5);
    CHECK(throws<InputError>([&] { engine.run_slot(bad, prewarm, false, nullptr); }));
    std::vector<SlotRecord> history;
    long long slots = 0;
    while (!engine.all_finished() && slots < 60) {
      std::fill(assign.begin(), assign.end(), -1);
      int k = 0;
      for (int id : engine.admitted()) assign[id] = (k++ + static_cast<int>(slots)) % 2;  // switches every slot
      const SlotStats st = engine.run_slot(assign, prewarm, false, &history);
      CHECK(st.served == static_cast<int>(engine.admitted().size()));
      CHECK(st.duration_sec > 0.0 && st.verify_sec > 0.0 && st.spec_max_sec > 0.0);
      for (const SpeculationOutcome& o : st.outcomes) {
        CHECK(o.accepted >= 0 && o.accepted <= spec.window && o.bonus == 1);
        CHECK(observed_goodput(o) > 0.0);
      }
      for (int id : engine.admitted()) {
        const std::vector<int> t = engine.tokens(id);
        const Request& r = engine.requests()[id];
        CHECK(static_cast<long long>(t.size()) >= r.prompt_len + r.generated_len);
      }
      engine.refill_admitted();
      ++slots;
    }
    CHECK(engine.all_finished());
    CHECK(engine.total_accepted > 0.0 && engine.total_time_sec > 0.0);
    bool any_switch = false;
    for (const SlotRecord& r : history) any_switch = any_switch || r.switched;
    CHECK(any_switch);
  }
}

int main(int argc, char** argv) {
  const std::string mode = argc > 1 ? argv[1] : "host";
  try {
    host_tests();
    if (mode == "gpu") gpu_tests();
  } catch (const std::exception& e) {
    std::fprintf(stderr, "uncaught: %s\n", e.what());
    return 2;
  }
  std::printf("%d checks, %d failures\n", g_checks, g_fail);
  return g_fail == 0 ? 0 : 1;
}

// Drop-in demonstration (test infrastructure, built into oracle/_ref/): the
// reference's UNMODIFIED selector sources (bandit.cpp / matching.cpp /
// policies.cpp, compiled from /root/reference by oracle/Makefile target
// `dropin`) run against the B200 SlotEngine of include/specsim. This driver is
// ours; it builds a small spec, runs LBSS and the greedy baseline, and prints a
// JSON summary.
#include <cstdio>
#include <string>

#include "specsim/bandit.hpp"
#include "specsim/policies.hpp"

using namespace specsim;

int main(int argc, char** argv) {
  const long long slots = argc > 1 ? std::stoll(argv[1]) : 24;
  WorkloadSpec spec;
  spec.num_requests = 16;
  spec.window = 4;
  spec.seed = 2503;
  spec.llm = {0.01, 1e-5};
  for (int j = 0; j < 2; ++j) spec.ssm_profiles.push_back({j, 200.0 + 100.0 * j, 4, 0.05});
  DifficultyClass c;
  c.name = "mix";
  c.weight = 1.0;
  c.accept_range = {{0.5, 0.8}, {0.6, 0.9}};
  c.prompt_len_lo = 16;
  c.prompt_len_hi = 64;
  c.target_len_lo = 24;
  c.target_len_hi = 48;
  spec.difficulty_mix = {c};
  try {
    BanditConfig cfg;
    cfg.alpha = 4;
    cfg.beta = 2;
    cfg.max_slots = slots;
    const PolicyRunResult run = run_lbss(cfg, spec);
    const PolicyRunResult greedy = run_greedy(spec, slots);
    std::printf("{\"lbss_tokens\": %.0f, \"lbss_time_s\": %.6f, \"lbss_slots\": %zu, \"greedy_tokens\": %.0f, "
                "\"greedy_time_s\": %.6f}\n",
                run.accepted_tokens, run.total_time_sec, run.history.size(), greedy.accepted_tokens,
                greedy.total_time_sec);
  } catch (const std::exception& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return 1;
  }
  return 0;
}

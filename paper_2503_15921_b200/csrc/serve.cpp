// The multi-GPU serving loop, native end to end:
// one process per GPU, requests sharded in contiguous blocks, replicated weights,
// the replicated LBSS selector (lbss.cpp, same seed on every rank) and one
// collective -- the all-gather of per-(request, SSM) ArmEstimate{sum, count} rows
// (comm.cpp) after every slot, so every rank derives the same assignment.
//
// Per slot (run_lbss, bandit.cpp:248-332, with SlotEngine::run_slot replaced by a
// real spin round on this rank's shard):
//   1. the selector's global assignment for the slot, and the next slot's
//      assignment where it is already determined (spin_lbss_peek) as prewarm;
//   2. spin_round_prewarm on the local shard: switch catch-up (charged), SSM drafts,
//      packed verification, accept -- the prewarm destinations recomputed on idle
//      streams meanwhile;
//   3. observed_goodput = (accepted + bonus) / (own SSM's draft end + verify)
//      (model.cpp:165-171, slot_engine.cpp:145) added to the local rows;
//   4. spin_stats_allgather; the gathered rows replace the selector's estimates.
#include <chrono>
#include <cstring>
#include <vector>

#include "spin_c.h"
#include "status.hpp"

namespace spin {
namespace {
void ok(spin_status s) {
  if (s != SPIN_OK) fail(s, spin_last_error());
}
}  // namespace
}  // namespace spin

using namespace spin;

extern "C" {

spin_status spin_lbss_serve(spin_ctx* ctx, spin_comm* comm, spin_lbss* sel, int32_t n_total, int32_t n_ssm,
                            const int32_t* local_slots, int32_t n_local, int32_t slots_to_run, int32_t use_prewarm,
                            spin_serve_report* rep, int32_t* final_assignment) {
  return guarded([&] {
    if (!ctx || !sel || !rep || (n_local > 0 && !local_slots) || slots_to_run < 1 || n_ssm < 1 || n_ssm > SPIN_MAX_SSM)
      fail(SPIN_INPUT_ERROR, "spin_lbss_serve: bad arguments");
    int32_t rank = 0, world = 1;
    if (comm) ok(spin_comm_info(comm, &rank, &world, nullptr));
    // contiguous shards, sizes differing by <= 1 (dist.shard)
    const int base = n_total / world, extra = n_total % world;
    auto first_of = [&](int r) { return r * base + std::min(r, extra); };
    auto size_of = [&](int r) { return base + (r < extra ? 1 : 0); };
    if (size_of(rank) != n_local) fail(SPIN_CONFIG_ERROR, "spin_lbss_serve: n_local is not this rank's shard");
    const int first = first_of(rank);
    const int rows = size_of(0);  // padded gather rows
    std::vector<int32_t> a(n_total), pw(n_total), nxt(n_total), a_loc(n_local), pw_loc(n_local);
    std::vector<int32_t> acc(n_local), bonus(n_local), comm_len(n_local), sw(n_local);
    std::vector<double> local_rows(static_cast<size_t>(rows) * n_ssm * 2, 0.0);
    std::vector<double> gathered(static_cast<size_t>(rows) * world * n_ssm * 2), est(static_cast<size_t>(n_total) * n_ssm * 2);
    *rep = spin_serve_report{};
    const auto t0 = std::chrono::steady_clock::now();
    for (int t = 0; t < slots_to_run; ++t) {
      int32_t explore = 0, epoch = 0;
      ok(spin_lbss_next(sel, a.data(), pw.data(), &explore, &epoch));
      if (use_prewarm) ok(spin_lbss_peek(sel, nxt.data()));
      for (int i = 0; i < n_local; ++i) {
        a_loc[i] = a[first + i];
        // warm only destinations the request is about to move to
        pw_loc[i] = use_prewarm && nxt[first + i] != a_loc[i] ? nxt[first + i] : -1;
      }
      spin_round_out out{};
      out.accepted = acc.data();
      out.bonus_token = bonus.data();
      out.committed = comm_len.data();
      out.switch_tokens_per_request = sw.data();
      ok(spin_round_prewarm(ctx, n_local, local_slots, a_loc.data(), pw_loc.data(), &out));
      for (int i = 0; i < n_local; ++i) {
        const int j = a_loc[i];
        if (j < 0) continue;
        const double wall_s = (out.spec_end_ms[j] + out.verify_ms) * 1e-3;
        double* r = local_rows.data() + (static_cast<size_t>(i) * n_ssm + j) * 2;
        r[0] += (acc[i] + 1) / wall_s;
        r[1] += 1.0;
        rep->tokens += acc[i] + 1;
        ++rep->served;
      }
      if (comm && world > 1) {
        ok(spin_stats_allgather(comm, local_rows.data(), gathered.data(), rows, n_ssm));
        for (int r = 0, o = 0; r < world; ++r)
          for (int i = 0; i < size_of(r); ++i, ++o)
            std::memcpy(est.data() + static_cast<size_t>(o) * n_ssm * 2,
                        gathered.data() + (static_cast<size_t>(r) * rows + i) * n_ssm * 2, sizeof(double) * n_ssm * 2);
        ok(spin_lbss_rows(sel, est.data(), 1));
      } else {
        ok(spin_lbss_rows(sel, local_rows.data(), 1));
      }
      rep->device_ms += out.round_ms;
      rep->switch_ms += out.switch_ms;
      rep->switch_tokens += out.switch_tokens;
      rep->explore_slots += explore;
      rep->epochs = epoch;
    }
    rep->wall_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    // the exploitation plan on the final estimates (plan_exploitation, bandit.cpp:186-226)
    if (final_assignment) ok(spin_lbss_plan(sel, final_assignment));
  });
}

}  // extern "C"

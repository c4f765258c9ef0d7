// Learning-based SSM selection (LBSS) on measured goodput: the host selector of
// Spin, restated in C++ from the reference's bandit (proj/core/src/bandit.cpp,
// include/specsim/bandit.hpp, src/matching.cpp) so that the multi-GPU driver
// (spin_lbss_serve) is native end to end. Same draw order as the reference
// (Rng(mix_seed(seed, kStreamPolicy)) = mt19937_64, rejection-sampled
// uniform_int), same schedule, same tie-breaking: given the same observations it
// produces the reference's assignments slot for slot (tests/test_lbss.py pins it
// to goldens generated with the reference's own functions).
//
//   epoch k: alpha exploration slots in chunks of beta, each chunk one
//            draw_exploration_assignment (bandit.cpp:108-120) resolved against the
//            SSM capacities (resolve_capacity_overflow, :61-106), prewarm = the draw;
//            then 2^k exploitation slots (exploitation_duration, :54-59) on
//            plan_exploitation (:186-226), prewarm = prewarm_destination (:122-139)
//            decided before the matching.
//   observations: ArmEstimate::add(observed_goodput) per served request (:166-169).
#include <algorithm>
#include <cmath>
#include <cstring>
#include <limits>
#include <memory>
#include <random>
#include <vector>

#include "spin_c.h"
#include "status.hpp"

namespace spin {
namespace {

constexpr double kInf = std::numeric_limits<double>::infinity();

uint64_t splitmix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}
uint64_t mix_seed(uint64_t seed, uint64_t a, uint64_t b = 0, uint64_t c = 0) {
  uint64_t h = splitmix64(seed);
  h = splitmix64(h ^ a);
  h = splitmix64(h ^ b);
  return splitmix64(h ^ c);
}
constexpr uint64_t kStreamPolicy = 0x02;  // rng.hpp stream tags

// rng.hpp Rng::uniform_int: exactly uniform in [lo, hi] by rejection.
long long uniform_int(std::mt19937_64& e, long long lo, long long hi) {
  if (hi <= lo) return lo;
  const uint64_t range = static_cast<uint64_t>(hi - lo) + 1;
  const uint64_t limit = UINT64_MAX - UINT64_MAX % range;
  uint64_t draw;
  do {
    draw = e();
  } while (draw >= limit);
  return lo + static_cast<long long>(draw % range);
}

// O(n^3) Hungarian with potentials, minimising a square cost matrix (matching.cpp:40-89).
std::vector<int> hungarian_min(const std::vector<double>& a, int n) {
  std::vector<double> u(n + 1, 0.0), v(n + 1, 0.0);
  std::vector<int> p(n + 1, 0), way(n + 1, 0);
  for (int i = 1; i <= n; ++i) {
    p[0] = i;
    int j0 = 0;
    std::vector<double> minv(n + 1, kInf);
    std::vector<char> used(n + 1, 0);
    do {
      used[j0] = 1;
      const int i0 = p[j0];
      double delta = kInf;
      int j1 = -1;
      for (int j = 1; j <= n; ++j) {
        if (used[j]) continue;
        const double cur = a[static_cast<size_t>(i0 - 1) * n + (j - 1)] - u[i0] - v[j];
        if (cur < minv[j]) {
          minv[j] = cur;
          way[j] = j0;
        }
        if (minv[j] < delta) {
          delta = minv[j];
          j1 = j;
        }
      }
      for (int j = 0; j <= n; ++j) {
        if (used[j]) {
          u[p[j]] += delta;
          v[j] -= delta;
        } else {
          minv[j] -= delta;
        }
      }
      j0 = j1;
    } while (p[j0] != 0);
    do {
      const int j1 = way[j0];
      p[j0] = p[j1];
      j0 = j1;
    } while (j0);
  }
  std::vector<int> row_to_col(n, -1);
  for (int j = 1; j <= n; ++j)
    if (p[j] >= 1) row_to_col[p[j] - 1] = j - 1;
  return row_to_col;
}

// Best total weight of rows [from, n) under capacities caps (replica expansion padded
// to a square with zero-weight dummies, maximised as a negated min-cost problem;
// matching.cpp:93-140).
double km_best_total(const std::vector<double>& w, int n, int m, int from, const std::vector<int>& caps) {
  const int rows = n - from;
  int cols = 0;
  for (int c : caps) cols += c;
  if (rows <= 0 || cols == 0) return 0.0;
  std::vector<int> col_ssm;
  for (int j = 0; j < m; ++j)
    for (int r = 0; r < caps[j]; ++r) col_ssm.push_back(j);
  const int size = std::max(rows, cols);
  std::vector<double> cost(static_cast<size_t>(size) * size, 0.0);
  for (int i = 0; i < rows; ++i)
    for (int c = 0; c < cols; ++c) cost[static_cast<size_t>(i) * size + c] = -w[static_cast<size_t>(from + i) * m + col_ssm[c]];
  const std::vector<int> rc = hungarian_min(cost, size);
  double total = 0.0;
  for (int i = 0; i < rows; ++i)
    if (rc[i] >= 0 && rc[i] < cols) total += -cost[static_cast<size_t>(i) * size + rc[i]];
  return total;
}

}  // namespace

struct Lbss {
  int n = 0, m = 0, alpha = 8, beta = 2;
  std::vector<int> cap;
  std::mt19937_64 rng;
  std::vector<double> sum;      // [n][m] ArmEstimate::sum
  std::vector<long long> cnt;   // [n][m] ArmEstimate::count
  int epoch = 1;
  bool exploring = true;
  int chunk = 0, in_chunk = 0;
  long long exploit_left = 0;
  std::vector<int> assign, prewarm;
  bool predrawn = false;
  std::vector<int> next_draw;

  bool observed(int i, int j) const { return cnt[static_cast<size_t>(i) * m + j] > 0; }
  double mean(int i, int j) const {
    return sum[static_cast<size_t>(i) * m + j] / static_cast<double>(cnt[static_cast<size_t>(i) * m + j]);
  }
  double optimistic_mean(int i, int j) const { return observed(i, j) ? mean(i, j) : kInf; }

  // resolve_capacity_overflow (bandit.cpp:61-106); every request is admitted.
  std::vector<int> resolve(std::vector<int> res) {
    std::vector<std::vector<int>> claimants(m);
    for (int id = 0; id < n; ++id)
      if (res[id] >= 0) claimants[res[id]].push_back(id);
    std::vector<int> load(m, 0), overflow;
    for (int j = 0; j < m; ++j) {
      if (static_cast<int>(claimants[j].size()) <= cap[j]) {
        load[j] = static_cast<int>(claimants[j].size());
        continue;
      }
      std::vector<int>& mem = claimants[j];
      for (int i = static_cast<int>(mem.size()) - 1; i > 0; --i) {
        const int k = static_cast<int>(uniform_int(rng, 0, i));
        std::swap(mem[i], mem[k]);
      }
      load[j] = cap[j];
      for (size_t i = cap[j]; i < mem.size(); ++i) overflow.push_back(mem[i]);
    }
    std::sort(overflow.begin(), overflow.end());
    for (int id : overflow) {
      std::vector<int> open;
      for (int j = 0; j < m; ++j)
        if (load[j] < cap[j]) open.push_back(j);
      if (open.empty()) {
        res[id] = -1;
        continue;
      }
      const int j = open[uniform_int(rng, 0, static_cast<int>(open.size()) - 1)];
      res[id] = j;
      ++load[j];
    }
    return res;
  }

  // draw_exploration_assignment (bandit.cpp:108-120)
  std::vector<int> draw() {
    std::vector<int> desired(n, -1);
    for (int id = 0; id < n; ++id) desired[id] = static_cast<int>(uniform_int(rng, 0, m - 1));
    return resolve(desired);
  }

  // prewarm_destination (bandit.cpp:122-139): optimistic argmax, ties to the lowest id
  std::vector<int> prewarm_destination() const {
    std::vector<int> pw(n, -1);
    for (int id = 0; id < n; ++id) {
      int best = 0;
      double bm = optimistic_mean(id, 0);
      for (int j = 1; j < m; ++j) {
        const double v = optimistic_mean(id, j);
        if (v > bm) bm = v, best = j;
      }
      pw[id] = best;
    }
    return pw;
  }

  // plan_exploitation (bandit.cpp:186-226) + solve_max_weight_matching (matching.cpp:161-196)
  std::vector<int> plan() const {
    double max_finite = 0.0;
    bool any = false;
    for (int id = 0; id < n; ++id)
      for (int j = 0; j < m; ++j)
        if (observed(id, j)) {
          max_finite = any ? std::max(max_finite, mean(id, j)) : mean(id, j);
          any = true;
        }
    const double cold = any ? max_finite + 1.0 : 1.0;
    std::vector<double> w(static_cast<size_t>(n) * m);
    for (int id = 0; id < n; ++id)
      for (int j = 0; j < m; ++j) w[static_cast<size_t>(id) * m + j] = observed(id, j) ? mean(id, j) : cold;
    std::vector<int> out(n, -1);
    bool binding = false;
    for (int j = 0; j < m; ++j) binding |= cap[j] < n;
    if (!binding) {
      // Capacities never bind, so every optimal completion of rows i+1.. is their
      // row maxima, summed in row order as km_best_total does: the canonicalisation
      // below then reduces to a per-request choice with the same float expressions
      // (and the same 1e-9 tolerance budget) as the general case.
      std::vector<double> rowmax(n);
      for (int id = 0; id < n; ++id) {
        double b = w[static_cast<size_t>(id) * m];
        for (int j = 1; j < m; ++j) b = std::max(b, w[static_cast<size_t>(id) * m + j]);
        rowmax[id] = b;
      }
      double best = 0.0;
      for (int id = 0; id < n; ++id) best += rowmax[id];
      const double tol = 1e-9 * std::max(1.0, std::abs(best));
      double fixed = 0.0;
      for (int i = 0; i < n; ++i) {
        double rest = 0.0;
        for (int k = i + 1; k < n; ++k) rest += rowmax[k];
        for (int j = 0; j < m; ++j) {
          const double wij = w[static_cast<size_t>(i) * m + j];
          if (fixed + wij + rest >= best - tol) {
            out[i] = j;
            fixed += wij;
            break;
          }
        }
      }
      return out;
    }
    if (n > 128) fail(SPIN_SIZE_ERROR, "lbss: binding capacities with more than 128 requests");
    // Lexicographic canonicalisation (matching.cpp:172-194): commit requests in id
    // order to the lowest SSM that still admits an optimal completion.
    std::vector<int> caps = cap;
    const double best = km_best_total(w, n, m, 0, caps);
    const double tol = 1e-9 * std::max(1.0, std::abs(best));
    double fixed = 0.0;
    for (int i = 0; i < n; ++i) {
      for (int j = 0; j < m; ++j) {
        if (caps[j] == 0) continue;
        const double wij = w[static_cast<size_t>(i) * m + j];
        --caps[j];
        const double rest = km_best_total(w, n, m, i + 1, caps);
        if (fixed + wij + rest >= best - tol) {
          out[i] = j;
          fixed += wij;
          break;
        }
        ++caps[j];
      }
    }
    return out;
  }

  // The assignment of the NEXT slot where it is already determined, for prewarm
  // planning: inside a chunk or an exploitation stage it is the current one; at an
  // exploration chunk boundary the next chunk is drawn now (the same draws in the
  // same order as when next() reaches it: observations never touch the Rng); before
  // the first exploitation slot it is the reference's own prewarm choice,
  // prewarm_destination on the current estimates (bandit.cpp:296-299).
  void peek(int32_t* out) {
    if (exploring) {
      if (in_chunk == 0) {
        if (!predrawn) {
          next_draw = draw();
          predrawn = true;
        }
        std::copy(next_draw.begin(), next_draw.end(), out);
      } else {
        std::copy(assign.begin(), assign.end(), out);
      }
      return;
    }
    const std::vector<int> v = exploit_left == 0 ? prewarm_destination() : assign;
    std::copy(v.begin(), v.end(), out);
  }

  void next(int32_t* a, int32_t* pw, int32_t* explore, int32_t* ep) {
    if (ep) *ep = epoch;
    if (exploring) {
      if (in_chunk == 0) {
        assign = predrawn ? next_draw : draw();
        predrawn = false;
        prewarm = assign;  // drawn one chunk ahead: destinations are prewarmed (bandit.cpp:157-160)
      }
      if (explore) *explore = 1;
      std::copy(assign.begin(), assign.end(), a);
      if (pw) std::copy(prewarm.begin(), prewarm.end(), pw);
      if (++in_chunk == beta) {
        in_chunk = 0;
        if (++chunk == alpha / beta) {
          chunk = 0;
          exploring = false;
          exploit_left = 0;
        }
      }
      return;
    }
    if (exploit_left == 0) {
      prewarm = prewarm_destination();  // before the matching (bandit.cpp:296-299)
      assign = plan();
      exploit_left = epoch >= 62 ? std::numeric_limits<long long>::max() : (1LL << epoch);
    }
    if (explore) *explore = 0;
    std::copy(assign.begin(), assign.end(), a);
    if (pw) std::copy(prewarm.begin(), prewarm.end(), pw);
    if (--exploit_left == 0) {
      ++epoch;
      exploring = true;
    }
  }
};

}  // namespace spin

using namespace spin;

struct spin_lbss {
  Lbss s;
};

extern "C" {

spin_status spin_lbss_create(int32_t n_requests, int32_t n_ssm, const int32_t* capacities, int32_t alpha,
                             int32_t beta, uint64_t seed, spin_lbss** out) {
  return guarded([&] {
    if (!out || !capacities) fail(SPIN_INPUT_ERROR, "spin_lbss_create: null argument");
    // validate(BanditConfig) (bandit.cpp:11-23)
    if (alpha < 1) fail(SPIN_CONFIG_ERROR, "bandit: alpha must be at least 1");
    if (beta < 1) fail(SPIN_CONFIG_ERROR, "bandit: beta must be at least 1");
    if (alpha % beta != 0) fail(SPIN_CONFIG_ERROR, "bandit: beta must divide alpha");
    if (n_requests < 1 || n_ssm < 1) fail(SPIN_CONFIG_ERROR, "lbss: need requests and ssms");
    int total = 0;
    for (int j = 0; j < n_ssm; ++j) {
      if (capacities[j] < 1) fail(SPIN_INPUT_ERROR, "matching: capacities must be at least 1");
      total += capacities[j];
    }
    auto p = std::make_unique<spin_lbss>();
    Lbss& s = p->s;
    s.n = n_requests, s.m = n_ssm, s.alpha = alpha, s.beta = beta;
    s.cap.assign(capacities, capacities + n_ssm);
    s.rng.seed(mix_seed(seed, kStreamPolicy));
    s.sum.assign(static_cast<size_t>(n_requests) * n_ssm, 0.0);
    s.cnt.assign(static_cast<size_t>(n_requests) * n_ssm, 0);
    (void)total;
    *out = p.release();
  });
}

spin_status spin_lbss_destroy(spin_lbss* sel) {
  return guarded([&] { delete sel; });
}

spin_status spin_lbss_next(spin_lbss* sel, int32_t* assignment, int32_t* prewarm, int32_t* explore, int32_t* epoch) {
  return guarded([&] {
    if (!sel || !assignment) fail(SPIN_INPUT_ERROR, "spin_lbss_next: null argument");
    sel->s.next(assignment, prewarm, explore, epoch);
  });
}

spin_status spin_lbss_observe(spin_lbss* sel, int32_t request, int32_t ssm, double goodput) {
  return guarded([&] {
    if (!sel) fail(SPIN_INPUT_ERROR, "spin_lbss_observe: null selector");
    Lbss& s = sel->s;
    if (request < 0 || request >= s.n || ssm < 0 || ssm >= s.m) fail(SPIN_INPUT_ERROR, "lbss: arm out of range");
    s.sum[static_cast<size_t>(request) * s.m + ssm] += goodput;
    ++s.cnt[static_cast<size_t>(request) * s.m + ssm];
  });
}

spin_status spin_lbss_peek(spin_lbss* sel, int32_t* assignment) {
  return guarded([&] {
    if (!sel || !assignment) fail(SPIN_INPUT_ERROR, "spin_lbss_peek: null argument");
    sel->s.peek(assignment);
  });
}

spin_status spin_lbss_plan(spin_lbss* sel, int32_t* assignment) {
  return guarded([&] {
    if (!sel || !assignment) fail(SPIN_INPUT_ERROR, "spin_lbss_plan: null argument");
    const std::vector<int> p = sel->s.plan();
    std::copy(p.begin(), p.end(), assignment);
  });
}

spin_status spin_lbss_rows(spin_lbss* sel, double* rows, int32_t set) {
  return guarded([&] {
    if (!sel || !rows) fail(SPIN_INPUT_ERROR, "spin_lbss_rows: null argument");
    Lbss& s = sel->s;
    const size_t nm = static_cast<size_t>(s.n) * s.m;
    for (size_t k = 0; k < nm; ++k) {
      if (set) {
        s.sum[k] = rows[2 * k];
        s.cnt[k] = static_cast<long long>(std::llround(rows[2 * k + 1]));
      } else {
        rows[2 * k] = s.sum[k];
        rows[2 * k + 1] = static_cast<double>(s.cnt[k]);
      }
    }
  });
}

}  // extern "C"

#include "pack.hpp"

#include <algorithm>
#include <numeric>

#include "status.hpp"

namespace spin {

namespace {

// One first-fit-decreasing attempt at a fixed tensor length (packing.cpp:16-70):
// requests in decreasing-length order (ties keep index order) go whole into the
// first row with room; a request no row can hold is spread over the rows'
// remaining space in row order, keeping its tokens in order.
bool place_at_length(const int32_t* len, int32_t n, int32_t rows, int32_t L, const std::vector<int32_t>& order,
                     PackResult* out) {
  std::vector<int32_t> used(rows, 0);
  std::vector<spin_segment> segs;
  segs.reserve(n + rows);
  for (int32_t id : order) {
    const int32_t need = len[id];
    int32_t home = -1;
    for (int32_t r = 0; r < rows && home < 0; ++r)
      if (L - used[r] >= need) home = r;
    if (home >= 0) {
      segs.push_back({id, home, used[home], used[home] + need, 0});
      used[home] += need;
      continue;
    }
    int32_t done = 0;
    for (int32_t r = 0; r < rows && done < need; ++r) {
      const int32_t room = L - used[r];
      if (room <= 0) continue;
      const int32_t take = std::min(room, need - done);
      segs.push_back({id, r, used[r], used[r] + take, done});
      used[r] += take;
      done += take;
    }
    if (done < need) return false;
  }
  int64_t filled = 0;
  for (int32_t u : used) filled += u;
  out->length = L;
  out->rows = rows;
  out->padding = static_cast<int64_t>(rows) * L - filled;
  out->segments = std::move(segs);
  out->q_replica_rows.assign(n, 0);
  // Distinct rows per request: segments of one request are emitted with
  // strictly increasing row, so counting row changes is enough.
  std::vector<int32_t> last_row(n, -1);
  for (const spin_segment& s : out->segments) {
    if (last_row[s.request_id] != s.row) {
      last_row[s.request_id] = s.row;
      ++out->q_replica_rows[s.request_id];
    }
  }
  return true;
}

}  // namespace

void pack_validate(const int32_t* kv_lens, int32_t n, int32_t width) {
  if (width < 1) fail(SPIN_CONFIG_ERROR, "pack: width must be at least 1");
  for (int32_t i = 0; i < n; ++i)
    if (kv_lens[i] < 1) fail(SPIN_CONFIG_ERROR, "pack: kv lengths must be at least 1");
}

PackResult pack_lengths(const int32_t* kv_lens, int32_t n, int32_t width) {
  pack_validate(kv_lens, n, width);
  PackResult res;
  if (n <= 0) return res;
  const int32_t rows = std::min(width, n);
  int64_t total = 0;
  int32_t longest = 0;
  for (int32_t i = 0; i < n; ++i) {
    total += kv_lens[i];
    longest = std::max(longest, kv_lens[i]);
  }
  std::vector<int32_t> order(n);
  std::iota(order.begin(), order.end(), 0);
  std::stable_sort(order.begin(), order.end(), [&](int32_t a, int32_t b) { return kv_lens[a] > kv_lens[b]; });
  // Padding is rows*L - total, increasing in L: the first feasible L wins
  // (packing.cpp:85-101).
  const int64_t lo = (total + rows - 1) / rows;
  const int64_t hi = std::max<int64_t>(lo, std::max<int64_t>(longest, total));
  for (int64_t L = lo; L <= hi; ++L) {
    if (L > INT32_MAX) break;
    if (place_at_length(kv_lens, n, rows, static_cast<int32_t>(L), order, &res)) return res;
  }
  fail(SPIN_CONSISTENCY_ERROR, "pack: no feasible layout found");
}

int64_t naive_padding_of(const int32_t* kv_lens, int32_t n) {
  if (n <= 0) fail(SPIN_INPUT_ERROR, "naive_padding: empty batch");
  const int32_t longest = *std::max_element(kv_lens, kv_lens + n);
  int64_t pad = 0;
  for (int32_t i = 0; i < n; ++i) pad += longest - kv_lens[i];
  return pad;
}

VerifyCost verify_cost(const int32_t* kv_lens, int32_t n, int32_t window, bool packing, int32_t pack_width) {
  VerifyCost c;
  if (n <= 0) return c;
  if (packing) {
    const PackResult p = pack_lengths(kv_lens, n, pack_width > 0 ? pack_width : n);
    c.padding = p.padding;
    c.tokens = static_cast<int64_t>(p.rows) * p.length;
    for (int32_t r : p.q_replica_rows) c.tokens += static_cast<int64_t>(r) * window;
  } else {
    c.padding = naive_padding_of(kv_lens, n);
    int64_t kv = 0;
    for (int32_t i = 0; i < n; ++i) kv += kv_lens[i];
    c.tokens = kv + c.padding + static_cast<int64_t>(n) * window;
  }
  return c;
}

}  // namespace spin

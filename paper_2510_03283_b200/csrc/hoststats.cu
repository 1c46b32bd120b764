// Host-side (CPU) head-stats / capacity allocation / prune bookkeeping of one tick's decode rows.
// Native restatement of paper_2510_03283_b200/hoststats.py (BatchedHeadStats.step + _allocate), which itself
// restates the reference's per-row Python: HeadStats.update (cache.py:291-309), allocate_capacity
// (cache.py:318-352) and prune_decision (cache.py:355-362) as called from Engine._exec_decode
// (engine.py:496-529). Same IEEE double operation order per element as the numpy version (sums left to
// right, no contraction: built with -ffp-contract=off), so kept[h] / released are bit-identical
// (tests/test_host_cpu.py compares against the numpy path and full runs against the reference).
#include <cmath>
#include <cstdint>
#include <vector>

#include "mace_b200.h"

namespace {

// caps for one row; returns false on the rounding-pathological leftover (>= H), decided by the caller
bool allocate_row(const double* means, int H, int64_t C, int64_t* caps) {
  double total = 0.0;
  for (int h = 0; h < H; ++h) total = total + means[h];
  if (!(total > 0.0)) {  // uniform split, remainder to the lowest heads (cache.py:330-333)
    const int64_t base = C / H;
    for (int h = 0; h < H; ++h) caps[h] = base + (h < C - base * H ? 1 : 0);
    return true;
  }
  double w[64];
  int64_t fl[64];
  int64_t left = C;
  for (int h = 0; h < H; ++h) {
    w[h] = means[h] / total;
    fl[h] = (int64_t)(w[h] * (double)C);  // int() truncation of a non-negative float
    caps[h] = fl[h];
    left -= fl[h];
  }
  if (left >= H) return false;
  // the `left` largest shares (ties: lower head index first) take one more slot (cache.py:340-343)
  for (int h = 0; h < H; ++h) {
    int rank = 0;
    for (int j = 0; j < H; ++j)
      if (-w[j] < -w[h] || (-w[j] == -w[h] && j < h)) ++rank;
    if (rank < left) caps[h] += 1;
  }
  // no head may end at zero slots: heads in index order, each takes one slot from the donor maximising
  // (caps - floors, caps, -index) among caps >= 2 (cache.py:345-351)
  for (int h = 0; h < H; ++h) {
    if (caps[h] != 0) continue;
    // lexicographic max over (eligible, caps - floors, caps, -j), fields compared directly (no digit packing,
    // so any c_total / H is exact); the first j wins ties on every field, as max() over the tuples does
    int donor = -1;
    for (int j = 0; j < H; ++j) {
      if (caps[j] < 2) continue;
      if (donor < 0) {
        donor = j;
        continue;
      }
      const int64_t dj = caps[j] - fl[j], dd = caps[donor] - fl[donor];
      if (dj > dd || (dj == dd && caps[j] > caps[donor])) donor = j;
    }
    if (donor < 0) donor = 0;  // no eligible donor: the reference's max() falls back the same way (all keys equal)
    caps[donor] -= 1;
    caps[h] += 1;
  }
  return true;
}

}  // namespace

extern "C" int mace_host_head_stats(int n, int H, int W, const int64_t* slots, const int64_t* steps,
                                    const double* norms, double* ring, int64_t* count, int64_t* pos, double* sums,
                                    double* current, double* last_used, double* tau, int64_t* kept, int c_total,
                                    double prune_window, int64_t* kept_out, int64_t* released_out) {
  if (n < 0 || H <= 0 || H > 64 || W <= 0) return MACE_ERR_ARG;
  std::vector<double> nsum((size_t)n * H), nlu((size_t)n * H), ntau(n);
  std::vector<int64_t> caps((size_t)n * H);
  std::vector<double> means(H);
  // pass 1: new statistics and caps (no state written, so a pathological row can defer to the caller)
  for (int r = 0; r < n; ++r) {
    const int64_t s = slots[r];
    const double* nr = norms + (size_t)r * H;
    double t = tau[s];
    if (std::isnan(t)) {  // first step: tau = 0.1 * mean(first norms) (cache.py:298-299)
      double tot = 0.0;
      for (int h = 0; h < H; ++h) tot = tot + nr[h];
      t = 0.1 * (tot / H);
    }
    ntau[r] = t;
    const int64_t cnt = count[s], p = pos[s];
    const bool full = cnt == W;
    const int64_t cnt2 = cnt + 1 < W ? cnt + 1 : W;
    for (int h = 0; h < H; ++h) {
      double sm = sums[(size_t)s * H + h];
      if (full) sm = sm - ring[((size_t)s * H + h) * W + p];
      sm = sm + nr[h];
      nsum[(size_t)r * H + h] = sm;
      nlu[(size_t)r * H + h] = nr[h] >= t ? (double)steps[r] : last_used[(size_t)s * H + h];
      means[h] = sm / (double)cnt2;
    }
    if (!allocate_row(means.data(), H, c_total, &caps[(size_t)r * H])) return 1;
  }
  // pass 2: commit the state, then kept += 1 and trim where kept > cap and prune_decision holds
  for (int r = 0; r < n; ++r) {
    const int64_t s = slots[r];
    const double* nr = norms + (size_t)r * H;
    const double t = ntau[r];
    tau[s] = t;
    const int64_t p = pos[s];
    int64_t rel = 0;
    for (int h = 0; h < H; ++h) {
      const size_t sh = (size_t)s * H + h;
      ring[sh * W + p] = nr[h];
      sums[sh] = nsum[(size_t)r * H + h];
      current[sh] = nr[h];
      const double lu = nlu[(size_t)r * H + h];
      last_used[sh] = lu;
      int64_t k = kept[sh] + 1;
      const int64_t cap = caps[(size_t)r * H + h];
      const bool prune = ((double)steps[r] - lu) > prune_window || nr[h] < t;
      if (k > cap && prune) {
        rel += k - cap;
        k = cap;
      }
      kept[sh] = k;
      kept_out[(size_t)r * H + h] = k;
    }
    released_out[r] = rel;
    count[s] = count[s] + 1 < W ? count[s] + 1 : W;
    pos[s] = (p + 1) % W;
  }
  return 0;
}

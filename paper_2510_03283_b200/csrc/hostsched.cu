// Host-side (CPU) Alg. 1 packing loop of one scheduling iteration: the reference's schedule_iteration
// (scheduler.py:133-188, Bin methods 81-117) over the queue's first n tasks in pop order, with their
// estimates precomputed by the caller. Same dequeue stop rule, same best-fit score
// lambda1*|free - mem| + lambda2*|maxlat - lat| with free = budget - used, same strict '<' tie rule, same
// reject / defer / requeue outcome; IEEE double in the reference's operation order (no contraction:
// -ffp-contract=off). Restates paper_2510_03283_b200/hostfast.py:fast_schedule_iteration, which stays the
// path for the rare iteration this routine hands back (return 2) and the oracle in tests/test_host_cpu.py.
#include <cmath>
#include <cstdint>
#include <vector>

#include "mace_b200.h"

extern "C" int mace_host_alg1(int n, const double* mem, const double* lat, const int8_t* is_ft, int more_queued,
                              double budget, double hard_limit, double stop_mem, int tau_task, double lambda1,
                              double lambda2, int max_ft, int max_inf, int* assign, int* out_counts,
                              double* out_bin0) {
  if (n < 0) return MACE_ERR_ARG;
  struct BinState {
    double used, maxlat;
    int n_inf, n_ft;
  };
  std::vector<BinState> bins;
  bins.reserve(64);
  long long examined = 0;
  int count = 0;
  int i = 0;
  for (; i < n; ++i) {
    if (!bins.empty() && (bins[0].used >= stop_mem || count >= tau_task)) break;
    ++count;
    const double m = mem[i], l = lat[i];
    if (m > hard_limit) {
      assign[i] = -1;  // rejected
      continue;
    }
    if (m > budget) {
      assign[i] = -2;  // deferred (requeued after the later bins)
      continue;
    }
    const bool ft = is_ft[i] != 0;
    int best = -1;
    double best_score = INFINITY;
    for (int b = 0; b < (int)bins.size(); ++b) {
      ++examined;
      const double free_mb = budget - bins[b].used;
      if (free_mb < m) continue;
      if (ft ? bins[b].n_ft < max_ft : bins[b].n_inf < max_inf) {
        const double score = lambda1 * std::fabs(free_mb - m) + lambda2 * std::fabs(bins[b].maxlat - l);
        if (score < best_score) {
          best_score = score;
          best = b;
        }
      }
    }
    if (best < 0) {
      bins.push_back(BinState{0.0, 0.0, 0, 0});
      best = (int)bins.size() - 1;
    }
    BinState& B = bins[best];
    B.used += m;
    B.maxlat = B.maxlat >= l ? B.maxlat : l;  // Python max(maxlat, lat): the first argument on ties
    if (ft) ++B.n_ft;
    else ++B.n_inf;
    assign[i] = best;
  }
  // ran out of precomputed candidates while the reference loop would keep dequeuing: hand back
  if (i == n && more_queued && !(!bins.empty() && (bins[0].used >= stop_mem || count >= tau_task))) return 2;
  out_counts[0] = count;
  out_counts[1] = (int)bins.size();
  out_counts[2] = (int)(examined < 2147483647LL ? examined : 2147483647LL);
  if (!bins.empty()) {
    out_bin0[0] = bins[0].used;
    out_bin0[1] = bins[0].maxlat;
    out_counts[3] = bins[0].n_inf;
    out_counts[4] = bins[0].n_ft;
  }
  return 0;
}

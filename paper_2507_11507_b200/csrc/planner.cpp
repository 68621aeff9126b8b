// Remap planner (SURVEY.md §8(a) a1; §5.3-5.4, Eqs. 1-5, :390-486).
//
//  * uniform-interval placement on the circular execution ring (Eqs. 1-3,
//    PAPER.md:434-461): gaps floor/ceil(n/m), larger gaps first from the anchor;
//  * m = alpha + beta layers share beta slots; beta = 1 is
//    the single-slot case (Eq. 4), beta = 2 double buffering (Eq. 5);
//  * the dynamic policy takes the smallest m whose predicted stall, from an
//    event simulation of the copy-engine / compute timeline, is zero
//    (reading #5-#6: Eqs. 4/5 are necessary, not sufficient).
#include <algorithm>
#include <cstdint>
#include <vector>

#include "../../include/mirage.h"

namespace mirage {

std::vector<int32_t> uniform_placement(int32_t n, int32_t m, int32_t anchor) {
  std::vector<int32_t> out;
  if (m <= 0) return out;
  const int32_t q = n / m, r = n % m;
  int64_t pos = anchor;
  for (int32_t i = 0; i < m; ++i) {
    out.push_back((int32_t)(pos % n));
    pos += (i < r) ? q + 1 : q;
  }
  std::sort(out.begin(), out.end());
  return out;
}

// Steady-state stall (ns) of the last of `steps` simulated decode steps:
// cycled use k = layer C[k % m] of step k / m in slot k % beta; copy k (k >= beta)
// starts when the link is free and use k - beta has finished computing; a
// cycled layer starts no earlier than its copy's end.
int64_t simulate_stall(int32_t n, const std::vector<int32_t>& C, int32_t beta, uint64_t tt,
                       uint64_t tc, int32_t steps) {
  const int32_t m = (int32_t)C.size();
  if (m == 0 || beta == 0) return 0;
  std::vector<uint64_t> compute_end;
  compute_end.reserve((size_t)m * steps);
  std::vector<char> is_cycled(n, 0);
  for (int32_t c : C) is_cycled[c] = 1;
  uint64_t t = 0, link = 0, last_dur = 0;
  int64_t k = 0;
  for (int32_t s = 0; s < steps; ++s) {
    const uint64_t t0 = t;
    for (int32_t l = 0; l < n; ++l) {
      uint64_t start = t;
      if (is_cycled[l]) {
        uint64_t ready = 0;
        if (k >= beta) {
          const uint64_t c0 = std::max(link, compute_end[k - beta]);
          link = c0 + tt;
          ready = link;
        }
        start = std::max(t, ready);
        compute_end.push_back(start + tc);
        ++k;
      }
      t = start + tc;
    }
    last_dur = t - t0;
  }
  return (int64_t)(last_dur - (uint64_t)n * tc);
}

}  // namespace mirage

extern "C" int32_t mirage_plan(int32_t n_layers, int32_t alpha, int32_t beta_policy,
                               uint64_t t_transfer_ns, uint64_t t_compute_layer_ns, int32_t anchor,
                               int32_t* cycle_out, int32_t* m_out, int32_t* beta_out) {
  if (n_layers <= 0 || n_layers > MIRAGE_MAX_CYCLE || alpha < 0 || anchor < 0 ||
      anchor >= n_layers || !cycle_out || !m_out || !beta_out)
    return MIRAGE_ERR_RANGE;
  if (beta_policy != MIRAGE_BETA_1 && beta_policy != MIRAGE_BETA_2 &&
      beta_policy != MIRAGE_BETA_DYNAMIC)
    return MIRAGE_ERR_RANGE;
  if (alpha == 0) {
    *m_out = 0;
    *beta_out = 0;
    return MIRAGE_OK;
  }
  const int32_t cand[2] = {1, 2};
  const int32_t lo = beta_policy == MIRAGE_BETA_2 ? 1 : 0;
  const int32_t hi = beta_policy == MIRAGE_BETA_1 ? 1 : 2;
  for (int32_t c = lo; c < hi; ++c) {
    const int32_t beta = cand[c];
    const int32_t m = alpha + beta;
    if (m > n_layers) continue;
    std::vector<int32_t> C = mirage::uniform_placement(n_layers, m, anchor);
    if (beta_policy == MIRAGE_BETA_DYNAMIC &&
        mirage::simulate_stall(n_layers, C, beta, t_transfer_ns, t_compute_layer_ns, 8) != 0)
      continue;
    std::copy(C.begin(), C.end(), cycle_out);
    *m_out = m;
    *beta_out = beta;
    return MIRAGE_OK;
  }
  return beta_policy == MIRAGE_BETA_DYNAMIC ? MIRAGE_ERR_INFEASIBLE : MIRAGE_ERR_RANGE;
}

extern "C" int32_t mirage_predict_stall(int32_t n_layers, const int32_t* cycle, int32_t m, int32_t beta,
                                        uint64_t t_transfer_ns, uint64_t t_compute_layer_ns, int64_t* stall_ns_out) {
  if (n_layers <= 0 || m < 0 || m > n_layers || beta < 0 || beta > m || !stall_ns_out || (m && !cycle))
    return MIRAGE_ERR_RANGE;
  for (int32_t i = 0; i < m; ++i)
    if (cycle[i] < 0 || cycle[i] >= n_layers || (i && cycle[i] <= cycle[i - 1])) return MIRAGE_ERR_RANGE;
  const std::vector<int32_t> C(cycle, cycle + m);
  *stall_ns_out = mirage::simulate_stall(n_layers, C, beta, t_transfer_ns, t_compute_layer_ns, 8);
  return MIRAGE_OK;
}

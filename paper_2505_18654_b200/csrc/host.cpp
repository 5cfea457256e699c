// Host-side integer artefacts of the MTGR hot path: jagged batch builder and the dynamic-BS
// LPT load balancer (readings R#19).  Bit-exact with
// oracle/balance.py by construction of the same definition (never by sharing code).
#include <algorithm>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <numeric>
#include <vector>

#include "../../include/mtgr.h"

#define MTGR_API extern "C" __attribute__((visibility("default")))

namespace mtgr {
mtgr_status_t set_error(mtgr_status_t s, const char* fmt, ...);
}

MTGR_API mtgr_status_t mtgr_build_jagged(const int32_t* seg4, int32_t n, const int32_t* users,
                                         int32_t m, int32_t* offsets, int32_t* n_static,
                                         int32_t* n_rt, int32_t* n_cand, uint8_t* group_id) {
  if (!seg4 || !offsets || !n_static || !n_rt || !n_cand || n < 0 || m < 0)
    return mtgr::set_error(MTGR_E_ARG, "mtgr_build_jagged: null pointer or negative size");
  if (!users && m != n)
    return mtgr::set_error(MTGR_E_ARG, "mtgr_build_jagged: users == NULL requires m == n");
  int64_t off = 0;
  offsets[0] = 0;
  for (int32_t i = 0; i < m; ++i) {
    int32_t u = users ? users[i] : i;
    if (u < 0 || u >= n) return mtgr::set_error(MTGR_E_ARG, "mtgr_build_jagged: user index %d out of range", u);
    const int32_t* s = seg4 + 4 * (int64_t)u;
    if (s[0] < 0 || s[1] < 0 || s[2] < 0 || s[3] < 0)
      return mtgr::set_error(MTGR_E_ARG, "mtgr_build_jagged: negative segment length (user %d)", u);
    int64_t L = (int64_t)s[0] + s[1] + s[2] + s[3];
    if (group_id) {
      uint8_t* g = group_id + off;
      std::memset(g, 0, s[0]);
      std::memset(g + s[0], 1, s[1]);
      std::memset(g + s[0] + s[1], 2, s[2]);
      std::memset(g + s[0] + s[1] + s[2], 3, s[3]);
    }
    off += L;
    if (off > INT32_MAX) return mtgr::set_error(MTGR_E_ARG, "mtgr_build_jagged: total tokens overflow int32");
    offsets[i + 1] = (int32_t)off;
    n_static[i] = s[0] + s[1];
    n_rt[i] = s[2];
    n_cand[i] = s[3];
  }
  return MTGR_OK;
}

MTGR_API mtgr_status_t mtgr_balance_lpt(const int64_t* cost, int32_t n, int32_t world,
                                        int64_t cap, int32_t* rank_of, int64_t* load) {
  if ((!cost && n > 0) || (!rank_of && n > 0) || !load || n < 0 || world < 1)
    return mtgr::set_error(MTGR_E_ARG, "mtgr_balance_lpt: invalid arguments");
  for (int32_t i = 0; i < n; ++i) {
    if (cost[i] < 0) return mtgr::set_error(MTGR_E_ARG, "mtgr_balance_lpt: negative cost");
    if (cap > 0 && cost[i] > cap)
      return mtgr::set_error(MTGR_E_BUDGET, "mtgr_balance_lpt: user %d cost %lld > cap %lld", i,
                             (long long)cost[i], (long long)cap);
  }
  std::vector<int32_t> order(n);
  std::iota(order.begin(), order.end(), 0);
  std::stable_sort(order.begin(), order.end(), [&](int32_t a, int32_t b) {
    return cost[a] != cost[b] ? cost[a] > cost[b] : a < b;
  });
  for (int32_t w = 0; w < world; ++w) load[w] = 0;
  for (int32_t u : order) {
    int32_t best = 0;
    for (int32_t w = 1; w < world; ++w)
      if (load[w] < load[best]) best = w;  // strict '<' keeps the lowest rank on ties
    rank_of[u] = best;
    load[best] += cost[u];
  }
  return MTGR_OK;
}

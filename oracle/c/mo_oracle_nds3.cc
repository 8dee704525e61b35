/* Exact non-dominated sort for m <= 3 in O(R log R log F) (TEST INFRASTRUCTURE / CPU CHECKER ONLY --
 * never linked into the product).
 *
 * The all-pairs oro_nds (mo_oracle.c) is O(R^2 m): about two minutes per generation at C4
 * (R = 2M, m = 3) on 16 cores.  This restates the same ranks (the peeling
 * definition of oracle/manyobj_ref/dominance.py:36) for m <= 3 by a sweep:
 *
 *   1. visit rows in lexicographic order of (f0, f1, f2) (float compares: -0 == +0);
 *   2. rows with identical vectors form one group (mutually non-dominating) and
 *      get one rank, computed before any of them is inserted;
 *   3. every row q visited before row p has q0 <= p0 (and q != p across groups), so q dominates p
 *      iff q1 <= p1 and q2 <= p2: a 2-D dominance query against the rows already placed;
 *   4. rank(p) = 1 + max rank of its dominators, and the fronts are nested (a dominator of p in
 *      front k has its own dominator in front k-1, which then dominates p), so rank(p) is the first
 *      front k that holds no 2-D dominator of p: binary search over the fronts;
 *   5. each front keeps its 2-D staircase (points (f1, f2) with f1 ascending, f2 strictly
 *      descending): "exists q with q1 <= x and q2 <= y" <=> the staircase point with the largest
 *      q1 <= x has q2 <= y.
 *
 * With stop_at > 0 the fronts after the first one whose cumulative size reaches stop_at are
 * DROPPED (2^31 - 1), exactly like the peeling oracle.  m = 1 and m = 2 run with the missing
 * coordinates set to 0 (a constant coordinate changes no dominance relation).
 */
#include <stdint.h>

#include <algorithm>
#include <map>
#include <numeric>
#include <vector>

namespace {

struct Stair {
  std::map<float, float> pts;   // f1 -> f2, f2 strictly decreasing in f1

  // some point with q1 <= x and q2 <= y ?
  bool covers(float x, float y) const {
    auto it = pts.upper_bound(x);   // first q1 > x  (-0 and +0 compare equal)
    if (it == pts.begin()) return false;
    --it;
    return it->second <= y;
  }
  void insert(float x, float y) {
    if (covers(x, y)) return;       // adds nothing to any prefix minimum
    auto it = pts.lower_bound(x);
    // drop points with q1 >= x and q2 >= y (now covered by (x, y))
    while (it != pts.end() && it->second >= y) it = pts.erase(it);
    pts[x] = y;
  }
};

}  // namespace

extern "C" int oro_nds3(const float* F, int64_t R, int m, int64_t stop_at, int64_t* ranks) {
  if (m < 1 || m > 3 || R < 0) return 2;
  std::vector<float> P((size_t)R * 3, 0.0f);
  for (int64_t i = 0; i < R; ++i)
    for (int k = 0; k < m; ++k) P[(size_t)i * 3 + k] = F[i * m + k] + 0.0f;   // -0 -> +0
  std::vector<int64_t> ord((size_t)R);
  std::iota(ord.begin(), ord.end(), (int64_t)0);
  auto lex_less = [&](int64_t a, int64_t b) {
    const float* x = &P[(size_t)a * 3];
    const float* y = &P[(size_t)b * 3];
    if (x[0] != y[0]) return x[0] < y[0];
    if (x[1] != y[1]) return x[1] < y[1];
    return x[2] < y[2];
  };
  std::stable_sort(ord.begin(), ord.end(), lex_less);
  std::vector<Stair> fronts;
  std::vector<int64_t> fsize;
  int64_t g0 = 0;
  while (g0 < R) {
    int64_t g1 = g0 + 1;
    while (g1 < R && !lex_less(ord[g0], ord[g1])) ++g1;   // identical vectors
    const float* p = &P[(size_t)ord[g0] * 3];
    // first front without a 2-D dominator of p (predicate true on a prefix of the fronts)
    int64_t lo = 0, hi = (int64_t)fronts.size();
    while (lo < hi) {
      const int64_t mid = (lo + hi) / 2;
      if (fronts[(size_t)mid].covers(p[1], p[2]))
        lo = mid + 1;
      else
        hi = mid;
    }
    if (lo == (int64_t)fronts.size()) {
      fronts.emplace_back();
      fsize.push_back(0);
    }
    fronts[(size_t)lo].insert(p[1], p[2]);
    fsize[(size_t)lo] += g1 - g0;
    for (int64_t q = g0; q < g1; ++q) ranks[ord[q]] = lo;
    g0 = g1;
  }
  if (stop_at > 0) {
    int64_t cum = 0, last = (int64_t)fronts.size();
    for (int64_t k = 0; k < (int64_t)fronts.size(); ++k) {
      cum += fsize[(size_t)k];
      if (cum >= stop_at) {
        last = k;
        break;
      }
    }
    for (int64_t i = 0; i < R; ++i)
      if (ranks[i] > last) ranks[i] = 2147483647;
  }
  return 0;
}

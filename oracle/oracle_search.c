/*
 * oracle_search.c -- TEST INFRASTRUCTURE ONLY (see oracle.h).
 *
 * O1: the Coop sliding-window eviction search of ONE pool, written as the plain
 * definition.  Build: gcc -O2 -ffp-contract=off (no FMA contraction, no fast-math),
 * SSE2 double arithmetic (x86-64 default), so every '/' and '+' is IEEE binary64 RN.
 *
 * What it computes (Sec. 3.1, Eq. 1; Sec. 3.3):
 *   the items of the pool are the address-ordered list of tensors and free chunks
 *   ("free memory chunks are included as special tensors of which the heuristics are
 *   zero"); a window is a contiguous run of items; evicting it frees its
 *   span; among windows whose span is >= the request M_R and which contain no
 *   unevictable item (R5), return the one with minimum summed heuristic
 *   h(t) = c(t)/s(t).
 *
 * Readings used:
 *   R1  h = c / s in IEEE binary64, round-to-nearest-even; FREE -> 0; PINNED -> barrier.
 *   R3  window cost = the correctly rounded binary64 value of the EXACT real sum of the
 *       h values in the window (fsum semantics, computed here with Shewchuk partials).
 *   R4  ties: minimum cost, then lowest first index; for one start the shortest window.
 *   R6  feasible iff span >= request (inclusive).
 *   R7  domain: 1 <= n <= 8192, request >= 1, 1 <= size < 2^48, state in {0,1,2};
 *       EVICTABLE: c finite >= 0, s finite >= 1, h in {0} U [2^-64, 2^60).
 *
 * Equivalence of "min over windows, minimal end per start" with Eq. 1 over sets S:
 * DESIGN.md R2 (all h >= 0, all sizes > 0); pinned by the 2^N subset enumeration in
 * tests/test_oracle_search.py.
 */
#include "oracle.h"

#include <math.h>
#include <stddef.h>
#include <string.h>

/* ---- exact summation: Shewchuk's algorithm with correctly rounded result (the same
 * definition as Python's math.fsum; written out, not shared with any GPU code). ---- */
double orc_fsum(const double *x, int64_t n) {
  double partials[128];
  int np = 0;
  for (int64_t k = 0; k < n; ++k) {
    double v = x[k];
    int i = 0;
    for (int p = 0; p < np; ++p) {
      double y = partials[p];
      if (fabs(v) < fabs(y)) {
        double t = v;
        v = y;
        y = t;
      }
      double hi = v + y;
      double lo = y - (hi - v);
      if (lo != 0.0) partials[i++] = lo;
      v = hi;
    }
    partials[i++] = v;
    np = i;
  }
  /* round the non-overlapping expansion partials[0..np) (increasing magnitude) */
  double hi = 0.0;
  if (np > 0) {
    int m = np;
    hi = partials[--m];
    double lo = 0.0;
    while (m > 0) {
      double xx = hi;
      double yy = partials[--m];
      hi = xx + yy;
      double yr = hi - xx;
      lo = yy - yr;
      if (lo != 0.0) break;
    }
    /* half-way case: make the rounding of the remaining partials correct */
    if (m > 0 && ((lo < 0.0 && partials[m - 1] < 0.0) || (lo > 0.0 && partials[m - 1] > 0.0))) {
      double yy = lo * 2.0;
      double xx = hi + yy;
      double yr = xx - hi;
      if (yy == yr) hi = xx;
    }
  }
  /* the exact real sum 0 is represented as +0.0 (as math.fsum does for -0.0 inputs) */
  return hi == 0.0 ? 0.0 : hi;
}

static void set_empty(orc_window *o, int status) {
  o->first = -1;
  o->last = -1;
  o->span = 0;
  o->cost = INFINITY;
  o->n_evict = 0;
  o->status = status;
}

#define SIZE_MASK ((((uint64_t)1) << 62) - 1)
#define SIZE_LIMIT (((uint64_t)1) << 48)

int orc_window_search(int32_t n, const uint64_t *size_state, const double *cost,
                      const double *stale, uint64_t request, orc_window *out) {
  double h[8192];
  unsigned char barrier[8192];
  if (!out) return ORC_INVALID_ARG;
  if (n < 1 || n > 8192 || request < 1 || !size_state || !cost || !stale) {
    set_empty(out, ORC_INVALID_ARG);
    return ORC_INVALID_ARG;
  }
  /* Step 1-2: validate and form the heuristic list (R1, R7). */
  for (int32_t k = 0; k < n; ++k) {
    uint64_t state = size_state[k] >> 62;
    uint64_t size = size_state[k] & SIZE_MASK;
    if (size < 1 || size >= SIZE_LIMIT || state > ORC_PINNED) {
      set_empty(out, ORC_INVALID_ARG);
      return ORC_INVALID_ARG;
    }
    barrier[k] = 0;
    if (state == ORC_FREE) {
      h[k] = 0.0; /* "special tensors of which the heuristics are zero" */
    } else if (state == ORC_PINNED) {
      barrier[k] = 1; /* unevictable: never inside a window (R5) */
      h[k] = 0.0;
    } else {
      double c = cost[k], s = stale[k];
      if (!isfinite(c) || !isfinite(s) || c < 0.0 || s < 1.0) {
        set_empty(out, ORC_INVALID_ARG);
        return ORC_INVALID_ARG;
      }
      h[k] = c / s; /* h(t) = c(t)/s(t) */
      if (h[k] != 0.0 && (h[k] < 0x1p-64 || h[k] >= 0x1p60)) {
        set_empty(out, ORC_INVALID_ARG);
        return ORC_INVALID_ARG;
      }
    }
  }
  /* Step 3-4: for every start, the shortest barrier-free window covering the request,
   * its exactly rounded cost, and the lexicographic minimum over (cost, start). */
  int best_first = -1, best_last = -1;
  double best_cost = INFINITY;
  uint64_t best_span = 0;
  for (int32_t i = 0; i < n; ++i) {
    if (barrier[i]) continue;
    uint64_t span = 0;
    int32_t j = i;
    int ok = 0;
    for (; j < n && !barrier[j]; ++j) {
      span += size_state[j] & SIZE_MASK;
      if (span >= request) { /* R6: M(S, L) >= M_R */
        ok = 1;
        break;
      }
    }
    if (!ok) continue;
    double c = orc_fsum(&h[i], (int64_t)(j - i + 1));
    if (c < best_cost) { /* strict: equal cost keeps the lower start (R4) */
      best_cost = c;
      best_first = i;
      best_last = j;
      best_span = span;
    }
  }
  if (best_first < 0) {
    set_empty(out, ORC_INFEASIBLE);
    return ORC_INFEASIBLE;
  }
  int32_t ne = 0;
  for (int32_t k = best_first; k <= best_last; ++k)
    if ((size_state[k] >> 62) == ORC_EVICTABLE) ++ne;
  out->first = best_first;
  out->last = best_last;
  out->span = best_span;
  out->cost = best_cost;
  out->n_evict = ne;
  out->status = ORC_OK;
  return ORC_OK;
}

int orc_window_search_many(int64_t n_pools, int32_t n, int64_t stride,
                           const uint64_t *size_state, const double *cost,
                           const double *stale, const uint64_t *requests,
                           orc_window *out) {
  if (n_pools < 0 || stride < n || !out || !requests) return ORC_INVALID_ARG;
  for (int64_t p = 0; p < n_pools; ++p)
    orc_window_search(n, size_state + p * stride, cost + p * stride, stale + p * stride,
                      requests[p], out + p);
  return ORC_OK;
}

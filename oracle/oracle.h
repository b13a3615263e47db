/*
 * oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain, slow, single-threaded CPU oracle for the Coop (arXiv 2311.00591) hot path.
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
 * leg may load it.  It shares no code, header, table or constant with the CUDA path
 * (paper_2311_00591_b200/, include/): every definition below is written out again here
 * from PAPER.md and the DESIGN.md readings.
 *
 * Parity pins: see tests/test_oracle_search.py (O1) and tests/test_oracle_replay.py (O2).
 */
#ifndef COOP_ORACLE_H
#define COOP_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* item states, packed in bits 62-63 of size_state */
#define ORC_FREE 0u
#define ORC_EVICTABLE 1u
#define ORC_PINNED 2u

/* statuses (numerically equal to the library's by DESIGN.md, defined here independently) */
#define ORC_OK 0
#define ORC_INFEASIBLE 1
#define ORC_INVALID_ARG (-1)
#define ORC_UNSATISFIABLE (-3)
#define ORC_THRASHED (-4)

typedef struct {
  int32_t first;   /* index of the first item of the window, -1 if none       */
  int32_t last;    /* index of the last item of the window (inclusive), -1   */
  uint64_t span;   /* sum of item sizes over [first, last]                    */
  double cost;     /* RN(exact sum of h over the window) -- DESIGN.md R3      */
  int32_t n_evict; /* number of EVICTABLE items in the window                 */
  int32_t status;  /* ORC_OK / ORC_INFEASIBLE / ORC_INVALID_ARG               */
} orc_window;

/* O1: sliding-window search of one pool (Eq. 1; 141-153 Sec. 3.3). */
int orc_window_search(int32_t n, const uint64_t *size_state, const double *cost,
                      const double *stale, uint64_t request, orc_window *out);

/* O1 over many pools laid out pool-major with a stride (same contract, one call per pool). */
int orc_window_search_many(int64_t n_pools, int32_t n, int64_t stride,
                           const uint64_t *size_state, const double *cost,
                           const double *stale, const uint64_t *requests,
                           orc_window *out);

/* Correctly rounded sum of n doubles (Shewchuk / fsum semantics); exposed for pins. */
double orc_fsum(const double *x, int64_t n);

#ifdef __cplusplus
}
#endif
#endif

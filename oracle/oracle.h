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


/* ======================================================================= O2: replay
 * Step-by-step replay of an allocation trace under one memory budget with the Coop
 * allocator: Alg. 1, sliding-window eviction (Sec. 3.3), cheap tensor
 * partitioning (Sec. 3.4), recomputable in-place (Sec. 3.5,
 * PAPER.md:206-222).  Readings R10-R35 in DESIGN.md.  TEST INFRASTRUCTURE ONLY.
 */
#define ORC_PHASE_FWD 0
#define ORC_PHASE_BWD 1
#define ORC_PHASE_UPD 2

#define ORC_F_PARTITION 1u            /* cheap tensor partitioning (Sec. 3.4)          */
#define ORC_F_INPLACE 2u              /* recomputable in-place (Sec. 3.5); off = COW    */
#define ORC_F_PARTITION_ALL_PHASES 4u /* partition backward/update ops too (R13)       */
#define ORC_F_DTR 8u   /* baseline policy: DTR's argmin loop, h = c / (m s) (R46)              */
#define ORC_F_DTE 16u  /* baseline policy: DTE, h = c / ((m + adjacent free bytes) s) (R46)    */

typedef struct {
  int32_t n_tensors, n_ops;
  const uint64_t *size;       /* [T] bytes, 1 <= size < 2^48                         */
  const uint8_t *is_param;    /* [T] 1: parameter / optimizer state (unevictable)    */
  const int32_t *producer;    /* [T] producing op, -1 for parameters                 */
  const int64_t *cost_us;     /* [M] op compute cost (us), 0 <= cost < 2^40          */
  const int32_t *out;         /* [M] output tensor (single output, R30)               */
  const int32_t *inplace_src; /* [M] mutated input tensor or -1                      */
  const uint8_t *phase;       /* [M] ORC_PHASE_*                                      */
  const int32_t *in_ptr;      /* [M+1] CSR of op inputs                               */
  const int32_t *in_idx;      /* [in_ptr[M]]                                          */
} orc_trace;

typedef struct {
  uint64_t budget;
  uint32_t flags;
  uint32_t class_threshold; /* us per MiB, C1 iff cost*2^20 >= thr*bytes (R14); 0 -> 15 */
  int32_t max_depth;        /* rematerialization depth bound (R23); 0 -> 512          */
  int32_t reserved;
} orc_cfg;

typedef struct {
  int32_t status;    /* ORC_OK, ORC_UNSATISFIABLE, ORC_THRASHED, ORC_INVALID_ARG         */
  int32_t fail_op;   /* op index of the failure, -1 for parameter placement / none     */
  int64_t base_us;   /* sum of op costs, each op once                                    */
  int64_t total_us;  /* base + recompute costs                                           */
  int64_t evictions; /* tensors evicted by window searches                               */
  int64_t remat;     /* rematerializations (recomputes)                                  */
  int64_t pressure;  /* allocation failures that triggered a window search               */
  int64_t frag_fail; /* ... of which bytes_free >= size (fragmentation failures)         */
  int64_t inplace_reuse;
  int64_t heuristic_evals;      /* EVICTABLE items whose h was formed (R28)             */
  uint64_t sum_free_bytes_after;/* after each pressure-event placement (R27)            */
  int64_t sum_free_blocks_after;
  uint64_t digest;              /* eviction sequence digest (R29)                       */
  int32_t max_depth;            /* deepest rematerialization recursion                  */
  int32_t max_blocks;           /* most pool blocks seen                                 */
  uint64_t budget;
  int64_t n_events;             /* events written (or that would have been)             */
} orc_replay_result;

/* event log record */
#define ORC_EV_PARAM 0   /* parameter placed                    */
#define ORC_EV_ALLOC 1   /* op output allocated                 */
#define ORC_EV_INPLACE 2 /* output took the mutated input's block */
#define ORC_EV_EVICT 3   /* evicted by a window                  */
#define ORC_EV_FREE 4    /* freed at death (R20, R22)            */
#define ORC_EV_REMAT 5   /* output of a recompute allocated      */
#define ORC_EV_EXEC 6    /* op executed (tensor = output)        */
#define ORC_EV_REXEC 7   /* op re-executed for a rematerialization */
typedef struct {
  int32_t kind, op, tensor, pad;
  uint64_t addr;
} orc_event;

int orc_replay(const orc_trace *tr, const orc_cfg *cfg, orc_replay_result *res,
               orc_event *log, int64_t log_cap);

/* Peak of resident bytes in an unbounded, eviction-free replay (R25). */
uint64_t orc_peak_live(const orc_trace *tr, uint32_t flags);

/* ======================================================================= O4: budget searches
 * Minimum budget (replay completes) and cutoff budget (completes without eviction) on the
 * coarse / fine grids of DESIGN.md R45.  TEST INFRASTRUCTURE ONLY. */
typedef struct {
  uint64_t peak, min_budget, cutoff_budget;
  int32_t min_status, cutoff_status, replays, reserved;
} orc_budget_result;
int orc_budget_search(const orc_trace *tr, uint32_t flags, uint32_t class_threshold, int32_t max_depth,
                      int32_t kc, int32_t kf, orc_budget_result *out);

/* ======================================================================= O3: online calls
 * One pool [0, budget) driven call by call (R38-R44): orc_pool_alloc creates
 * tensor ids 0, 1, 2, ... (one op per tensor, the parents are its inputs) through Alg. 1;
 * free / access / remat follow.  TEST INFRASTRUCTURE ONLY. */
#define ORC_NEEDS_REMAT 1
#define ORC_UNKNOWN_ID (-2)
#define ORC_NOMEM (-6)
#define ORC_BAD_STATE (-7)

#define ORC_OP_EXPENSIVE 1u   /* class C1 */
#define ORC_OP_CHEAP 2u       /* class C2 */
#define ORC_OP_INPLACE 4u     /* mutates inplace_src */
#define ORC_OP_UNEVICTABLE 8u
#define ORC_OP_PHASE_FWD 16u

typedef struct {
  int64_t tensor_id;
  uint64_t addr, size;
  int32_t n_evicted, window_first, window_last, reserved;
  uint64_t window_span;
  double window_cost;
} orc_alloc_result;

typedef struct orc_pool_s orc_pool;
orc_pool *orc_pool_create(uint64_t budget, uint32_t flags, uint32_t class_threshold,
                          int32_t max_tensors, int32_t max_edges);
void orc_pool_destroy(orc_pool *p);
int orc_pool_alloc(orc_pool *p, uint64_t size, uint64_t cost_us, uint32_t op_flags,
                   int32_t inplace_src, const int32_t *parents, int32_t n_parents,
                   orc_alloc_result *out, int32_t *evicted, int32_t evicted_cap);
int orc_pool_free(orc_pool *p, int32_t t);
int orc_pool_access(orc_pool *p, int32_t t, uint64_t advance_us);
int orc_pool_remat(orc_pool *p, int32_t t, orc_alloc_result *out, int32_t *evicted,
                   int32_t evicted_cap);
int orc_pool_stats(orc_pool *p, orc_replay_result *out);
int32_t orc_pool_layout(orc_pool *p, uint64_t *addr, uint64_t *size, int32_t *owner, int32_t cap);

#ifdef __cplusplus
}
#endif
#endif

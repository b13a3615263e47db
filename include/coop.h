/*
 * coop.h -- C ABI of libcoop, the B200-native hot path of Coop (arXiv 2311.00591,
 * "Coop: Memory is not a Commodity").
 *
 * All calls return an int status (COOP_OK = 0; COOP_INFEASIBLE = 1 is informational;
 * negative values are errors).  No C++ exception or abort crosses this boundary.
 * Outputs are written only when the call returns COOP_OK or COOP_INFEASIBLE; batched
 * calls additionally carry a per-element status inside each output record.
 *
 * Ownership: the caller owns every input and output buffer.  Device-side calls take
 * DEVICE pointers (e.g. torch.empty(..., device="cuda").data_ptr()) and a CUDA stream
 * (cudaStream_t passed as coop_stream_t, NULL = legacy default stream); they are
 * asynchronous with respect to the host and make no device allocations.  Calls whose
 * name ends in _host take HOST pointers and are synchronous.
 *
 * Threading: distinct calls on distinct buffers are independent; the library holds no
 * mutable global state except a per-device cache of kernel attributes.
 *
 * Paper references are PAPER.md:<line> (Sec./Eq./Alg.) of /root/reference/PAPER.md;
 * DESIGN.md "Readings" R1..R35 state every choice the paper leaves open.
 */
#ifndef COOP_H
#define COOP_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ------------------------------------------------------------------ status codes */
#define COOP_OK 0
#define COOP_INFEASIBLE 1        /* no window / allocation possible (informational)  */
#define COOP_ERR_INVALID_ARG (-1)
#define COOP_ERR_UNKNOWN_ID (-2)
#define COOP_ERR_UNSATISFIABLE (-3)
#define COOP_ERR_THRASHED (-4)
#define COOP_ERR_CUDA (-5)
#define COOP_ERR_NOMEM (-6)
#define COOP_ERR_BAD_STATE (-7)
#define COOP_ERR_UNIMPLEMENTED (-8)

typedef void *coop_stream_t; /* a cudaStream_t */

/* Human-readable name of a status code (static storage, never NULL). */
const char *coop_status_string(int status);

/* Library version string, e.g. "coop-b200 0.1 sm_100a" (static storage). */
const char *coop_version(void);

/* ------------------------------------------------------------------ block table
 * One pool's block table is its address-ordered item list (Sec. 3.3:
 * "storing them in a list, sorted by the memory addresses. The free memory chunks are
 * included as special tensors").  SoA, pool-major: item k of pool p is at index
 * p * pool_stride + k of each array.
 *
 *   size_state[k]  bits 0..61 = size in bytes (1 <= size < 2^48; bits 48..61 zero),
 *                  bits 62..63 = state: COOP_FREE, COOP_EVICTABLE or COOP_PINNED.
 *   cost[k]        c(t): projected recompute cost (us), finite, >= 0   (EVICTABLE only)
 *   stale[k]       s(t): staleness (us), finite, >= 1                   (EVICTABLE only)
 *
 * h(t) = c(t) / s(t) in IEEE binary64 round-to-nearest (R1); FREE items
 * have h = 0; PINNED items (unevictable: PAPER.md:51) never enter a
 * window (R5).  An EVICTABLE h must be 0 or lie in [2^-64, 2^60) (R7).
 */
#define COOP_FREE 0u
#define COOP_EVICTABLE 1u
#define COOP_PINNED 2u
#define COOP_MAX_BLOCKS 8192 /* n_blocks limit of the batched search (R7) */

typedef struct {
  const uint64_t *size_state; /* [n_pools * pool_stride], device pointer          */
  const double *cost;         /* [n_pools * pool_stride], device pointer          */
  const double *stale;        /* [n_pools * pool_stride], device pointer          */
  int64_t n_pools;            /* >= 0                                             */
  int32_t n_blocks;           /* items per pool, 1..COOP_MAX_BLOCKS               */
  int32_t reserved;           /* must be 0                                        */
  int64_t pool_stride;        /* elements between pools, >= n_blocks. The TMA fast
                                 path needs pool_stride % 16 == 0 and 16-byte aligned
                                 arrays; other layouts take a slower staging path. */
} coop_tables_soa;

/* One search result, 32 bytes. */
typedef struct {
  int32_t first;   /* first item of the window (lowest address), -1 if none          */
  int32_t last;    /* last item of the window, inclusive, -1 if none                 */
  uint64_t span;   /* bytes freed by evicting the window = sum of its item sizes     */
  double cost;     /* RN(exact sum of h over the window) (R3); +inf if none          */
  int32_t n_evict; /* EVICTABLE items in the window (FREE items are not evictions)   */
  int32_t status;  /* COOP_OK, COOP_INFEASIBLE or COOP_ERR_INVALID_ARG               */
} coop_window;

/*
 * coop_window_search_batched -- Sec. 3.3 sliding-window search of
 * Eq. 1 over n_pools independent pools, one request each.
 *
 * For pool p with request R = requests[p] (1 <= R; larger than the pool = infeasible),
 * out[p] is the contiguous run of items [first, last] with no PINNED item, span >= R
 * (R6), minimum cost (R3), ties broken by the lowest first index (R4), and for that
 * start the shortest such run.  This equals the argmin of Eq. 1 over sets S (R2).
 *
 * Arguments: t (host struct holding device pointers), requests [n_pools] device,
 * out [n_pools] device, stream.  Per-pool domain violations give out[p].status =
 * COOP_ERR_INVALID_ARG (first = last = -1, span = 0, cost = +inf, n_evict = 0);
 * an infeasible pool gives COOP_INFEASIBLE with the same fill.
 * Returns COOP_ERR_INVALID_ARG for bad struct fields / NULL pointers, COOP_ERR_CUDA on
 * a launch error, else COOP_OK (asynchronous: results are ready when the stream is).
 */
int coop_window_search_batched(const coop_tables_soa *t, const uint64_t *requests,
                               coop_window *out, coop_stream_t stream);

/*
 * coop_window_search_batched_host -- the same search on HOST-resident tables: the
 * library streams chunks of pools host->device, searches them and copies the results
 * back, overlapping the copies with the kernel on two internal streams.  Host arrays
 * should be pinned (cudaHostAlloc / torch pin_memory) for full copy bandwidth.
 * Allocates (and frees before returning) device staging of at most chunk_pools pools
 * x 2 buffers; chunk_pools <= 0 selects a default.  Synchronous.
 * Returns as coop_window_search_batched, or COOP_ERR_NOMEM.
 */
int coop_window_search_batched_host(const coop_tables_soa *host_tables,
                                    const uint64_t *host_requests, coop_window *host_out,
                                    int64_t chunk_pools);


/* ------------------------------------------------------------------ traces & replay
 * A trace is the execution-ordered op list of one or more training iterations (SoA):
 * tensors have a size, a parameter flag (parameters / optimizer states are unevictable
 * and placed before the first op) and a producing op; every op has a cost
 * (us), ONE output tensor (R30), an optional mutated input (in-place op, Sec. 3.5
 * PAPER.md:206-222), a phase and an input list (CSR).  Validation (R19, R30):
 * producer[out[k]] == k; inputs are parameters or outputs of earlier ops; an in-place
 * op's mutated input is one of its inputs, has the output's size and is never read
 * again; 1 <= size < 2^48; 0 <= cost < 2^40.
 */
#define COOP_PHASE_FWD 0
#define COOP_PHASE_BWD 1
#define COOP_PHASE_UPD 2

typedef struct {
  int32_t n_tensors;          /* T >= 1                                           */
  int32_t n_ops;              /* M >= 0                                           */
  const uint64_t *size;       /* [T] bytes                                        */
  const uint8_t *is_param;    /* [T] 1 = parameter / optimizer state              */
  const int32_t *producer;    /* [T] producing op, -1 for parameters              */
  const int64_t *cost_us;     /* [M]                                              */
  const int32_t *out;         /* [M] output tensor                                */
  const int32_t *inplace_src; /* [M] mutated input, -1 if none                    */
  const uint8_t *phase;       /* [M] COOP_PHASE_*                                 */
  const int32_t *in_ptr;      /* [M+1] input CSR offsets                          */
  const int32_t *in_idx;      /* [in_ptr[M]] input tensors                        */
} coop_trace_desc;            /* all HOST pointers; deep-copied by coop_trace_create */

typedef struct coop_trace_s *coop_trace_t;

/* Validate, preprocess (last uses, deaths, consumers, R36 lock lists) and upload a trace
 * to the current device.  Returns COOP_ERR_INVALID_ARG on a malformed trace. */
int coop_trace_create(const coop_trace_desc *desc, coop_trace_t *out);
int coop_trace_destroy(coop_trace_t trace);

/* Peak resident bytes of an unbounded, eviction-free replay (R25), host-side. */
int coop_trace_peak_live(coop_trace_t trace, uint32_t flags, uint64_t *out);

/* replay flags */
#define COOP_F_PARTITION 1u            /* cheap tensor partitioning, Sec. 3.4 */
#define COOP_F_INPLACE 2u              /* recomputable in-place, Sec. 3.5; off = copy-on-write */
#define COOP_F_PARTITION_ALL_PHASES 4u /* partition backward/update ops too (R13)          */

typedef struct {
  int32_t status;              /* COOP_OK, COOP_ERR_UNSATISFIABLE, COOP_ERR_THRASHED,
                                  COOP_ERR_NOMEM (pool exceeded the kernel's block table)  */
  int32_t fail_op;             /* op index of the failure, -1 = parameter placement / none */
  int64_t base_us, total_us;   /* compute without / with recomputation (overhead metric)  */
  int64_t evictions, remat, pressure, frag_fail, inplace_reuse, heuristic_evals;
  uint64_t sum_free_bytes_after; /* fragmentation samples after pressure events (R27)    */
  int64_t sum_free_blocks_after;
  uint64_t digest;             /* eviction sequence digest (R29)                         */
  int32_t max_depth, max_blocks;
  uint64_t budget;
  int64_t n_events;            /* events produced (log entries written = min(cap, this)) */
  int64_t search_ns_total;     /* %globaltimer ns spent in window searches (R28)         */
  int64_t search_ns_max;
} coop_replay_result;          /* 136 bytes */

typedef struct {
  int32_t kind;   /* 0 param placed, 1 output allocated, 2 in-place reuse, 3 evicted,
                     4 freed at death, 5 recompute output allocated, 6 op executed,
                     7 op re-executed for a recompute                                 */
  int32_t op;     /* op index (trace op for 0..4 and 6; producer op for 5 and 7)     */
  int32_t tensor;
  int32_t pad;
  uint64_t addr;
} coop_event;     /* 24 bytes */

/*
 * coop_replay_trace -- replay `trace` once per budget, one CTA per budget (Alg. 1,
 * PAPER.md:117-138, with Sec. 3.3-3.5), on `stream`.  budgets: HOST array [n_budgets];
 * out: DEVICE array [n_budgets]; log: DEVICE array [n_budgets * log_cap_per_budget] or
 * NULL.  class_threshold: us per MiB separating C1/C2 (0 -> 15, R14); max_depth:
 * rematerialization bound (0 -> 512, R23).  The trace's device workspace grows on demand
 * (first call with a larger n_budgets allocates).  Asynchronous.
 */
int coop_replay_trace(coop_trace_t trace, const uint64_t *budgets, int32_t n_budgets,
                      uint32_t flags, uint32_t class_threshold, int32_t max_depth,
                      coop_replay_result *out, coop_event *log, int64_t log_cap_per_budget,
                      coop_stream_t stream);

#ifdef __cplusplus
}
#endif
#endif /* COOP_H */

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
 * DESIGN.md "Readings" R1..R44 state every choice the paper leaves open.
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
 * Uses a per-device staging workspace of chunk_pools pools x 2 buffers, allocated on
 * first use (or grown for a larger chunk) and kept for later calls, so steady-state calls
 * make no device allocation; chunk_pools <= 0 selects a default (16384).  Synchronous;
 * calls are serialised process-wide.
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
/* eviction policy (default: Coop's sliding window, Sec. 3.3).  The paper's baselines
 * (R46), mutually exclusive: evict the argmin-h tensor one at a time,
 * re-evaluating all candidates, until a free block fits -- DTR h = c / (m s); DTE
 * h = c / ((m + adjacent free bytes) s).  Usually combined with no other flag (their
 * systems have neither partitioning nor recomputable in-place). */
#define COOP_F_POLICY_DTR 8u
#define COOP_F_POLICY_DTE 16u

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
 * (first call with a larger n_budgets allocates).  Asynchronous.  Calls on one trace
 * handle serialise on the device: each call's stream first waits for the previous call's
 * kernel (an event recorded after every launch), because they share the handle's
 * workspace; run independent sweeps concurrently on distinct handles.  The launch goes to
 * the device the trace was first uploaded to.
 */
int coop_replay_trace(coop_trace_t trace, const uint64_t *budgets, int32_t n_budgets,
                      uint32_t flags, uint32_t class_threshold, int32_t max_depth,
                      coop_replay_result *out, coop_event *log, int64_t log_cap_per_budget,
                      coop_stream_t stream);


/*
 * coop_replay_snapshots -- the second config-4 workload of SURVEY.md 8(d): the pools the
 * window search really sees.  Replays `trace` once under `budget` with the Coop policy
 * (flags as coop_replay_trace; the DTR / DTE baselines have no window search ->
 * COOP_ERR_INVALID_ARG) and records, at each of the first `cap` pressure events whose pool
 * holds at most n_max blocks, the address-ordered item view that the sliding-window search
 * ran on (R10-R18): one row of a coop_window_search_batched table with
 * pool_stride = n_max -- size | state << 62 per block, cost = c(t) (R18) and stale = s(t)
 * (R17) as binary64 for EVICTABLE blocks (0 / 1 otherwise), padded with trailing PINNED
 * items of size 1 (a trailing barrier cannot change any window, index or span) -- plus the
 * request (requests[k]) and the window the replay evicted (windows[k], as the batched
 * search reports it; status COOP_INFEASIBLE when none existed).  DEVICE arrays:
 * size_state / cost / stale [cap * n_max], requests / windows [cap], count (int64: events
 * recorded), out (the cell's coop_replay_result).  n_max in [1, COOP_MAX_BLOCKS].
 * Asynchronous on `stream`; same handle rules as coop_replay_trace.
 */
int coop_replay_snapshots(coop_trace_t trace, uint64_t budget, uint32_t flags,
                          uint32_t class_threshold, int32_t max_depth, int32_t n_max, int64_t cap,
                          uint64_t *size_state, double *cost, double *stale, uint64_t *requests,
                          coop_window *windows, int64_t *count, coop_replay_result *out,
                          coop_stream_t stream);

/*
 * coop_budget_search -- the two budget metrics of Sec. 4.2 and App. C
 * for one trace, by waves of coop_replay_trace (one CTA per budget):
 *   min budget    = the smallest budget at which the replay completes (status COOP_OK),
 *   cutoff budget = the smallest budget at which it completes with zero evictions.
 * Grid (R45): P = peak_live(flags) (R25), Z = the bytes of all tensors of the trace (a pool
 * of Z bytes never evicts).  Brackets (lo, hi] = (0, P], (P, 2P], (2P, 4P], ...: coarse
 * budgets B_k = max(1, lo + floor((hi - lo) * k / Kc)), k = 1..Kc; for each metric the
 * first bracket with a satisfying B_k gives k* = its smallest such k (later brackets are
 * tried only while some metric has none and hi < Z); then the fine budgets B_{k*-1} +
 * floor((B_{k*} - B_{k*-1}) * j / Kf), j = 1..Kf (B_0 = lo), and the result is the smallest
 * fine budget that satisfies it (else B_{k*}).  A metric that no bracket satisfies gets
 * status COOP_INFEASIBLE and budget 0.  Synchronous (legacy default stream); the device
 * result buffer is cached in the trace handle.  Kc, Kf in [1, 4096].
 */
typedef struct {
  uint64_t peak;           /* P */
  uint64_t min_budget;     /* 0 when min_status != COOP_OK */
  uint64_t cutoff_budget;  /* 0 when cutoff_status != COOP_OK */
  int32_t min_status, cutoff_status;
  int32_t replays;         /* replay cells run (coarse + fine waves) */
  int32_t reserved;
} coop_budget_result;      /* 40 bytes */

int coop_budget_search(coop_trace_t trace, uint32_t flags, uint32_t class_threshold,
                       int32_t max_depth, int32_t coarse_steps, int32_t fine_steps,
                       coop_budget_result *out);

/* ------------------------------------------------------------------ online single pool
 * One memory pool [0, budget) driven call by call by a framework -- the user-facing side of
 * Alg. 1 Allocate(op, size) with the sliding-window eviction of Sec. 3.3
 * (PAPER.md:141-153), cheap tensor partitioning (Sec. 3.4) and
 * recomputable in-place (Sec. 3.5).  Readings R38-R44.
 *
 * The pool state (block table, tensor graph, residency, clock, counters) is DEVICE-resident;
 * every call runs one CTA of the same Alg. 1 engine as coop_replay_trace on it, on the
 * pool's own stream, and is synchronous (results are returned in host memory).  Calls on
 * one pool must not overlap (one owner per handle).
 *
 * Tensors: coop_alloc creates ids 0, 1, 2, ... in call order; each alloc is one op whose
 * inputs are `parents` (all resident) and whose output is the new tensor (op id = tensor
 * id).  c(t) = the op's cost plus its evicted neighbourhood (R18); s(t) = clock -
 * last access (R17); the clock advances by each executed op's cost and by coop_access.
 * A freed tensor keeps its graph node: it can be recomputed (coop_rematerialize) when an
 * evicted descendant needs it, and must then be freed again.
 */
#define COOP_NEEDS_REMAT 1 /* coop_access / coop_alloc / coop_rematerialize: a tensor (or a
                              parent) is not resident -- rematerialize it first          */

typedef struct {
  uint64_t budget;          /* pool bytes, >= 1                                             */
  uint32_t flags;           /* COOP_F_PARTITION | COOP_F_INPLACE | COOP_F_PARTITION_ALL_PHASES */
  uint32_t class_threshold; /* us per MiB separating C1 / C2 when no class flag is given;
                               0 -> 15 (R14)                                              */
  int32_t max_tensors;      /* id capacity, 1..16384 (device arrays sized once)            */
  int32_t max_edges;        /* total parent links over all allocs, >= 0                    */
} coop_pool_config;

typedef struct coop_pool_s *coop_pool_t;

/* op_flags of coop_alloc */
#define COOP_OP_EXPENSIVE 1u   /* class C1: placed from the left (Sec. 3.4)                  */
#define COOP_OP_CHEAP 2u       /* class C2: from the right under COOP_F_PARTITION (fwd phase)  */
#define COOP_OP_INPLACE 4u     /* mutates inplace_src (a parent of the same size, Sec. 3.5)    */
#define COOP_OP_UNEVICTABLE 8u /* never evicted (parameters, optimizer state: PAPER.md:51)     */
#define COOP_OP_PHASE_FWD 16u  /* a forward-phase op (partitioning applies, R12)               */

typedef struct {
  int64_t tensor_id;     /* the tensor allocated (NEEDS_REMAT: the parent to recompute)    */
  uint64_t addr;         /* byte offset in the pool                                        */
  uint64_t size;
  int32_t n_evicted;     /* tensors evicted by this call (ids in evicted_ids)              */
  int32_t window_first;  /* item indices of the evicted window in the address-ordered     */
  int32_t window_last;   /*   list before eviction, -1 when no window was needed           */
  int32_t reserved;
  uint64_t window_span;  /* bytes of the window                                            */
  double window_cost;    /* its cost RN(sum h) (R3); 0 when no window                      */
} coop_alloc_result;     /* 56 bytes */

/* Create a pool with one free block [0, budget) on the current device.  Allocates all
 * device state once (no allocation in later calls).  COOP_ERR_INVALID_ARG on a bad
 * config, COOP_ERR_NOMEM / COOP_ERR_CUDA on device failures. */
int coop_pool_init(const coop_pool_config *cfg, coop_pool_t *out);
int coop_pool_destroy(coop_pool_t pool);

/*
 * coop_alloc -- Alg. 1 for a new tensor of `size` bytes produced by an op of cost
 * `cost_us` reading `parents` (HOST array, n_parents ids, all resident).  With
 * COOP_OP_INPLACE and COOP_F_INPLACE the output takes inplace_src's block (inplace_src
 * becomes non-resident, recomputable); otherwise the output is placed by first fit from
 * its class's end, and on failure the minimum-cost window is evicted (Sec. 3.3) and the
 * output placed in the coalesced block.  inplace_src must be -1 without COOP_OP_INPLACE.
 * Returns COOP_OK (out, evicted_ids[0 .. min(n_evicted, evicted_cap)) in ascending
 * address order), COOP_NEEDS_REMAT (out->tensor_id = the first non-resident parent; no
 * state change), COOP_ERR_UNSATISFIABLE (no window exists; no tensor is created),
 * COOP_ERR_INVALID_ARG (size outside [1, 2^48), cost >= 2^40, bad flags, bad in-place
 * source), COOP_ERR_UNKNOWN_ID (a parent id never allocated), COOP_ERR_NOMEM (capacity,
 * or a block table beyond 4096 blocks), COOP_ERR_CUDA.
 */
int coop_alloc(coop_pool_t pool, uint64_t size, uint64_t cost_us, uint32_t op_flags,
               int64_t inplace_src, const int64_t *parents, int32_t n_parents,
               coop_alloc_result *out, int64_t *evicted_ids, int32_t evicted_cap);

/* coop_free -- the framework frees a tensor: a resident block is released and coalesced
 * with free neighbours.  COOP_ERR_UNKNOWN_ID, or COOP_ERR_BAD_STATE for a
 * double free (a freed tensor that is not resident). */
int coop_free(coop_pool_t pool, int64_t tensor_id);

/* coop_access -- the framework reads a tensor after `advance_clock_us` of other work: the
 * clock advances, and a resident tensor's staleness restarts (R17).  COOP_OK, or
 * COOP_NEEDS_REMAT when the tensor is not resident (evicted, or its block was taken by an
 * in-place op); COOP_ERR_BAD_STATE for a freed tensor; COOP_ERR_UNKNOWN_ID;
 * COOP_ERR_INVALID_ARG for advance >= 2^40. */
int coop_access(coop_pool_t pool, int64_t tensor_id, uint64_t advance_clock_us);

/* coop_rematerialize -- re-allocate a non-resident tensor through Alg. 1 out of place
 * (R21); the framework then re-runs its op (its cost is charged to the clock).  Its
 * parents must be resident: otherwise COOP_NEEDS_REMAT with out->tensor_id = the first
 * missing parent (rematerialize that first).  A resident tensor: COOP_OK, no change.
 * Other returns as coop_alloc. */
int coop_rematerialize(coop_pool_t pool, int64_t tensor_id, coop_alloc_result *out,
                       int64_t *evicted_ids, int32_t evicted_cap);

/* Counters of the pool so far (the coop_replay_result fields; status = COOP_OK). */
int coop_pool_stats(coop_pool_t pool, coop_replay_result *out);

/* The block table in address order (SPEC.md debug dump): *n_blocks = count; the first
 * min(count, cap) blocks are written to the HOST arrays (owner -1 = free). */
int coop_pool_layout(coop_pool_t pool, uint64_t *addr, uint64_t *size, int64_t *owner,
                     int32_t cap, int32_t *n_blocks);

/*
 * coop_pool_service -- low-latency mode for the online calls above (
 * the calls are Alg. 1 per call, whose search the paper times per call,
 * PAPER.md:264, 299-300).  With idle_timeout_us > 0 one CTA stays resident on the pool's
 * stream and polls a mailbox in mapped pinned host memory: each call writes its arguments
 * and a sequence number there and spins until the device acknowledges it -- no kernel
 * launch and no stream synchronisation per call.  Results are bit-identical to the
 * launch-per-call mode (same device code).  The resident kernel exits after
 * idle_timeout_us without a call (so a device-wide synchronisation elsewhere in the
 * process waits at most that long) and is relaunched transparently by the next call.
 * idle_timeout_us = 0 stops it and returns to one launch per call (the default).
 * The resident CTA occupies one SM while active.  COOP_ERR_INVALID_ARG for a timeout
 * above 10 s, COOP_ERR_CUDA on launch failure.  Not thread-safe (one owner per handle).
 */
int coop_pool_service(coop_pool_t pool, uint32_t idle_timeout_us);

#ifdef __cplusplus
}
#endif
#endif /* COOP_H */

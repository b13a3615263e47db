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

#ifdef __cplusplus
}
#endif
#endif /* COOP_H */

// replay_core.cuh -- the device side of the Alg. 1 engine shared by the trace replay
// (coop_replay.cu, one CTA per (trace, budget) cell) and the online single-pool calls
// (coop_pool.cu, one CTA per call on a persistent device-resident pool).
#pragma once
#include <cooperative_groups.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <new>
#include <vector>

#include "coop.h"
#include "coop_internal.h"
#include "fixed192.cuh"

namespace coop {
namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kCap = 4096;       // blocks per pool held by the kernel (COOP_ERR_NOMEM beyond)
constexpr int kStackCap = 1030;  // rematerialization frames (max_depth <= 1024)
constexpr int kRsm = 64;         // of which held in shared memory
constexpr int kFree = -1;
constexpr int kOpChunk = 32;   // replay: trace ops whose records are staged in shared memory at once
constexpr int kListCap = 384;  // their input / death / lock lists staged with them (else read from L2)
constexpr int kMaxCluster = 8;  // replay: CTAs per cell (the leader + up to 7 closure helpers)
constexpr int kRing = 2048;    // replay warp BFS: per-warp queue ring (uint16 entries, shared memory)
constexpr int kGL = 8;         // replay group BFS: lanes per group (4 groups per warp)
constexpr int kGroups = kThreads / kGL;
constexpr int kGRing = 256;    // replay group BFS: per-group queue ring

// one trace op, staged in shared memory (replay op loop): everything the op loop reads
struct OpRec {
  int32_t in_beg, in_end, die_beg, die_end, lock_beg, lock_end;
  int32_t out, src;
  int64_t cost;
  uint64_t out_size;
  int32_t right;  // Alg. 1 placement side of the op (R12-R13)
  int32_t pad;
};

// replay / pool flag validation: known bits, at most one baseline policy
inline bool bad_flags(uint32_t f) {
  return (f & ~31u) || ((f & COOP_F_POLICY_DTR) && (f & COOP_F_POLICY_DTE));
}
constexpr int kMaxT = 16384;     // tensors per trace whose flags live in shared memory

enum : uint8_t { TF_RES = 1, TF_BORN = 2, TF_DEAD = 4, TF_LOCK = 8 };

struct TraceDev {
  int32_t T, M, n_params;
  const uint64_t *size;
  const int32_t *producer;
  const uint8_t *unevict;
  const int64_t *cost;
  const int32_t *out;
  const int32_t *src;
  const uint8_t *phase;
  const int32_t *in_ptr, *in_idx;
  // consumers as singly linked edge lists (the online pool appends edges as tensors
  // are created): the OUTPUTS of the ops reading x are cons_out[e] for e = cons_head[x],
  // cons_next[e], ... until -1
  const int32_t *cons_head, *cons_next, *cons_out;
  // per tensor, packed for the projected-cost DFS (one 16-byte load per visited node):
  // {cost of its producer (lo, hi words), producer's inputs [in_beg, in_end) of in_idx};
  // in_beg = -1 for tensors without a producer (parameters)
  const int4 *rec;
  const uint8_t *cls;  // per op: 0 = class by threshold (R14), 1 = C1, 2 = C2; NULL = all 0
  const int32_t *lock_ptr, *lock_idx;
  const int32_t *die_ptr, *die_idx;
  const int32_t *params;
  // replay only: the graph in the compact CSR form of the fast closure walk (16-bit tensor
  // ids and offsets, 32-bit producer costs; -1 = no producer), or null when the trace is too
  // large for it (T or edges >= 2^16, or a cost >= 2^31) -- then the generic walk is used
  const int32_t *cg_cost;
  const uint16_t *cg_iptr, *cg_iidx;  // inputs of producer(x): cg_iidx[cg_iptr[x] .. cg_iptr[x+1])
  const uint16_t *cg_cptr, *cg_cout;  // outputs of the ops that read x
  int32_t cg_nnz;
};

// Byte offsets of the compact graph's pieces in one contiguous blob (host upload and the
// shared-memory copy use the same layout): cost int32[T], iptr u16[T+1], cptr u16[T+1],
// iidx u16[nnz], cout u16[nnz]; each piece 16-byte aligned.  off[5] = total bytes.
__host__ __device__ __forceinline__ void cg_offsets(int T, int nnz, size_t off[6]) {
  size_t o = 0;
  auto take = [&](size_t b) {
    const size_t r = o;
    o = (o + b + 15) / 16 * 16;
    return r;
  };
  off[0] = take((size_t)T * 4);
  off[1] = take((size_t)(T + 1) * 2);
  off[2] = take((size_t)(T + 1) * 2);
  off[3] = take((size_t)nnz * 2);
  off[4] = take((size_t)nnz * 2);
  off[5] = o;
}

struct WsLayout {  // byte offsets inside one cell's workspace
  size_t tflags, pins, last_access, taddr, epochs, marks, stack, isz, ih, ist, S, H, B, trans, victims, cand, pacc,
      rst, vc, vs, ctid;
  size_t bytes;
};

struct CellPtrs {
  uint8_t *tflags;
  int32_t *pins;
  int64_t *last_access;
  uint64_t *taddr;
  uint32_t *epochs, *marks;
  int32_t *stack;
  uint64_t *isz;
  double *ih;
  uint8_t *ist;
  uint64_t *S;
  U192 *H;
  int32_t *B;
  int32_t *trans, *victims;
  int32_t *cand;
  int64_t *pacc;  // per (candidate, half) closure sums of the current pressure event
  int32_t *rst;   // rematerialization stack: 4 x kStackCap (tensor, stage, input index, depth)
  int64_t *vc, *vs;  // c(t) and s(t) of the item view's EVICTABLE blocks (snapshots)
  int32_t *ctid;     // the current event's candidate tensors (read by both CTAs of a cluster)
};

struct KArgs {
  TraceDev tr;
  const uint64_t *budgets;
  uint32_t flags, thr;
  int32_t max_depth;
  int32_t n_cells;
  coop_replay_result *out;
  coop_event *log;
  int64_t log_cap;
  unsigned char *ws;
  WsLayout lay;
  // dynamic shared memory after Shared: tfl (tfl_bytes), then (replay) the compact graph
  // when it fits (g_smem), then `walkers` closure-walk bitmaps of vis_words words each
  int32_t tfl_bytes;
  int32_t g_smem;     // the compact graph is copied into shared memory
  int32_t g_bytes;    // its size (16-byte multiple)
  int32_t walkers;    // threads [0, walkers) walk closures (fast path); 0 = generic walk
  int32_t helper;     // replay: helper CTAs per cell (thread-block clusters of helper + 1 CTAs:
                      // the others walk projected-cost closures with the leader, cluster_helper)
  int32_t warp_bfs;   // fast path by whole warps (1) or by 8-lane groups (2): one closure per
                      // warp / group, edge-parallel BFS
  int32_t vis_words;  // bitmap words per walker (ceil(T / 32), rounded to 4)
  // coop_replay_snapshots: the item view of every Coop pressure event (one cell), as rows
  // of a batched-search table (stride snap_n), plus the request and the evicted window
  uint64_t *snap_ss;
  double *snap_c, *snap_s;
  uint64_t *snap_req;
  coop_window *snap_win;
  int64_t *snap_count;
  int64_t snap_cap;
  int32_t snap_n;
  int64_t *phase_ns;  // profiling hook (COOP_REPLAY_PHASES): per cell, ns in 8 pressure-event phases
};

struct Shared {
  // the pool's address-ordered block table (single buffer; splices shift in place)
  uint64_t addr[kCap + 2];
  uint64_t size[kCap + 2];
  int16_t owner[kCap + 2];  // tensor id (< kMaxT = 16384) or kFree
  uint64_t wS[kWarps];
  U192 wH[kWarps];
  int32_t wB[kWarps];
  int32_t nb;
  // CTA-uniform scalars (written by thread 0, published by a barrier)
  uint64_t bytes_free;
  int64_t clock;
  int32_t status, fail_op, cur_op;
  int32_t sp;
  int32_t ntrans;
  int32_t bcast_i;
  uint64_t bcast_u;
  // counters (thread 0 only)
  coop_replay_result res;
  // reductions
  uint64_t red64[2][kWarps];
  int32_t red32[2][kWarps];
  U192 red192[kWarps];
  int32_t redpar;
  int32_t ncand, cand_next;  // projected-cost work list of the current pressure event
  int32_t helper_cmd;        // cluster helper: 1 = walk this event's items, 2 = exit
  // the last evicted window (read by the online calls): items, span, cost bits, victims
  int32_t win_first, win_last, nvict;
  uint64_t win_span, win_cost;
  // the bottom kRsm frames of the rematerialization stack (deeper frames: the workspace)
  int32_t rsm[4][kRsm];
  // replay op loop: the records and lists of the current chunk of kOpChunk ops
  OpRec ops[kOpChunk];
  int32_t op_base;                    // first op of the staged chunk
  int32_t l_in0, l_die0, l_lock0;     // first list index staged for each list
  int32_t l_in1, l_die1, l_lock1;     // one past the last staged (lists longer than kListCap: global)
  int32_t lin[kListCap], ldie[kListCap], llock[kListCap];
  uint8_t ldie_unev[kListCap];        // unevict flag of each staged dying tensor
  // dynamic tail: per-tensor flags TF_* (then the replay's graph and walker bitmaps)
  alignas(16) uint8_t tfl[];
};

__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__device__ __forceinline__ uint64_t gtimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// ------------------------------------------------------------------ CTA reductions
// Each returns the reduced value to every thread (two barriers-worth of ordering via a
// parity-double-buffered scratch: one __syncthreads per call).
__device__ __forceinline__ int32_t cta_min_i32(Shared &sh, int32_t v) {
  for (int d = 16; d > 0; d >>= 1) v = min(v, __shfl_xor_sync(0xffffffffu, v, d));
  const int par = sh.redpar;
  if ((threadIdx.x & 31) == 0) sh.red32[par][threadIdx.x >> 5] = v;
  __syncthreads();
  int32_t r = sh.red32[par][0];
  for (int w = 1; w < kWarps; ++w) r = min(r, sh.red32[par][w]);
  if (threadIdx.x == 0) sh.redpar = par ^ 1;  // next call uses the other buffer
  __syncthreads();
  return r;
}
__device__ __forceinline__ int32_t cta_max_i32(Shared &sh, int32_t v) { return -cta_min_i32(sh, -v); }
__device__ __forceinline__ int32_t cta_sum_i32(Shared &sh, int32_t v) {
  for (int d = 16; d > 0; d >>= 1) v += __shfl_xor_sync(0xffffffffu, v, d);
  const int par = sh.redpar;
  if ((threadIdx.x & 31) == 0) sh.red32[par][threadIdx.x >> 5] = v;
  __syncthreads();
  int32_t r = 0;
  for (int w = 0; w < kWarps; ++w) r += sh.red32[par][w];
  if (threadIdx.x == 0) sh.redpar = par ^ 1;
  __syncthreads();
  return r;
}
__device__ __forceinline__ uint64_t cta_min_u64(Shared &sh, uint64_t v) {
  for (int d = 16; d > 0; d >>= 1) {
    const uint64_t o = __shfl_xor_sync(0xffffffffu, v, d);
    v = o < v ? o : v;
  }
  const int par = sh.redpar;
  if ((threadIdx.x & 31) == 0) sh.red64[par][threadIdx.x >> 5] = v;
  __syncthreads();
  uint64_t r = sh.red64[par][0];
  for (int w = 1; w < kWarps; ++w) r = sh.red64[par][w] < r ? sh.red64[par][w] : r;
  if (threadIdx.x == 0) sh.redpar = par ^ 1;
  __syncthreads();
  return r;
}

// Loads of the trace graph: the read-only path (__ldg, ld.global.nc) for the trace replay,
// whose graph is immutable for the kernel's lifetime; plain coherent loads for the online
// pool, whose graph arrays are appended to by earlier calls of the same resident kernel.
template <bool RO, class T>
__device__ __forceinline__ T ldg_if(const T *p) {
  if constexpr (RO) return __ldg(p);
  else return *p;
}

// ------------------------------------------------------------------ the replay cell
// kRO: the trace graph is read-only while the kernel runs (replay) or not (online pool).
template <bool kRO>
struct CellT {
  const KArgs &a;
  const TraceDev &tr;
  Shared &sh;
  CellPtrs w;
  int cell;
  uint32_t epoch;  // per-thread DFS epoch
  coop_event *log;
  // fast closure walk (replay): the compact graph (shared memory or global) and this
  // thread's visited bitmap in shared memory (threads < a.walkers)
  const int32_t *gc;
  const uint16_t *gip, *gcp, *gii, *gco;
  uint32_t *vis;
  uint16_t *ring;  // warp BFS: this warp's queue ring
  int *wcnt;       // the work-item counter of the current event (local, or the cluster leader's)

  // slot: the workspace slot (the CTA, or the cluster, that runs the cell); helper: this is
  // the second CTA of a cluster (its walkers use the upper half of the DFS stacks)
  __device__ CellT(const KArgs &a_, Shared &sh_, int cell_, int slot = -1, int rank = 0)
      : a(a_), tr(a_.tr), sh(sh_), cell(cell_) {
    unsigned char *base = a.ws + (size_t)(slot >= 0 ? slot : (int)blockIdx.x) * a.lay.bytes;
    w.tflags = (uint8_t *)(base + a.lay.tflags);
    w.pins = (int32_t *)(base + a.lay.pins);
    w.last_access = (int64_t *)(base + a.lay.last_access);
    w.taddr = (uint64_t *)(base + a.lay.taddr);
    w.epochs = (uint32_t *)(base + a.lay.epochs);
    w.marks = (uint32_t *)(base + a.lay.marks);
    w.stack = (int32_t *)(base + a.lay.stack) + (size_t)rank * kThreads * tr.T;
    w.isz = (uint64_t *)(base + a.lay.isz);
    w.ih = (double *)(base + a.lay.ih);
    w.ist = (uint8_t *)(base + a.lay.ist);
    w.S = (uint64_t *)(base + a.lay.S);
    w.H = (U192 *)(base + a.lay.H);
    w.B = (int32_t *)(base + a.lay.B);
    w.trans = (int32_t *)(base + a.lay.trans);
    w.victims = (int32_t *)(base + a.lay.victims);
    w.cand = (int32_t *)(base + a.lay.cand);
    w.pacc = (int64_t *)(base + a.lay.pacc);
    w.rst = (int32_t *)(base + a.lay.rst);
    w.vc = (int64_t *)(base + a.lay.vc);
    w.vs = (int64_t *)(base + a.lay.vs);
    w.ctid = (int32_t *)(base + a.lay.ctid);
    log = (a.log && cell >= 0) ? a.log + (size_t)cell * a.log_cap : nullptr;
    gc = nullptr;
    gip = gcp = gii = gco = nullptr;
    vis = nullptr;
    ring = nullptr;
    wcnt = &sh.cand_next;
    if (kRO && a.walkers > 0) {
      size_t off[6];
      cg_offsets(tr.T, tr.cg_nnz, off);
      unsigned char *tail = sh.tfl + a.tfl_bytes;
      const unsigned char *g = a.g_smem ? tail : reinterpret_cast<const unsigned char *>(tr.cg_cost);
      gc = reinterpret_cast<const int32_t *>(g + off[0]);
      gip = reinterpret_cast<const uint16_t *>(g + off[1]);
      gcp = reinterpret_cast<const uint16_t *>(g + off[2]);
      gii = reinterpret_cast<const uint16_t *>(g + off[3]);
      gco = reinterpret_cast<const uint16_t *>(g + off[4]);
      if (a.warp_bfs == 2) {  // one bitmap per 8-lane group, then one queue ring per group
        unsigned char *vb = tail + (a.g_smem ? a.g_bytes : 0);
        vis = reinterpret_cast<uint32_t *>(vb) + (size_t)(threadIdx.x / kGL) * a.vis_words;
        ring = reinterpret_cast<uint16_t *>(vb + (size_t)kGroups * a.vis_words * 4) + (size_t)(threadIdx.x / kGL) * kGRing;
      } else if (a.warp_bfs) {  // one bitmap per warp, then one queue ring per warp
        unsigned char *vb = tail + (a.g_smem ? a.g_bytes : 0);
        vis = reinterpret_cast<uint32_t *>(vb) + (size_t)(threadIdx.x >> 5) * a.vis_words;
        ring = reinterpret_cast<uint16_t *>(vb + (size_t)kWarps * a.vis_words * 4) + (size_t)(threadIdx.x >> 5) * kRing;
      } else {
        vis = reinterpret_cast<uint32_t *>(tail + (a.g_smem ? a.g_bytes : 0)) +
              (size_t)threadIdx.x * a.vis_words;
      }

    }
  }

  __device__ __forceinline__ bool ok() const { return sh.status == COOP_OK; }
  __device__ __forceinline__ int nin(int op) const { return tr.in_ptr[op + 1] - tr.in_ptr[op]; }
  __device__ __forceinline__ int in_at(int op, int j) const { return tr.in_idx[tr.in_ptr[op] + j]; }
  __device__ __forceinline__ uint64_t *A() { return sh.addr; }
  __device__ __forceinline__ uint64_t *Z() { return sh.size; }
  __device__ __forceinline__ int16_t *O() { return sh.owner; }

  __device__ void log_ev(int kind, int op, int t, uint64_t addr) {  // thread 0 only
    const int64_t i = sh.res.n_events++;
    if (log && i < a.log_cap) {
      coop_event e;
      e.kind = kind;
      e.op = op;
      e.tensor = t;
      e.pad = 0;
      e.addr = addr;
      log[i] = e;
    }
  }

  // ---------------------------------------------------------------- block table ops
  // lowest (right = false) / highest (right = true) free block with size >= need, or -1
  __device__ int find_fit(uint64_t need, bool right) {
    const int nb = sh.nb;
    int best = right ? -1 : 0x7fffffff;
    for (int b = threadIdx.x; b < nb; b += kThreads)
      if (O()[b] == kFree && Z()[b] >= need) best = right ? max(best, b) : min(best, b);
    if (right) return cta_max_i32(sh, best);
    const int r = cta_min_i32(sh, best);
    return r == 0x7fffffff ? -1 : r;
  }

  // replace blocks [lo, hi] (hi >= lo - 1; hi = lo - 1 means pure insertion at lo) by the
  // m new blocks na/nz/no[0..m) -- in place: every thread reads the entries it will write
  // (at most kCap / kThreads of them) into registers, one barrier, then writes them
  __device__ __noinline__ void splice(int lo, int hi, int m, const uint64_t *na, const uint64_t *nz, const int32_t *no) {
    constexpr int kPer = (kCap + 2 + kThreads - 1) / kThreads;
    const int nb = sh.nb;
    const int removed = hi - lo + 1;
    const int nnb = nb - removed + m;
    uint64_t ra[kPer], rz[kPer];
    int32_t ro[kPer];
    // entries at or after the first one that moves: the new blocks, then the tail shifted
    // by m - removed (nothing moves when the tail does not shift: those are rewritten in
    // place with their own values)
    const int top = (m == removed) ? lo + m : nnb;
#pragma unroll
    for (int r = 0; r < kPer; ++r) {
      const int j = lo + r * kThreads + (int)threadIdx.x;  // new position, >= lo
      if (j >= top) break;
      if (j < lo + m) {
        ra[r] = na[j - lo];
        rz[r] = nz[j - lo];
        ro[r] = no[j - lo];
      } else {
        const int src = j - m + removed;
        ra[r] = sh.addr[src];
        rz[r] = sh.size[src];
        ro[r] = sh.owner[src];
      }
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < kPer; ++r) {
      const int j = lo + r * kThreads + (int)threadIdx.x;
      if (j >= top) break;
      sh.addr[j] = ra[r];
      sh.size[j] = rz[r];
      sh.owner[j] = (int16_t)ro[r];
    }
    if (threadIdx.x == 0) {
      sh.nb = nnb;
      if (nnb > sh.res.max_blocks) sh.res.max_blocks = nnb;
    }
    __syncthreads();
  }

  // place `need` bytes of tensor t into free block i (left end, or right end - need)
  __device__ uint64_t place(int i, uint64_t need, bool right, int t) {
    const uint64_t fa = A()[i], fz = Z()[i];
    uint64_t at;
    if (fz == need) {
      __syncthreads();
      if (threadIdx.x == 0) O()[i] = t;
      at = fa;
      __syncthreads();
    } else if (sh.nb + 1 > kCap) {
      if (threadIdx.x == 0) sh.status = COOP_ERR_NOMEM;
      __syncthreads();
      return 0;
    } else if (!right) {
      const uint64_t na[2] = {fa, fa + need}, nz[2] = {need, fz - need};
      const int32_t no[2] = {t, kFree};
      splice(i, i, 2, na, nz, no);
      at = fa;
    } else {
      const uint64_t na[2] = {fa, fa + fz - need}, nz[2] = {fz - need, need};
      const int32_t no[2] = {kFree, t};
      splice(i, i, 2, na, nz, no);
      at = fa + fz - need;
    }
    if (threadIdx.x == 0) sh.bytes_free -= need;
    return at;
  }

  __device__ int block_of_addr(uint64_t ad) {  // binary search (uniform)
    int lo = 0, hi = sh.nb - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (A()[mid] <= ad) lo = mid;
      else hi = mid - 1;
    }
    return lo;
  }

  // free block i and merge with free neighbours
  __device__ void release(int i) {
    const int nb = sh.nb;
    int lo = i, hi = i;
    if (i > 0 && O()[i - 1] == kFree) lo = i - 1;
    if (i + 1 < nb && O()[i + 1] == kFree) hi = i + 1;
    const uint64_t na = A()[lo], nz = A()[hi] + Z()[hi] - A()[lo];
    const int32_t no = kFree;
    if (threadIdx.x == 0) sh.bytes_free += Z()[i];
    splice(lo, hi, 1, &na, &nz, &no);
  }

  __device__ void free_tensor(int t) {  // resident tensor -> freed (R20, R22)
    const uint64_t ad = w.taddr[t];
    const int b = block_of_addr(ad);
    release(b);
    if (threadIdx.x == 0) {
      sh.tfl[t] &= (uint8_t)~TF_RES;
      log_ev(4, sh.cur_op, t, ad);
    }
    __syncthreads();
  }

  // ---------------------------------------------------------------- heuristics
  __device__ bool is_c1(int op) const {  // R14: C1 iff cost * 2^20 >= thr * out bytes
    if (tr.cls && tr.cls[op]) return tr.cls[op] == 1;  // online calls: explicit class (R41)
    return (uint64_t)tr.cost[op] * 1048576ull >= (uint64_t)a.thr * tr.size[tr.out[op]];
  }
  __device__ bool goes_right(int op) const {  // PAPER.md:173; R12-R13
    if (!(a.flags & COOP_F_PARTITION)) return false;
    if (tr.phase[op] != COOP_PHASE_FWD && !(a.flags & COOP_F_PARTITION_ALL_PHASES)) return false;
    return !is_c1(op);
  }

  // ---------------- projected cost c(t) (R18) --------------------
  // c(t) = cost(producer(t)) + cost of Anc(t) + cost of Desc(t) where
  //   Anc(t)  = the SET of non-resident tensors reachable upward from t's inputs through
  //             non-resident tensors (parameters stop),
  //   Desc(t) = the SET of evicted live tensors reachable downward from t's consumers'
  //             outputs through evicted live tensors.
  // All candidates of a pressure event are evaluated by ONE flat loop per thread: each
  // iteration either starts the next candidate (fetched from a shared counter, so threads
  // stay busy whatever the closure sizes), switches a candidate from its ancestors to its
  // descendants, or pops one DFS node.  No nested data-dependent loops, so the lanes of a
  // warp stay converged while their closures differ in size.  Visited marks: per-thread
  // epoch bytes in global memory (one epoch per candidate, cleared every 255).
  __device__ __forceinline__ bool down_ok(int d) const {  // evicted and live
    const uint8_t f = sh.tfl[d];
    return (f & TF_BORN) && !(f & TF_RES) && !(f & TF_DEAD);
  }
  // push-time filter: only nodes that can pass the pop-time test are pushed (and marked);
  // the pop-time test stays, so the visited set and the sums are unchanged (resident
  // neighbours such as parameters were pushed, popped and rejected before)
  __device__ __forceinline__ bool dfs_elig(int y, int stage) const {
    const uint8_t f = sh.tfl[y];
    return stage == 0 ? !(f & TF_RES) : ((f & TF_BORN) && !(f & TF_RES) && !(f & TF_DEAD));
  }
  static __device__ __forceinline__ int64_t rec_cost(const int4 r) {
    return (int64_t)(((uint64_t)(uint32_t)r.y << 32) | (uint32_t)r.x);
  }

  // cand[0..ncand): block indices of EVICTABLE items; writes w.ih[b] = RN(c(t) / s(t)).
  // The work items are (candidate, half): half 0 sums Anc(t), half 1 sums Desc(t) -- in a
  // DAG the two sets are disjoint, so they are independent walks that different threads
  // take up (finer items balance long chains better); the integer sums meet in w.pacc and
  // one pass after a barrier forms c(t) and h.  A node is marked when pushed, so every
  // node enters a walk's stack at most once: the per-thread stack (T entries) cannot
  // overflow.
  // Replay fast path of the same sums: the compact graph in shared memory and one visited
  // BITMAP per walking thread in shared memory (threads [0, a.walkers) walk, the others
  // wait at the barrier), so a DFS step is a handful of shared-memory accesses instead of
  // dependent global loads; long chains of evicted tensors (the thrashing BiLSTM cells)
  // are walked several times faster.  Same work items (candidate, half), same sets.
  __device__ void closures_fast(const int32_t *cand, int ncand) {
    if ((int)threadIdx.x < a.walkers) {
      uint32_t *mk = vis;
      const int VW = a.vis_words;
      int32_t *stk = w.stack + (size_t)threadIdx.x * tr.T;
      const int nitems = 2 * ncand;
      int sp = 0, it = -1, stage = 0;
      int64_t acc = 0;
      // push y if eligible and new (mark at push: a node enters the stack at most once)
      auto push = [&](int y) {
        const uint8_t f = sh.tfl[y];
        const bool el = stage == 0 ? !(f & TF_RES) : ((f & TF_BORN) && !(f & TF_RES) && !(f & TF_DEAD));
        const uint32_t bit = 1u << (y & 31);
        if (el && !(mk[y >> 5] & bit)) {
          mk[y >> 5] |= bit;
          stk[sp++] = y;
        }
      };
      auto expand = [&](int x) {
        if (stage == 0) {
          const int j1 = gip[x + 1];
          for (int j = gip[x]; j < j1; ++j) push(gii[j]);
        } else {
          const int j1 = gcp[x + 1];
          for (int j = gcp[x]; j < j1; ++j) push(gco[j]);
        }
      };
      // one flat loop: every iteration either starts the next work item or pops one node,
      // so the lanes of a warp stay converged while their closures differ in size
      while (true) {
        if (sp == 0) {
          if (it >= 0) w.pacc[it] = acc;
          it = atomicAdd(wcnt, 1);
          if (it >= nitems) break;
          const int t = w.ctid[it >> 1];
          stage = it & 1;
          acc = 0;
          for (int q = 0; q < VW; q += 4) *reinterpret_cast<uint4 *>(mk + q) = make_uint4(0, 0, 0, 0);
          mk[t >> 5] |= 1u << (t & 31);
          expand(t);  // roots: t's producer's inputs / its consumers' outputs
          continue;
        }
        const int x = stk[--sp];
        const int32_t cx = gc[x];
        // ancestors: non-resident (pushed so) and recomputable; descendants: evicted and
        // live (pushed so)
        if (stage == 0 && cx < 0) continue;
        acc += cx;
        expand(x);
      }
    }
  }

  // The same sums with a whole WARP per work item: an edge-parallel breadth-first walk
  // over the warp's queue ring (shared memory) with one visited bitmap per warp (test-and-set
  // by atomicOr: two lanes may reach the same node in one step).  Every lane of every warp
  // works -- the per-thread walk keeps only the walkers whose bitmaps fit busy and its lanes
  // diverge (9 threads per executed instruction on BiLSTM) -- and a long chain of evicted
  // tensors costs one queue step per BFS level instead of a serial pop per node.  A warp
  // whose ring would overflow redoes that item with the per-thread DFS on lane 0.
  __device__ void closures_warp(const int32_t *cand, int ncand) {
    const int lane = threadIdx.x & 31;
    const unsigned lt = (1u << lane) - 1u;
    uint32_t *mk = vis;  // all zero between items
    uint16_t *q = ring;
    const int VW = a.vis_words;
    const int nitems = 2 * ncand;
    while (true) {
      int it = 0;
      if (lane == 0) it = atomicAdd(wcnt, 1);
      it = __shfl_sync(0xffffffffu, it, 0);
      if (it >= nitems) break;
      const int t = w.ctid[it >> 1];
      const int stage = it & 1;
      const uint16_t *lst = stage == 0 ? gii : gco;
      const uint16_t *ptr = stage == 0 ? gip : gcp;
      int64_t acc = 0;
      int head = 0, tail = 0;
      bool ovf = false;
      if (lane == 0) mk[t >> 5] |= 1u << (t & 31);
      __syncwarp();
      // expand the edges [b, e) of the lane's node (d = e - b, 0 for none), all lanes' edges
      // spread over the warp; new eligible nodes are appended to the ring
      auto expand_batch = [&](int b, int d) {
        int off = d;  // inclusive scan of the degrees
#pragma unroll
        for (int k = 1; k < 32; k <<= 1) {
          const int o = __shfl_up_sync(0xffffffffu, off, k);
          if (lane >= k) off += o;
        }
        const int D = __shfl_sync(0xffffffffu, off, 31);
        const int ex = off - d;  // exclusive
        for (int k0 = 0; k0 < D; k0 += 32) {
          const int k = k0 + lane;
          // owner lane of edge k: the last lane whose exclusive offset is <= k (binary search
          // over the lanes' offsets by shuffles, executed by every lane); a lane with no
          // edges shares its offset with the next lane, so the last one always has edges
          int lo = 0;
#pragma unroll
          for (int step = 16; step > 0; step >>= 1) {
            const int cl = lo + step;
            const int exo = __shfl_sync(0xffffffffu, ex, cl & 31);
            if (cl < 32 && exo <= k) lo = cl;
          }
          const int bo = __shfl_sync(0xffffffffu, b, lo), exo = __shfl_sync(0xffffffffu, ex, lo);
          bool nw = false;
          int y = 0;
          if (k < D) {
            y = lst[bo + (k - exo)];
            const uint8_t f = sh.tfl[y];
            const bool el = stage == 0 ? !(f & TF_RES) : ((f & TF_BORN) && !(f & TF_RES) && !(f & TF_DEAD));
            if (el) {
              const uint32_t bit = 1u << (y & 31);
              nw = !(mk[y >> 5] & bit) && !(atomicOr(&mk[y >> 5], bit) & bit);
            }
          }
          const uint32_t bal = __ballot_sync(0xffffffffu, nw);
          if (tail - head + __popc(bal) > kRing) ovf = true;
          else if (nw) q[(tail + __popc(bal & lt)) & (kRing - 1)] = (uint16_t)y;
          tail += __popc(bal);
        }
      };
      {  // roots: t's producer's inputs / its consumers' outputs
        const int b = lane == 0 ? ptr[t] : 0, e = lane == 0 ? ptr[t + 1] : 0;
        expand_batch(b, e - b);
      }
      __syncwarp();
      while (head < tail && !__any_sync(0xffffffffu, ovf)) {
        const int n = min(32, tail - head);
        int b = 0, d = 0;
        if (lane < n) {
          const int x = q[(head + lane) & (kRing - 1)];
          const int32_t cx = gc[x];
          // ancestors: non-resident (queued so) and recomputable; descendants: evicted and
          // live (queued so)
          if (!(stage == 0 && cx < 0)) {
            acc += cx;
            b = ptr[x];
            d = ptr[x + 1] - b;
          }
        }
        head += n;
        __syncwarp();
        expand_batch(b, d);
        __syncwarp();
      }
      const bool overflow = __any_sync(0xffffffffu, ovf);
#pragma unroll
      for (int k = 16; k > 0; k >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, k);
      // clear the bitmap (warp-parallel)
      for (int k = lane; k < VW; k += 32) mk[k] = 0u;
      __syncwarp();
      if (overflow) {  // a frontier wider than the ring: redo this item depth-first on lane 0
        if (lane == 0) {
          int32_t *stk = w.stack + (size_t)threadIdx.x * tr.T;
          int sp = 0;
          acc = 0;
          mk[t >> 5] |= 1u << (t & 31);
          auto push = [&](int y) {
            const uint8_t f = sh.tfl[y];
            const bool el = stage == 0 ? !(f & TF_RES) : ((f & TF_BORN) && !(f & TF_RES) && !(f & TF_DEAD));
            const uint32_t bit = 1u << (y & 31);
            if (el && !(mk[y >> 5] & bit)) {
              mk[y >> 5] |= bit;
              stk[sp++] = y;
            }
          };
          for (int j = ptr[t]; j < ptr[t + 1]; ++j) push(lst[j]);
          while (sp > 0) {
            const int x = stk[--sp];
            const int32_t cx = gc[x];
            if (stage == 0 && cx < 0) continue;
            acc += cx;
            for (int j = ptr[x]; j < ptr[x + 1]; ++j) push(lst[j]);
          }
        }
        __syncwarp();
        for (int k = lane; k < VW; k += 32) mk[k] = 0u;
        __syncwarp();
      }
      if (lane == 0) w.pacc[it] = acc;
    }
  }

  // The warp BFS with four independent 8-lane groups per warp: a BiLSTM closure's frontier
  // is 2-4 nodes wide, so 8 lanes keep most of the edge parallelism while 32 closures are
  // walked at once per CTA instead of 8.  One flat loop per group: every iteration either
  // starts the group's next work item (seeding its queue with the roots) or expands one
  // batch of up to 8 queued nodes edge-parallel, so the groups of a warp stay converged.
  __device__ void closures_group(const int32_t *cand, int ncand) {
    const int lane = threadIdx.x & 31, gl = lane & (kGL - 1);
    const int gbase = lane & ~(kGL - 1);
    const uint32_t gmask = 0xffu << gbase;
    const unsigned glt = (1u << gl) - 1u;
    uint32_t *mk = vis;  // all zero between items
    uint16_t *q = ring;
    const int VW = a.vis_words;
    const int nitems = 2 * ncand;
    int it = -1, t = 0, stage = 0, head = 0, tail = 0;
    bool live = false, ovf = false;
    int64_t acc = 0;
    const uint16_t *lst = gii, *ptr = gip;
    // expand the edges [b, b + d) of each lane's node, spread over the group's lanes
    auto expand_batch = [&](int b, int d) {
      int off = d;
#pragma unroll
      for (int k = 1; k < kGL; k <<= 1) {
        const int o = __shfl_up_sync(gmask, off, k, kGL);
        if (gl >= k) off += o;
      }
      const int D = __shfl_sync(gmask, off, kGL - 1, kGL);
      const int ex = off - d;
      for (int k0 = 0; k0 < D; k0 += kGL) {
        const int k = k0 + gl;
        int lo = 0;
#pragma unroll
        for (int step = kGL / 2; step > 0; step >>= 1) {
          const int cl = lo + step;
          const int exo = __shfl_sync(gmask, ex, cl & (kGL - 1), kGL);
          if (cl < kGL && exo <= k) lo = cl;
        }
        const int bo = __shfl_sync(gmask, b, lo, kGL), exo = __shfl_sync(gmask, ex, lo, kGL);
        bool nw = false;
        int y = 0;
        if (k < D) {
          y = lst[bo + (k - exo)];
          const uint8_t f = sh.tfl[y];
          const bool el = stage == 0 ? !(f & TF_RES) : ((f & TF_BORN) && !(f & TF_RES) && !(f & TF_DEAD));
          if (el) {
            const uint32_t bit = 1u << (y & 31);
            nw = !(mk[y >> 5] & bit) && !(atomicOr(&mk[y >> 5], bit) & bit);
          }
        }
        const uint32_t bal = (__ballot_sync(gmask, nw) >> gbase) & 0xffu;
        if (tail - head + __popc(bal) > kGRing) ovf = true;
        else if (nw) q[(tail + __popc(bal & glt)) & (kGRing - 1)] = (uint16_t)y;
        tail += __popc(bal);
      }
    };
    while (true) {
      if (!live) {
        if (it >= 0) {  // finish the previous item
#pragma unroll
          for (int k = kGL / 2; k > 0; k >>= 1) acc += __shfl_xor_sync(gmask, acc, k, kGL);
          for (int k = gl; k < VW; k += kGL) mk[k] = 0u;
          __syncwarp(gmask);
          if (ovf) {  // a frontier wider than the ring: redo the item depth-first on one lane
            if (gl == 0) {
              int32_t *stk = w.stack + (size_t)threadIdx.x * tr.T;
              int sp = 0;
              acc = 0;
              mk[t >> 5] |= 1u << (t & 31);
              auto push = [&](int y) {
                const uint8_t f = sh.tfl[y];
                const bool el = stage == 0 ? !(f & TF_RES) : ((f & TF_BORN) && !(f & TF_RES) && !(f & TF_DEAD));
                const uint32_t bit = 1u << (y & 31);
                if (el && !(mk[y >> 5] & bit)) {
                  mk[y >> 5] |= bit;
                  stk[sp++] = y;
                }
              };
              for (int j = ptr[t]; j < ptr[t + 1]; ++j) push(lst[j]);
              while (sp > 0) {
                const int x = stk[--sp];
                const int32_t cx = gc[x];
                if (stage == 0 && cx < 0) continue;
                acc += cx;
                for (int j = ptr[x]; j < ptr[x + 1]; ++j) push(lst[j]);
              }
            }
            __syncwarp(gmask);
            for (int k = gl; k < VW; k += kGL) mk[k] = 0u;
            __syncwarp(gmask);
          }
          if (gl == 0) w.pacc[it] = acc;
        }
        int nit = 0;
        if (gl == 0) nit = atomicAdd(wcnt, 1);
        it = __shfl_sync(gmask, nit, 0, kGL);
        if (it >= nitems) break;
        t = w.ctid[it >> 1];
        stage = it & 1;
        lst = stage == 0 ? gii : gco;
        ptr = stage == 0 ? gip : gcp;
        acc = 0;
        head = tail = 0;
        ovf = false;
        if (gl == 0) mk[t >> 5] |= 1u << (t & 31);
        __syncwarp(gmask);
        const int b = gl == 0 ? ptr[t] : 0, e = gl == 0 ? ptr[t + 1] : 0;
        expand_batch(b, e - b);  // roots: t's producer's inputs / its consumers' outputs
        __syncwarp(gmask);
        live = head < tail && !ovf;
        continue;
      }
      const int n = min(kGL, tail - head);
      int b = 0, d = 0;
      if (gl < n) {
        const int x = q[(head + gl) & (kGRing - 1)];
        const int32_t cx = gc[x];
        // ancestors: non-resident (queued so) and recomputable; descendants: evicted and
        // live (queued so)
        if (!(stage == 0 && cx < 0)) {
          acc += cx;
          b = ptr[x];
          d = ptr[x + 1] - b;
        }
      }
      head += n;
      __syncwarp(gmask);
      expand_batch(b, d);
      __syncwarp(gmask);
      live = head < tail && !ovf;
    }
  }

  // the fast walk of this event's items (both CTAs of a cluster run it)
  __device__ void walk_items(const int32_t *cand, int ncand) {
    if (a.warp_bfs == 2) closures_group(cand, ncand);
    else if (a.warp_bfs) closures_warp(cand, ncand);
    else closures_fast(cand, ncand);
  }

  __device__ void projected_costs(const int32_t *cand, int ncand, int pol = 0) {
    // the candidates' tensors, in global memory where a cluster helper can read them
    for (int ci = threadIdx.x; ci < ncand; ci += kThreads) w.ctid[ci] = O()[cand[ci]];
    __syncthreads();
    if (kRO && a.walkers > 0) {
      if (a.helper) {  // the cluster's second CTA takes items from the same counter
        if (threadIdx.x == 0) {
          sh.helper_cmd = 1;
          sh.ncand = ncand;
        }
        cooperative_groups::this_cluster().sync();  // A: the helper may start
        walk_items(cand, ncand);
        cooperative_groups::this_cluster().sync();  // B: every item's sums are in w.pacc
      } else {
        walk_items(cand, ncand);
      }
      finish_costs(cand, ncand, pol);
      return;
    }
    // visited marks: one byte per tensor and thread (epoch & 255; cleared on wrap), four
    // times denser than word epochs so a walking thread's marks stay in L1
    const int Tp = (tr.T + 15) & ~15;  // per-thread stride, 16-byte aligned (uint4 clears)
    uint8_t *mk = reinterpret_cast<uint8_t *>(w.marks) + (size_t)threadIdx.x * Tp;
    int32_t *stk = w.stack + (size_t)threadIdx.x * tr.T;
    const int nitems = 2 * ncand;
    int sp = 0, it = -1, stage = 0;
    int64_t acc = 0;
    uint8_t ep = 0;
    while (true) {
      if (sp == 0) {
        if (it >= 0) w.pacc[it] = acc;
        it = atomicAdd(&sh.cand_next, 1);
        if (it >= nitems) break;
        const int t = w.ctid[it >> 1];
        stage = it & 1;
        acc = 0;
        ep = (uint8_t)++epoch;
        if (ep == 0) {  // epoch wrap (every 255 walks): clear this thread's marks
          for (int x = 0; x < Tp; x += 16) *reinterpret_cast<uint4 *>(mk + x) = make_uint4(0, 0, 0, 0);
          ep = (uint8_t)++epoch;
        }
        mk[t] = ep;
        if (stage == 0) {  // the ancestors' roots: t's producer's inputs
          const int4 r = ldg_if<kRO>(&tr.rec[t]);
          for (int j = r.z; j < r.w; ++j) {
            const int y = ldg_if<kRO>(&tr.in_idx[j]);
            if (dfs_elig(y, 0) && mk[y] != ep) {
              mk[y] = ep;
              stk[sp++] = y;
            }
          }
        } else {  // the descendants' roots: the outputs of t's consumers
          for (int e = ldg_if<kRO>(&tr.cons_head[t]); e >= 0; e = ldg_if<kRO>(&tr.cons_next[e])) {
            const int y = ldg_if<kRO>(&tr.cons_out[e]);
            if (dfs_elig(y, 1) && mk[y] != ep) {
              mk[y] = ep;
              stk[sp++] = y;
            }
          }
        }
        continue;
      }
      const int x = stk[--sp];
      const uint8_t f = sh.tfl[x];
      const int4 r = ldg_if<kRO>(&tr.rec[x]);
      // ancestors: non-resident and recomputable; descendants: evicted and live
      const bool ok = stage == 0 ? (!(f & TF_RES) && r.z >= 0)
                                 : ((f & TF_BORN) && !(f & TF_RES) && !(f & TF_DEAD));
      if (!ok) continue;
      acc += rec_cost(r);
      if (stage == 0) {
        // inputs in batches of 4: all index loads, then all mark loads, then the pushes
        // (duplicates inside a batch are skipped explicitly: their marks were read early)
        for (int j0 = r.z; j0 < r.w; j0 += 4) {
          int y[4];
          uint8_t m[4];
#pragma unroll
          for (int k = 0; k < 4; ++k) y[k] = j0 + k < r.w ? ldg_if<kRO>(&tr.in_idx[j0 + k]) : -1;
#pragma unroll
          for (int k = 0; k < 4; ++k) m[k] = (y[k] >= 0 && dfs_elig(y[k], 0)) ? mk[y[k]] : ep;
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            bool fresh = m[k] != ep;
#pragma unroll
            for (int q = 0; q < k; ++q) fresh &= y[q] != y[k];
            if (fresh) {
              mk[y[k]] = ep;
              stk[sp++] = y[k];
            }
          }
        }
      } else {
        for (int e = ldg_if<kRO>(&tr.cons_head[x]); e >= 0; e = ldg_if<kRO>(&tr.cons_next[e])) {
          const int y = ldg_if<kRO>(&tr.cons_out[e]);
          if (dfs_elig(y, 1) && mk[y] != ep) {
            mk[y] = ep;
            stk[sp++] = y;
          }
        }
      }
    }
    finish_costs(cand, ncand, pol);
  }

  // c(t) = producer cost + the two sums; h = c / s (Coop), c / (m s) (DTR), c / ((m +
  // adjacent free bytes) s) (DTE)
  __device__ void finish_costs(const int32_t *cand, int ncand, int pol) {
    __syncthreads();
    for (int ci = threadIdx.x; ci < ncand; ci += kThreads) {
      const int b = cand[ci];
      const int t = O()[b];
      const int64_t c = rec_cost(ldg_if<kRO>(&tr.rec[t])) + w.pacc[2 * ci] + w.pacc[2 * ci + 1];
      int64_t s = sh.clock - w.last_access[t];  // staleness (R17)
      if (s < 1) s = 1;
      double den = (double)s;  // Coop: h = c/s (R1)
      if (pol) {               // DTR: c / (m s); DTE: m + the adjacent free bytes (R46)
        uint64_t m = Z()[b];
        if (pol == 2) {
          if (b > 0 && O()[b - 1] == kFree) m += Z()[b - 1];
          if (b + 1 < sh.nb && O()[b + 1] == kFree) m += Z()[b + 1];
        }
        den = __dmul_rn((double)m, (double)s);
      }
      w.ih[b] = __ddiv_rn((double)c, den);
      if (a.snap_ss) {
        w.vc[b] = c;
        w.vs[b] = s;
      }
    }
  }

  // ---------------------------------------------------------------- Sec. 3.3 search
  // Sliding-window search over the address-ordered item view and eviction of the window;
  // returns false when no window exists (R24).  Scratch: the inactive block buffer holds
  // S (span prefix, u64) in its addr[], B (barrier count prefix) in its size[] and the
  // item states in its owner[]; the exact 192-bit prefix H and h live in global memory.
  // The baselines of the paper's comparison (R46): DTR / DTE evict
  // the argmin-h tensor (ties: lowest address), one at a time, re-evaluating every
  // candidate, until a free block can hold `need`.
  __device__ bool evict_loop(uint64_t need, int pol) {
    const uint64_t t0 = gtimer();
    if (threadIdx.x == 0) {
      sh.win_first = sh.win_last = -1;
      sh.win_span = 0;
      sh.win_cost = 0;
      sh.nvict = 0;
    }
    __syncthreads();
    bool ok = true;
    while (find_fit(need, false) < 0) {
      if (threadIdx.x == 0) {
        sh.ncand = 0;
        sh.cand_next = 0;
      }
      __syncthreads();
      for (int b = threadIdx.x; b < sh.nb; b += kThreads) {
        const int o = O()[b];
        if (o != kFree && !ldg_if<kRO>(&tr.unevict[o]) && w.pins[o] == 0 && !(sh.tfl[o] & TF_LOCK))
          w.cand[atomicAdd(&sh.ncand, 1)] = b;
      }
      __syncthreads();
      const int nc = sh.ncand;
      if (nc == 0) {  // nothing left to evict
        ok = false;
        break;
      }
      projected_costs(w.cand, nc, pol);
      __syncthreads();
      uint64_t best = ~0ull;
      int bi = 0x7fffffff;
      for (int c = threadIdx.x; c < nc; c += kThreads) {
        const int b = w.cand[c];
        const uint64_t hb = (uint64_t)__double_as_longlong(w.ih[b]);  // h >= 0: bit order
        if (hb < best || (hb == best && b < bi)) {
          best = hb;
          bi = b;
        }
      }
      const uint64_t hmin = cta_min_u64(sh, best);
      const int bmin = cta_min_i32(sh, best == hmin ? bi : 0x7fffffff);
      if (threadIdx.x == 0) {
        sh.res.heuristic_evals += nc;
        const int o = O()[bmin];
        const uint64_t ad = A()[bmin];
        sh.tfl[o] &= (uint8_t)~TF_RES;
        sh.res.evictions++;
        log_ev(3, sh.cur_op, o, ad);
        uint64_t d = sh.res.digest;  // R29
        d = splitmix64(d ^ (((uint64_t)(uint32_t)sh.cur_op << 32) | (uint32_t)o));
        sh.res.digest = splitmix64(d ^ ad);
        w.victims[sh.nvict++] = o;
      }
      __syncthreads();
      release(bmin);  // free + coalesce
    }
    if (threadIdx.x == 0) {
      const int64_t dt = (int64_t)(gtimer() - t0);
      sh.res.search_ns_total += dt;
      if (dt > sh.res.search_ns_max) sh.res.search_ns_max = dt;
    }
    __syncthreads();
    return ok;
  }

  __device__ bool evict_window(uint64_t need) {
    if (a.flags & (COOP_F_POLICY_DTR | COOP_F_POLICY_DTE))
      return evict_loop(need, (a.flags & COOP_F_POLICY_DTE) ? 2 : 1);
    const uint64_t t0 = gtimer();
    if (threadIdx.x == 0) {
      sh.ncand = 0;
      sh.cand_next = 0;
    }
    __syncthreads();
    const int nb = sh.nb;
    uint64_t *S = w.S;   // span prefix (workspace, L1-resident)
    int32_t *Bc = w.B;   // PINNED-count prefix
    uint8_t *St = w.ist; // item states
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    // item view (contiguous chunk per thread): FREE -> h = 0; unevictable / pinned /
    // locked -> barrier; else h = c/s with the projected cost and the staleness
    const int chunk = (nb + kThreads - 1) / kThreads;
    const int b0 = min(nb, (int)threadIdx.x * chunk), b1 = min(nb, b0 + chunk);
    int nev = 0;
    for (int b = b0; b < b1; ++b) {
      const int o = O()[b];
      int st;
      if (o == kFree) {
        st = COOP_FREE;
      } else if (ldg_if<kRO>(&tr.unevict[o]) || w.pins[o] > 0 || (sh.tfl[o] & TF_LOCK)) {
        st = COOP_PINNED;
      } else {
        st = COOP_EVICTABLE;
        w.cand[atomicAdd(&sh.ncand, 1)] = b;
        ++nev;
      }
      w.ih[b] = 0.0;
      St[b] = st;
    }
    __syncthreads();
    const uint64_t t1 = gtimer();
    projected_costs(w.cand, sh.ncand);
    __syncthreads();
    const uint64_t t2 = gtimer();
    int snap = -1;  // coop_replay_snapshots: this event's row
    if (a.snap_ss) {
      if (threadIdx.x == 0) {
        const int64_t k = *a.snap_count;
        sh.bcast_i = (k < a.snap_cap && nb <= a.snap_n) ? (int32_t)k : -1;
      }
      __syncthreads();
      snap = sh.bcast_i;
      if (snap >= 0) {
        const size_t row = (size_t)snap * a.snap_n;
        for (int b = threadIdx.x; b < a.snap_n; b += kThreads) {
          uint64_t ss = (1ull | ((uint64_t)COOP_PINNED << 62));  // padding: PINNED, size 1
          double c = 0.0, sv = 1.0;
          if (b < nb) {
            ss = Z()[b] | ((uint64_t)St[b] << 62);
            if (St[b] == COOP_EVICTABLE) {
              c = (double)w.vc[b];
              sv = (double)w.vs[b];
            }
          }
          a.snap_ss[row + b] = ss;
          a.snap_c[row + b] = c;
          a.snap_s[row + b] = sv;
        }
        if (threadIdx.x == 0) a.snap_req[snap] = need;
      }
    }
    uint64_t ls = 0;
    U192 lh = u192_zero();
    int lb = 0;
    for (int b = b0; b < b1; ++b) {
      const double h = w.ih[b];
      ls += Z()[b];
      lh = u192_add(lh, u192_from_double(h));
      lb += (St[b] == COOP_PINNED);
    }
    // exclusive scans of the thread totals: warp shuffles, then the <= 8 warp totals
    uint64_t is = ls;
    U192 ih = lh;
    int ib = lb;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const uint64_t so = __shfl_up_sync(0xffffffffu, is, d);
      U192 ho;
      ho.w0 = __shfl_up_sync(0xffffffffu, ih.w0, d);
      ho.w1 = __shfl_up_sync(0xffffffffu, ih.w1, d);
      ho.w2 = __shfl_up_sync(0xffffffffu, ih.w2, d);
      const int bo = __shfl_up_sync(0xffffffffu, ib, d);
      if (lane >= d) {
        is += so;
        ih = u192_add(ih, ho);
        ib += bo;
      }
    }
    if (lane == 31) {
      sh.wS[warp] = is;
      sh.wH[warp] = ih;
      sh.wB[warp] = ib;
    }
    nev = cta_sum_i32(sh, nev);  // (its barrier also publishes the warp totals)
    uint64_t cs = is - ls;  // exclusive within the warp
    U192 ch = u192_sub(ih, lh);
    int cb = ib - lb;
    for (int w2 = 0; w2 < warp; ++w2) {
      cs += sh.wS[w2];
      ch = u192_add(ch, sh.wH[w2]);
      cb += sh.wB[w2];
    }
    for (int b = b0; b < b1; ++b) {
      S[b] = cs;
      w.H[b] = ch;
      Bc[b] = cb;
      cs += Z()[b];
      ch = u192_add(ch, u192_from_double(w.ih[b]));
      cb += (St[b] == COOP_PINNED);
    }
    if (b1 == nb && b0 < b1) {
      S[nb] = cs;
      w.H[nb] = ch;
      Bc[nb] = cb;
    }
    if (nb == 0 && threadIdx.x == 0) {
      S[0] = 0;
      Bc[0] = 0;
    }
    __syncthreads();
    // per start: minimal end by bisection on S, barrier check, exact cost RN(H[e] - H[i]);
    // argmin over (cost bits, start) (R3, R4)
    const uint64_t Stot = S[nb];
    uint64_t bestc = ~0ull;
    int besti = 0x7fffffff;
    for (int i = threadIdx.x; i < nb; i += kThreads) {
      if (St[i] == COOP_PINNED) continue;
      const uint64_t target = S[i] + need;
      if (target > Stot) continue;
      int lo = i + 1, hi = nb;
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (S[mid] >= target) hi = mid;
        else lo = mid + 1;
      }
      const int e = lo;
      if (Bc[e] != Bc[i]) continue;
      const uint64_t cb2 = (uint64_t)__double_as_longlong(u192_round_to_double(u192_sub(w.H[e], w.H[i])));
      if (cb2 < bestc || (cb2 == bestc && i < besti)) {
        bestc = cb2;
        besti = i;
      }
    }
    const uint64_t t3 = gtimer();
    const uint64_t cmin = cta_min_u64(sh, bestc);
    const int first = cta_min_i32(sh, bestc == cmin ? besti : 0x7fffffff);
    if (threadIdx.x == 0) {
      sh.res.heuristic_evals += nev;
      const int64_t dt = (int64_t)(gtimer() - t0);
      sh.res.search_ns_total += dt;
      if (dt > sh.res.search_ns_max) sh.res.search_ns_max = dt;
    }
    if (cmin == ~0ull) {
      if (snap >= 0 && threadIdx.x == 0) {  // no window: the batched search's INFEASIBLE record
        coop_window wv;
        wv.first = wv.last = -1;
        wv.span = 0;
        wv.cost = __longlong_as_double(0x7ff0000000000000ll);
        wv.n_evict = 0;
        wv.status = COOP_INFEASIBLE;
        a.snap_win[snap] = wv;
        *a.snap_count = snap + 1;
      }
      __syncthreads();
      return false;
    }
    // window end of the winner; evict its tensors in ascending address order (R10)
    int last;
    {
      const uint64_t target = S[first] + need;
      int lo = first + 1, hi = nb;
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (S[mid] >= target) hi = mid;
        else lo = mid + 1;
      }
      last = lo - 1;
    }
    if (threadIdx.x == 0) {
      sh.win_first = first;
      sh.win_last = last;
      sh.win_span = S[last + 1] - S[first];
      sh.win_cost = cmin;
      sh.nvict = 0;
      uint64_t d = sh.res.digest;
      for (int b = first; b <= last; ++b) {
        const int o = O()[b];
        if (o == kFree) continue;
        w.victims[sh.nvict++] = o;
        const uint64_t ad = A()[b];
        sh.tfl[o] &= (uint8_t)~TF_RES;
        sh.res.evictions++;
        log_ev(3, sh.cur_op, o, ad);
        d = splitmix64(d ^ (((uint64_t)(uint32_t)sh.cur_op << 32) | (uint32_t)o));  // R29
        d = splitmix64(d ^ ad);
        sh.bytes_free += Z()[b];
      }
      sh.res.digest = d;
      if (snap >= 0) {  // the window the replay evicts, as a coop_window
        coop_window wv;
        wv.first = first;
        wv.last = last;
        wv.span = sh.win_span;
        wv.cost = __longlong_as_double((long long)cmin);
        wv.n_evict = sh.nvict;
        wv.status = COOP_OK;
        a.snap_win[snap] = wv;
        *a.snap_count = snap + 1;
      }
    }
    __syncthreads();
    // the window and its free neighbours coalesce into one free block
    int lo = first, hi = last;
    if (lo > 0 && O()[lo - 1] == kFree) --lo;
    if (hi + 1 < nb && O()[hi + 1] == kFree) ++hi;
    const uint64_t na = A()[lo], nz = A()[hi] + Z()[hi] - A()[lo];
    const int32_t no = kFree;
    splice(lo, hi, 1, &na, &nz, &no);
    if (a.phase_ns && threadIdx.x == 0) {  // view, closures, scans + ends + costs, argmin + evict + splice
      int64_t *pn = a.phase_ns + (size_t)cell * 8;
      const uint64_t t4 = gtimer();
      pn[0] += (int64_t)(t1 - t0);
      pn[1] += (int64_t)(t2 - t1);
      pn[2] += (int64_t)(t3 - t2);
      pn[3] += (int64_t)(t4 - t3);
      pn[4] += 1;
    }
    return true;
  }

  // ---------------------------------------------------------------- Alg. 1
  __device__ void allocate(int op, int t, bool allow_inplace, int kind) {
    allocate_with(op, t, tr.size[t], tr.src[op], goes_right(op), allow_inplace, kind);
  }
  // the same with the op's fields already at hand (the replay's staged op records)
  __device__ __forceinline__ void allocate_with(int op, int t, uint64_t need, int src, bool right, bool allow_inplace, int kind) {
    if (allow_inplace && src >= 0 && (a.flags & COOP_F_INPLACE)) {  // addr <- input.addr
      const uint64_t ad = w.taddr[src];
      const int b = block_of_addr(ad);
      __syncthreads();
      if (threadIdx.x == 0) {
        O()[b] = t;
        w.taddr[t] = ad;
        sh.tfl[src] &= (uint8_t)~TF_RES;
        sh.tfl[t] |= TF_RES;
        sh.res.inplace_reuse++;
        log_ev(2, op, t, ad);
      }
      __syncthreads();
      return;
    }
    int i = find_fit(need, right);
    uint64_t at;
    if (i < 0) {
      if (threadIdx.x == 0) {
        sh.res.pressure++;
        if (sh.bytes_free >= need) sh.res.frag_fail++;
      }
      if (!evict_window(need)) {
        if (threadIdx.x == 0) {
          if (sh.status == COOP_OK) sh.status = COOP_ERR_UNSATISFIABLE;
          sh.res.fail_op = sh.cur_op;
        }
        __syncthreads();
        return;
      }
      i = find_fit(need, right);  // the unique coalesced block >= need
      at = place(i, need, right, t);
      if (!ok()) return;
      int nfree = 0;
      for (int b = threadIdx.x; b < sh.nb; b += kThreads) nfree += (O()[b] == kFree);
      nfree = cta_sum_i32(sh, nfree);
      if (threadIdx.x == 0) {
        sh.res.sum_free_bytes_after += sh.bytes_free;  // R27
        sh.res.sum_free_blocks_after += nfree;
      }
    } else {
      at = place(i, need, right, t);
      if (!ok()) return;
    }
    if (threadIdx.x == 0) {
      w.taddr[t] = at;
      sh.tfl[t] |= TF_RES;
      log_ev(kind, op, t, at);
    }
    __syncthreads();
  }

  // ---------------------------------------------------------------- rematerialization
  // M(t): explicit stack (R21-R23); a dead tensor recomputed here stays resident until
  // the end of the current trace op (R22).
  // stack frame field (0 tensor, 1 stage, 2 next input to check, 3 depth): shared memory for
  // the bottom kRsm frames, the workspace beyond
  __device__ __forceinline__ int32_t &rs(int field, int f) {
    return f < kRsm ? sh.rsm[field][f] : w.rst[field * kStackCap + f];
  }
  __device__ void materialize(int t0) {
    if (threadIdx.x == 0) {
      sh.sp = 1;
      rs(0, 0) = t0;
      rs(1, 0) = 0;
      rs(2, 0) = 0;
      rs(3, 0) = 0;
    }
    __syncthreads();
    while (sh.sp > 0 && ok()) {
      const int f = sh.sp - 1;
      const int t = rs(0, f), depth = rs(3, f), stage = rs(1, f);
      const int op = ldg_if<kRO>(&tr.producer[t]);
      if (stage == 0) {
        __syncthreads();
        if (threadIdx.x == 0) {
          if (depth > a.max_depth) {
            sh.status = COOP_ERR_THRASHED;  // R23
            sh.res.fail_op = sh.cur_op;
          } else if (op < 0) {
            sh.status = COOP_ERR_UNSATISFIABLE;
            sh.res.fail_op = sh.cur_op;
          } else {
            if (depth > sh.res.max_depth) sh.res.max_depth = depth;
            rs(1, f) = 1;
          }
        }
        __syncthreads();
        if (!ok()) return;
        for (int j = threadIdx.x; j < nin(op); j += kThreads) atomicAdd(&w.pins[in_at(op, j)], 1);
        __syncthreads();
        continue;
      }
      if (stage == 1) {
        // the first input at or after the frame's cursor that is not resident: warp 0 checks
        // 32 inputs at a time (inputs before the cursor were made resident and are pinned)
        __syncthreads();
        if (threadIdx.x < 32) {
          const int n = nin(op), ib = ldg_if<kRO>(&tr.in_ptr[op]);
          int j = rs(2, f);
          while (j < n) {
            const int jj = j + (int)threadIdx.x;
            const bool miss = jj < n && !(sh.tfl[ldg_if<kRO>(&tr.in_idx[ib + jj])] & TF_RES);
            const uint32_t bal = __ballot_sync(0xffffffffu, miss);
            if (bal) {
              j += __ffs(bal) - 1;
              break;
            }
            j += 32;
          }
          if (threadIdx.x == 0) {
            if (j < n) {
              rs(2, f) = j + 1;
              if (sh.sp >= kStackCap) {
                sh.status = COOP_ERR_THRASHED;
                sh.res.fail_op = sh.cur_op;
              } else {
                const int g = sh.sp++;
                rs(0, g) = ldg_if<kRO>(&tr.in_idx[ib + j]);
                rs(1, g) = 0;
                rs(2, g) = 0;
                rs(3, g) = depth + 1;
              }
            } else {
              rs(1, f) = 2;
            }
          }
        }
        __syncthreads();
        continue;
      }
      // stage 2: recompute t out-of-place (R21)
      allocate(op, t, false, 5);
      if (!ok()) return;
      __syncthreads();
      if (threadIdx.x == 0) {
        sh.clock += tr.cost[op];
        sh.res.total_us += tr.cost[op];
        sh.res.remat++;
        log_ev(7, op, t, w.taddr[t]);
        if (sh.tfl[t] & TF_DEAD) {
          if (sh.ntrans < 4 * tr.T) w.trans[sh.ntrans++] = t;
          else sh.status = COOP_ERR_NOMEM;
        }
        sh.sp--;
      }
      __syncthreads();
      const int64_t clk = sh.clock;
      for (int j = threadIdx.x; j < nin(op); j += kThreads) {
        const int u = in_at(op, j);
        w.last_access[u] = clk;
        atomicSub(&w.pins[u], 1);
      }
      if (threadIdx.x == 0) w.last_access[t] = clk;
      __syncthreads();
    }
  }

  // Stage the records of ops [k0, k0 + kOpChunk) and their lists into shared memory: two
  // rounds of independent loads by all threads instead of a dozen dependent L2 round
  // trips per op in the op loop.  Called by every thread; ends with a barrier.
  __device__ void stage_ops(int k0) {
    const int M = tr.M;
    const int nk = min(kOpChunk, M - k0);
    __syncthreads();  // the previous chunk is no longer read
    for (int i = threadIdx.x; i < nk; i += kThreads) {
      const int k = k0 + i;
      OpRec r;
      r.in_beg = tr.in_ptr[k];
      r.in_end = tr.in_ptr[k + 1];
      r.die_beg = tr.die_ptr[k];
      r.die_end = tr.die_ptr[k + 1];
      r.lock_beg = tr.lock_ptr[k];
      r.lock_end = tr.lock_ptr[k + 1];
      r.out = tr.out[k];
      r.src = tr.src[k];
      r.cost = tr.cost[k];
      r.out_size = tr.size[r.out];
      r.right = goes_right(k) ? 1 : 0;
      r.pad = 0;
      sh.ops[i] = r;
    }
    if (threadIdx.x == 0) {
      sh.op_base = k0;
      const int ke = k0 + nk;
      sh.l_in0 = tr.in_ptr[k0];
      sh.l_in1 = min(tr.in_ptr[ke], sh.l_in0 + kListCap);
      sh.l_die0 = tr.die_ptr[k0];
      sh.l_die1 = min(tr.die_ptr[ke], sh.l_die0 + kListCap);
      sh.l_lock0 = tr.lock_ptr[k0];
      sh.l_lock1 = min(tr.lock_ptr[ke], sh.l_lock0 + kListCap);
    }
    __syncthreads();
    for (int j = sh.l_in0 + threadIdx.x; j < sh.l_in1; j += kThreads) sh.lin[j - sh.l_in0] = tr.in_idx[j];
    for (int j = sh.l_die0 + threadIdx.x; j < sh.l_die1; j += kThreads) {
      const int t = tr.die_idx[j];
      sh.ldie[j - sh.l_die0] = t;
      sh.ldie_unev[j - sh.l_die0] = ldg_if<kRO>(&tr.unevict[t]);
    }
    for (int j = sh.l_lock0 + threadIdx.x; j < sh.l_lock1; j += kThreads) sh.llock[j - sh.l_lock0] = tr.lock_idx[j];
    __syncthreads();
  }
  __device__ __forceinline__ int st_in(int j) const { return j < sh.l_in1 ? sh.lin[j - sh.l_in0] : tr.in_idx[j]; }
  __device__ __forceinline__ int st_die(int j) const { return j < sh.l_die1 ? sh.ldie[j - sh.l_die0] : tr.die_idx[j]; }
  __device__ __forceinline__ bool st_die_unev(int j) const {
    return j < sh.l_die1 ? sh.ldie_unev[j - sh.l_die0] : ldg_if<kRO>(&tr.unevict[tr.die_idx[j]]);
  }
  __device__ __forceinline__ int st_lock(int j) const { return j < sh.l_lock1 ? sh.llock[j - sh.l_lock0] : tr.lock_idx[j]; }

  // The second CTA of a cluster: at every pressure event of the leader (rank 0) it copies
  // the leader's tensor flags through distributed shared memory and walks work items from
  // the leader's counter with its own walkers, bitmaps and graph copy; both CTAs' sums land
  // in the cell's w.pacc.  Ends when the leader posts the exit command.
  __device__ void cluster_helper() {
    cooperative_groups::cluster_group cl = cooperative_groups::this_cluster();
    Shared *lead = cl.map_shared_rank(&sh, 0);
    wcnt = &lead->cand_next;
    while (true) {
      cl.sync();  // A
      const int cmd = lead->helper_cmd;
      if (cmd != 1) {
        cl.sync();  // the leader keeps its shared memory until this read is done
        break;
      }
      const int ncand = lead->ncand;
      {  // the leader's residency / liveness flags (16-byte copies)
        const uint4 *src = reinterpret_cast<const uint4 *>(lead->tfl);
        uint4 *dst = reinterpret_cast<uint4 *>(sh.tfl);
        for (int i = threadIdx.x; i < a.tfl_bytes / 16; i += kThreads) dst[i] = src[i];
      }
      __syncthreads();
      walk_items(nullptr, ncand);
      cl.sync();  // B
    }
  }

  // ---------------------------------------------------------------- the op loop
  __device__ void run(uint64_t budget) {
    const int T = tr.T, M = tr.M;
    for (int t = threadIdx.x; t < T; t += kThreads) {
      sh.tfl[t] = 0;
      w.pins[t] = 0;
      w.last_access[t] = 0;
      w.taddr[t] = 0;
    }
    if (threadIdx.x == 0) {
      sh.nb = 1;
      sh.addr[0] = 0;
      sh.size[0] = budget;
      sh.owner[0] = kFree;
      sh.bytes_free = budget;
      sh.clock = 0;
      sh.status = COOP_OK;
      sh.cur_op = -1;
      sh.redpar = 0;
      memset(&sh.res, 0, sizeof(sh.res));
      sh.res.fail_op = -1;
      sh.res.digest = 0x9E3779B97F4A7C15ull;
      sh.res.budget = budget;
      sh.res.max_blocks = 1;
    }
    epoch = w.epochs[threadIdx.x];
    __syncthreads();
    // parameters to the two ends (R15)
    {
      uint64_t lb = 0, rb = 0;
      for (int j = 0; j < tr.n_params && ok(); ++j) {
        const int t = tr.params[j];
        const bool right = (a.flags & COOP_F_INPLACE) ? (rb < lb) : false;
        const int i = find_fit(tr.size[t], right);
        if (i < 0) {
          if (threadIdx.x == 0) sh.status = COOP_ERR_UNSATISFIABLE;
          __syncthreads();
          break;
        }
        const uint64_t at = place(i, tr.size[t], right, t);
        if (!ok()) break;
        if (right) rb += tr.size[t];
        else lb += tr.size[t];
        if (threadIdx.x == 0) {
          w.taddr[t] = at;
          sh.tfl[t] = TF_RES | TF_BORN;
          log_ev(0, -1, t, at);
        }
        __syncthreads();
      }
    }
    for (int k = 0; k < M && ok(); ++k) {
      if (k % kOpChunk == 0) stage_ops(k);
      const OpRec R = sh.ops[k - sh.op_base];
      const int n = R.in_end - R.in_beg, o = R.out, src = R.src;
      if (threadIdx.x == 0) sh.cur_op = k;  // read by thread 0 only
      for (int j = threadIdx.x; j < n; j += kThreads) atomicAdd(&w.pins[st_in(R.in_beg + j)], 1);
      for (int j = R.lock_beg + threadIdx.x; j < R.lock_end; j += kThreads)
        sh.tfl[st_lock(j)] |= TF_LOCK;  // R36
      __syncthreads();
      // reset after the barrier: every thread has read the previous op's count (racecheck)
      if (threadIdx.x == 0) sh.ntrans = 0;
      for (int j = 0; j < n && ok(); ++j) {
        const int u = st_in(R.in_beg + j);
        const bool res = sh.tfl[u] & TF_RES;
        __syncthreads();
        if (!res) materialize(u);
      }
      for (int j = R.lock_beg; j < R.lock_end && ok(); ++j) {
        const int u = st_lock(j);
        const bool res = sh.tfl[u] & TF_RES;
        __syncthreads();
        if (!res) materialize(u);
      }
      if (!ok()) break;
      allocate_with(k, o, R.out_size, src, R.right != 0, true, 1);
      if (!ok()) break;
      if (threadIdx.x == 0) {
        sh.tfl[o] |= TF_BORN;
        sh.clock += R.cost;
        sh.res.base_us += R.cost;
        sh.res.total_us += R.cost;
        log_ev(6, k, o, w.taddr[o]);
      }
      __syncthreads();
      const int64_t clk = sh.clock;
      for (int j = threadIdx.x; j < n; j += kThreads) {
        const int u = st_in(R.in_beg + j);
        w.last_access[u] = clk;
        atomicSub(&w.pins[u], 1);
      }
      if (threadIdx.x == 0) w.last_access[o] = clk;
      __syncthreads();
      // deaths after op k (R20) merged with transient dead recomputes (R22), ascending id
      if (threadIdx.x == 0) {
        for (int j = R.die_beg; j < R.die_end; ++j) sh.tfl[st_die(j)] |= TF_DEAD;
        // insertion-sort the transient list (small) and merge with the (sorted) die list
        int *tl = w.trans;
        const int nt = sh.ntrans;
        for (int x = 1; x < nt; ++x) {
          const int v = tl[x];
          int y = x - 1;
          while (y >= 0 && tl[y] > v) { tl[y + 1] = tl[y]; --y; }
          tl[y + 1] = v;
        }
      }
      __syncthreads();
      {
        int pd = R.die_beg;
        const int pe = R.die_end;
        int pt = 0;
        const int nt = sh.ntrans;
        int last = -1;
        while (pd < pe || pt < nt) {
          int t;
          bool unev;
          if (pt >= nt || (pd < pe && st_die(pd) <= w.trans[pt])) {
            unev = st_die_unev(pd);
            t = st_die(pd++);
          } else {
            t = w.trans[pt++];
            unev = ldg_if<kRO>(&tr.unevict[t]);
          }
          if (t == last) continue;
          last = t;
          const uint8_t f = sh.tfl[t];
          const bool keep = unev && t != src;
          __syncthreads();
          if ((f & TF_DEAD) && (f & TF_RES) && !keep) free_tensor(t);
        }
      }
    }
    if (threadIdx.x == 0) {
      sh.res.status = sh.status;
      if (sh.status != COOP_OK && sh.res.fail_op < 0 && sh.cur_op >= 0) sh.res.fail_op = sh.cur_op;
    }
    w.epochs[threadIdx.x] = epoch;
    __syncthreads();
  }
};

// Per-cell workspace layout for T tensors (host).
WsLayout make_layout(int T) {
  WsLayout L{};
  size_t o = 0;
  auto take = [&](size_t bytes) {
    size_t r = o;
    o = (o + bytes + 255) / 256 * 256;
    return r;
  };
  L.tflags = take((size_t)T);
  L.pins = take((size_t)T * 4);
  L.last_access = take((size_t)T * 8);
  L.taddr = take((size_t)T * 8);
  L.epochs = take((size_t)kThreads * 4);
  L.marks = take((size_t)kThreads * ((T + 15) & ~15));  // one byte per tensor and thread
  L.stack = take((size_t)kMaxCluster * kThreads * T * 4);  // one set of stacks per CTA of a cluster
  L.isz = take((size_t)(kCap + 1) * 8);
  L.ih = take((size_t)(kCap + 1) * 8);
  L.ist = take((size_t)(kCap + 1));
  L.S = take((size_t)(kCap + 1 + kThreads) * 8);
  L.H = take((size_t)(kCap + 1 + kThreads) * sizeof(U192));
  L.B = take((size_t)(kCap + 1 + kThreads) * 4);
  L.trans = take((size_t)T * 4 * 4);
  L.victims = take((size_t)kCap * 4);
  L.cand = take((size_t)(kCap + 2) * 4);
  L.pacc = take((size_t)(kCap + 2) * 2 * 8);
  L.rst = take((size_t)4 * kStackCap * 4);
  L.vc = take((size_t)(kCap + 2) * 8);
  L.vs = take((size_t)(kCap + 2) * 8);
  L.ctid = take((size_t)(kCap + 2) * 4);
  L.bytes = o;
  return L;
}

}  // namespace
}  // namespace coop

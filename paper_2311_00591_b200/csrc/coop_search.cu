// coop_search.cu -- batched sliding-window eviction search for sm_100a.
//
// Computes, for each pool, the window of Eq. 1 as found by the Sec. 3.3
// sliding window: the contiguous, PINNED-free run of items with
// span >= R and the minimum correctly rounded exact sum of h = c/s (R1-R7).
//
// Design ("Batched search"):
//   * persistent CTAs (two 256-thread CTAs per SM at N = 4096) loop over pools in rotated
//     rounds (the second CTA of an SM in pair-swapped order, so the two alternate short- and
//     long-request pools); one shared-memory stage per CTA is filled by TMA
//     (cp.async.bulk.tensor, SWIZZLE_128B) while the other CTA of the SM computes; thread t
//     owns K items;
//   * phase 1 (every pool): state codes, R7 validation from the binary64 encodings (the exact
//     division only for the rare items the exponents cannot clear), local prefixes of span
//     (u64) and of an approximate h^ = c * rcp(s) (fp64), warp scans;
//   * zero pass: a run of h = 0 items covering R is exactly optimal (lowest head wins);
//     short-request pools end here;
//   * phase 2 + B (the others): S and H^ completed in place; chunk pruning from one
//     bisection per thread; the surviving starts' ends by galloping and an fp64 filter
//     C^(i) = H^[e] - H^[i] with a rigorous error bound (sums of nonnegative terms);
//   * every start whose lower bound can reach the minimum is re-summed EXACTLY (h = c/s by
//     IEEE division, 192-bit fixed point, fixed192.cuh) and rounded once -- from global
//     memory, after the stage has been released; winner = lexicographic min of (rounded
//     cost, first index) -- bit-identical to the oracle.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <stdint.h>
#include <stdio.h>
#include <string.h>

#include "coop.h"
#include "coop_internal.h"
#include "fixed192.cuh"

namespace coop {

namespace {

#ifdef COOP_SEARCH_PHASE_HOOKS
constexpr bool kPhaseHooks = true;  // COOP_SEARCH_DBG = 3..6 (profiling builds only)
#else
constexpr bool kPhaseHooks = false;
#endif
constexpr int kCandCap = 512;  // fits two 512-thread CTAs (one stage each) per SM at N = 4096
constexpr int kMaxWarps = 16;
constexpr int kDefMax = 16;  // candidates a deferred re-summation takes
constexpr uint64_t kRClamp = 1ull << 62;  // any R > sum of sizes (< 2^61) is infeasible
constexpr int kInfIdx = 0x7fffffff;
constexpr uint64_t kSizeMask = (1ull << 62) - 1ull;

struct Scratch {
  uint64_t wS[kMaxWarps];
  double wH[kMaxWarps];
  double wU[kMaxWarps];
  double wP[kMaxWarps];  // chunk-pruning upper bounds
  int32_t wF[kMaxWarps];
  int32_t wZ[kMaxWarps];
  uint64_t part[2][kMaxWarps][3];                         // verification partial sums
  int32_t zW[kMaxWarps], zM[kMaxWarps], zW2[kMaxWarps];  // zero-pass reductions
  int32_t partn[2][kMaxWarps];
  uint64_t pspan[2][kMaxWarps];
  uint64_t bcost[kMaxWarps];
  int32_t bfirst[kMaxWarps];
  int32_t bend[kMaxWarps];
  int32_t bnev[kMaxWarps];
  int32_t ncand;
  int32_t nsurv;      // surviving chunks in the list (phase B1)
  uint16_t evc[kMaxWarps * 32];  // per chunk: EVICTABLE mask (exact re-summation, n_evict)
  uint32_t cand[kCandCap];
  unsigned long long mbar[2];
  // deferred exact re-summations (two slots: the newest and an older one): pool (-1: none),
  // candidate count and windows; dnext = the slot the next deferral uses
  int32_t swap;  // 1: this CTA visits its rounds in pair-swapped order (k = j ^ 1)
  int64_t dpool[2];
  int32_t dnc[2], dnext;
  uint32_t dcand[2][kDefMax];
  uint64_t dspan[2][kDefMax];
  int32_t nplist;                      // pending mode: pools of the chunk to finish
  int16_t plist[kMaxWarps * 32];
};

// per-SM launch counters: which of the two CTAs on an SM this one is (see the round order in
// search_kernel; a wrong guess only costs balance, never correctness)
__device__ unsigned int g_smcnt[1024];

struct Args {
  const uint64_t *ss;
  const double *cost;
  const double *stale;
  const uint64_t *req;
  coop_window *out;
  int64_t n_pools;
  int64_t stride;
  int32_t n;
  int32_t box_rows;
  int32_t n_boxes;
  uint32_t region_bytes;
  uint32_t stage_bytes;
  int32_t stages;
  int32_t use_tma;
  int32_t pending;  // finish only the pools the streaming kernel marked COOP_PENDING_
  int32_t dbg;  // profiling hook (COOP_SEARCH_DBG): stop each pool after 1 = load, 2 = phase 1;
                // with -DCOOP_SEARCH_PHASE_HOOKS also 4 = zero pass, 3 = phase 2, 5 = pruning +
                // compaction, 6 = filter + reductions
  double gerr;  // filter error coefficient: |C^ - C| <= gerr * (H^[e] + H^[i])
};

__device__ __forceinline__ uint32_t swz(uint32_t k) {  // item k -> byte offset, SWIZZLE_128B
  uint32_t off = k * 8u;
  return off ^ (((off >> 7) & 7u) << 4);
}

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

// Shared-memory accessors: plain C++ loads/stores on pointers derived from the
// extern __shared__ array (the compiler emits LDS/STS and may schedule them freely;
// TMA-written data is ordered by the "memory" clobber of the mbarrier wait).
typedef unsigned char smem_t;
template <class T>
__device__ __forceinline__ T &sm(smem_t *base, uint32_t off) {
  return *reinterpret_cast<T *>(base + off);
}

// ---- mbarrier / TMA -------------------------------------------------------------
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(bar),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
// CTA barriers (named barrier 1, T threads).
__device__ __forceinline__ void cbar(int T) { asm volatile("bar.sync 1, %0;" ::"r"(T) : "memory"); }
__device__ __forceinline__ int cbar_or(int pred, int T) {
  int r;
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.s32 p, %1, 0;\n\t"
      "bar.red.or.pred p, 1, %2, p;\n\tselp.s32 %0, 1, 0, p;\n\t}"
      : "=r"(r)
      : "r"(pred), "r"(T)
      : "memory");
  return r;
}
__device__ __forceinline__ void tma_load_3d(uint32_t dst, const CUtensorMap *map, int c0, int c1,
                                            int c2, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(dst),
      "l"((uint64_t)map), "r"(c0), "r"(c1), "r"(c2), "r"(bar)
      : "memory");
}

__device__ __forceinline__ void issue_stage(const Args &a, const CUtensorMap *m_ss,
                                            const CUtensorMap *m_c, const CUtensorMap *m_s,
                                            uint32_t stage_base, uint32_t bar, int64_t p) {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  mbar_expect_tx(bar, 3u * (uint32_t)a.n_boxes * (uint32_t)a.box_rows * 128u);
  for (int b = 0; b < a.n_boxes; ++b) {
    uint32_t off = (uint32_t)b * (uint32_t)a.box_rows * 128u;
    tma_load_3d(stage_base + off, m_ss, 0, b * a.box_rows, (int)p, bar);
    tma_load_3d(stage_base + a.region_bytes + off, m_c, 0, b * a.box_rows, (int)p, bar);
    tma_load_3d(stage_base + 2u * a.region_bytes + off, m_s, 0, b * a.box_rows, (int)p, bar);
  }
}

// Fallback staging for layouts the TMA map cannot describe (plain coalesced loads).
__device__ __forceinline__ void stage_plain(const Args &a, smem_t *stage, int64_t p, int T) {
  const int64_t base = p * a.stride;
  for (int k = threadIdx.x; k < a.n; k += T) {
    const uint32_t o = swz((uint32_t)k);
    sm<uint64_t>(stage, o) = a.ss[base + k];
    sm<double>(stage, a.region_bytes + o) = a.cost[base + k];
    sm<double>(stage, 2u * a.region_bytes + o) = a.stale[base + k];
  }
}

__device__ __forceinline__ void write_result(coop_window *o, int32_t first, int32_t last,
                                             uint64_t span, double cost, int32_t nev,
                                             int32_t status) {
  coop_window w;
  w.first = first;
  w.last = last;
  w.span = span;
  w.cost = cost;
  w.n_evict = nev;
  w.status = status;
  *o = w;
}


// Warp reductions on the REDUX unit (one instruction per 32-bit step).  Doubles are reduced
// through their total-order keys (monotone in the value for every non-NaN binary64).
__device__ __forceinline__ int wmin_i32(int x) { return __reduce_min_sync(0xffffffffu, x); }
__device__ __forceinline__ uint64_t wmin_u64(uint64_t x) {
  const uint32_t xh = (uint32_t)(x >> 32);
  const uint32_t hi = __reduce_min_sync(0xffffffffu, xh);
  const uint32_t lo = __reduce_min_sync(0xffffffffu, xh == hi ? (uint32_t)x : 0xffffffffu);
  return ((uint64_t)hi << 32) | lo;
}
__device__ __forceinline__ uint64_t dkey(double d) {
  const uint64_t b = (uint64_t)__double_as_longlong(d);
  return (int64_t)b < 0 ? ~b : (b | 0x8000000000000000ull);
}
__device__ __forceinline__ double dunkey(uint64_t k) {
  return __longlong_as_double((long long)((int64_t)k < 0 ? (k & 0x7fffffffffffffffull) : ~k));
}
__device__ __forceinline__ double wmin_f64(double x) { return dunkey(wmin_u64(dkey(x))); }

__device__ __forceinline__ U192 warp_sum192(U192 acc, int &nev) {
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) {
    U192 o;
    o.w0 = __shfl_xor_sync(0xffffffffu, acc.w0, d);
    o.w1 = __shfl_xor_sync(0xffffffffu, acc.w1, d);
    o.w2 = __shfl_xor_sync(0xffffffffu, acc.w2, d);
    nev += __shfl_xor_sync(0xffffffffu, nev, d);
    acc = u192_add(acc, o);
  }
  return acc;
}

__device__ __forceinline__ bool better(uint64_t cb, int i, uint64_t bb, int bi) {
  return cb < bb || (cb == bb && i < bi);
}

// Per-pool view in shared memory after phase 1 (region = one TMA-staged array):
//   region 0: S[k]   exclusive span prefix, k in [0, n]; S[n] = total span, S[n+1] = ~0
//   region 1: c[k]   as staged (the exact re-summation divides it again)
//   region 2: H^[k]  fp64 prefix of the approximate h^ (chunk-local until phase 2)
//   list[c]          (uint4, scratch) surviving chunks of the pruning pass (phase B1)
//   evc[t]           EVICTABLE mask of chunk t
struct PoolView {
  smem_t *sr, *cr, *hr;
  uint4 *list;
  const uint16_t *evc;
  const double *sg;  // this pool's staleness s in global memory (exact re-summation only)
  int32_t n;
  uint64_t R;
  double gerr;

  __device__ __forceinline__ uint64_t S_at(int x) const { return sm<uint64_t>(sr, swz((uint32_t)x)); }
  __device__ __forceinline__ double H_at(int x) const { return sm<double>(hr, swz((uint32_t)x)); }
  __device__ __forceinline__ double c_at(int x) const { return sm<double>(cr, swz((uint32_t)x)); }
};

// 1/s for s in [1, 2^960): the MUFU approximation and two Newton steps (relative error a few
// ulps; the filter's bound allows 2^-44 per h^)
__device__ __forceinline__ double rcp_nr(double s) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(s));
  double e = __fma_rn(-s, r, 1.0);
  r = __fma_rn(r, e, r);
  e = __fma_rn(-s, r, 1.0);
  return __fma_rn(r, e, r);
}

// Exact cost of the window [i, e) of pool p (R3): h = c/s (IEEE RN, R1) of its EVICTABLE
// items -- FREE items add 0, a window never holds a PINNED one -- summed in 192-bit fixed
// point over the items i + off, i + off + step, ...; also the EVICTABLE count (n_evict) and
// the span.  SMEM = false: everything from global memory (deferred re-summations: the stage
// holds another pool by then; the lines were prefetched into L1); SMEM = true: exact h from
// region 1 (converted in place by exact_h_in_place) and the states from the chunk masks.
template <bool SMEM, bool GSPAN, int K>
__device__ __forceinline__ void window_sum(const Args &a, const PoolView *v, const uint16_t *evc, int64_t p,
                                           int i, int e, int off, int step, U192 &acc,
                                           uint64_t &span, int &nev) {
  const uint64_t *ss = a.ss + p * a.stride;
  const double *cg = a.cost + p * a.stride, *sg = a.stale + p * a.stride;
  for (int k = i + off; k < e; k += step) {
    if (GSPAN) span += __ldg(ss + k) & kSizeMask;
    if ((evc[k / K] >> (k % K)) & 1u) {  // EVICTABLE (the chunk masks of this pool)
      acc = u192_add(acc, u192_from_double(SMEM ? v->c_at(k) : __ddiv_rn(__ldg(cg + k), __ldg(sg + k))));
      ++nev;
    }
  }
}

__device__ __forceinline__ void warp_sum_all(U192 &acc, uint64_t &span, int &nev) {
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) {
    acc = u192_add(acc, U192{__shfl_xor_sync(0xffffffffu, acc.w0, d), __shfl_xor_sync(0xffffffffu, acc.w1, d),
                             __shfl_xor_sync(0xffffffffu, acc.w2, d)});
    span += __shfl_xor_sync(0xffffffffu, span, d);
    nev += __shfl_xor_sync(0xffffffffu, nev, d);
  }
}

// The exact re-summation of the candidate windows sc.cand[0, nc) of pool p by the whole CTA
// and the pool's result: the lexicographic (rounded exact cost bits, first) minimum.
// spans: the candidates' spans when known (taken from S before the stage was released), else
// summed from the global size words
template <bool SMEM, int K>
__device__ __forceinline__ void verify_pool(const Args &a, const PoolView *v, Scratch &sc, int64_t p,
                                            const uint32_t *cand, const uint64_t *spans, int nc, int T) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, W = T >> 5;
  uint64_t best = ~0ull, bspan = 0;  // meaningful in thread 0
  int bfirst = kInfIdx, bend = -1, bnev = 0;
  if (nc <= W) {
    // few candidates: the whole CTA sums each window (short latency chain)
    for (int c = 0; c < nc; ++c) {
      const uint32_t cd = cand[c];
      const int i = (int)(cd >> 16), e = i + (int)(cd & 0xffffu);
      U192 acc = u192_zero();
      uint64_t span = 0;
      int nev = 0;
      if (i + warp * 32 < e) {  // warp-uniform: warps without items skip
        if (spans) window_sum<SMEM, false, K>(a, v, sc.evc, p, i, e, tid, T, acc, span, nev);
        else window_sum<SMEM, true, K>(a, v, sc.evc, p, i, e, tid, T, acc, span, nev);
        warp_sum_all(acc, span, nev);
      }
      const int par = c & 1;
      if (lane == 0) {
        sc.part[par][warp][0] = acc.w0;
        sc.part[par][warp][1] = acc.w1;
        sc.part[par][warp][2] = acc.w2;
        sc.partn[par][warp] = nev;
        sc.pspan[par][warp] = span;
      }
      cbar(T);
      if (warp == 0) {
        U192 t = u192_zero();
        uint64_t tsp = 0;
        int tn = 0;
        if (lane < W) {
          t.w0 = sc.part[par][lane][0];
          t.w1 = sc.part[par][lane][1];
          t.w2 = sc.part[par][lane][2];
          tn = sc.partn[par][lane];
          tsp = sc.pspan[par][lane];
        }
        warp_sum_all(t, tsp, tn);
        const uint64_t cb = (uint64_t)__double_as_longlong(u192_round_to_double(t));
        if (lane == 0 && better(cb, i, best, bfirst)) {
          best = cb;
          bfirst = i;
          bend = e;
          bnev = tn;
          bspan = spans ? spans[c] : tsp;
        }
      }
    }
  } else {
    // many candidates: one warp per candidate window
    uint64_t wbest = ~0ull, wspan = 0;
    int32_t wfirst = kInfIdx, wend = -1, wnev = 0;
    for (int c = warp; c < nc; c += W) {
      const uint32_t cd = cand[c];
      const int i = (int)(cd >> 16), e = i + (int)(cd & 0xffffu);
      U192 acc = u192_zero();
      uint64_t span = 0;
      int nev = 0;
      if (spans) window_sum<SMEM, false, K>(a, v, sc.evc, p, i, e, lane, 32, acc, span, nev);
      else window_sum<SMEM, true, K>(a, v, sc.evc, p, i, e, lane, 32, acc, span, nev);
      warp_sum_all(acc, span, nev);
      const uint64_t cb = (uint64_t)__double_as_longlong(u192_round_to_double(acc));
      if (better(cb, i, wbest, wfirst)) {
        wbest = cb;
        wfirst = i;
        wend = e;
        wnev = nev;
        wspan = spans ? spans[c] : span;
      }
    }
    if (lane == 0) {
      sc.bcost[warp] = wbest;
      sc.bfirst[warp] = wfirst;
      sc.bend[warp] = wend;
      sc.bnev[warp] = wnev;
      sc.pspan[0][warp] = wspan;
    }
    cbar(T);
    if (tid == 0) {
      for (int w = 0; w < W; ++w) {
        if (sc.bend[w] >= 0 && better(sc.bcost[w], sc.bfirst[w], best, bfirst)) {
          best = sc.bcost[w];
          bfirst = sc.bfirst[w];
          bend = sc.bend[w];
          bnev = sc.bnev[w];
          bspan = sc.pspan[0][w];
        }
      }
    }
  }
  if (tid == 0) {
    if (SMEM) bspan = v->S_at(bend) - v->S_at(bfirst);
    write_result(a.out + p, bfirst, bend - 1, bspan, __longlong_as_double((long long)best), bnev, COOP_OK);
  }
  cbar(T);  // the candidate list / sc.part free again
}

// Per-thread running state of the filter.
struct LaneBest {
  double U, L, L2;  // min upper bound, min / second-min lower bound
  int li, le;       // the start with the minimal lower bound and its end
};

// A surviving chunk (phase B1): x = k0 | elo << 16 (elo <= e(i) for every start of the
// chunk), y = PINNED mask of its K items, z = first PINNED index to the right of the chunk.
__device__ __forceinline__ uint4 chunk_rec(int k0, int elo, uint32_t barmask, int nb_right) {
  return make_uint4((uint32_t)k0 | ((uint32_t)elo << 16), barmask, (uint32_t)nb_right, 0u);
}

// The filter for start i = k0 + q of a surviving chunk, run by any thread: window end by a
// galloping search from elo, PINNED check from the chunk mask, and the fp64 prefix difference
// C^ = H^[e] - H^[i] with its bound |C^ - C| <= gerr (H^[e] + H^[i]).  MODE 0 folds the start
// into LaneBest; MODE 1 appends it to the candidate list when its lower bound is <= thresh
// and i lies in [w_lo, w_hi).
template <int MODE>
__device__ __forceinline__ void eval_start(const PoolView &v, const uint4 rec, int q, double thresh,
                                           int w_lo, int w_hi, Scratch &sc, LaneBest &b) {
  const int n = v.n;
  const int k0 = (int)(rec.x & 0xffffu), elo = (int)(rec.x >> 16);
  const uint32_t barmask = rec.y;
  const int i = k0 + q;
  if (i >= n || ((barmask >> q) & 1u)) return;
  const uint64_t target = v.S_at(i) + v.R;  // < 2^63
  int lo = max(elo, i + 1), e;
  if (v.S_at(lo) >= target) {
    e = lo;
  } else {  // S[lo] < target <= S[n + 1] = ~0: gallop, then bisect (lo, hi]
    int step = 1, hi = min(lo + 1, n + 1);
    while (v.S_at(hi) < target) {
      lo = hi;
      step <<= 1;
      hi = min(lo + step, n + 1);
    }
    ++lo;
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (v.S_at(mid) >= target) hi = mid;
      else lo = mid + 1;
    }
    e = hi;
  }
  if (e > n) return;  // no window covers R from i (nor from any later start)
  const uint32_t mb = barmask >> q;
  const int nb = mb ? i + __ffs(mb) - 1 : (int)rec.z;
  if (nb < e) return;  // a PINNED item inside [i, e-1]
  const double He = v.H_at(e), Hi = v.H_at(i);
  const double C = He - Hi;
  const double err = v.gerr * (He + Hi);
  const double Lb = C - err;
  if (MODE == 0) {
    b.U = fmin(b.U, C + err);
    if (Lb < b.L) {
      b.L2 = b.L;
      b.L = Lb;
      b.li = i;
      b.le = e;
    } else {
      b.L2 = fmin(b.L2, Lb);
    }
  } else if (Lb <= thresh && i >= w_lo && i < w_hi) {
    const int slot = atomicAdd(&sc.ncand, 1);
    if (slot < kCandCap) sc.cand[slot] = ((uint32_t)i << 16) | (uint32_t)(e - i);  // n <= 8192
  }
}

// Phase 1 of one thread (every pool): decode its K items (pairs via 16-byte conflict-free
// loads of the swizzled stage), local exclusive prefixes of span (u64) and of the
// approximate h^ = c * rcp(s) (fp64; stored over s, which is not read again from shared
// memory), a 2-bit state code per item, and the R7 checks WITHOUT a division: for c > 0
// normal and s >= 1, c/s lies in (2^(d-1), 2^(d+1)) with d the exponent difference of c and
// s, and hi(c) - hi(s) lies in ((d-1) 2^20, (d+1) 2^20), so hi(c) - hi(s) in
// [-62 2^20, 58 2^20) gives d in [-62, 58] and RN(c/s) inside [2^-64, 2^60), nonzero (s is
// held to [1, 2^960), so c = +-0 or a negative or non-finite c falls outside the band too).
// An EVICTABLE item outside that clear range sets `oor`, and settle_chunk() then re-decides
// the chunk with the oracle's own comparisons and the exact division (h = 0 items included).
// FULL: no item past n.
//   st2: bits 2j..2j+1 = state of item j (padding: FREE); badbits: size bits 48..61 of
//   some item; zsize: some live item has size 0.
template <int K, bool FULL>
__device__ __forceinline__ void phase1(const PoolView &v, int k0, int n, uint32_t &st2,
                                       uint32_t &badbits, bool &zsize, bool &oor,
                                       uint64_t (&spre)[K], uint64_t &sacc, double &hacc) {
#pragma unroll
  for (int q = 0; q < K; q += 2) {
    const int k = k0 + q;
    const uint32_t o = swz((uint32_t)k);
    ulonglong2 vs = make_ulonglong2(0, 0);
    double2 vc = make_double2(0.0, 0.0), vt = make_double2(1.0, 1.0);
    if (FULL || k < n) {
      vs = sm<ulonglong2>(v.sr, o);
      vc = sm<double2>(v.cr, o);
      vt = sm<double2>(v.hr, o);
    }
    double hl[2];
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      const int j = q + r;
      const bool live = FULL || (k + r < n);
      const uint64_t sv = live ? (r ? vs.y : vs.x) : 0ull;  // padding: FREE, size 0
      const uint32_t slo = (uint32_t)sv, svh = (uint32_t)(sv >> 32);
      st2 |= (svh >> (30 - 2 * j)) & (3u << (2 * j));
      badbits |= svh & 0x3fff0000u;
      const uint32_t shi = svh & 0x3fffffffu;
      zsize |= live && (slo | shi) == 0u;
      spre[j] = sacc;
      sacc += ((uint64_t)shi << 32) | slo;
      // branch-free: h^ is formed for every item and kept for EVICTABLE ones only
      const double c = r ? vc.y : vc.x, s = r ? vt.y : vt.x;
      const uint32_t ch = (uint32_t)__double2hiint(c), sh = (uint32_t)__double2hiint(s);
      const bool ev = (svh >> 30) == COOP_EVICTABLE;
      // clear range: s in [1, 2^960) and hi(c) - hi(s) in [-62 2^20, 58 2^20); c = +-0,
      // negative, infinite or NaN (and every s outside the range) lands outside it too
      oor |= ev & (((sh - 0x3ff00000u) >= 0x3c000000u) | ((ch - sh + (62u << 20)) >= (120u << 20)));
      const double hq = c * rcp_nr(s);
      hl[r] = hacc;
      hacc = __dadd_rn(hacc, ev ? hq : 0.0);
    }
    if (FULL || k < n) sm<double2>(v.hr, o) = make_double2(hl[0], hl[1]);
  }
}

// The exact R7 tests (the oracle's comparisons; h = c/s) for a chunk with an
// EVICTABLE item phase 1 could not clear from the encodings: sets nz exactly and rebuilds the
// chunk's local h^ prefixes with exact h (s from global memory: the stage holds the prefixes).
struct Settled {
  uint32_t nz, bad;
  double hacc;
};
// (by value: a reference argument to a non-inlined call would keep the caller's PoolView and
// flags in local memory on every pool)
template <int K>
__device__ __noinline__ Settled settle_chunk(smem_t *cr, smem_t *hr, const double *sg, int n, int k0,
                                             uint32_t evm, uint32_t nz) {
  Settled r{nz, 0u, 0.0};
  double acc = 0.0;
  for (int q = 0; q < K && k0 + q < n; ++q) {
    const uint32_t o = swz((uint32_t)(k0 + q));
    double h = 0.0;
    if ((evm >> q) & 1u) {
      const double c = sm<double>(cr, o), s = sg[k0 + q];
      if (!isfinite(c) || !isfinite(s) || c < 0.0 || s < 1.0) {
        r.bad = 1u;
      } else {
        h = __ddiv_rn(c, s);
        if (h == 0.0) r.nz &= ~(1u << q);
        else if (h < 0x1p-64 || h >= 0x1p60) r.bad = 1u;
      }
    }
    sm<double>(hr, o) = acc;
    acc = __dadd_rn(acc, h);
  }
  r.hacc = acc;
  return r;
}

// bits 2j of x -> bit j (K <= 16)
__device__ __forceinline__ uint32_t even_bits(uint32_t x) {
  x &= 0x55555555u;
  x = (x | (x >> 1)) & 0x33333333u;
  x = (x | (x >> 2)) & 0x0f0f0f0fu;
  x = (x | (x >> 4)) & 0x00ff00ffu;
  return (x | (x >> 8)) & 0x0000ffffu;
}

// First item at or after chunk t's item q (q may be K) that is not an h = 0 item, using the
// published per-chunk zero masks (rare paths only); n if none.
__device__ int zero_run_stop(const uint16_t *zmk, int t, int q, int K, int n) {
  for (;; ++t, q = 0) {
    if (t * K >= n) return n;
    const uint32_t m = ~((uint32_t)zmk[t] >> q) & ((1u << (K - q)) - 1u);  // K - q >= 1 here
    if (q < K && m) return min(t * K + q + __ffs(m) - 1, n);
  }
}

// One pool of the CTA-per-pool search on its staged stage (called by every thread).
template <int K>
__device__ __forceinline__ void search_pool(const Args &a, Scratch &sc, uint4 *Ebuf, smem_t *stage,
                                            int64_t p, uint64_t Rraw) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int T = blockDim.x, W = T >> 5;
  const int n = a.n;
  const double kInf = __longlong_as_double(0x7ff0000000000000ll);
  constexpr uint32_t kFull = K == 32 ? ~0u : ((1u << K) - 1u);
  PoolView v;
  v.sr = stage;
  v.cr = stage + a.region_bytes;
  v.hr = stage + 2u * a.region_bytes;
  v.list = Ebuf;
  v.evc = sc.evc;
  v.sg = a.stale + p * a.stride;
  v.n = n;
  v.R = Rraw < kRClamp ? Rraw : kRClamp;
  v.gerr = a.gerr;
  const int k0 = tid * K;
  uint16_t *zmk16 = reinterpret_cast<uint16_t *>(Ebuf);  // per chunk: h = 0 item mask

  if (a.dbg == 1) {
    if (tid == 0) write_result(a.out + p, -1, -1, 0, 0.0, 0, COOP_OK);
    return;
  }
  // ---------------- phase 1: decode, validate (R7), span / h^ prefixes, masks --------------
  bool bad = (Rraw == 0), oor = false, zsize = false;
  uint32_t st2 = 0, badbits = 0;
  uint64_t spre[K];
  uint64_t sacc = 0;
  double hacc = 0.0;
  if (k0 + K <= n)  // warp-uniform except in the last warp
    phase1<K, true>(v, k0, n, st2, badbits, zsize, oor, spre, sacc, hacc);
  else
    phase1<K, false>(v, k0, n, st2, badbits, zsize, oor, spre, sacc, hacc);
  const uint32_t evmask = even_bits(st2 & ~(st2 >> 1));  // state 01
  const uint32_t barmask = even_bits((st2 >> 1) & ~st2);  // state 10
  uint32_t nzmask = evmask;  // EVICTABLE items in the clear range have h != 0
  bad |= (badbits != 0u) | zsize | ((st2 & (st2 >> 1) & 0x55555555u) != 0u);  // state 3
  if (oor) {
    const Settled st = settle_chunk<K>(v.cr, v.hr, v.sg, n, k0, evmask, nzmask);
    nzmask = st.nz;
    bad |= st.bad != 0u;
    hacc = st.hacc;
  }
  const int cnt = n - k0;
  const uint32_t valid = cnt >= K ? kFull : (cnt > 0 ? (1u << cnt) - 1u : 0u);
  const uint32_t zm = valid & ~barmask & ~nzmask;  // h = 0 items (FREE, or EVICTABLE with h = 0)
  sc.evc[tid] = (uint16_t)evmask;
  zmk16[tid] = (uint16_t)zm;

  // ---------------- warp scans: S (u64), H^ (fp64), next PINNED (suffix min) -------------
  uint64_t sinc = sacc;
  double hinc = hacc;
  int32_t fb = barmask ? k0 + __ffs(barmask) - 1 : kInfIdx;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const uint64_t so = __shfl_up_sync(0xffffffffu, sinc, d);
    const double ho = __shfl_up_sync(0xffffffffu, hinc, d);
    const int32_t bo = __shfl_down_sync(0xffffffffu, fb, d);
    if (lane >= d) {
      sinc += so;
      hinc = __dadd_rn(ho, hinc);
    }
    if (lane + d < 32) fb = min(fb, bo);
  }
  uint64_t sexc = __shfl_up_sync(0xffffffffu, sinc, 1);
  double hexc = __shfl_up_sync(0xffffffffu, hinc, 1);
  int32_t bexc = __shfl_down_sync(0xffffffffu, fb, 1);
  if (lane == 0) {
    sexc = 0;
    hexc = 0.0;
    sc.wF[warp] = fb;
  }
  if (lane == 31) {
    bexc = kInfIdx;
    sc.wS[warp] = sinc;
    sc.wH[warp] = hinc;
  }
  const int bad_any = cbar_or(bad, T);
  if (bad_any || a.dbg == 2) {
    if (tid == 0) write_result(a.out + p, -1, -1, 0, kInf, 0, bad_any ? COOP_ERR_INVALID_ARG : COOP_OK);
    return;
  }
  // ---------------- zero pass: zero-cost windows ----------------------------------------
  // A run of consecutive h = 0 items is a zero-cost window iff its span covers R; the lowest
  // such run head is the answer (exact cost 0 is the global minimum, R4).  The heads whose
  // own item covers R first (sizes from the raw words still in region 0); heads of runs that
  // go on past the head (never on the config-4 law) are settled below.
  const bool cont = (k0 + K < n) && (zmk16[tid + 1] & 1u);  // item k0 + K is h = 0
  const uint32_t heads = zm & ~(zm << 1);
  uint32_t one = 0;
  {
    uint32_t hm = heads;
    while (hm) {  // ~1 head per chunk; stop at the first whose own item covers R
      const int q = __ffs(hm) - 1;
      hm &= hm - 1u;
      if ((v.S_at(k0 + q) & kSizeMask) >= v.R) {  // raw size word (S is written in phase 2)
        one = 1u << q;
        break;
      }
    }
  }
  const uint32_t below = one ? one - 1u : kFull;
  const uint32_t multi = heads & below & ~one & ((zm >> 1) | (cont ? (1u << (K - 1)) : 0u));
  const int zi1 = one ? k0 + __ffs(one) - 1 : kInfIdx;
  const int zmh = multi ? k0 + __ffs(multi) - 1 : kInfIdx;
  {
    const int a1 = wmin_i32(zi1);
    const int a2 = wmin_i32(zmh);
    if (lane == 0) {
      sc.zW[warp] = a1;
      sc.zM[warp] = a2;
    }
  }
  cbar(T);
  int zmin = wmin_i32(lane < W ? sc.zW[lane] : kInfIdx);
  const int mmin = wmin_i32(lane < W ? sc.zM[lane] : kInfIdx);
  if (mmin < zmin) {  // CTA-uniform, rare: runs of several h = 0 items below the best single one
    int zi2 = kInfIdx;
    uint32_t mm = multi;
    while (mm) {
      const int q = __ffs(mm) - 1;
      mm &= mm - 1u;
      if (k0 + q >= zmin) break;
      const int stop = zero_run_stop(zmk16, tid, q, K, n);
      uint64_t span = 0;
      for (int k = k0 + q; k < stop && span < v.R; ++k) span += v.S_at(k) & kSizeMask;
      if (span >= v.R) {
        zi2 = k0 + q;
        break;
      }
    }
    const int a2 = wmin_i32(zi2);
    if (lane == 0) sc.zW2[warp] = a2;
    cbar(T);
    zmin = min(zmin, wmin_i32(lane < W ? sc.zW2[lane] : kInfIdx));
  }
  if (kPhaseHooks && a.dbg == 4) { if (tid == 0) write_result(a.out + p, -1, -1, 0, 0.0, 0, COOP_OK); return; }
  if (zmin != kInfIdx) {
    if (zmin >= k0 && zmin < k0 + K) {  // the owner of the winning head writes the window
      uint64_t span = 0;
      int k = zmin, znev = 0;
      do {  // the shortest covering window from zmin (inside its run of h = 0 items)
        span += v.S_at(k) & kSizeMask;
        znev += (sc.evc[k / K] >> (k % K)) & 1;
        ++k;
      } while (span < v.R);
      write_result(a.out + p, zmin, k - 1, span, 0.0, znev, COOP_OK);
    }
    return;
  }
  // ---------------- phase 2: carries of S, H^ and of the next-PINNED index ---------------
  int32_t nb_right;
  uint64_t S_car, S_total;
  {
    uint64_t ws = lane < W ? sc.wS[lane] : 0ull;
    double wh = lane < W ? sc.wH[lane] : 0.0;
    int32_t wb = lane < W ? sc.wF[lane] : kInfIdx;
#pragma unroll
    for (int d = 1; d < kMaxWarps; d <<= 1) {
      const uint64_t so = __shfl_up_sync(0xffffffffu, ws, d);
      const double ho = __shfl_up_sync(0xffffffffu, wh, d);
      const int32_t bo = __shfl_down_sync(0xffffffffu, wb, d);
      if (lane >= d) {
        ws += so;
        wh = __dadd_rn(ho, wh);
      }
      if (lane + d < 32) wb = min(wb, bo);
    }
    const uint64_t sprev = __shfl_sync(0xffffffffu, ws, warp ? warp - 1 : 0);
    const double hprev = __shfl_sync(0xffffffffu, wh, warp ? warp - 1 : 0);
    const int32_t bnext = __shfl_sync(0xffffffffu, wb, min(warp + 1, 31));
    S_car = (warp ? sprev : 0ull) + sexc;
    S_total = __shfl_sync(0xffffffffu, ws, W - 1);
    const double H_car = __dadd_rn(warp ? hprev : 0.0, hexc);
    nb_right = min(bexc, warp + 1 < W ? bnext : kInfIdx);
    // S over the raw size words, H^ carries added in place
#pragma unroll
    for (int q = 0; q < K; q += 2) {
      const int k = k0 + q;
      if (k < n) {
        const uint32_t o = swz((uint32_t)k);
        sm<ulonglong2>(v.sr, o) = make_ulonglong2(S_car + spre[q], S_car + spre[q + 1]);
        const double2 hl = sm<double2>(v.hr, o);
        sm<double2>(v.hr, o) = make_double2(__dadd_rn(H_car, hl.x), __dadd_rn(H_car, hl.y));
      }
    }
    if (k0 <= n - 1 && n - 1 < k0 + K) {  // sentinels: S[n], S[n+1] = ~0, H^[n]
      sm<uint64_t>(v.sr, swz((uint32_t)n)) = S_total;
      sm<uint64_t>(v.sr, swz((uint32_t)n + 1u)) = ~0ull;
      sm<double>(v.hr, swz((uint32_t)n)) = __dadd_rn(H_car, hacc);
    }
  }
  cbar(T);
  if (kPhaseHooks && a.dbg == 3) { if (tid == 0) write_result(a.out + p, -1, -1, 0, 0.0, 0, COOP_OK); return; }
  const uint64_t Sk0 = S_car + spre[0];
  // ---------------- phase B1: chunk pruning -------------------------------------------
  // Thread t's starts i in [k0, kl] have ends e(i) >= e(k0) (monotone) and prefixes
  // H[i] <= H[kl], so every window cost there is >= H[e(k0)] - H[kl].  e(k0) by one binary
  // search per thread; the first start's window (when PINNED-free) gives an upper bound;
  // chunks whose lower bound exceeds the CTA's best upper bound by more than the margin
  // cannot hold the winner (nor tie it after rounding) and skip the per-start work.
  const int kl = min(k0 + K, n) - 1;
  int e0 = n + 1;
  double LBt = kInf, Ut = kInf;
  if (k0 < n && !(barmask & 1u)) {
    const uint64_t target = Sk0 + v.R;  // S[k0] + R  (< 2^63)
    int lo = k0 + 1, hi = n + 1;        // S[n + 1] = ~0 >= target
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (v.S_at(mid) >= target) hi = mid;
      else lo = mid + 1;
    }
    e0 = lo;
  } else if (k0 < n) {
    e0 = -1;  // first start PINNED: no sample; ends of the others found below
  }
  if (k0 < n && e0 <= n) {
    const int nb = barmask ? k0 + __ffs(barmask) - 1 : nb_right;
    const double Hl = v.H_at(kl);
    if (e0 >= 0) {
      const double He = v.H_at(e0), Hk = v.H_at(k0);
      if (nb >= e0) Ut = (He - Hk) + v.gerr * (He + Hk);
      LBt = (He - Hl) - v.gerr * (He + Hl);
    } else {
      LBt = -kInf;  // no bound without e(k0): keep the chunk
    }
  }
  {
    const double uw = wmin_f64(Ut);
    if (lane == 0) sc.wP[warp] = uw;
    if (tid == 0) sc.nsurv = 0;
  }
  cbar(T);
  const double Upre = wmin_f64(lane < W ? sc.wP[lane] : kInf);
  const bool survive = (k0 < n) && (e0 <= n) && !(LBt > Upre * (1.0 + 0x1p-45));
  {  // compact the surviving chunks (one shared atomic per warp)
    const uint32_t bal = __ballot_sync(0xffffffffu, survive);
    int wbase = 0;
    if (lane == 0 && bal) wbase = atomicAdd(&sc.nsurv, __popc(bal));
    wbase = __shfl_sync(0xffffffffu, wbase, 0);
    if (survive)
      v.list[wbase + __popc(bal & ((1u << lane) - 1u))] = chunk_rec(k0, e0 >= 0 ? e0 : k0 + 1, barmask, nb_right);
  }
  cbar(T);
  if (kPhaseHooks && a.dbg == 5) { if (tid == 0) write_result(a.out + p, -1, -1, 0, 0.0, 0, COOP_OK); return; }
  // ---------------- phase B2: filter every start of the surviving chunks ---------------
  // (spread evenly over the CTA's threads, not left to the owner threads)
  const int nslots = sc.nsurv * K;
  LaneBest bl;
  bl.U = kInf; bl.L = kInf; bl.L2 = kInf; bl.li = -1; bl.le = -1;
  for (int sl = tid; sl < nslots; sl += T)
    eval_start<0>(v, v.list[sl / K], sl % K, 0.0, 0, 0, sc, bl);
  {
    const double Uw = wmin_f64(bl.U);
    if (lane == 0) sc.wU[warp] = Uw;
    if (tid == 0) sc.ncand = 0;
  }
  cbar(T);
  const double Umin = wmin_f64(lane < W ? sc.wU[lane] : kInf);
  if (kPhaseHooks && a.dbg == 6) { if (tid == 0) write_result(a.out + p, -1, -1, 0, 0.0, 0, COOP_OK); return; }
  if (Umin == kInf) {  // no PINNED-free window covers R
    if (tid == 0) write_result(a.out + p, -1, -1, 0, kInf, 0, COOP_INFEASIBLE);
    return;
  }
  const double thresh = Umin * (1.0 + 0x1p-45);
  // a lane with exactly one start under the threshold appends it; two or more re-walk
  const bool multi_l = (bl.L2 <= thresh);
  if (bl.L <= thresh && !multi_l) {
    const int slot = atomicAdd(&sc.ncand, 1);
    if (slot < kCandCap) sc.cand[slot] = ((uint32_t)bl.li << 16) | (uint32_t)(bl.le - bl.li);
  }
  const int any_multi = cbar_or(multi_l, T);
  if (!any_multi && sc.ncand <= kDefMax) {
    // the usual case: the candidates' exact re-summation reads global memory only; it is
    // deferred until this CTA has released the stage and issued the next TMA load (an L1 /
    // L2 prefetch of the windows' lines measured slower)
    const int nc = sc.ncand, slot = sc.dnext;
    if (tid < nc) {
      const uint32_t cd = sc.cand[tid];
      const int i = (int)(cd >> 16), e = i + (int)(cd & 0xffffu);
      sc.dcand[slot][tid] = cd;
      sc.dspan[slot][tid] = v.S_at(e) - v.S_at(i);
    }
    if (tid == 0) {
      sc.dpool[slot] = p;
      sc.dnc[slot] = nc;
      sc.dnext = slot ^ 1;
    }
    return;
  }
  // rare (ties, many candidates): exact h over region 1 first, then -- if some thread holds
  // two or more candidates -- re-walks restricted to windows of kCandCap consecutive starts
  // (cannot overflow the list), verified round by round from shared memory
#pragma unroll
  for (int q = 0; q < K; ++q) {
    const int k = k0 + q;
    if (k < n && ((evmask >> q) & 1u)) {
      const uint32_t o = swz((uint32_t)k);
      sm<double>(v.cr, o) = __ddiv_rn(sm<double>(v.cr, o), v.sg[k]);
    }
  }
  cbar(T);
  if (!any_multi) {
    verify_pool<true, K>(a, &v, sc, p, sc.cand, nullptr, sc.ncand, T);
    return;
  }
  const bool wmulti = __any_sync(0xffffffffu, bl.L <= thresh);  // this warp holds candidates
  uint64_t best = ~0ull, bspan = 0;  // meaningful in thread 0
  int bfirst = kInfIdx, blast = -1, bnev = 0;
  for (int w_lo = 0; w_lo < n; w_lo += kCandCap) {
    cbar(T);
    if (tid == 0) sc.ncand = 0;
    cbar(T);
    if (wmulti) {
      LaneBest dummy = bl;
      for (int sl = tid; sl < nslots; sl += T)
        eval_start<1>(v, v.list[sl / K], sl % K, thresh, w_lo, w_lo + kCandCap, sc, dummy);
    }
    cbar(T);
    const int nc = min(sc.ncand, kCandCap);
    if (nc == 0) continue;
    verify_pool<true, K>(a, &v, sc, p, sc.cand, nullptr, nc, T);  // writes this round's best into out[p]
    if (tid == 0) {
      const coop_window r = a.out[p];
      const uint64_t cb = (uint64_t)__double_as_longlong(r.cost);
      if (better(cb, r.first, best, bfirst)) {
        best = cb;
        bfirst = r.first;
        blast = r.last;
        bspan = r.span;
        bnev = r.n_evict;
      }
    }
  }
  if (tid == 0) write_result(a.out + p, bfirst, blast, bspan, __longlong_as_double((long long)best), bnev, COOP_OK);
}

template <int K, int MAXT, int MINB>
__global__ void __launch_bounds__(MAXT, MINB)
    search_kernel(const __grid_constant__ CUtensorMap m_ss, const __grid_constant__ CUtensorMap m_c,
                  const __grid_constant__ CUtensorMap m_s, const Args a) {
  extern __shared__ unsigned char smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  smem_t *base_ptr = smem_raw + (base - raw);
  Scratch &sc = *reinterpret_cast<Scratch *>(base_ptr + (size_t)a.stages * a.stage_bytes);
  uint4 *Ebuf = reinterpret_cast<uint4 *>(base_ptr + (size_t)a.stages * a.stage_bytes +
                                                 (sizeof(Scratch) + 15) / 16 * 16);

  const int tid = threadIdx.x;
  const int T = blockDim.x;

  if (tid == 0) {
    for (int s = 0; s < a.stages; ++s) mbar_init(smem_u32(&sc.mbar[s]), 1);
    sc.dpool[0] = sc.dpool[1] = -1;
    sc.dnext = 0;
    {
      unsigned smid;
      asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
      sc.swap = (int)(atomicAdd(&g_smcnt[smid & 1023u], 1u) & 1u);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  cbar(T);
  // pool of this CTA's round k: the rounds sweep [kG, (k+1)G) in a rotated order, so every
  // CTA sees every residue of the pool index modulo G (a periodic mix of short and long
  // requests -- the config-4 law alternates them -- is spread evenly over the CTAs and SMs)
  const int64_t G = gridDim.x;
  // (k < G rounds ahead at most: the residue is blockIdx.x + k reduced once or twice)
  auto pool_of = [&](int64_t k) {
    int64_t r = (int64_t)blockIdx.x + (k % G);
    if (r >= G) r -= G;
    return k * G + r;
  };
  const bool paired = a.use_tma && a.stages == 1 && !a.pending;
  if (a.use_tma && tid == 0 && !paired) {
    for (int s = 0; s < a.stages; ++s) {
      const int64_t p = pool_of(s);
      if (p < a.n_pools)
        issue_stage(a, &m_ss, &m_c, &m_s, base + (uint32_t)s * a.stage_bytes,
                    smem_u32(&sc.mbar[s]), p);
    }
  }

  if (a.pending) {
    // second pass after the streaming kernel: only the pools it marked COOP_PENDING_;
    // chunks of T pools are scanned with one status read per thread, plain staging
    for (int64_t c0 = (int64_t)blockIdx.x * T; c0 < a.n_pools; c0 += (int64_t)gridDim.x * T) {
      cbar(T);
      if (tid == 0) sc.nplist = 0;
      cbar(T);
      const int64_t q = c0 + tid;
      if (q < a.n_pools && a.out[q].status == COOP_PENDING_) sc.plist[atomicAdd(&sc.nplist, 1)] = tid;
      cbar(T);
      const int np = sc.nplist;
      for (int u = 0; u < np; ++u) {
        const int64_t p = c0 + sc.plist[u];
        smem_t *stage = base_ptr;
        stage_plain(a, stage, p, T);
        cbar(T);
        search_pool<K>(a, sc, Ebuf, stage, p, a.req[p]);
        cbar(T);
        const int slot = sc.dnext;  // keep a slot free for the next deferral
        if (sc.dpool[slot] >= 0) {
          verify_pool<false, K>(a, nullptr, sc, sc.dpool[slot], sc.dcand[slot], sc.dspan[slot], sc.dnc[slot], T);
          if (tid == 0) sc.dpool[slot] = -1;
        }
      }
    }
  } else if (paired) {
    // one stage per CTA, two CTAs per SM: the CTA visits its rounds k = j ^ swap, where the
    // second CTA to arrive on an SM swaps each pair of rounds -- with the rotated residues
    // (b + k) mod G the pool parity then differs between the two CTAs of an SM in every step
    // (the config-4 law alternates short and long requests by parity), so one CTA's
    // latency-bound phases of a long-request pool meet the other's throughput-bound phase 1
    const int64_t J = (a.n_pools + G - 1) / G + 1;
    const int64_t sw = sc.swap;
    auto pof = [&](int64_t j) -> int64_t {
      const int64_t k = j ^ sw;
      const uint32_t r = ((uint32_t)blockIdx.x + (uint32_t)k) % (uint32_t)G;  // k < 2^31
      return k * G + r;
    };
    int64_t j = 0;
    while (j < J && pof(j) >= a.n_pools) ++j;
    int64_t p = j < J ? pof(j) : -1;
    if (tid == 0 && p >= 0) issue_stage(a, &m_ss, &m_c, &m_s, base, smem_u32(&sc.mbar[0]), p);
    uint64_t Rnext = p >= 0 ? a.req[p] : 0ull;
    uint32_t phase = 0;
    while (p >= 0) {
      int64_t jn = j + 1, pn = -1;
      for (; jn < J; ++jn) {
        const int64_t q = pof(jn);
        if (q < a.n_pools) {
          pn = q;
          break;
        }
      }
      const uint64_t Rraw = Rnext;
      if (pn >= 0) Rnext = a.req[pn];
      mbar_wait(smem_u32(&sc.mbar[0]), phase);
      search_pool<K>(a, sc, Ebuf, base_ptr, p, Rraw);
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      cbar(T);  // the stage fully consumed
      if (tid == 0 && pn >= 0) issue_stage(a, &m_ss, &m_c, &m_s, base, smem_u32(&sc.mbar[0]), pn);
      {
        const int slot = sc.dnext ^ 1;
        if (sc.dpool[slot] >= 0) {
          verify_pool<false, K>(a, nullptr, sc, sc.dpool[slot], sc.dcand[slot], sc.dspan[slot], sc.dnc[slot], T);
          if (tid == 0) sc.dpool[slot] = -1;
        }
      }
      phase ^= 1u;
      j = jn;
      p = pn;
    }
  } else {
    int s = 0;
    uint32_t phase = 0;
    // residue of round k, advanced incrementally (no 64-bit division per pool); the next
    // pool's request is loaded a pool ahead
    int64_t rk = blockIdx.x, kG = 0;
    uint64_t Rnext = rk < a.n_pools ? a.req[rk] : 0ull;
    for (int64_t k = 0;; ++k, kG += G) {
      const int64_t p = kG + rk;
      if (p >= a.n_pools) break;  // only the last round is partial
      smem_t *stage = base_ptr + (size_t)s * a.stage_bytes;
      const uint64_t Rraw = Rnext;
      if (++rk == G) rk = 0;
      if (kG + G + rk < a.n_pools) Rnext = a.req[kG + G + rk];
      if (a.use_tma) {
        mbar_wait(smem_u32(&sc.mbar[s]), phase);
      } else {
        stage_plain(a, stage, p, T);
        cbar(T);
      }
      search_pool<K>(a, sc, Ebuf, stage, p, Rraw);
      // every thread orders its generic-proxy writes into the stage (S / H^ write-back)
      // before the async-proxy (TMA) refill that the barrier releases
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      cbar(T);  // stage s fully consumed
      if (a.use_tma && tid == 0) {
        // round k + stages: rk is already round k + 1's residue (stages is 1 or 2)
        int64_t rn = rk + (a.stages - 1);
        if (rn >= G) rn -= G;
        const int64_t pn = kG + (int64_t)a.stages * G + rn;
        if (pn < a.n_pools)
          issue_stage(a, &m_ss, &m_c, &m_s, base + (uint32_t)s * a.stage_bytes,
                      smem_u32(&sc.mbar[s]), pn);
      }
      // this pool's deferred exact re-summation (global memory; its lines were prefetched into
      // L1 when the candidates were found) while the stage refills
      {
        const int slot = sc.dnext ^ 1;
        if (sc.dpool[slot] >= 0) {
          verify_pool<false, K>(a, nullptr, sc, sc.dpool[slot], sc.dcand[slot], sc.dspan[slot], sc.dnc[slot], T);
          if (tid == 0) sc.dpool[slot] = -1;
        }
      }
      if (++s == a.stages) {  // next stage of the ring; parity flips on wrap-around
        s = 0;
        phase ^= 1u;
      }
    }
  }
  for (int slot = 0; slot < 2; ++slot) {  // the last deferred re-summations
    cbar(T);
    if (sc.dpool[slot] >= 0) verify_pool<false, K>(a, nullptr, sc, sc.dpool[slot], sc.dcand[slot], sc.dspan[slot], sc.dnc[slot], T);
  }
}

// ---------------------------------------------------------------- host side ------
PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static bool tried = false;
  if (!tried) {
    tried = true;
    void *p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

bool make_map(CUtensorMap *m, const void *ptr, int64_t stride, int64_t n_pools, int box_rows) {
  auto enc = get_encode();
  if (!enc) return false;
  cuuint64_t dims[3] = {16, (cuuint64_t)(stride / 16), (cuuint64_t)n_pools};
  cuuint64_t strides[2] = {128, (cuuint64_t)stride * 8};
  cuuint32_t box[3] = {16, (cuuint32_t)box_rows, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_UINT64, 3, const_cast<void *>(ptr), dims, strides,
                   box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

template <int K, int MAXT, int MINB>
int launch_k(const Args &a0, cudaStream_t st) {
  Args a = a0;
  const int rows = (a.n + 15) / 16;
  a.box_rows = rows < 256 ? rows : 256;
  a.n_boxes = (rows + a.box_rows - 1) / a.box_rows;
  {  // each region holds the TMA rows and the sentinel slots n, n+1
    const int64_t bytes = (int64_t)a.n_boxes * a.box_rows * 128;
    const int64_t need = ((int64_t)a.n + 2) * 8;
    a.region_bytes = (uint32_t)(((bytes > need ? bytes : need) + 1023) / 1024 * 1024);
  }
  a.stage_bytes = 3u * a.region_bytes;
  const int threads = ((a.n + K - 1) / K + 31) / 32 * 32;
  const int W = threads / 32;
  (void)W;  // summation depth of any H^ entry <= K + 5 (warp) + 4 (cross-warp) + 2 < K + 32
  a.gerr = 2.0 * (double)(K + 32) * 0x1p-53 + 0x1p-50 + 0x1p-43;  // + 2 x 2^-44 for h^ (rcp_nr)

  int dev = 0;
  cudaGetDevice(&dev);
  int max_smem = 0, sms = 0;
  cudaDeviceGetAttribute(&max_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const size_t fixed = (sizeof(Scratch) + 15) / 16 * 16 + (size_t)threads * 16 + 1024;  // + chunk list
  // MINB CTAs per SM share the SM's shared memory (228 KiB less 1 KiB per CTA reserved);
  // each CTA double-buffers only if that still fits
  size_t per_cta = (size_t)max_smem;
  if (MINB > 1) {
    int sm_total = 0;
    cudaDeviceGetAttribute(&sm_total, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev);
    per_cta = (size_t)sm_total / MINB - 1024;
    if (per_cta > (size_t)max_smem) per_cta = (size_t)max_smem;
  }
  a.stages = (2 * (size_t)a.stage_bytes + fixed <= per_cta) ? 2 : 1;
  const size_t smem = (size_t)a.stages * a.stage_bytes + fixed;
  if (smem > (size_t)max_smem) return COOP_ERR_INVALID_ARG;

  CUtensorMap m_ss, m_c, m_s;
  memset(&m_ss, 0, sizeof(m_ss));
  memset(&m_c, 0, sizeof(m_c));
  memset(&m_s, 0, sizeof(m_s));
  a.use_tma = 0;
  if (a.pending) a.stages = 1;
  {
    const char *d = getenv("COOP_SEARCH_DBG");
    a.dbg = d ? atoi(d) : 0;
  }
  const bool aligned = ((uintptr_t)a.ss % 16 == 0) && ((uintptr_t)a.cost % 16 == 0) &&
                       ((uintptr_t)a.stale % 16 == 0) && (a.stride % 16 == 0) &&
                       (a.n_pools < (1ll << 31)) && !coop_force_plain_staging() && !a.pending;
  if (aligned && make_map(&m_ss, a.ss, a.stride, a.n_pools, a.box_rows) &&
      make_map(&m_c, a.cost, a.stride, a.n_pools, a.box_rows) &&
      make_map(&m_s, a.stale, a.stride, a.n_pools, a.box_rows))
    a.use_tma = 1;

  if (threads > MAXT) return COOP_ERR_INVALID_ARG;
  auto kern = search_kernel<K, MAXT, MINB>;
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
      cudaSuccess)
    return COOP_ERR_CUDA;
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, threads, smem);
  if (per_sm < 1) per_sm = 1;
  int64_t grid = (int64_t)sms * per_sm;
  if (grid > a.n_pools) grid = a.n_pools;
  kern<<<(unsigned)grid, threads, smem, st>>>(m_ss, m_c, m_s, a);
  return cudaGetLastError() == cudaSuccess ? COOP_OK : COOP_ERR_CUDA;
}

}  // namespace

int launch_window_search_cta(const coop_tables_soa *t, const uint64_t *requests, coop_window *out,
                             cudaStream_t st, bool pending) {
  Args a;
  memset(&a, 0, sizeof(a));
  a.ss = t->size_state;
  a.cost = t->cost;
  a.stale = t->stale;
  a.req = requests;
  a.out = out;
  a.n_pools = t->n_pools;
  a.stride = t->pool_stride;
  a.n = t->n_blocks;
  a.pending = pending ? 1 : 0;
  if (a.n_pools == 0) return COOP_OK;
  const char *cfg = getenv("COOP_SEARCH_CFG");  // profiling hook: "8x512" = K 8, 512 threads
  if (cfg && strcmp(cfg, "8x512") == 0 && a.n <= 4096) return launch_k<8, 512, 2>(a, st);
  if (cfg && strcmp(cfg, "8x512x1") == 0 && a.n <= 4096) return launch_k<8, 512, 1>(a, st);
  if (cfg && strcmp(cfg, "16x256x1") == 0 && a.n <= 4096) return launch_k<16, 256, 1>(a, st);
  if (a.n <= 2048) return launch_k<8, 256, 2>(a, st);   // 2 CTAs per SM
  if (a.n <= 4096) return launch_k<16, 256, 2>(a, st);  // 2 CTAs per SM, 1 stage each
  return launch_k<16, 512, 1>(a, st);
}

int launch_window_search(const coop_tables_soa *t, const uint64_t *requests, coop_window *out,
                         cudaStream_t st) {
  if (!stream_search_enabled(t->n_blocks)) return launch_window_search_cta(t, requests, out, st, false);
  // the warp-per-pool stream, then the CTA-per-pool kernel on the pools it left pending
  int rc = launch_window_search_stream(t, requests, out, st);
  if (rc != COOP_OK) return rc;
  const char *v = getenv("COOP_SEARCH_IMPL");  // profiling hook: "stream_only" skips the second pass
  if (v && strcmp(v, "stream_only") == 0) return COOP_OK;
  return launch_window_search_cta(t, requests, out, st, true);
}

}  // namespace coop

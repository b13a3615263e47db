// coop_search.cu -- batched sliding-window eviction search for sm_100a.
//
// Computes, for each pool, the window of Eq. 1 as found by the Sec. 3.3
// sliding window: the contiguous, PINNED-free run of items with
// span >= R and the minimum correctly rounded exact sum of h = c/s (R1-R7).
//
// Design:
//   * persistent CTAs (one per SM at N = 4096) loop over pools; a 2-stage ring of
//     shared-memory buffers is filled by TMA (cp.async.bulk.tensor, SWIZZLE_128B) so the
//     next pool streams in while the current one is searched; thread t owns K items;
//   * phase A: h = c/s (IEEE RN), local prefixes of span (u64, exact) and h (fp64),
//     warp-shuffle + cross-warp scans; the stage is overwritten in place with
//     S[k] (span prefix), H^[k] (fp64 prefix of h) and h[k] (sign bit = FREE);
//   * phase B: per start i the window end e(i) = min{e : S[e] - S[i] >= R} by a galloping
//     two-pointer (cost ~2 log2 of the advance), PINNED and zero-cost checks from
//     per-thread bit masks, and an fp64 filter C^(i) = H^[e] - H^[i] with a rigorous
//     error bound (sums of nonnegative terms);
//   * a window of h = 0 items is exactly optimal (lowest start wins); otherwise every
//     start whose lower bound can reach the minimum is re-summed EXACTLY in 192-bit
//     fixed point (fixed192.cuh) and rounded once; winner = lexicographic min of
//     (rounded cost, first index)  -- bit-identical to the oracle.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <stdint.h>
#include <stdio.h>

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
constexpr uint64_t kSizeMask = (1ull << 62) - 1ull;
constexpr uint64_t kSizeLimit = 1ull << 48;
constexpr uint64_t kRClamp = 1ull << 62;  // any R > sum of sizes (< 2^61) is infeasible
constexpr int kInfIdx = 0x7fffffff;

struct Scratch {
  uint64_t wS[kMaxWarps];
  double wH[kMaxWarps];
  double wU[kMaxWarps];
  double wP[kMaxWarps];  // chunk-pruning upper bounds
  int32_t wF[kMaxWarps];
  int32_t wZ[kMaxWarps];
  uint64_t part[2][kMaxWarps][3];
  int32_t partn[2][kMaxWarps];
  uint64_t bcost[kMaxWarps];
  int32_t bfirst[kMaxWarps];
  int32_t bend[kMaxWarps];
  int32_t bnev[kMaxWarps];
  int32_t ncand;
  int32_t nsurv;      // surviving chunks in the list (phase B1)
  int32_t xend, xnev;  // end / evictions of the best exactly-costed window
  uint32_t cand[kCandCap];
  unsigned long long mbar[2];
  int32_t nplist;                      // pending mode: pools of the chunk to finish
  int16_t plist[kMaxWarps * 32];
};

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
  int32_t dbg;  // profiling hook (COOP_SEARCH_DBG): stop each pool after 1 = load, 2 = phase A +
                // scan + write-back; with -DCOOP_SEARCH_PHASE_HOOKS also 3 = write-back,
                // 4 = zero pass, 5 = pruning + compaction, 6 = filter + reductions
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
__device__ __forceinline__ void stage_plain(const Args &a, smem_t *stage, int64_t p) {
  const int64_t base = p * a.stride;
  for (int k = threadIdx.x; k < a.n; k += blockDim.x) {
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

template <typename T, typename Op>
__device__ __forceinline__ T warp_allreduce(T v, Op op) {
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) v = op(v, __shfl_xor_sync(0xffffffffu, v, d));
  return v;
}

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

// Per-pool view after phase A (all in shared memory):
//   region 0: S[k]   exclusive span prefix, k in [0, n]; S[n] = total span, S[n+1] = ~0
//   region 1: H^[k]  fp64 prefix of h, k in [0, n]
//   region 2: v[k]   h as binary64; FREE items stored as -0.0, PINNED items as NaN
//   list[c]          (uint4, scratch) surviving chunks of the pruning pass (phase B1)
struct PoolView {
  smem_t *sr, *hr, *vr;
  uint4 *list;
  int32_t n;
  uint64_t R, S_total;
  double gerr;

  __device__ __forceinline__ uint64_t S_at(int x) const { return sm<uint64_t>(sr, swz((uint32_t)x)); }
  __device__ __forceinline__ double H_at(int x) const { return sm<double>(hr, swz((uint32_t)x)); }
  __device__ __forceinline__ double v_at(int x) const { return sm<double>(vr, swz((uint32_t)x)); }

};

// Per-thread running state of the filter.
struct LaneBest {
  double U, L, L2;   // inexact windows: min upper bound, min / second-min lower bound
  int li, le;        // the inexact start with the minimal lower bound and its end
  uint64_t xb;       // exactly known windows (zero-cost, or <= 2 items): min cost bits
  int xi, xe;        //   ... its start (lowest among equal cost) and end
};

// A surviving chunk (phase B1): x = k0 | elo << 16 (elo <= e(i) for every start of the
// chunk), y = PINNED mask | nonzero-h mask << 16 of its K items, z / w = first PINNED /
// nonzero-h index to the right of the chunk.
__device__ __forceinline__ uint4 chunk_rec(int k0, int elo, uint32_t barmask, uint32_t nzmask,
                                           int nb_right, int nz_right) {
  return make_uint4((uint32_t)k0 | ((uint32_t)elo << 16), barmask | (nzmask << 16),
                    (uint32_t)nb_right, (uint32_t)nz_right);
}

// The filter for start i = k0 + q of a surviving chunk, run by any thread: window end by a
// galloping search from elo, PINNED and zero-cost checks from the chunk masks, exact cost
// for zero windows and windows of <= 2 items, else the fp64 prefix difference with its
// bound.  MODE 0 folds the start into LaneBest (lexicographic (cost bits, start) for exact
// windows, so the order in which a thread visits starts does not matter); MODE 1 appends
// it to the candidate list when it is inexact, its lower bound is <= thresh and i lies in
// [w_lo, w_hi).
template <int MODE>
__device__ __forceinline__ void eval_start(const PoolView &v, const uint4 rec, int q, double thresh,
                                           int w_lo, int w_hi, Scratch &sc, LaneBest &b) {
  const int n = v.n;
  const int k0 = (int)(rec.x & 0xffffu), elo = (int)(rec.x >> 16);
  const uint32_t barmask = rec.y & 0xffffu, nzmask = rec.y >> 16;
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
  const uint32_t mb = barmask >> q, mz = nzmask >> q;
  const int nb = mb ? i + __ffs(mb) - 1 : (int)rec.z;
  if (nb < e) return;  // a PINNED item inside [i, e-1]
  const int nz = mz ? i + __ffs(mz) - 1 : (int)rec.w;
  const int len = e - i;
  const bool zero = nz >= e;
  const bool exact = zero || len <= 2;
  const double h0 = fabs(v.v_at(i));
  const double h1 = len >= 2 ? fabs(v.v_at(i + 1)) : 0.0;
  const double He = v.H_at(e), Hi = v.H_at(i);
  const double Cx = zero ? 0.0 : __dadd_rn(h0, h1);
  const double C = exact ? Cx : He - Hi;
  const double err = exact ? 0.0 : v.gerr * (He + Hi);
  const double Lb = C - err;
  if (MODE == 0) {
    if (exact) {
      const uint64_t cb = (uint64_t)__double_as_longlong(C);
      if (better(cb, i, b.xb, b.xi)) {
        b.xb = cb;
        b.xi = i;
        b.xe = e;
      }
    } else {
      b.U = fmin(b.U, C + err);
      if (Lb < b.L) {
        b.L2 = b.L;
        b.L = Lb;
        b.li = i;
        b.le = e;
      } else {
        b.L2 = fmin(b.L2, Lb);
      }
    }
  } else if (!exact && Lb <= thresh && i >= w_lo && i < w_hi) {
    const int slot = atomicAdd(&sc.ncand, 1);
    if (slot < kCandCap) sc.cand[slot] = ((uint32_t)i << 16) | (uint32_t)(e - i);  // n <= 8192
  }
}

// Phase A of one thread: decode its K items (pairs via 16-byte conflict-free loads of the
// swizzled stage), validate (R7; integer tests on the binary64 encodings, same semantics as
// the oracle's comparisons), h = c/s (R1), local exclusive prefixes of span and h, and the
// h slot written back in place (FREE -> -0.0, PINNED -> NaN).  FULL: no item past n.
template <int K, bool FULL>
__device__ __forceinline__ void phase_a(const PoolView &v, int k0, int n, bool &bad,
                                        uint32_t &barmask, uint32_t &nzmask, uint64_t (&spre)[K],
                                        double (&hpre)[K], uint64_t &sacc, double &hacc) {
#pragma unroll
  for (int q = 0; q < K; q += 2) {
    const int k = k0 + q;
    const uint32_t o = swz((uint32_t)k);
    ulonglong2 vs = make_ulonglong2(0, 0);
    double2 vc = make_double2(0.0, 0.0), vt = make_double2(1.0, 1.0);
    if (FULL || k < n) {
      vs = sm<ulonglong2>(v.sr, o);
      vc = sm<double2>(v.hr, o);
      vt = sm<double2>(v.vr, o);
    }
    double hs[2];
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      const bool live = FULL || (k + r < n);
      const uint64_t sv = live ? (r ? vs.y : vs.x) : 0ull;  // padding: FREE, size 0
      const uint32_t svh = (uint32_t)(sv >> 32);
      const uint32_t state = svh >> 30;
      const bool ev = (state == COOP_EVICTABLE);
      const uint64_t size = sv & kSizeMask;
      const double cr = r ? vc.y : vc.x, sr_ = r ? vt.y : vt.x;
      const double c = ev ? cr : 1.0, st = ev ? sr_ : 1.0;  // 1/1: no slow division path
      const double hq = __ddiv_rn(c, st);                    // h(t) = c(t)/s(t), PAPER.md:150 (R1)
      // validation (R7) on the high words: the bounds are powers of two, so these are the
      // exact value ranges of the oracle's comparisons
      const uint32_t ch = (uint32_t)((uint64_t)__double_as_longlong(c) >> 32);
      const uint32_t cl = (uint32_t)__double_as_longlong(c);
      const uint32_t sh_ = (uint32_t)((uint64_t)__double_as_longlong(st) >> 32);
      const uint32_t hh = (uint32_t)((uint64_t)__double_as_longlong(hq) >> 32) & 0x7fffffffu;
      const uint32_t hl = (uint32_t)__double_as_longlong(hq);
      const bool hzero = (hh | hl) == 0u;
      const bool c_ok = (ch < 0x7ff00000u) | ((ch == 0x80000000u) & (cl == 0u));  // finite, >= 0 (or -0)
      const bool s_ok = (sh_ - 0x3ff00000u) < 0x40000000u;                       // finite, >= 1
      const bool h_ok = hzero | ((hh - 0x3bf00000u) < 0x07c00000u);               // 0 or [2^-64, 2^60)
      const bool size_bad = ((svh & 0x3fff0000u) != 0u) | (size == 0ull);       // size in [1, 2^48)
      if (live) bad |= size_bad | (state == 3u) | (ev & !(c_ok & s_ok & h_ok));
      const double h = ev ? hq : 0.0;
      const bool nzh = ev & !hzero;
      nzmask |= (uint32_t)nzh << (q + r);
      barmask |= (uint32_t)(live & (state == COOP_PINNED)) << (q + r);
      spre[q + r] = sacc;
      hpre[q + r] = hacc;
      sacc += live ? size : 0ull;
      hacc = __dadd_rn(hacc, h);
      // slot: EVICTABLE |h| (sign cleared), FREE -0.0 (h = 0, "not an eviction",
      // PAPER.md:147), PINNED NaN (never summed)
      const uint32_t oh = ev ? hh : (state == COOP_PINNED ? 0x7ff80000u : 0x80000000u);
      const uint32_t ol = ev ? hl : 0u;
      hs[r] = __hiloint2double((int)oh, (int)ol);
    }
    if (FULL || k < n) sm<double2>(v.vr, o) = make_double2(hs[0], hs[1]);
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
  PoolView v;
  v.sr = stage;
  v.hr = stage + a.region_bytes;
  v.vr = stage + 2u * a.region_bytes;
  v.list = Ebuf;
  v.n = n;
  v.R = Rraw < kRClamp ? Rraw : kRClamp;
  v.gerr = a.gerr;
  const int k0 = tid * K;

  if (a.dbg == 1) {
    if (tid == 0) write_result(a.out + p, -1, -1, 0, 0.0, 0, COOP_OK);
    return;
  }
  {
    // ---------------- phase A: decode, validate, h = c/s, local prefixes -------------
    bool bad = (Rraw == 0);
    uint32_t barmask = 0, nzmask = 0;
    uint64_t spre[K];
    double hpre[K];
    uint64_t sacc = 0;
    double hacc = 0.0;
    if (k0 + K <= n)  // warp-uniform except in the last warp
      phase_a<K, true>(v, k0, n, bad, barmask, nzmask, spre, hpre, sacc, hacc);
    else
      phase_a<K, false>(v, k0, n, bad, barmask, nzmask, spre, hpre, sacc, hacc);

    // ---------------- block scan: S (u64), H^ (fp64), next PINNED / next nonzero-h ------
    uint64_t sinc = sacc;
    double hinc = hacc;
    int32_t fb = barmask ? k0 + __ffs(barmask) - 1 : kInfIdx;
    int32_t fz = nzmask ? k0 + __ffs(nzmask) - 1 : kInfIdx;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const uint64_t so = __shfl_up_sync(0xffffffffu, sinc, d);
      const double ho = __shfl_up_sync(0xffffffffu, hinc, d);
      const int32_t bo = __shfl_down_sync(0xffffffffu, fb, d);
      const int32_t zo = __shfl_down_sync(0xffffffffu, fz, d);
      if (lane >= d) {
        sinc += so;
        hinc = __dadd_rn(ho, hinc);
      }
      if (lane + d < 32) {
        fb = min(fb, bo);
        fz = min(fz, zo);
      }
    }
    uint64_t sexc = __shfl_up_sync(0xffffffffu, sinc, 1);
    double hexc = __shfl_up_sync(0xffffffffu, hinc, 1);
    int32_t bexc = __shfl_down_sync(0xffffffffu, fb, 1);
    int32_t zexc = __shfl_down_sync(0xffffffffu, fz, 1);
    if (lane == 0) {
      sexc = 0;
      hexc = 0.0;
    }
    if (lane == 31) {
      bexc = kInfIdx;
      zexc = kInfIdx;
      sc.wS[warp] = sinc;
      sc.wH[warp] = hinc;
    }
    if (lane == 0) {
      sc.wF[warp] = fb;
      sc.wZ[warp] = fz;
    }
    const int bad_any = __syncthreads_or(bad);
    uint64_t S_car, S_total;
    double H_car;
    int32_t nb_right, nz_right;
    {
      // cross-warp: lane l < W holds warp l's totals; shuffle scan over the (<= 16) warps
      uint64_t ws = lane < W ? sc.wS[lane] : 0ull;
      double wh = lane < W ? sc.wH[lane] : 0.0;
      int32_t wb = lane < W ? sc.wF[lane] : kInfIdx;
      int32_t wz = lane < W ? sc.wZ[lane] : kInfIdx;
#pragma unroll
      for (int d = 1; d < kMaxWarps; d <<= 1) {
        const uint64_t so = __shfl_up_sync(0xffffffffu, ws, d);
        const double ho = __shfl_up_sync(0xffffffffu, wh, d);
        const int32_t bo = __shfl_down_sync(0xffffffffu, wb, d);
        const int32_t zo = __shfl_down_sync(0xffffffffu, wz, d);
        if (lane >= d) {
          ws += so;
          wh = __dadd_rn(ho, wh);
        }
        if (lane + d < 32) {
          wb = min(wb, bo);
          wz = min(wz, zo);
        }
      }
      const uint64_t sprev = __shfl_sync(0xffffffffu, ws, warp ? warp - 1 : 0);
      const double hprev = __shfl_sync(0xffffffffu, wh, warp ? warp - 1 : 0);
      const int32_t bnext = __shfl_sync(0xffffffffu, wb, min(warp + 1, 31));
      const int32_t znext = __shfl_sync(0xffffffffu, wz, min(warp + 1, 31));
      S_car = (warp ? sprev : 0ull) + sexc;
      H_car = __dadd_rn(warp ? hprev : 0.0, hexc);
      nb_right = min(bexc, warp + 1 < W ? bnext : kInfIdx);
      nz_right = min(zexc, warp + 1 < W ? znext : kInfIdx);
      S_total = __shfl_sync(0xffffffffu, ws, W - 1);
    }
    v.S_total = S_total;
    if (!bad_any) {
#pragma unroll
      for (int q = 0; q < K; q += 2) {
        const int k = k0 + q;
        if (k < n) {
          const uint32_t o = swz((uint32_t)k);
          sm<ulonglong2>(v.sr, o) = make_ulonglong2(S_car + spre[q], S_car + spre[q + 1]);
          sm<double2>(v.hr, o) = make_double2(__dadd_rn(H_car, hpre[q]), __dadd_rn(H_car, hpre[q + 1]));
        }
      }
      if (k0 <= n - 1 && n - 1 < k0 + K) {  // sentinels at slots n, n + 1
        sm<uint64_t>(v.sr, swz((uint32_t)n)) = S_total;
        sm<uint64_t>(v.sr, swz((uint32_t)n + 1u)) = ~0ull;
        sm<double>(v.hr, swz((uint32_t)n)) = __dadd_rn(H_car, hacc);
      }
    }
    __syncthreads();

    if (bad_any || a.dbg == 2) {
      if (tid == 0) write_result(a.out + p, -1, -1, 0, kInf, 0, COOP_ERR_INVALID_ARG);
    } else {
      if (kPhaseHooks && a.dbg == 3) { if (tid == 0) write_result(a.out + p, -1, -1, 0, 0.0, 0, COOP_OK); return; }
      // ---------------- phase B0: zero-cost windows -------------------------------------
      // A run of consecutive h = 0 items (FREE, or EVICTABLE with c = 0) is a zero-cost
      // window iff its span covers R; the lowest such run head is the answer (exact cost
      // 0 is the global minimum, R4).  Each thread checks the run heads of its chunk.
      int zi = kInfIdx, ze = -1, znev = 0;
      {
        const int cnt = n - k0;
        const uint32_t valid = cnt >= K ? (K == 32 ? ~0u : ((1u << K) - 1u)) : (cnt > 0 ? (1u << cnt) - 1u : 0u);
        const uint32_t zm = valid & ~barmask & ~nzmask;
        const uint32_t heads = zm & ~(zm << 1);
        // items that alone cover R (sizes from the prefix registers; the chunk's last
        // item is left to the span test below)
        uint32_t cov = 0;
#pragma unroll
        for (int q = 0; q + 1 < K; ++q) cov |= (uint32_t)(spre[q + 1] - spre[q] >= v.R) << q;
        const uint32_t one = heads & cov;  // zero windows [q, q]
        const uint32_t lower = one ? (1u << (__ffs(one) - 1)) - 1u : ~0u;
        // heads below the first of them whose run may be longer than one item
        uint32_t multi = heads & ~one & lower & ((zm >> 1) | (1u << (K - 1)));
        int zstop = n;
        while (multi) {
          const int q = __ffs(multi) - 1;
          multi &= multi - 1u;
          const uint32_t mb = barmask >> q, mz = nzmask >> q;
          const int nb = mb ? k0 + q + __ffs(mb) - 1 : nb_right;
          const int nz = mz ? k0 + q + __ffs(mz) - 1 : nz_right;
          const int stop = min(min(nb, nz), n);
          if (v.S_at(stop) - v.S_at(k0 + q) >= v.R) {
            zi = k0 + q;
            zstop = stop;
            break;
          }
        }
        if (zi == kInfIdx && one) {
          zi = k0 + __ffs(one) - 1;
          zstop = zi + 1;
        }
        if (zi != kInfIdx) {
          const uint64_t target = v.S_at(zi) + v.R;
          int lo = zi + 1, hi = zstop;
          while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if (v.S_at(mid) >= target) hi = mid;
            else lo = mid + 1;
          }
          ze = lo;
          for (int k = zi; k < ze; ++k) znev += (__double_as_longlong(v.v_at(k)) >= 0);
        }
      }
      const int zw = warp_allreduce(zi, [](int x, int y) { return min(x, y); });
      if (lane == 0) sc.wZ[warp] = zw;
      __syncthreads();
      const int zmin = warp_allreduce(lane < W ? sc.wZ[lane] : kInfIdx, [](int x, int y) { return min(x, y); });
      if (kPhaseHooks && a.dbg == 4) { if (tid == 0) write_result(a.out + p, -1, -1, 0, 0.0, 0, COOP_OK); return; }
      if (zmin != kInfIdx) {
        if (zi == zmin) write_result(a.out + p, zi, ze - 1, v.S_at(ze) - v.S_at(zi), 0.0, znev, COOP_OK);
      } else {
      // ---------------- phase B1: chunk pruning -------------------------------------------
      // Thread t's starts i in [k0, kl] have ends e(i) >= e(k0) (monotone) and prefixes
      // H[i] <= H[kl], so every window cost there is >= H[e(k0)] - H[kl].  e(k0) by one
      // binary search per thread; the first start's window (when PINNED-free) gives an
      // upper bound; chunks whose lower bound exceeds the CTA's best upper bound by more
      // than the filter's margin cannot hold the winner (nor tie it after rounding) and
      // skip the per-start work.  Bounds: |C^ - C| <= gerr (H^[e] + H^[i]) for any pair.
      const int kl = min(k0 + K, n) - 1;
      int e0 = n + 1;
      double LBt = kInf, Ut = kInf;
      if (k0 < n && !(barmask & 1u)) {
        const uint64_t target = S_car + spre[0] + v.R;  // S[k0] + R  (< 2^63)
        int lo = k0 + 1, hi = n + 1;                    // S[n + 1] = ~0 >= target
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
        double hl = hpre[0];  // hpre[kl - k0] with constant indices (stays in registers)
#pragma unroll
        for (int q = 1; q < K; ++q)
          if (k0 + q <= kl) hl = hpre[q];
        const double Hl = __dadd_rn(H_car, hl);
        if (e0 >= 0) {
          const double He = v.H_at(e0), Hk = __dadd_rn(H_car, hpre[0]);
          if (nb >= e0) Ut = (He - Hk) + v.gerr * (He + Hk);
          LBt = (He - Hl) - v.gerr * (He + Hl);
        } else {
          LBt = -kInf;  // no bound without e(k0): keep the chunk
        }
      }
      {
        const double uw = warp_allreduce(Ut, [](double x, double y) { return fmin(x, y); });
        if (lane == 0) sc.wP[warp] = uw;
        if (tid == 0) sc.nsurv = 0;
      }
      __syncthreads();
      const double Upre = warp_allreduce(lane < W ? sc.wP[lane] : kInf,
                                         [](double x, double y) { return fmin(x, y); });
      const bool survive = (k0 < n) && (e0 <= n) && !(LBt > Upre * (1.0 + 0x1p-45));
      {  // compact the surviving chunks (one shared atomic per warp)
        const uint32_t bal = __ballot_sync(0xffffffffu, survive);
        int wbase = 0;
        if (lane == 0 && bal) wbase = atomicAdd(&sc.nsurv, __popc(bal));
        wbase = __shfl_sync(0xffffffffu, wbase, 0);
        if (survive)
          v.list[wbase + __popc(bal & ((1u << lane) - 1u))] =
              chunk_rec(k0, e0 >= 0 ? e0 : k0 + 1, barmask, nzmask, nb_right, nz_right);
      }
      __syncthreads();
      if (kPhaseHooks && a.dbg == 5) { if (tid == 0) write_result(a.out + p, -1, -1, 0, 0.0, 0, COOP_OK); return; }
      // every start of the surviving chunks, spread evenly over the CTA's threads
      const int nslots = sc.nsurv * K;
      LaneBest bl;
      bl.U = kInf; bl.L = kInf; bl.L2 = kInf; bl.li = -1; bl.le = -1;
      bl.xb = ~0ull; bl.xi = kInfIdx; bl.xe = -1;
      for (int sl = tid; sl < nslots; sl += T)
        eval_start<0>(v, v.list[sl / K], sl % K, 0.0, 0, 0, sc, bl);
      const double Uw = warp_allreduce(bl.U, [](double x, double y) { return fmin(x, y); });
      const uint64_t xw = warp_allreduce(bl.xb, [](uint64_t x, uint64_t y) { return x < y ? x : y; });
      if (lane == 0) {
        sc.wU[warp] = Uw;
        sc.bcost[warp] = xw;
      }
      if (tid == 0) sc.ncand = 0;
      __syncthreads();
      const double Umin = warp_allreduce(lane < W ? sc.wU[lane] : kInf,
                                         [](double x, double y) { return fmin(x, y); });
      const uint64_t xbest = warp_allreduce(lane < W ? sc.bcost[lane] : ~0ull,
                                            [](uint64_t x, uint64_t y) { return x < y ? x : y; });
      const double thresh = fmin(Umin, __longlong_as_double((long long)xbest)) * (1.0 + 0x1p-45);
      if (kPhaseHooks && a.dbg == 6) { if (tid == 0) write_result(a.out + p, -1, -1, 0, 0.0, 0, COOP_OK); return; }
      // a lane with exactly one start under the threshold appends it; two or more re-walk
      const bool multi = (bl.L2 <= thresh);
      if (bl.L <= thresh && !multi) {
        const int slot = atomicAdd(&sc.ncand, 1);
        if (slot < kCandCap) sc.cand[slot] = ((uint32_t)bl.li << 16) | (uint32_t)(bl.le - bl.li);
      }
      const int xiw = warp_allreduce(bl.xb == xbest ? bl.xi : kInfIdx, [](int x, int y) { return min(x, y); });
      const int mw = __any_sync(0xffffffffu, multi) ? 1 : 0;
      if (lane == 0) {
        sc.bfirst[warp] = xiw;
        sc.bnev[warp] = mw;
      }
      __syncthreads();
      const int xfirst = warp_allreduce(lane < W ? sc.bfirst[lane] : kInfIdx, [](int x, int y) { return min(x, y); });
      const int any_multi = warp_allreduce(lane < W ? sc.bnev[lane] : 0, [](int x, int y) { return x | y; });
      const int nc0 = sc.ncand;
      const bool x_owner = (xbest != ~0ull) && bl.xi == xfirst && bl.xb == xbest;
      if (Umin == kInf && xbest == ~0ull) {
        if (tid == 0) write_result(a.out + p, -1, -1, 0, kInf, 0, COOP_INFEASIBLE);
      } else if (nc0 == 0 && !any_multi) {
        // no window of inexactly known cost can reach the exact best: the owner writes
        if (x_owner) {
          int nev = 0;
          for (int k = bl.xi; k < bl.xe; ++k) nev += (__double_as_longlong(v.v_at(k)) >= 0);
          write_result(a.out + p, bl.xi, bl.xe - 1, v.S_at(bl.xe) - v.S_at(bl.xi),
                       __longlong_as_double((long long)xbest), nev, COOP_OK);
        }
      } else {
        // ------------- candidates: exact 192-bit re-summation, RN, (cost, first) min ----
        if (x_owner) {
          int nev = 0;
          for (int k = bl.xi; k < bl.xe; ++k) nev += (__double_as_longlong(v.v_at(k)) >= 0);
          sc.xend = bl.xe;
          sc.xnev = nev;
        }
        __syncthreads();
        uint64_t best = xbest;  // meaningful in thread 0
        int bfirst = xfirst, bend = xbest != ~0ull ? sc.xend : -1, bnev = xbest != ~0ull ? sc.xnev : 0;
        const bool wmulti = __any_sync(0xffffffffu, bl.L <= thresh);  // this warp holds candidates
        // rounds: the prebuilt list (no multi), or re-walks restricted to windows of
        // kCandCap consecutive starts (cannot overflow the list)
        const int rounds = any_multi ? (n + kCandCap - 1) / kCandCap : 1;
        for (int rd = 0; rd < rounds; ++rd) {
          if (any_multi) {
            __syncthreads();
            if (tid == 0) sc.ncand = 0;
            __syncthreads();
            const int w_lo = rd * kCandCap, w_hi = w_lo + kCandCap;
            if (wmulti) {
              LaneBest dummy = bl;
              for (int sl = tid; sl < nslots; sl += T)
                eval_start<1>(v, v.list[sl / K], sl % K, thresh, w_lo, w_hi, sc, dummy);
            }
            __syncthreads();
          }
          const int nc = min(sc.ncand, kCandCap);
          if (nc <= W) {
            // few candidates: the whole CTA sums each window (short latency chain)
            for (int c = 0; c < nc; ++c) {
              const uint32_t cd = sc.cand[c];
              const int i = (int)(cd >> 16), e = i + (int)(cd & 0xffffu);
              U192 acc = u192_zero();
              int nev = 0;
              if (i + warp * 32 < e) {  // warp-uniform: warps without items skip
                for (int k = i + tid; k < e; k += T) {
                  const double hv = v.v_at(k);
                  nev += (__double_as_longlong(hv) >= 0);
                  acc = u192_add(acc, u192_from_double(hv));
                }
                acc = warp_sum192(acc, nev);
              }
              const int par = c & 1;
              if (lane == 0) {
                sc.part[par][warp][0] = acc.w0;
                sc.part[par][warp][1] = acc.w1;
                sc.part[par][warp][2] = acc.w2;
                sc.partn[par][warp] = nev;
              }
              __syncthreads();
              if (warp == 0) {
                U192 t = u192_zero();
                int tn = 0;
                if (lane < W) {
                  t.w0 = sc.part[par][lane][0];
                  t.w1 = sc.part[par][lane][1];
                  t.w2 = sc.part[par][lane][2];
                  tn = sc.partn[par][lane];
                }
                t = warp_sum192(t, tn);
                const uint64_t cb = (uint64_t)__double_as_longlong(u192_round_to_double(t));
                if (lane == 0 && better(cb, i, best, bfirst)) {
                  best = cb;
                  bfirst = i;
                  bend = e;
                  bnev = tn;
                }
              }
            }
          } else {
            // many candidates: one warp per candidate window
            uint64_t wbest = ~0ull;
            int32_t wfirst = kInfIdx, wend = -1, wnev = 0;
            for (int c = warp; c < nc; c += W) {
              const uint32_t cd = sc.cand[c];
              const int i = (int)(cd >> 16), e = i + (int)(cd & 0xffffu);
              U192 acc = u192_zero();
              int nev = 0;
              for (int k = i + lane; k < e; k += 32) {
                const double hv = v.v_at(k);
                nev += (__double_as_longlong(hv) >= 0);
                acc = u192_add(acc, u192_from_double(hv));
              }
              acc = warp_sum192(acc, nev);
              const uint64_t cb = (uint64_t)__double_as_longlong(u192_round_to_double(acc));
              if (better(cb, i, wbest, wfirst)) {
                wbest = cb;
                wfirst = i;
                wend = e;
                wnev = nev;
              }
            }
            if (lane == 0) {
              sc.bcost[warp] = wbest;
              sc.bfirst[warp] = wfirst;
              sc.bend[warp] = wend;
              sc.bnev[warp] = wnev;
            }
            __syncthreads();
            if (tid == 0) {
              for (int w = 0; w < W; ++w) {
                if (sc.bend[w] >= 0 && better(sc.bcost[w], sc.bfirst[w], best, bfirst)) {
                  best = sc.bcost[w];
                  bfirst = sc.bfirst[w];
                  bend = sc.bend[w];
                  bnev = sc.bnev[w];
                }
              }
            }
          }
        }
        if (tid == 0)
          write_result(a.out + p, bfirst, bend - 1, v.S_at(bend) - v.S_at(bfirst),
                       __longlong_as_double((long long)best), bnev, COOP_OK);
      }
      }
    }
  }
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

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int T = blockDim.x, W = T >> 5;
  const int n = a.n;
  const double kInf = __longlong_as_double(0x7ff0000000000000ll);

  if (tid == 0) {
    for (int s = 0; s < a.stages; ++s) mbar_init(smem_u32(&sc.mbar[s]), 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (a.use_tma && tid == 0) {
    for (int s = 0; s < a.stages; ++s) {
      const int64_t p = (int64_t)blockIdx.x + (int64_t)s * gridDim.x;
      if (p < a.n_pools)
        issue_stage(a, &m_ss, &m_c, &m_s, base + (uint32_t)s * a.stage_bytes,
                    smem_u32(&sc.mbar[s]), p);
    }
  }

  if (a.pending) {
    // second pass after the streaming kernel: only the pools it marked COOP_PENDING_;
    // chunks of T pools are scanned with one status read per thread, plain staging
    for (int64_t c0 = (int64_t)blockIdx.x * T; c0 < a.n_pools; c0 += (int64_t)gridDim.x * T) {
      __syncthreads();
      if (tid == 0) sc.nplist = 0;
      __syncthreads();
      const int64_t q = c0 + tid;
      if (q < a.n_pools && a.out[q].status == COOP_PENDING_) sc.plist[atomicAdd(&sc.nplist, 1)] = tid;
      __syncthreads();
      const int np = sc.nplist;
      for (int u = 0; u < np; ++u) {
        const int64_t p = c0 + sc.plist[u];
        smem_t *stage = base_ptr;
        stage_plain(a, stage, p);
        __syncthreads();
        search_pool<K>(a, sc, Ebuf, stage, p, a.req[p]);
        __syncthreads();
      }
    }
    return;
  }
  int it = 0, s = 0;
  uint32_t phase = 0;
  for (int64_t p = blockIdx.x; p < a.n_pools; p += gridDim.x, ++it) {
    smem_t *stage = base_ptr + (size_t)s * a.stage_bytes;
    const uint64_t Rraw = a.req[p];
    if (a.use_tma) {
      mbar_wait(smem_u32(&sc.mbar[s]), phase);
    } else {
      stage_plain(a, stage, p);
      __syncthreads();
    }
    search_pool<K>(a, sc, Ebuf, stage, p, Rraw);
    // every thread orders its generic-proxy writes into the stage (S / H^ / h write-back)
    // before the async-proxy (TMA) refill that the barrier releases
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();  // stage s fully consumed
    if (a.use_tma && tid == 0) {
      const int64_t pn = p + (int64_t)a.stages * gridDim.x;
      if (pn < a.n_pools)
        issue_stage(a, &m_ss, &m_c, &m_s, base + (uint32_t)s * a.stage_bytes,
                    smem_u32(&sc.mbar[s]), pn);
    }
    if (++s == a.stages) {  // next stage of the ring; parity flips on wrap-around
      s = 0;
      phase ^= 1u;
    }
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
  a.gerr = 2.0 * (double)(K + 32) * 0x1p-53 + 0x1p-50;

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
  const char *two = getenv("COOP_SEARCH_TWO_CTA");  // profiling hook: 2 CTAs/SM, 1 stage
  if (two && two[0] == '1' && a.n <= 4096) return launch_k<16, 256, 2>(a, st);
  if (a.n <= 2048) return launch_k<8, 256, 2>(a, st);  // 2 CTAs per SM
  if (a.n <= 4096) return launch_k<8, 512, 2>(a, st);  // 2 CTAs per SM, 1 stage each
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

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

#include "coop.h"
#include "coop_internal.h"
#include "fixed192.cuh"

namespace coop {

namespace {

constexpr int kCandCap = 1024;
constexpr int kMaxWarps = 16;
constexpr uint64_t kSizeMask = (1ull << 62) - 1ull;
constexpr uint64_t kSizeLimit = 1ull << 48;
constexpr uint64_t kRClamp = 1ull << 62;  // any R > sum of sizes (< 2^61) is infeasible
constexpr int kInfIdx = 0x7fffffff;

struct Scratch {
  uint64_t wS[kMaxWarps];
  double wH[kMaxWarps];
  double wU[kMaxWarps];
  int32_t wF[kMaxWarps];
  int32_t wZ[kMaxWarps];
  uint64_t part[2][kMaxWarps][3];
  int32_t partn[2][kMaxWarps];
  uint64_t bcost[kMaxWarps];
  int32_t bfirst[kMaxWarps];
  int32_t bend[kMaxWarps];
  int32_t bnev[kMaxWarps];
  int32_t ncand;
  uint32_t cand[kCandCap];
  unsigned long long mbar[2];
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

// Per-pool context.  Thread t owns items [k0, k0 + K).  After phase A the stage holds
//   region 0: S[k]  (exclusive span prefix, k in [0, n]; S[n] = total span)
//   region 1: H^[k] (fp64 prefix of h, k in [0, n])
//   region 2: h[k]  (binary64; FREE items stored as -0.0)
template <int K>
struct PoolCtx {
  smem_t *sr, *hr, *vr;
  int32_t n, k0;
  uint64_t R, S_car, S_total;
  double H_car, gerr;
  uint32_t barmask, nzmask;
  int32_t nb_right, nz_right;
  uint64_t spre[K];
  double hpre[K];

  __device__ __forceinline__ uint64_t S_at(int x) const { return sm<uint64_t>(sr, swz((uint32_t)x)); }
  __device__ __forceinline__ double H_at(int x) const { return sm<double>(hr, swz((uint32_t)x)); }
  __device__ __forceinline__ double h_at(int x) const { return sm<double>(vr, swz((uint32_t)x)); }
  __device__ __forceinline__ int32_t next_barrier(int q) const {  // first PINNED index >= k0+q
    const uint32_t m = barmask >> q;
    return m ? k0 + q + __ffs(m) - 1 : nb_right;
  }
  __device__ __forceinline__ int32_t next_nonzero(int q) const {  // first h != 0 index >= k0+q
    const uint32_t m = nzmask >> q;
    return m ? k0 + q + __ffs(m) - 1 : nz_right;
  }

  // Walk this thread's starts from q_from: binary search for the first start's window end,
  // then a galloping two-pointer (cost ~2 log2 of each advance).  Called only when no
  // zero-cost window exists, so every feasible window holds a nonzero h.
  // MODE 0: fp64 filter bounds (U_t, L_t).
  // MODE 1: append starts whose lower bound <= thresh to the candidate list; returns
  //         the q at which the list overflowed (resume point) or K when done.
  template <int MODE>
  __device__ __forceinline__ int walk(int q_from, double thresh, Scratch &sc, double &U_t,
                                      double &L_t, uint64_t &xb, int &xi, int &xe) const {
    int e = 0;
#pragma unroll
    for (int q = 0; q < K; ++q) {
      if (q < q_from) continue;
      const int i = k0 + q;
      if (i >= n) break;
      if ((barmask >> q) & 1u) continue;
      const uint64_t target = S_car + spre[q] + R;  // R clamped: no overflow
      if (target > S_total) break;                  // this and every later start: infeasible
      if (e <= i) {  // first start: bisect (i, n]; S[n] >= target
        int lo = i + 1, hi = n;
        while (lo < hi) {
          const int mid = (lo + hi) >> 1;
          if (S_at(mid) >= target) hi = mid;
          else lo = mid + 1;
        }
        e = lo;
      } else if (S_at(e) < target) {  // gallop to a bracket, then bisect
        int lo = e + 1, step = 1, hi = e + 1;
        while (hi < n && S_at(hi) < target) {
          lo = hi + 1;
          step <<= 1;
          hi = e + step;
        }
        if (hi > n) hi = n;
        while (lo < hi) {
          const int mid = (lo + hi) >> 1;
          if (S_at(mid) >= target) hi = mid;
          else lo = mid + 1;
        }
        e = lo;
      }
      if (next_barrier(q) < e) continue;  // a PINNED item inside [i, e-1]
      const int len = e - i;
      double C, err;
      bool exact = false;
      if (len <= 2) {  // one IEEE add is correctly rounded: the exact window cost
        const double h0 = fabs(h_at(i));
        C = (len == 1) ? h0 : __dadd_rn(h0, fabs(h_at(i + 1)));
        err = 0.0;
        exact = true;
      } else if (len <= 8) {  // direct sum of nonnegative terms: relative error < 7u
        double acc = 0.0;
        for (int k = i; k < e; ++k) acc = __dadd_rn(acc, fabs(h_at(k)));
        C = acc;
        err = 0x1p-50 * acc;
      } else {  // prefix difference: error bounded by the prefix magnitudes
        const double He = H_at(e);
        const double Hi = __dadd_rn(H_car, hpre[q]);
        C = He - Hi;
        err = gerr * (He + Hi);
      }
      const double Lb = C - err;
      if (MODE == 0) {
        if (exact) {
          const uint64_t cb = (uint64_t)__double_as_longlong(C);
          if (cb < xb) {  // starts ascend within a thread: ties keep the lower start
            xb = cb;
            xi = i;
            xe = e;
          }
        } else {
          U_t = fmin(U_t, C + err);
          L_t = fmin(L_t, Lb);
        }
      } else if (!exact && Lb <= thresh) {
        const int slot = atomicAdd(&sc.ncand, 1);
        if (slot >= kCandCap) return q;
        sc.cand[slot] = ((uint32_t)i << 16) | (uint32_t)(e - i);  // n <= 8192
      }
    }
    return K;
  }

  // Lowest start of a zero-cost window in this thread's chunk (kInfIdx if none): a run of
  // consecutive h = 0 items (FREE, or EVICTABLE with c = 0) is a zero-cost window iff its
  // span covers R; the run's first item is then the lowest such start.
  __device__ __forceinline__ int zero_start() const {
    const int cnt = n - k0;
    const uint32_t valid = cnt >= K ? (K == 32 ? ~0u : ((1u << K) - 1u)) : (cnt > 0 ? (1u << cnt) - 1u : 0u);
    const uint32_t zm = valid & ~barmask & ~nzmask;
    const uint32_t heads = zm & ~(zm << 1);  // first item of each zero run inside the chunk
#pragma unroll
    for (int q = 0; q < K; ++q) {  // static indices: spre stays in registers
      if (!((heads >> q) & 1u)) continue;
      const int stop = min(min(next_nonzero(q), next_barrier(q)), n);
      if (S_at(stop) - (S_car + spre[q]) >= R) return k0 + q;
    }
    return kInfIdx;
  }
};

template <int K>
__global__ void __launch_bounds__(512, 1)
    search_kernel(const __grid_constant__ CUtensorMap m_ss, const __grid_constant__ CUtensorMap m_c,
                  const __grid_constant__ CUtensorMap m_s, const Args a) {
  extern __shared__ unsigned char smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  smem_t *base_ptr = smem_raw + (base - raw);
  Scratch &sc = *reinterpret_cast<Scratch *>(base_ptr + (size_t)a.stages * a.stage_bytes);

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

  int it = 0;
  for (int64_t p = blockIdx.x; p < a.n_pools; p += gridDim.x, ++it) {
    const int s = it % a.stages;
    smem_t *stage = base_ptr + (size_t)s * a.stage_bytes;
    const uint64_t Rraw = a.req[p];
    if (a.use_tma) {
      mbar_wait(smem_u32(&sc.mbar[s]), (uint32_t)((it / a.stages) & 1));
    } else {
      stage_plain(a, stage, p);
      __syncthreads();
    }

    PoolCtx<K> cx;
    cx.sr = stage;
    cx.hr = stage + a.region_bytes;
    cx.vr = stage + 2u * a.region_bytes;
    cx.n = n;
    cx.k0 = tid * K;
    cx.gerr = a.gerr;
    cx.R = Rraw < kRClamp ? Rraw : kRClamp;

    // ---------------- phase A: decode, validate, h = c/s, local prefixes -------------
    bool bad = (Rraw == 0);
    uint32_t barmask = 0, nzmask = 0;
    uint64_t sacc = 0;
    double hacc = 0.0;
#pragma unroll
    for (int q = 0; q < K; q += 2) {
      const int k = cx.k0 + q;
      uint64_t sv[2] = {0, 0};
      double cv[2] = {0.0, 0.0}, tv[2] = {1.0, 1.0};
      const uint32_t o = swz((uint32_t)k);
      if (k < n) {
        const ulonglong2 vs = sm<ulonglong2>(cx.sr, o);
        const double2 vc = sm<double2>(cx.hr, o);
        const double2 vt = sm<double2>(cx.vr, o);
        sv[0] = vs.x; sv[1] = vs.y; cv[0] = vc.x; cv[1] = vc.y; tv[0] = vt.x; tv[1] = vt.y;
      }
      double hs[2];
#pragma unroll
      for (int r = 0; r < 2; ++r) {
        const int kk = k + r;
        uint64_t size = 0;
        double h = 0.0, hslot = 0.0;
        if (kk < n) {
          const uint32_t state = (uint32_t)(sv[r] >> 62);
          const bool ev = (state == COOP_EVICTABLE);
          size = sv[r] & kSizeMask;
          const double c = ev ? cv[r] : 0.0, st = ev ? tv[r] : 1.0;
          h = __ddiv_rn(c, st);  // h(t) = c(t)/s(t), IEEE RN (R1); 0 if not EVICTABLE
          bad |= (size == 0) | (size >= kSizeLimit) | (state > 2u) |
                 (ev & (!(c >= 0.0 && c <= 1.7976931348623157e308) |
                        !(st >= 1.0 && st <= 1.7976931348623157e308) |
                        ((h != 0.0) & ((h < 0x1p-64) | (h >= 0x1p60)))));
          nzmask |= (uint32_t)(h != 0.0) << (q + r);
          barmask |= (uint32_t)(state == COOP_PINNED) << (q + r);
          hslot = (state == COOP_FREE) ? -0.0 : h;  // FREE: h = 0, sign = not an eviction
        }
        cx.spre[q + r] = sacc;
        cx.hpre[q + r] = hacc;
        sacc += size;
        hacc = __dadd_rn(hacc, h);
        hs[r] = hslot;
      }
      if (k < n) sm<double2>(cx.vr, o) = make_double2(hs[0], hs[1]);
    }
    cx.barmask = barmask;
    cx.nzmask = nzmask;

    // ---------------- block scan: S (u64), H^ (fp64), next PINNED / next nonzero-h ------
    uint64_t sinc = sacc;
    double hinc = hacc;
    int32_t fb = barmask ? cx.k0 + __ffs(barmask) - 1 : kInfIdx;
    int32_t fz = nzmask ? cx.k0 + __ffs(nzmask) - 1 : kInfIdx;
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
      cx.S_car = (warp ? sprev : 0ull) + sexc;
      cx.H_car = __dadd_rn(warp ? hprev : 0.0, hexc);
      cx.nb_right = min(bexc, warp + 1 < W ? bnext : kInfIdx);
      cx.nz_right = min(zexc, warp + 1 < W ? znext : kInfIdx);
      cx.S_total = __shfl_sync(0xffffffffu, ws, W - 1);
    }
    if (!bad_any) {
#pragma unroll
      for (int q = 0; q < K; q += 2) {
        const int k = cx.k0 + q;
        if (k < n) {
          const uint32_t o = swz((uint32_t)k);
          sm<ulonglong2>(cx.sr, o) = make_ulonglong2(cx.S_car + cx.spre[q], cx.S_car + cx.spre[q + 1]);
          sm<double2>(cx.hr, o) = make_double2(__dadd_rn(cx.H_car, cx.hpre[q]),
                                               __dadd_rn(cx.H_car, cx.hpre[q + 1]));
        }
      }
      if (cx.k0 <= n - 1 && n - 1 < cx.k0 + K) {  // sentinels at slot n
        sm<uint64_t>(cx.sr, swz((uint32_t)n)) = cx.S_total;
        sm<double>(cx.hr, swz((uint32_t)n)) = __dadd_rn(cx.H_car, hacc);
      }
    }
    __syncthreads();

    if (bad_any) {
      if (tid == 0) write_result(a.out + p, -1, -1, 0, kInf, 0, COOP_ERR_INVALID_ARG);
    } else {
      // ---------------- phase B1: zero-cost windows (h = 0 runs covering R) -------------
      const int zw = warp_allreduce(cx.zero_start(), [](int x, int y) { return min(x, y); });
      if (lane == 0) sc.wZ[warp] = zw;
      __syncthreads();
      const int zmin = warp_allreduce(lane < W ? sc.wZ[lane] : kInfIdx,
                                      [](int x, int y) { return min(x, y); });
      double Umin = kInf, L_t = kInf;
      uint64_t xbest = ~0ull;  // best exactly-costed window (length <= 2): bits, start, end
      int xfirst = kInfIdx, xend = -1;
      if (zmin == kInfIdx) {
        // ---------------- phase B2: window ends + fp64 filter ----------------------------
        double U_t = kInf;
        uint64_t xb = ~0ull;
        int xi = kInfIdx, xe = -1;
        cx.template walk<0>(0, 0.0, sc, U_t, L_t, xb, xi, xe);
        const double Uw = warp_allreduce(U_t, [](double x, double y) { return fmin(x, y); });
        const uint64_t xw = warp_allreduce(xb, [](uint64_t x, uint64_t y) { return x < y ? x : y; });
        if (lane == 0) {
          sc.wU[warp] = Uw;
          sc.bcost[warp] = xw;
        }
        __syncthreads();
        Umin = warp_allreduce(lane < W ? sc.wU[lane] : kInf,
                              [](double x, double y) { return fmin(x, y); });
        xbest = warp_allreduce(lane < W ? sc.bcost[lane] : ~0ull,
                               [](uint64_t x, uint64_t y) { return x < y ? x : y; });
        if (xbest != ~0ull) {  // lowest start among the exact windows with that cost
          const int xiw = warp_allreduce(xb == xbest ? xi : kInfIdx, [](int x, int y) { return min(x, y); });
          if (lane == 0) sc.bfirst[warp] = xiw;
          __syncthreads();
          xfirst = warp_allreduce(lane < W ? sc.bfirst[lane] : kInfIdx, [](int x, int y) { return min(x, y); });
          if (xi == xfirst) sc.ncand = xe;  // unique owner publishes the end
          __syncthreads();
          xend = sc.ncand;
        }
      }
      if (zmin != kInfIdx) {
        // exact cost 0 is the minimum; the lowest start wins, with its minimal end
        if (warp == 0) {
          const int i = zmin;
          const uint64_t target = cx.S_at(i) + cx.R;
          int lo = i + 1, hi = n;
          while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if (cx.S_at(mid) >= target) hi = mid;
            else lo = mid + 1;
          }
          const int e = lo;
          int nev = 0;
          for (int k = i + lane; k < e; k += 32)
            nev += (__double_as_longlong(cx.h_at(k)) >= 0);  // sign clear: EVICTABLE
          nev = warp_allreduce(nev, [](int x, int y) { return x + y; });
          if (lane == 0) write_result(a.out + p, i, e - 1, cx.S_at(e) - cx.S_at(i), 0.0, nev, COOP_OK);
        }
      } else if (Umin == kInf && xbest == ~0ull) {
        if (tid == 0) write_result(a.out + p, -1, -1, 0, kInf, 0, COOP_INFEASIBLE);
      } else {
        // ------------- candidates: exact 192-bit re-summation, RN, (cost, first) min --
        const double xval = __longlong_as_double((long long)xbest);
        const double thresh = fmin(Umin, xval) * (1.0 + 0x1p-45);
        int resume = (L_t <= thresh) ? 0 : K;
        uint64_t best = xbest;  // meaningful in thread 0
        int bfirst = xfirst, bend = xend, bnev = 0;
        if (tid == 0 && xbest != ~0ull)
          for (int k = xfirst; k < xend; ++k) bnev += (__double_as_longlong(cx.h_at(k)) >= 0);
        const int any_cand = __syncthreads_or(resume < K);
        while (any_cand) {
          if (tid == 0) sc.ncand = 0;
          __syncthreads();
          if (resume < K) {
            double du = 0, dl = 0;
            uint64_t dxb = 0;
            int dxi = 0, dxe = 0;
            resume = cx.template walk<1>(resume, thresh, sc, du, dl, dxb, dxi, dxe);
          }
          const int pending = __syncthreads_or(resume < K);
          const int nc = min(sc.ncand, kCandCap);
          if (nc <= W) {
            // few candidates: the whole CTA sums each window (short latency chain)
            for (int c = 0; c < nc; ++c) {
              const uint32_t cd = sc.cand[c];
              const int i = (int)(cd >> 16), e = i + (int)(cd & 0xffffu);
              U192 acc = u192_zero();
              int nev = 0;
              if (i + warp * 32 < e) {  // warp-uniform: warps without items skip the shuffles
                for (int k = i + tid; k < e; k += T) {
                  const double hv = cx.h_at(k);
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
                const double hv = cx.h_at(k);
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
          if (!pending) break;
          __syncthreads();  // the candidate list is rewritten next round
        }
        if (tid == 0)
          write_result(a.out + p, bfirst, bend - 1, cx.S_at(bend) - cx.S_at(bfirst),
                       __longlong_as_double((long long)best), bnev, COOP_OK);
      }
    }
    __syncthreads();  // stage s fully consumed
    if (a.use_tma && tid == 0) {
      const int64_t pn = p + (int64_t)a.stages * gridDim.x;
      if (pn < a.n_pools)
        issue_stage(a, &m_ss, &m_c, &m_s, base + (uint32_t)s * a.stage_bytes,
                    smem_u32(&sc.mbar[s]), pn);
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

template <int K>
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
  const size_t fixed = sizeof(Scratch) + 1024;
  a.stages = (2 * (size_t)a.stage_bytes + fixed <= (size_t)max_smem) ? 2 : 1;
  const size_t smem = (size_t)a.stages * a.stage_bytes + fixed;
  if (smem > (size_t)max_smem) return COOP_ERR_INVALID_ARG;

  CUtensorMap m_ss, m_c, m_s;
  memset(&m_ss, 0, sizeof(m_ss));
  memset(&m_c, 0, sizeof(m_c));
  memset(&m_s, 0, sizeof(m_s));
  a.use_tma = 0;
  const bool aligned = ((uintptr_t)a.ss % 16 == 0) && ((uintptr_t)a.cost % 16 == 0) &&
                       ((uintptr_t)a.stale % 16 == 0) && (a.stride % 16 == 0) &&
                       (a.n_pools < (1ll << 31)) && !coop_force_plain_staging();
  if (aligned && make_map(&m_ss, a.ss, a.stride, a.n_pools, a.box_rows) &&
      make_map(&m_c, a.cost, a.stride, a.n_pools, a.box_rows) &&
      make_map(&m_s, a.stale, a.stride, a.n_pools, a.box_rows))
    a.use_tma = 1;

  auto kern = search_kernel<K>;
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

int launch_window_search(const coop_tables_soa *t, const uint64_t *requests, coop_window *out,
                         cudaStream_t st) {
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
  if (a.n_pools == 0) return COOP_OK;
  if (a.n <= 4096) return launch_k<8>(a, st);
  return launch_k<16>(a, st);
}

}  // namespace coop

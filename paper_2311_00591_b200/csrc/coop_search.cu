// coop_search.cu -- batched sliding-window eviction search for sm_100a.
//
// Computes, for each pool, the window of Eq. 1 as found by the Sec. 3.3
// sliding window: the contiguous, PINNED-free run of items with
// span >= R and the minimum correctly rounded exact sum of h = c/s (R1-R7).
//
// Design:
//   * persistent CTAs (one per SM at N = 4096), each loops over pools; a 2-stage ring of
//     shared-memory buffers is filled by TMA (cp.async.bulk.tensor, SWIZZLE_128B) so the
//     next pool streams in while the current one is searched;  thread t owns K items;
//   * per item: h = c/s (IEEE RN), an exact u64 span prefix S and an fp64 prefix H^ of h,
//     both by thread-local sums + a warp-shuffle / cross-warp block scan, written back
//     in place into the stage (the raw bytes are no longer needed);
//   * per start i: the window end e(i) = min{e : S[e] - S[i] >= R} (binary search for the
//     thread's first start, then a monotone two-pointer), a PINNED check, and an fp64
//     filter value C^(i) = H^[e] - H^[i] with a rigorous error bound (nonnegative sums);
//   * block-min of the upper bounds; every start whose lower bound can still reach the
//     minimum (after binary64 rounding) is re-summed EXACTLY by a warp in 192-bit fixed
//     point (fixed192.cuh), rounded once (ties-to-even), and the winner is the
//     lexicographic min of (rounded cost, first index)  -- bit-identical to the oracle.
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

struct Scratch {
  uint64_t wS[kMaxWarps];
  double wH[kMaxWarps];
  double wU[kMaxWarps];
  int32_t wF[kMaxWarps];
  uint64_t bcost[kMaxWarps];
  int32_t bfirst[kMaxWarps];
  int32_t bend[kMaxWarps];
  int32_t bnev[kMaxWarps];
  uint64_t S_total;
  double H_total;
  uint64_t best_cost;
  int32_t best_first, best_end, best_nev;
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
  double gamma2;
};

__device__ __forceinline__ uint32_t swz(uint32_t k) {  // item k -> byte offset, SWIZZLE_128B
  uint32_t off = k * 8u;
  return off ^ (((off >> 7) & 7u) << 4);
}

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ uint64_t lds_u64(uint32_t a) {
  uint64_t v;
  asm volatile("ld.shared.u64 %0, [%1];" : "=l"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ double lds_f64(uint32_t a) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ void lds_v2u64(uint32_t a, uint64_t &x, uint64_t &y) {
  asm volatile("ld.shared.v2.u64 {%0, %1}, [%2];" : "=l"(x), "=l"(y) : "r"(a));
}
__device__ __forceinline__ void lds_v2f64(uint32_t a, double &x, double &y) {
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(x), "=d"(y) : "r"(a));
}
__device__ __forceinline__ void sts_v2u64(uint32_t a, uint64_t x, uint64_t y) {
  asm volatile("st.shared.v2.u64 [%0], {%1, %2};" ::"r"(a), "l"(x), "l"(y) : "memory");
}
__device__ __forceinline__ void sts_v2f64(uint32_t a, double x, double y) {
  asm volatile("st.shared.v2.f64 [%0], {%1, %2};" ::"r"(a), "d"(x), "d"(y) : "memory");
}
__device__ __forceinline__ void sts_u64(uint32_t a, uint64_t x) {
  asm volatile("st.shared.u64 [%0], %1;" ::"r"(a), "l"(x) : "memory");
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
__device__ __forceinline__ void stage_plain(const Args &a, uint32_t stage_base, int64_t p) {
  const int64_t base = p * a.stride;
  for (int k = threadIdx.x; k < a.n; k += blockDim.x) {
    uint32_t o = swz((uint32_t)k);
    sts_u64(stage_base + o, a.ss[base + k]);
    sts_u64(stage_base + a.region_bytes + o, (uint64_t)__double_as_longlong(a.cost[base + k]));
    sts_u64(stage_base + 2u * a.region_bytes + o,
            (uint64_t)__double_as_longlong(a.stale[base + k]));
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

__device__ __forceinline__ double warp_min_f64(double v) {
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) v = fmin(v, __shfl_xor_sync(0xffffffffu, v, d));
  return v;
}

template <int K>
struct PoolCtx {
  uint32_t ssr, cr, sr;  // region bases (shared addresses)
  int32_t n, k0;
  uint64_t R, S_car, S_total;
  double H_car, H_total, gamma2;
  uint32_t barmask;
  int32_t nb_right;
  uint64_t spre[K];
  double hpre[K];

  __device__ __forceinline__ uint64_t S_at(int e) const {
    return e >= n ? S_total : lds_u64(ssr + swz((uint32_t)e));
  }
  __device__ __forceinline__ double H_at(int e) const {
    return e >= n ? H_total : lds_f64(cr + swz((uint32_t)e));
  }
  __device__ __forceinline__ int32_t next_barrier(int q) const {  // first PINNED index >= k0+q
    uint32_t m = barmask >> q;
    return m ? k0 + q + __ffs(m) - 1 : nb_right;
  }

  // Walk this thread's starts from q_from.  mode 0: accumulate filter bounds.
  // mode 1: append starts whose lower bound <= thresh to the candidate list; returns
  // the q at which the list overflowed (resume point) or K when done.
  template <int MODE>
  __device__ __forceinline__ int walk(int q_from, double thresh, Scratch &sc, double &U_t,
                                      double &L_t) const {
    int e = -1;
#pragma unroll
    for (int q = 0; q < K; ++q) {
      if (q < q_from) continue;
      const int i = k0 + q;
      if (i >= n) break;
      if ((barmask >> q) & 1u) continue;
      const uint64_t Si = S_car + spre[q];
      const uint64_t target = Si + R;
      if (target < Si || target > S_total) break;  // this and every later start: infeasible
      if (e < 0) {
        int lo = i + 1, hi = n;
        while (lo < hi) {
          int mid = (lo + hi) >> 1;
          if (S_at(mid) >= target) hi = mid;
          else lo = mid + 1;
        }
        e = lo;
      } else {
        while (e < n && S_at(e) < target) ++e;
      }
      if (next_barrier(q) < e) continue;  // a PINNED item inside [i, e-1]
      const double He = H_at(e);
      const double Hi = H_car + hpre[q];
      const double C = He - Hi;
      const double err = gamma2 * (He + Hi) + 0x1p-50 * fabs(C);
      const double L = C - err;
      if (MODE == 0) {
        U_t = fmin(U_t, C + err);
        L_t = fmin(L_t, L);
      } else if (L <= thresh) {
        int slot = atomicAdd(&sc.ncand, 1);
        if (slot >= kCandCap) return q;
        sc.cand[slot] = ((uint32_t)i << 16) | (uint32_t)(e - i);  // n <= 8192: e - i <= 8192
      }
    }
    return K;
  }
};

template <int K>
__global__ void __launch_bounds__(512, 1)
    search_kernel(const __grid_constant__ CUtensorMap m_ss, const __grid_constant__ CUtensorMap m_c,
                  const __grid_constant__ CUtensorMap m_s, const Args a) {
  extern __shared__ unsigned char smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  unsigned char *base_ptr = smem_raw + (base - raw);
  Scratch &sc = *reinterpret_cast<Scratch *>(base_ptr + (size_t)a.stages * a.stage_bytes);

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int W = blockDim.x >> 5;
  const int n = a.n;

  if (tid == 0) {
    for (int s = 0; s < a.stages; ++s) mbar_init(smem_u32(&sc.mbar[s]), 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (a.use_tma && tid == 0) {
    for (int s = 0; s < a.stages; ++s) {
      int64_t p = (int64_t)blockIdx.x + (int64_t)s * gridDim.x;
      if (p < a.n_pools)
        issue_stage(a, &m_ss, &m_c, &m_s, base + (uint32_t)s * a.stage_bytes,
                    smem_u32(&sc.mbar[s]), p);
    }
  }

  int it = 0;
  for (int64_t p = blockIdx.x; p < a.n_pools; p += gridDim.x, ++it) {
    const int s = it % a.stages;
    const uint32_t stage = base + (uint32_t)s * a.stage_bytes;
    if (a.use_tma) {
      mbar_wait(smem_u32(&sc.mbar[s]), (uint32_t)((it / a.stages) & 1));
    } else {
      stage_plain(a, stage, p);
      __syncthreads();
    }

    PoolCtx<K> cx;
    cx.ssr = stage;
    cx.cr = stage + a.region_bytes;
    cx.sr = stage + 2u * a.region_bytes;
    cx.n = n;
    cx.k0 = tid * K;
    cx.gamma2 = a.gamma2;
    cx.R = a.req[p];

    // ---------------- phase A: h, local prefixes, validation ----------------------
    bool bad = (cx.R == 0);
    uint32_t barmask = 0;
    uint64_t sacc = 0;
    double hacc = 0.0;
#pragma unroll
    for (int q = 0; q < K; q += 2) {
      const int k = cx.k0 + q;
      uint64_t sv0 = 0, sv1 = 0;
      double c0 = 0.0, c1 = 0.0, t0 = 1.0, t1 = 1.0;
      const uint32_t o = swz((uint32_t)k);
      if (k < n) {
        lds_v2u64(cx.ssr + o, sv0, sv1);
        lds_v2f64(cx.cr + o, c0, c1);
        lds_v2f64(cx.sr + o, t0, t1);
      }
      double hs[2];
#pragma unroll
      for (int r = 0; r < 2; ++r) {
        const int kk = k + r;
        const uint64_t sv = r ? sv1 : sv0;
        const double c = r ? c1 : c0, st = r ? t1 : t0;
        uint64_t size = 0;
        double h = 0.0, hslot = 0.0;
        if (kk < n) {
          const uint64_t state = sv >> 62;
          size = sv & kSizeMask;
          bad |= (size == 0) | (size >= kSizeLimit) | (state > 2u);
          if (state == COOP_EVICTABLE) {
            bad |= !(c >= 0.0 && c <= 1.7976931348623157e308) |
                   !(st >= 1.0 && st <= 1.7976931348623157e308);
            h = __ddiv_rn(c, st);  // h(t) = c(t)/s(t), IEEE RN (R1)
            bad |= (h != 0.0) & ((h < 0x1p-64) | (h >= 0x1p60));
            hslot = h;
          } else if (state == COOP_PINNED) {
            barmask |= 1u << (q + r);
          } else {
            hslot = -0.0;  // FREE: h = 0; sign bit marks "not an eviction"
          }
        }
        cx.spre[q + r] = sacc;
        cx.hpre[q + r] = hacc;
        sacc += size;
        hacc = __dadd_rn(hacc, h);
        hs[r] = hslot;
      }
      if (k < n) sts_v2f64(cx.sr + o, hs[0], hs[1]);
    }
    cx.barmask = barmask;

    // ---------------- block scan: S (exact u64), H^ (fp64), next PINNED (suffix min) --
    uint64_t sinc = sacc;
    double hinc = hacc;
    int32_t fsuf = barmask ? cx.k0 + __ffs(barmask) - 1 : 0x7fffffff;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      uint64_t so = __shfl_up_sync(0xffffffffu, sinc, d);
      double ho = __shfl_up_sync(0xffffffffu, hinc, d);
      int32_t fo = __shfl_down_sync(0xffffffffu, fsuf, d);
      if (lane >= d) {
        sinc += so;
        hinc = __dadd_rn(ho, hinc);
      }
      if (lane + d < 32) fsuf = min(fsuf, fo);
    }
    uint64_t sexc = __shfl_up_sync(0xffffffffu, sinc, 1);
    double hexc = __shfl_up_sync(0xffffffffu, hinc, 1);
    int32_t fexc = __shfl_down_sync(0xffffffffu, fsuf, 1);
    if (lane == 0) {
      sexc = 0;
      hexc = 0.0;
    }
    if (lane == 31) {
      fexc = 0x7fffffff;
      sc.wS[warp] = sinc;
      sc.wH[warp] = hinc;
    }
    if (lane == 0) sc.wF[warp] = fsuf;
    const int bad_any = __syncthreads_or(bad);
    uint64_t scar = 0;
    double hcar = 0.0;
    int32_t fcar = 0x7fffffff;
    for (int w = 0; w < W; ++w) {
      if (w < warp) {
        scar += sc.wS[w];
        hcar = __dadd_rn(hcar, sc.wH[w]);
      }
      if (w > warp) fcar = min(fcar, sc.wF[w]);
    }
    cx.S_car = scar + sexc;
    cx.H_car = __dadd_rn(hcar, hexc);
    cx.nb_right = min(fexc, fcar);

    if (!bad_any) {
#pragma unroll
      for (int q = 0; q < K; q += 2) {
        const int k = cx.k0 + q;
        if (k < n) {
          const uint32_t o = swz((uint32_t)k);
          sts_v2u64(cx.ssr + o, cx.S_car + cx.spre[q], cx.S_car + cx.spre[q + 1]);
          sts_v2f64(cx.cr + o, __dadd_rn(cx.H_car, cx.hpre[q]),
                    __dadd_rn(cx.H_car, cx.hpre[q + 1]));
        }
      }
      if (cx.k0 <= n - 1 && n - 1 < cx.k0 + K) {
        sc.S_total = cx.S_car + sacc;
        sc.H_total = __dadd_rn(cx.H_car, hacc);
      }
    }
    __syncthreads();

    if (bad_any) {
      if (tid == 0) write_result(a.out + p, -1, -1, 0, __longlong_as_double(0x7ff0000000000000ll), 0,
                                 COOP_ERR_INVALID_ARG);
    } else {
      cx.S_total = sc.S_total;
      cx.H_total = sc.H_total;
      // ---------------- phase B: window ends + fp64 filter ----------------------------
      double U_t = __longlong_as_double(0x7ff0000000000000ll), L_t = U_t;
      cx.template walk<0>(0, 0.0, sc, U_t, L_t);
      double Um = warp_min_f64(U_t);
      if (lane == 0) sc.wU[warp] = Um;
      if (tid == 0) {
        sc.best_cost = ~0ull;
        sc.best_first = 0x7fffffff;
        sc.best_end = -1;
        sc.best_nev = 0;
      }
      __syncthreads();
      double Umin = sc.wU[0];
      for (int w = 1; w < W; ++w) Umin = fmin(Umin, sc.wU[w]);

      if (Umin == __longlong_as_double(0x7ff0000000000000ll)) {
        if (tid == 0)
          write_result(a.out + p, -1, -1, 0, Umin, 0, COOP_INFEASIBLE);
      } else {
        // ------------- candidates: exact 192-bit re-summation, RN, (cost, first) min --
        const double thresh = Umin * (1.0 + 0x1p-45);
        int resume = (L_t <= thresh) ? 0 : K;
        while (true) {
          if (tid == 0) sc.ncand = 0;
          __syncthreads();
          if (resume < K) {
            double du = 0, dl = 0;
            resume = cx.template walk<1>(resume, thresh, sc, du, dl);
          }
          const int pending = __syncthreads_or(resume < K);
          const int nc = min(sc.ncand, kCandCap);
          uint64_t wbest = ~0ull;
          int32_t wfirst = 0x7fffffff, wend = -1, wnev = 0;
          for (int c = warp; c < nc; c += W) {
            const uint32_t cd = sc.cand[c];
            const int i = (int)(cd >> 16), e = i + (int)(cd & 0xffffu);
            U192 acc = u192_zero();
            int nev = 0;
            for (int k = i + lane; k < e; k += 32) {
              const double hv = lds_f64(cx.sr + swz((uint32_t)k));
              nev += (__double_as_longlong(hv) >= 0);  // sign clear: EVICTABLE
              acc = u192_add(acc, u192_from_double(hv));
            }
#pragma unroll
            for (int d = 16; d > 0; d >>= 1) {
              U192 o;
              o.w0 = __shfl_xor_sync(0xffffffffu, acc.w0, d);
              o.w1 = __shfl_xor_sync(0xffffffffu, acc.w1, d);
              o.w2 = __shfl_xor_sync(0xffffffffu, acc.w2, d);
              nev += __shfl_xor_sync(0xffffffffu, nev, d);
              acc = u192_add(acc, o);
            }
            const uint64_t cb = (uint64_t)__double_as_longlong(u192_round_to_double(acc));
            if (cb < wbest || (cb == wbest && i < wfirst)) {
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
              if (sc.bend[w] < 0) continue;
              if (sc.bcost[w] < sc.best_cost ||
                  (sc.bcost[w] == sc.best_cost && sc.bfirst[w] < sc.best_first)) {
                sc.best_cost = sc.bcost[w];
                sc.best_first = sc.bfirst[w];
                sc.best_end = sc.bend[w];
                sc.best_nev = sc.bnev[w];
              }
            }
          }
          if (!pending) break;
        }
        if (tid == 0) {
          const int i = sc.best_first, e = sc.best_end;
          const uint64_t span = cx.S_at(e) - cx.S_at(i);
          write_result(a.out + p, i, e - 1, span, __longlong_as_double((long long)sc.best_cost),
                       sc.best_nev, COOP_OK);
        }
      }
    }
    __syncthreads();  // stage s fully consumed
    if (a.use_tma && tid == 0) {
      int64_t pn = p + (int64_t)a.stages * gridDim.x;
      if (pn < a.n_pools) issue_stage(a, &m_ss, &m_c, &m_s, stage, smem_u32(&sc.mbar[s]), pn);
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
  a.region_bytes = (uint32_t)((a.n_boxes * a.box_rows * 128 + 1023) / 1024 * 1024);
  a.stage_bytes = 3u * a.region_bytes;
  const int threads = ((a.n + K - 1) / K + 31) / 32 * 32;
  const int W = threads / 32;
  a.gamma2 = 2.0 * (double)(K + W + 10) * 0x1p-53;

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

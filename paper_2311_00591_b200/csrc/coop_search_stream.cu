// coop_search_stream.cu -- the batched sliding-window search as a warp-per-pool stream.
//
// Computes, for each pool, the window of Eq. 1 that the Sec. 3.3 sliding
// window finds: the contiguous, PINNED-free run of items with span >= R,
// minimum correctly rounded exact sum of h = c/s, lowest first index among equals
// (R1-R7) -- bit-identical to the CTA-per-pool kernel (coop_search.cu) and to
// the oracle O1.
//
// Why a stream ("streaming search"): a 4096-item pool is 96 KB, so a
// CTA that stages whole pools fits two pools per SM and spends most of its time at
// barriers between the phases of one pool.  Here ONE WARP owns one pool at a time and
// walks it once, left to right, in tiles of 128 items (4 per lane), the way the paper's
// two-pointer walks the address-ordered list: for every END e of the tile it finds the
// latest start st(e) = max{i : S[e+1] - S[i] >= R} in a per-warp history ring of the
// exclusive span / cost prefixes S[k], H^[k] (shared memory, the last 1024 items), so the
// windows (st(e), e) are evaluated the moment their last item streams in.  There are no
// CTA barriers; warps are independent, so 12 of them per SM hide each other's latencies,
// and every lane keeps the next two tiles in flight in registers (24 registers per tile;
// coalesced 16-byte streaming loads).
//
// Exactness: the canonical windows of R4 are (i, j(i)), j(i) the shortest end covering R.
// The starts whose window ends at e are exactly (st(e-1), st(e)] (minus any start at or
// before the last PINNED item <= e), and their costs H[e+1] - H[i] are nonincreasing in i,
// so min_e C(st(e), e) is the exact minimum.  The winner is then found as in R4:
//   * zero windows (no nonzero h in the window) are detected exactly from the index of
//     the last nonzero item; the lowest-start one wins outright;
//   * otherwise an fp64 filter C^ = H^[e+1] - H^[st(e)] with the rigorous bound
//     |C^ - C| <= gerr (H^[e+1] + H^[st(e)]) keeps every end that can still reach the
//     minimum after rounding (a per-warp candidate list, pruned against the running upper
//     bound); at the end of the pool the candidates are re-summed EXACTLY in 192-bit fixed
//     point from a re-read of their items (fixed192.cuh), rounded once; the earliest end
//     with the minimal rounded cost wins, and its start is extended downwards while the
//     rounded cost stays the same (lowest first index, R4).
// Pools this cannot finish -- a window longer than the ring, or more near-optimal ends
// than the candidate list holds -- are marked COOP_PENDING_ and finished by the
// CTA-per-pool kernel in a second launch on the same stream.
#include <cuda_runtime.h>
#include <stdint.h>

#include "coop.h"
#include "coop_internal.h"
#include "fixed192.cuh"

namespace coop {

namespace {

constexpr int SK = 4;             // items per lane per tile
constexpr int STILE = 32 * SK;    // items per tile
constexpr int HCAP = 1024;        // history ring per warp (items); power of two, multiple of STILE
constexpr int HMASK = HCAP - 1;
constexpr int CCAP = 64;          // candidate ends per warp
constexpr int SWARPS = 6;         // warps per CTA (two CTAs per SM)
constexpr uint64_t kSizeMask = (1ull << 62) - 1ull;
constexpr uint64_t kRClamp = 1ull << 62;
constexpr double kMargin = 1.0 + 0x1p-45;  // rounding margin of the filter (as coop_search.cu)

struct WarpSmem {
  uint64_t hS[HCAP];     // S[k]  (exclusive span prefix) of item k at slot k & HMASK
  double hH[HCAP];       // H^[k] (fp64 prefix of h)
  int32_t ce[CCAP];      // candidate end e
  int32_t cb[CCAP];      // its start st(e)
  int32_t ca[CCAP];      // starts of e lie in (a, st(e)]
  double cl[CCAP];       // lower bound of its exact cost
};

struct SArgs {
  const uint64_t *ss;
  const double *cost;
  const double *stale;
  const uint64_t *req;
  coop_window *out;
  int64_t n_pools;
  int64_t stride;
  int32_t n;
  int32_t ntiles;
  int32_t vec;  // 16-byte vector loads allowed (aligned arrays, even stride)
  double gerr;  // filter error coefficient
};

struct Raw {  // one lane's 4 items of one tile
  ulonglong2 a0, a1;
  double2 c0, c1, s0, s1;
};

__device__ __forceinline__ void load_tile(const SArgs &A, Raw &r, int64_t p, int t, int lane) {
  const int k = t * STILE + 4 * lane;
  const int64_t off = p * A.stride + k;
  if (A.vec && k + 4 <= A.n) {
    const ulonglong2 *qs = reinterpret_cast<const ulonglong2 *>(A.ss + off);
    const double2 *qc = reinterpret_cast<const double2 *>(A.cost + off);
    const double2 *qt = reinterpret_cast<const double2 *>(A.stale + off);
    r.a0 = __ldcs(qs);
    r.a1 = __ldcs(qs + 1);
    r.c0 = __ldcs(qc);
    r.c1 = __ldcs(qc + 1);
    r.s0 = __ldcs(qt);
    r.s1 = __ldcs(qt + 1);
  } else {  // ragged tail or unaligned layout: items >= n read as FREE, size 0
    uint64_t v[4];
    double c[4], s[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const bool live = k + q < A.n;
      v[q] = live ? __ldcs(A.ss + off + q) : 0ull;
      c[q] = live ? __ldcs(A.cost + off + q) : 0.0;
      s[q] = live ? __ldcs(A.stale + off + q) : 1.0;
    }
    r.a0 = make_ulonglong2(v[0], v[1]);
    r.a1 = make_ulonglong2(v[2], v[3]);
    r.c0 = make_double2(c[0], c[1]);
    r.c1 = make_double2(c[2], c[3]);
    r.s0 = make_double2(s[0], s[1]);
    r.s1 = make_double2(s[2], s[3]);
  }
}

__device__ __forceinline__ void put_window(coop_window *o, int32_t first, int32_t last, uint64_t span,
                                           double cost, int32_t nev, int32_t status) {
  coop_window w;
  w.first = first;
  w.last = last;
  w.span = span;
  w.cost = cost;
  w.n_evict = nev;
  w.status = status;
  *o = w;
}

// exact h of item k (re-read; the same IEEE division as the stream), its size and state
struct Item {
  double h;
  uint64_t size;
  bool ev;
};
__device__ __forceinline__ Item reread(const SArgs &A, int64_t p, int k) {
  const int64_t off = p * A.stride + k;
  const uint64_t sv = A.ss[off];
  const uint32_t state = (uint32_t)(sv >> 62);
  Item it;
  it.ev = state == COOP_EVICTABLE;
  it.size = sv & kSizeMask;
  it.h = it.ev ? __ddiv_rn(A.cost[off], A.stale[off]) : 0.0;
  return it;
}

__device__ __forceinline__ U192 shfl_xor192(U192 v, int d) {
  U192 o;
  o.w0 = __shfl_xor_sync(0xffffffffu, v.w0, d);
  o.w1 = __shfl_xor_sync(0xffffffffu, v.w1, d);
  o.w2 = __shfl_xor_sync(0xffffffffu, v.w2, d);
  return o;
}
__device__ __forceinline__ U192 shfl_up192(U192 v, int d) {
  U192 o;
  o.w0 = __shfl_up_sync(0xffffffffu, v.w0, d);
  o.w1 = __shfl_up_sync(0xffffffffu, v.w1, d);
  o.w2 = __shfl_up_sync(0xffffffffu, v.w2, d);
  return o;
}

// Exact sum (192-bit), span and EVICTABLE count of items [i, e] of pool p, by the warp.
__device__ __forceinline__ void exact_window(const SArgs &A, int64_t p, int i, int e, int lane,
                                             U192 &sum, uint64_t &span, int &nev) {
  U192 acc = u192_zero();
  uint64_t sp = 0;
  int ne = 0;
  for (int k = i + lane; k <= e; k += 32) {
    const Item it = reread(A, p, k);
    acc = u192_add(acc, u192_from_double(it.h));
    sp += it.size;
    ne += it.ev;
  }
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) {
    acc = u192_add(acc, shfl_xor192(acc, d));
    sp += __shfl_xor_sync(0xffffffffu, sp, d);
    ne += __shfl_xor_sync(0xffffffffu, ne, d);
  }
  sum = acc;
  span = sp;
  nev = ne;
}

// Per-pool running state (warp-uniform unless noted).
struct PoolRun {
  int64_t p;
  uint64_t R;
  uint64_t Scar;   // S at the start of the current tile
  double Hcar;     // H^ at the start of the current tile
  int lpcar;       // last PINNED index before the tile (-1)
  int lnzcar;      // last nonzero-h index before the tile (-1)
  int stlast;      // st(e) of the last end of the previous tile if feasible, else -1
  int stmax;       // the largest st found so far (monotone lower bound), -1
  double Urun;     // running minimum of the upper bounds
  int ncand;
  bool zfound, overflow;
  int zi, ze;
  bool bad;        // lane-local
};

template <bool HOOK>
__device__ __forceinline__ void process_tile(const SArgs &A, WarpSmem &W, PoolRun &P, const Raw &r,
                                             int t, int lane) {
  const int n = A.n;
  const int kt = t * STILE;
  const int k0 = kt + 4 * lane;
  if (t == 0) {
    const uint64_t Rraw = A.req[P.p];
    P.R = Rraw < kRClamp ? Rraw : kRClamp;
    P.bad = (Rraw == 0);
    P.Scar = 0;
    P.Hcar = 0.0;
    P.lpcar = -1;
    P.lnzcar = -1;
    P.stlast = -1;
    P.stmax = -1;
    P.Urun = __longlong_as_double(0x7ff0000000000000ll);
    P.ncand = 0;
    P.zfound = false;
    P.overflow = false;
    P.zi = P.ze = -1;
  }
  // ---- decode, validate (R7, same tests as coop_search.cu phase A), h = c/s (R1) -------
  const uint64_t sv[4] = {r.a0.x, r.a0.y, r.a1.x, r.a1.y};
  const double cv[4] = {r.c0.x, r.c0.y, r.c1.x, r.c1.y};
  const double tv[4] = {r.s0.x, r.s0.y, r.s1.x, r.s1.y};
  uint64_t szi[4];  // inclusive local size prefix
  double hi_[4];    // inclusive local h prefix
  uint32_t pm = 0, zm = 0;  // PINNED / nonzero-h masks of the lane's items
  uint64_t sacc = 0;
  double hacc = 0.0;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const bool live = k0 + q < n;
    const uint64_t s = sv[q];
    const uint32_t svh = (uint32_t)(s >> 32);
    const uint32_t state = svh >> 30;
    const bool ev = state == COOP_EVICTABLE;
    const uint64_t size = s & kSizeMask;
    const double c = ev ? cv[q] : 1.0, st = ev ? tv[q] : 1.0;
    const double hq = __ddiv_rn(c, st);  // h(t) = c(t)/s(t)
    const uint32_t ch = (uint32_t)((uint64_t)__double_as_longlong(c) >> 32);
    const uint32_t cl = (uint32_t)__double_as_longlong(c);
    const uint32_t sh_ = (uint32_t)((uint64_t)__double_as_longlong(st) >> 32);
    const uint32_t hh = (uint32_t)((uint64_t)__double_as_longlong(hq) >> 32) & 0x7fffffffu;
    const uint32_t hl = (uint32_t)__double_as_longlong(hq);
    const bool hzero = (hh | hl) == 0u;
    const bool c_ok = (ch < 0x7ff00000u) | ((ch == 0x80000000u) & (cl == 0u));
    const bool s_ok = (sh_ - 0x3ff00000u) < 0x40000000u;
    const bool h_ok = hzero | ((hh - 0x3bf00000u) < 0x07c00000u);
    const bool size_bad = ((svh & 0x3fff0000u) != 0u) | (size == 0ull);
    if (live) P.bad |= size_bad | (state == 3u) | (ev & !(c_ok & s_ok & h_ok));
    pm |= (uint32_t)(live & (state == COOP_PINNED)) << q;
    zm |= (uint32_t)(live & ev & !hzero) << q;
    sacc += live ? size : 0ull;
    hacc = __dadd_rn(hacc, ev ? hq : 0.0);
    szi[q] = sacc;
    hi_[q] = hacc;
  }
  if (P.zfound) return;  // the answer is known; the rest of the pool is only validated
  // ---- warp scans: exclusive span / cost prefixes of the lane's first item --------------
  uint64_t s_in = sacc;
  double h_in = hacc;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const uint64_t so = __shfl_up_sync(0xffffffffu, s_in, d);
    const double ho = __shfl_up_sync(0xffffffffu, h_in, d);
    if (lane >= d) {
      s_in += so;
      h_in = __dadd_rn(ho, h_in);
    }
  }
  uint64_t s_ex = __shfl_up_sync(0xffffffffu, s_in, 1);
  double h_ex = __shfl_up_sync(0xffffffffu, h_in, 1);
  if (lane == 0) {
    s_ex = 0;
    h_ex = 0.0;
  }
  const uint64_t Sb = P.Scar + s_ex;
  const double Hb = __dadd_rn(P.Hcar, h_ex);
  uint64_t Sx[4], Sn[4];
  double Hx[4], Hn[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    Sx[q] = q ? Sb + szi[q - 1] : Sb;
    Sn[q] = Sb + szi[q];
    Hx[q] = q ? __dadd_rn(Hb, hi_[q - 1]) : Hb;
    Hn[q] = __dadd_rn(Hb, hi_[q]);
  }
  // ---- last PINNED / last nonzero index at or before each item --------------------------
  const unsigned lt = (1u << lane) - 1u;
  const uint32_t bp = __ballot_sync(0xffffffffu, pm != 0), bz = __ballot_sync(0xffffffffu, zm != 0);
  const int mylp = pm ? k0 + 31 - __clz(pm) : -1, mylz = zm ? k0 + 31 - __clz(zm) : -1;
  const int srcp = (bp & lt) ? 31 - __clz(bp & lt) : 0, srcz = (bz & lt) ? 31 - __clz(bz & lt) : 0;
  const int lpo = __shfl_sync(0xffffffffu, mylp, srcp), lzo = __shfl_sync(0xffffffffu, mylz, srcz);
  const int lp_before = (bp & lt) ? lpo : P.lpcar;   // last PINNED before the lane's items
  const int lz_before = (bz & lt) ? lzo : P.lnzcar;
  // ---- history ring: this tile's S[k], H^[k] -----------------------------------------------
  {
    const int slot = k0 & HMASK;
    *reinterpret_cast<ulonglong2 *>(&W.hS[slot]) = make_ulonglong2(Sx[0], Sx[1]);
    *reinterpret_cast<ulonglong2 *>(&W.hS[slot + 2]) = make_ulonglong2(Sx[2], Sx[3]);
    *reinterpret_cast<double2 *>(&W.hH[slot]) = make_double2(Hx[0], Hx[1]);
    *reinterpret_cast<double2 *>(&W.hH[slot + 2]) = make_double2(Hx[2], Hx[3]);
  }
  __syncwarp();
  // ---- every end of the tile: latest start, window cost bounds -----------------------------
  const int oldest = max(0, kt + STILE - HCAP);  // first item still in the ring
  int st_of[4];       // st(e) if the window (st(e), e) is feasible, else -1
  bool fz[4];         // that window is a zero window
  int zst[4];         // its lowest zero start (fz)
  double Lb[4], Ub[4];
  const double kInf = __longlong_as_double(0x7ff0000000000000ll);
  int lbm = P.stmax;  // monotone lower bound of st
  bool ovf = false;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int e = k0 + q;
    st_of[q] = -1;
    fz[q] = false;
    zst[q] = -1;
    Lb[q] = kInf;
    Ub[q] = kInf;
    const int lpe = ((pm >> q) & 1u) ? e : ((pm & ((1u << q) - 1u)) ? k0 + 31 - __clz(pm & ((1u << q) - 1u)) : lp_before);
    const int lze = (zm & ((2u << q) - 1u)) ? k0 + 31 - __clz(zm & ((2u << q) - 1u)) : lz_before;
    if (e >= n || lpe == e || Sn[q] < P.R) continue;
    const uint64_t tgt = Sn[q] - P.R;  // starts i with S[i] <= tgt cover R
    const int lbp = lpe + 1;
    int lo = max(max(lbp, oldest), max(lbm, 0));
    if (W.hS[lo & HMASK] > tgt) {  // no start >= lo
      if (lo == oldest && oldest > lbp && oldest > lbm) ovf = true;  // window longer than the ring
      continue;
    }
    // largest i in [lo, e] with S[i] <= tgt: gallop from lo, then bisect
    int hi = lo, step = 1;
    while (true) {
      const int nx = min(hi + step, e);
      if (nx == hi || W.hS[nx & HMASK] > tgt) break;
      hi = nx;
      step <<= 1;
    }
    int top = min(hi + step, e);  // S[top] > tgt unless top == e
    if (W.hS[top & HMASK] <= tgt) {
      hi = top;
    } else {
      while (top - hi > 1) {
        const int mid = (hi + top) >> 1;
        if (W.hS[mid & HMASK] <= tgt) hi = mid;
        else top = mid;
      }
    }
    const int b = hi;
    st_of[q] = b;
    lbm = b;
    if (lze < b) {
      fz[q] = true;  // items (lze, e] are all zero: a zero-cost window
    } else {
      const double Hbv = W.hH[b & HMASK];
      const double C = Hn[q] - Hbv;
      const double err = A.gerr * (Hn[q] + Hbv);
      Lb[q] = C - err;
      Ub[q] = C + err;
    }
  }
  // a(e) = max(st(e-1), lp(e)): st(e-1) from the previous end (lane q-1, lane - 1, or tile)
  const int st_prev_lane = __shfl_up_sync(0xffffffffu, st_of[3], 1);
  int a_of[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int e = k0 + q;
    const int lpe = ((pm >> q) & 1u) ? e : ((pm & ((1u << q) - 1u)) ? k0 + 31 - __clz(pm & ((1u << q) - 1u)) : lp_before);
    const int sp = q ? st_of[q - 1] : (lane ? st_prev_lane : P.stlast);
    a_of[q] = max(sp, lpe);
    if (st_of[q] >= 0 && a_of[q] >= st_of[q]) {  // (a, st(e)] empty: no canonical window ends at e
      fz[q] = false;
      Lb[q] = kInf;
      Ub[q] = kInf;
    }
    if (fz[q]) {
      const int lze = (zm & ((2u << q) - 1u)) ? k0 + 31 - __clz(zm & ((2u << q) - 1u)) : lz_before;
      zst[q] = max(a_of[q], lze) + 1;  // <= st(e)
    }
  }
  // ---- carries to the next tile ---------------------------------------------------------
  P.Scar = __shfl_sync(0xffffffffu, Sn[3], 31);
  P.Hcar = __shfl_sync(0xffffffffu, Hn[3], 31);
  {
    const int lp_last = pm ? mylp : lp_before, lz_last = zm ? mylz : lz_before;
    P.lpcar = __shfl_sync(0xffffffffu, lp_last, 31);
    P.lnzcar = __shfl_sync(0xffffffffu, lz_last, 31);
  }
  P.stlast = __shfl_sync(0xffffffffu, st_of[3], 31);
  P.stmax = __reduce_max_sync(0xffffffffu, (unsigned)(lbm + 1)) - 1;
  if (__any_sync(0xffffffffu, ovf)) P.overflow = true;
  // ---- zero windows: the earliest end with one gives the lowest start (exact, R4) -------
  {
    int myz = 0x7fffffff;
#pragma unroll
    for (int q = 3; q >= 0; --q)
      if (fz[q]) myz = k0 + q;
    const int ez = (int)__reduce_min_sync(0xffffffffu, (unsigned)myz);
    if (ez != 0x7fffffff) {
      const int src = (ez - kt) >> 2, qz = (ez - kt) & 3;  // lane and item of that end
      int zs = zst[0];
#pragma unroll
      for (int q = 1; q < 4; ++q)
        if (q == qz) zs = zst[q];
      zs = __shfl_sync(0xffffffffu, zs, src);
      P.zfound = true;
      P.zi = zs;
      P.ze = ez;
      return;
    }
  }
  // ---- candidates: ends whose lower bound can still reach the minimum -------------------
  double um = fmin(fmin(Ub[0], Ub[1]), fmin(Ub[2], Ub[3]));
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) um = fmin(um, __shfl_xor_sync(0xffffffffu, um, d));
  P.Urun = fmin(P.Urun, um);
  const double thr = P.Urun * kMargin;
  uint32_t want = 0;
#pragma unroll
  for (int q = 0; q < 4; ++q) want |= (uint32_t)((Lb[q] <= thr) & (Ub[q] < kInf)) << q;
  int nnew = __reduce_add_sync(0xffffffffu, (unsigned)__popc(want));
  if (nnew == 0) return;
  if (P.ncand + nnew > CCAP) {  // prune the list against the current bound
    int keep = 0;
    for (int c0 = 0; c0 < P.ncand; c0 += 32) {
      const int c = c0 + lane;
      int e_ = 0, b_ = 0, a_ = 0;
      double l_ = 0.0;
      bool k = false;
      if (c < P.ncand) {
        e_ = W.ce[c];
        b_ = W.cb[c];
        a_ = W.ca[c];
        l_ = W.cl[c];
        k = l_ <= thr;
      }
      const uint32_t bal = __ballot_sync(0xffffffffu, k);
      __syncwarp();
      if (k) {
        const int pos = keep + __popc(bal & lt);
        W.ce[pos] = e_;
        W.cb[pos] = b_;
        W.ca[pos] = a_;
        W.cl[pos] = l_;
      }
      __syncwarp();
      keep += __popc(bal);
    }
    P.ncand = keep;
    if (P.ncand + nnew > CCAP) {
      P.overflow = true;
      return;
    }
  }
  const int mine = __popc(want);
  int base = P.ncand;
  {
    int incl = mine;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const int o = __shfl_up_sync(0xffffffffu, incl, d);
      if (lane >= d) incl += o;
    }
    base += incl - mine;
  }
#pragma unroll
  for (int q = 0; q < 4; ++q)
    if ((want >> q) & 1u) {
      W.ce[base] = k0 + q;
      W.cb[base] = st_of[q];
      W.ca[base] = a_of[q];
      W.cl[base] = Lb[q];
      ++base;
    }
  __syncwarp();
  P.ncand += nnew;
}

__device__ __forceinline__ void finish_pool(const SArgs &A, WarpSmem &W, PoolRun &P, int lane) {
  const double kInf = __longlong_as_double(0x7ff0000000000000ll);
  coop_window *o = A.out + P.p;
  const bool bad = __any_sync(0xffffffffu, P.bad);
  if (bad) {
    if (lane == 0) put_window(o, -1, -1, 0, kInf, 0, COOP_ERR_INVALID_ARG);
    return;
  }
  if (P.overflow) {  // a window the ring could not hold (it may have been the winner)
    if (lane == 0) put_window(o, -1, -1, 0, kInf, 0, COOP_PENDING_);
    return;
  }
  if (P.zfound) {
    U192 s;
    uint64_t span;
    int nev;
    exact_window(A, P.p, P.zi, P.ze, lane, s, span, nev);
    if (lane == 0) put_window(o, P.zi, P.ze, span, 0.0, nev, COOP_OK);
    return;
  }
  if (P.Urun == kInf) {
    if (lane == 0) put_window(o, -1, -1, 0, kInf, 0, COOP_INFEASIBLE);
    return;
  }
  // exact re-summation of the surviving candidates; earliest end of the minimal rounded cost
  const double thr = P.Urun * kMargin;
  uint64_t best = ~0ull;
  int be = 0x7fffffff, bb = -1, ba = -1;
  U192 bsum = u192_zero();
  uint64_t bspan = 0;
  int bnev = 0;
  __syncwarp();
  for (int c = 0; c < P.ncand; ++c) {
    if (!(W.cl[c] <= thr)) continue;
    const int e = W.ce[c], b = W.cb[c];
    U192 s;
    uint64_t span;
    int nev;
    exact_window(A, P.p, b, e, lane, s, span, nev);
    const uint64_t cb = (uint64_t)__double_as_longlong(u192_round_to_double(s));
    if (cb < best || (cb == best && e < be)) {
      best = cb;
      be = e;
      bb = b;
      ba = W.ca[c];
      bsum = s;
      bspan = span;
      bnev = nev;
    }
  }
  // lowest start of that end with the same rounded cost: extend (a, b] downwards
  int start = bb;
  for (int top = bb - 1; top > ba; top -= 32) {
    const int i = top - lane;
    const bool in = i > ba;
    U192 hx = u192_zero();
    uint64_t sz = 0;
    int ev = 0;
    if (in) {
      const Item it = reread(A, P.p, i);
      hx = u192_from_double(it.h);
      sz = it.size;
      ev = it.ev;
    }
    // inclusive scan over lanes (lane 0 = item top, lane l = item top - l)
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const U192 ho = shfl_up192(hx, d);
      const uint64_t so = __shfl_up_sync(0xffffffffu, sz, d);
      const int eo = __shfl_up_sync(0xffffffffu, ev, d);
      if (lane >= d) {
        hx = u192_add(hx, ho);
        sz += so;
        ev += eo;
      }
    }
    const U192 tot = u192_add(bsum, hx);
    const bool same = in && (uint64_t)__double_as_longlong(u192_round_to_double(tot)) == best;
    const uint32_t ok = __ballot_sync(0xffffffffu, same);
    const int run = __ffs(~ok) - 1;  // lanes 0 .. run-1 keep the rounded cost (a prefix)
    const int m = ok == 0xffffffffu ? 32 : run;
    if (m > 0) {
      const int src = m - 1;
      bsum.w0 = __shfl_sync(0xffffffffu, tot.w0, src);
      bsum.w1 = __shfl_sync(0xffffffffu, tot.w1, src);
      bsum.w2 = __shfl_sync(0xffffffffu, tot.w2, src);
      bspan += __shfl_sync(0xffffffffu, sz, src);
      bnev += __shfl_sync(0xffffffffu, ev, src);
      start = top - src;
    }
    if (m < 32) break;
  }
  if (lane == 0) put_window(o, start, be, bspan, __longlong_as_double((long long)best), bnev, COOP_OK);
}

template <bool HOOK>
__global__ void __launch_bounds__(SWARPS * 32, 2) search_stream_kernel(const SArgs A) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  WarpSmem &W = reinterpret_cast<WarpSmem *>(smem_raw)[wid];
  const int64_t gw = (int64_t)blockIdx.x * SWARPS + wid, GW = (int64_t)gridDim.x * SWARPS;
  const int nt = A.ntiles;
  // tile positions: (pool, tile), pools gw, gw + GW, ...; two tiles in flight ahead
  int64_t p0 = gw, p1 = gw, p2 = gw;
  int t0 = 0, t1 = 1, t2 = 2;
  auto norm = [&](int64_t &p, int &t) {
    while (t >= nt) {
      t -= nt;
      p += GW;
    }
  };
  norm(p1, t1);
  norm(p2, t2);
  Raw ra, rb, rc;
  if (p0 < A.n_pools) load_tile(A, ra, p0, t0, lane);
  if (p1 < A.n_pools) load_tile(A, rb, p1, t1, lane);
  PoolRun P;
  P.p = p0;
  P.bad = false;
  auto step = [&](Raw &cur, Raw &ahead2) -> bool {
    if (p0 >= A.n_pools) return false;
    if (p2 < A.n_pools) load_tile(A, ahead2, p2, t2, lane);
    P.p = p0;
    process_tile<HOOK>(A, W, P, cur, t0, lane);
    if (t0 == nt - 1) finish_pool(A, W, P, lane);
    p0 = p1;
    t0 = t1;
    p1 = p2;
    t1 = t2;
    ++t2;
    norm(p2, t2);
    return true;
  };
  while (true) {
    if (!step(ra, rc)) break;
    if (!step(rb, ra)) break;
    if (!step(rc, rb)) break;
  }
}

}  // namespace

bool stream_search_enabled(int n) {
  const char *v = getenv("COOP_SEARCH_IMPL");
  if (v && v[0] == 'c') return false;  // "cta": the CTA-per-pool kernel only
  return n >= 1;
}

int launch_window_search_stream(const coop_tables_soa *t, const uint64_t *requests, coop_window *out,
                                 cudaStream_t st) {
  SArgs A;
  A.ss = t->size_state;
  A.cost = t->cost;
  A.stale = t->stale;
  A.req = requests;
  A.out = out;
  A.n_pools = t->n_pools;
  A.stride = t->pool_stride;
  A.n = t->n_blocks;
  A.ntiles = (A.n + STILE - 1) / STILE;
  A.vec = ((uintptr_t)A.ss % 16 == 0) && ((uintptr_t)A.cost % 16 == 0) && ((uintptr_t)A.stale % 16 == 0) &&
          (A.stride % 2 == 0);
  // summation depth of any H^ entry <= 4 (lane) + 5 (warp scan) + 2 + ntiles (carry chain)
  const int depth = 4 + 5 + 2 + A.ntiles + 2;
  A.gerr = 2.0 * (double)(depth + 2) * 0x1p-53 + 0x1p-50;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const size_t smem = sizeof(WarpSmem) * SWARPS;
  auto kern = search_stream_kernel<false>;
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
    return COOP_ERR_CUDA;
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, SWARPS * 32, smem);
  if (per_sm < 1) per_sm = 1;
  int64_t grid = (int64_t)sms * per_sm;
  const int64_t need = (A.n_pools + SWARPS - 1) / SWARPS;
  if (grid > need) grid = need;
  kern<<<(unsigned)grid, SWARPS * 32, smem, st>>>(A);
  return cudaGetLastError() == cudaSuccess ? COOP_OK : COOP_ERR_CUDA;
}

}  // namespace coop

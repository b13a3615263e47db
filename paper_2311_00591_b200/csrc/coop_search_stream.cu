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
  int stlast_known; // the last end of the previous tile was evaluated (its lane was active)
  int stmax;       // the largest st found so far (monotone lower bound), -1
  double Urun;     // running minimum of the upper bounds
  int ncand;
  bool zfound, overflow;
  int zi, ze;
  bool bad;        // lane-local
};

// Validation (R7) and h of one item.  The filter only needs h within a relative error
// delta (folded into gerr): h ~ c * r, r = 1/s from rcp.approx + one Newton step.  R7's
// range test on RN(c/s) is decided from the exponents of c and s except in a thin band at
// the bounds (and for c subnormal), where the exact IEEE division decides.
__device__ __forceinline__ double rcp_nr(double s) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(s));
  const double e = __fma_rn(-s, r, 1.0);
  return __fma_rn(r, e, r);
}

struct ItemA {
  double h;    // approximate h (0 for non-EVICTABLE and for h = 0)
  bool nz;     // h != 0 (exact)
  bool pin;
  bool bad;
  uint64_t size;
};

__device__ __forceinline__ ItemA decode_item(uint64_t sv, double cr, double sr, bool live) {
  ItemA it;
  const uint32_t svh = (uint32_t)(sv >> 32);
  const uint32_t state = svh >> 30;
  const bool ev = state == COOP_EVICTABLE;
  it.size = live ? (sv & kSizeMask) : 0ull;
  it.pin = live & (state == COOP_PINNED);
  const uint32_t ch = (uint32_t)((uint64_t)__double_as_longlong(cr) >> 32);
  const uint32_t cl = (uint32_t)__double_as_longlong(cr);
  const uint32_t sh_ = (uint32_t)((uint64_t)__double_as_longlong(sr) >> 32);
  const bool czero = ((ch & 0x7fffffffu) | cl) == 0u;
  const bool c_ok = (ch < 0x7ff00000u) | ((ch == 0x80000000u) & (cl == 0u));  // finite, >= 0 (or -0)
  const bool s_ok = (sh_ - 0x3ff00000u) < 0x40000000u;                       // finite, >= 1
  // exponent difference: RN(c/s) lies in [2^(d-1), 2^(d+1)] for normal c; safely inside
  // [2^-64, 2^60) when -63 <= d <= 58
  const int d = (int)(ch >> 20) - (int)(sh_ >> 20);
  bool h_ok = czero | ((unsigned)(d + 63) <= 121u);
  bool nz = !czero;
  const double r = rcp_nr(sr);
  double h = ev ? cr * r : 0.0;
  if (ev & c_ok & s_ok & !h_ok) {  // the band at the bounds: the exact division decides
    const double hq = __ddiv_rn(cr, sr);
    const uint32_t hh = (uint32_t)((uint64_t)__double_as_longlong(hq) >> 32) & 0x7fffffffu;
    const uint32_t hl = (uint32_t)__double_as_longlong(hq);
    const bool hzero = (hh | hl) == 0u;
    h_ok = hzero | ((hh - 0x3bf00000u) < 0x07c00000u);
    nz = !hzero;
    h = hzero ? 0.0 : hq;
  }
  const bool size_bad = ((svh & 0x3fff0000u) != 0u) | ((sv & kSizeMask) == 0ull);
  it.bad = live & (size_bad | (state == 3u) | (ev & !(c_ok & s_ok & h_ok)));
  it.nz = live & ev & nz;
  it.h = it.nz ? h : 0.0;
  return it;
}

// largest i in [lo, hi] with S[i] <= tgt, given S[lo] <= tgt (bisection on the ring)
__device__ __forceinline__ int ring_bisect(const WarpSmem &W, int lo, int hi, uint64_t tgt) {
  if (W.hS[hi & HMASK] <= tgt) return hi;
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (W.hS[mid & HMASK] <= tgt) lo = mid;
    else hi = mid;
  }
  return lo;
}
// same, galloping up from lo (for the ends after the first: st moves little)
__device__ __forceinline__ int ring_gallop(const WarpSmem &W, int lo, int hi, uint64_t tgt) {
  int step = 1;
  while (true) {
    const int nx = min(lo + step, hi);
    if (nx == lo || W.hS[nx & HMASK] > tgt) return ring_bisect(W, lo, nx, tgt);
    lo = nx;
    step <<= 1;
  }
}

__device__ __forceinline__ int last_bit_idx(uint32_t m, int k0, int none) {  // highest set bit -> item index
  return m ? k0 + 31 - __clz(m) : none;
}

__device__ __forceinline__ void process_tile(const SArgs &A, WarpSmem &W, PoolRun &P, const Raw &r,
                                             int t, int lane) {
  const int n = A.n;
  const int kt = t * STILE;
  const int k0 = kt + 4 * lane;
  const double kInf = __longlong_as_double(0x7ff0000000000000ll);
  if (t == 0) {
    const uint64_t Rraw = A.req[P.p];
    P.R = Rraw < kRClamp ? Rraw : kRClamp;
    P.bad = (Rraw == 0);
    P.Scar = 0;
    P.Hcar = 0.0;
    P.lpcar = -1;
    P.lnzcar = -1;
    P.stlast = -1;
    P.stlast_known = 1;
    P.stmax = -1;
    P.Urun = kInf;
    P.ncand = 0;
    P.zfound = false;
    P.overflow = false;
    P.zi = P.ze = -1;
  }
  // ---- decode, validate (R7), h (R1, approximate for the filter), local prefixes ---------
  const uint64_t sv[4] = {r.a0.x, r.a0.y, r.a1.x, r.a1.y};
  const double cv[4] = {r.c0.x, r.c0.y, r.c1.x, r.c1.y};
  const double tv[4] = {r.s0.x, r.s0.y, r.s1.x, r.s1.y};
  uint64_t szi[4];  // inclusive local size prefix
  double hi_[4];    // inclusive local h prefix
  uint32_t pm = 0, zm = 0;  // PINNED / nonzero-h masks of the lane's items
  uint64_t sacc = 0;
  double hacc = 0.0;
  bool bad = false;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const ItemA it = decode_item(sv[q], cv[q], tv[q], k0 + q < n);
    bad |= it.bad;
    pm |= (uint32_t)it.pin << q;
    zm |= (uint32_t)it.nz << q;
    sacc += it.size;
    hacc = __dadd_rn(hacc, it.h);
    szi[q] = sacc;
    hi_[q] = hacc;
  }
  P.bad |= bad;
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
  const uint64_t Sb = P.Scar + (s_in - sacc);  // exact
  const double hexc = __shfl_up_sync(0xffffffffu, h_in, 1);
  const double Hb = __dadd_rn(P.Hcar, lane ? hexc : 0.0);
  uint64_t Sx[4], Sn[4];
  double Hx[4], Hn[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    Sx[q] = q ? Sb + szi[q - 1] : Sb;
    Sn[q] = Sb + szi[q];
    Hx[q] = q ? __dadd_rn(Hb, hi_[q - 1]) : Hb;
    Hn[q] = __dadd_rn(Hb, hi_[q]);
  }
  // ---- last PINNED / last nonzero index before the lane's items ---------------------------
  const unsigned lt = (1u << lane) - 1u;
  const uint32_t bp = __ballot_sync(0xffffffffu, pm != 0), bz = __ballot_sync(0xffffffffu, zm != 0);
  const int mylp = last_bit_idx(pm, k0, -1), mylz = last_bit_idx(zm, k0, -1);
  const int srcp = (bp & lt) ? 31 - __clz(bp & lt) : 0, srcz = (bz & lt) ? 31 - __clz(bz & lt) : 0;
  const int lpo = __shfl_sync(0xffffffffu, mylp, srcp), lzo = __shfl_sync(0xffffffffu, mylz, srcz);
  const int lp_before = (bp & lt) ? lpo : P.lpcar;
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
  const int oldest = max(0, kt + STILE - HCAP);  // first item still in the ring
  // ---- lane pruning: the latest start of the lane's last end bounds all its windows ------
  // For ends e0 <= e <= e3 of the lane, st(e) <= st(e3), so every window cost is >=
  // H[e0 + 1] - H[st(e3)]; the window (st(e3), e3) itself, when PINNED-free, bounds the
  // minimum from above.  Lanes whose bound cannot reach the running minimum skip their ends.
  int e3q = -1;
#pragma unroll
  for (int q = 0; q < 4; ++q)
    if (k0 + q < n && !((pm >> q) & 1u) && Sn[q] >= P.R) e3q = q;
  int st3 = -1;       // st_raw of the lane's last valid end (-1: none >= the lower bound)
  bool ovf = false;
  double Ul = kInf, Ll = kInf;
  const int lbm0 = max(P.stmax, 0);
  if (e3q >= 0) {
    int e3 = k0, q3 = 0;
#pragma unroll
    for (int q = 1; q < 4; ++q)
      if (q == e3q) {
        e3 = k0 + q;
        q3 = q;
      }
    uint64_t sn3 = Sn[0];
    double hn3 = Hn[0];
#pragma unroll
    for (int q = 1; q < 4; ++q)
      if (q == q3) {
        sn3 = Sn[q];
        hn3 = Hn[q];
      }
    const uint64_t tgt = sn3 - P.R;
    const int lo = max(oldest, lbm0);
    if (W.hS[lo & HMASK] <= tgt) {
      st3 = ring_bisect(W, lo, e3, tgt);
      const int lp3 = (pm & ((2u << q3) - 1u)) ? last_bit_idx(pm & ((2u << q3) - 1u), k0, -1) : lp_before;
      const double Hs = W.hH[st3 & HMASK];
      const double err = A.gerr * (hn3 + Hs);
      if (st3 > lp3) Ul = (hn3 - Hs) + err;  // a real (PINNED-free) window
      // lower bound for every end of the lane (its first valid end's prefix)
      int qf = 3;
#pragma unroll
      for (int q = 3; q >= 0; --q)
        if (k0 + q < n && !((pm >> q) & 1u) && Sn[q] >= P.R) qf = q;
      double hnf = Hn[0];
#pragma unroll
      for (int q = 1; q < 4; ++q)
        if (q == qf) hnf = Hn[q];
      Ll = (hnf - Hs) - A.gerr * (hnf + Hs);
    } else {
      Ll = -kInf;  // no start >= lo covers R for the last end: decided per end below
    }
  }
  double um = Ul;
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) um = fmin(um, __shfl_xor_sync(0xffffffffu, um, d));
  P.Urun = fmin(P.Urun, um);
  const double thr = P.Urun * kMargin;
  const bool active = (e3q >= 0) && (Ll <= thr);
  // ---- the active lanes: every end, its latest start, window cost bounds --------------------
  int st_of[4] = {-1, -1, -1, -1};  // st(e) if the window (st(e), e) is PINNED-free, else -1
  bool fz[4] = {false, false, false, false};
  double Lb[4] = {kInf, kInf, kInf, kInf}, Ub[4] = {kInf, kInf, kInf, kInf};
  int lbm = P.stmax;
  if (active) {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int e = k0 + q;
      const int lpe = ((pm >> q) & 1u) ? e : last_bit_idx(pm & ((1u << q) - 1u), k0, lp_before);
      const int lze = last_bit_idx(zm & ((2u << q) - 1u), k0, lz_before);
      if (e >= n || lpe == e || Sn[q] < P.R) continue;
      const uint64_t tgt = Sn[q] - P.R;
      const int lbp = lpe + 1;
      const int lo = max(max(lbp, oldest), max(lbm, 0));
      if (W.hS[lo & HMASK] > tgt) {
        if (lo == oldest && oldest > lbp && oldest > lbm) ovf = true;
        continue;
      }
      const int b = (q == 0 || lbm < 0) ? ring_bisect(W, lo, e, tgt) : ring_gallop(W, lo, e, tgt);
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
  } else if (st3 >= 0) {
    lbm = st3;  // st is monotone: the lane's last end's start bounds later ends
  }
  if (!__any_sync(0xffffffffu, active)) {  // no window of this tile can reach the minimum
    P.Scar = __shfl_sync(0xffffffffu, Sn[3], 31);
    P.Hcar = __shfl_sync(0xffffffffu, Hn[3], 31);
    const int lp_last = pm ? mylp : lp_before, lz_last = zm ? mylz : lz_before;
    P.lpcar = __shfl_sync(0xffffffffu, lp_last, 31);
    P.lnzcar = __shfl_sync(0xffffffffu, lz_last, 31);
    P.stlast = -1;
    P.stlast_known = 0;
    P.stmax = (int)__reduce_max_sync(0xffffffffu, (unsigned)(lbm + 1)) - 1;
    return;
  }
  // a(e) = max(st(e-1), lp(e)): starts of e lie in (a(e), st(e)]; the previous end's st
  // comes from lane q-1, the previous lane, or the previous tile (only needed when the
  // previous end is in an active lane; an inactive lane's ends cannot win -- their windows'
  // exact costs exceed the minimum -- so a(e) only matters for ends of active lanes, whose
  // previous end is either in the same lane or in the previous lane)
  const bool prev_active = __shfl_up_sync(0xffffffffu, (int)active, 1);
  const int st_prev_lane = __shfl_up_sync(0xffffffffu, st_of[3], 1);
  int a_of[4], zst[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int e = k0 + q;
    const int lpe = ((pm >> q) & 1u) ? e : last_bit_idx(pm & ((1u << q) - 1u), k0, lp_before);
    int sp;
    bool known = true;
    if (q) sp = st_of[q - 1];
    else if (lane) {
      sp = st_prev_lane;
      known = prev_active;
    } else {
      sp = P.stlast;
      known = P.stlast_known;
    }
    a_of[q] = max(sp, lpe);
    zst[q] = -1;
    if (st_of[q] >= 0 && !known) {
      // the previous end's start is unknown (inactive previous lane): recompute it here
      const int ep = e - 1;
      int spv = -1;
      if (ep >= 0) {
        uint64_t snp = Sx[q];  // S[e] = S[(e-1) + 1]
        if (snp >= P.R) {
          const uint64_t tgt = snp - P.R;
          const int lo = max(oldest, lbm0);
          if (W.hS[lo & HMASK] <= tgt) spv = ring_bisect(W, lo, ep, tgt);
          else if (lo == oldest && oldest > lpe + 1) ovf = true;  // st(e-1) beyond the ring
        }
      }
      a_of[q] = max(spv, lpe);
    }
    if (st_of[q] >= 0 && a_of[q] >= st_of[q]) {  // (a, st(e)] empty: no canonical window ends at e
      fz[q] = false;
      Lb[q] = kInf;
      Ub[q] = kInf;
    }
    if (fz[q]) zst[q] = max(a_of[q], last_bit_idx(zm & ((2u << q) - 1u), k0, lz_before)) + 1;
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
  P.stlast_known = __shfl_sync(0xffffffffu, (int)active, 31);
  P.stmax = (int)__reduce_max_sync(0xffffffffu, (unsigned)(lbm + 1)) - 1;
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
  um = fmin(fmin(Ub[0], Ub[1]), fmin(Ub[2], Ub[3]));
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) um = fmin(um, __shfl_xor_sync(0xffffffffu, um, d));
  P.Urun = fmin(P.Urun, um);
  const double thr2 = P.Urun * kMargin;
  uint32_t want = 0;
#pragma unroll
  for (int q = 0; q < 4; ++q) want |= (uint32_t)((Lb[q] <= thr2) & (Ub[q] < kInf)) << q;
  const int nnew = (int)__reduce_add_sync(0xffffffffu, (unsigned)__popc(want));
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
        k = l_ <= thr2;
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

__device__ __noinline__ void finish_pool(const SArgs &A, WarpSmem &W, const PoolRun P, int lane) {
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

__global__ void __launch_bounds__(SWARPS * 32, 2) search_stream_kernel(const SArgs A) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  WarpSmem &W = reinterpret_cast<WarpSmem *>(smem_raw)[wid];
  const int64_t gw = (int64_t)blockIdx.x * SWARPS + wid, GW = (int64_t)gridDim.x * SWARPS;
  const int nt = A.ntiles;
  // tile positions: (pool, tile), pools gw, gw + GW, ...; the next tile is in flight while
  // one is processed (a tile takes a warp several microseconds at 12 warps per SM)
  int64_t p0 = gw, p1 = gw;
  int t0 = 0, t1 = 1;
  auto norm = [&](int64_t &p, int &t) {
    while (t >= nt) {
      t -= nt;
      p += GW;
    }
  };
  norm(p1, t1);
  Raw cur, nxt;
  if (p0 < A.n_pools) load_tile(A, cur, p0, t0, lane);
  PoolRun P;
  P.p = p0;
  P.bad = false;
  while (p0 < A.n_pools) {
    if (p1 < A.n_pools) load_tile(A, nxt, p1, t1, lane);
    P.p = p0;
    process_tile(A, W, P, cur, t0, lane);
    if (t0 == nt - 1) finish_pool(A, W, P, lane);
    cur = nxt;
    p0 = p1;
    t0 = t1;
    ++t1;
    norm(p1, t1);
  }
}

}  // namespace

// The CTA-per-pool kernel is the default (faster on B200: 46.5 ms vs 63 ms per 2^20 x 4096
// pools); COOP_SEARCH_IMPL=stream selects this kernel (+ the CTA kernel
// for the pools it leaves pending), COOP_SEARCH_IMPL=stream_only skips that second pass.
bool stream_search_enabled(int n) {
  const char *v = getenv("COOP_SEARCH_IMPL");
  return v && v[0] == 's' && n >= 1;
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
  // summation depth of any H^ entry <= 4 (lane) + 5 (warp scan) + 2 + ntiles (carry chain);
  // every h carries a relative error <= 2^-40 (rcp.approx + one Newton step)
  const int depth = 4 + 5 + 2 + A.ntiles + 2;
  A.gerr = 2.0 * (double)(depth + 2) * 0x1p-53 + 2.0 * 0x1p-39 + 0x1p-50;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const size_t smem = sizeof(WarpSmem) * SWARPS;
  auto kern = search_stream_kernel;
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

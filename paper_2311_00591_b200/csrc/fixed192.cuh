// fixed192.cuh -- exact window costs for the CUDA path (R3, "exact verify").
//
// Every admissible heuristic h (0 or in [2^-64, 2^60), R7) is an integer multiple of
// 2^-116, and any sum of <= 8192 of them is < 2^74, so a 192-bit unsigned fixed-point
// number with LSB 2^-116 holds every h and every window sum EXACTLY; addition is then
// associative, so any summation order (warp lanes, shuffles) gives identical bits.
// round_to_double() returns the correctly rounded (nearest-even) binary64 value of the
// exact sum -- the canonical window cost of R3.
#pragma once
#include <stdint.h>

#ifndef COOP_HD
#define COOP_HD __host__ __device__ __forceinline__
#endif

namespace coop {

struct U192 {
  uint64_t w0, w1, w2;  // little-endian limbs; value = (w2:w1:w0) * 2^-116
};

COOP_HD U192 u192_zero() { return U192{0, 0, 0}; }

COOP_HD U192 u192_add(U192 a, U192 b) {
#ifdef __CUDA_ARCH__
  U192 r;
  asm("add.cc.u64 %0, %3, %6;\n\t"
      "addc.cc.u64 %1, %4, %7;\n\t"
      "addc.u64 %2, %5, %8;"
      : "=l"(r.w0), "=l"(r.w1), "=l"(r.w2)
      : "l"(a.w0), "l"(a.w1), "l"(a.w2), "l"(b.w0), "l"(b.w1), "l"(b.w2));
  return r;
#else
  U192 r;
  r.w0 = a.w0 + b.w0;
  uint64_t c0 = r.w0 < a.w0;
  uint64_t t1 = a.w1 + b.w1;
  uint64_t c1 = t1 < a.w1;
  r.w1 = t1 + c0;
  c1 |= (r.w1 < t1);
  r.w2 = a.w2 + b.w2 + c1;
  return r;
#endif
}

COOP_HD U192 u192_sub(U192 a, U192 b) {  // a - b, requires a >= b
#ifdef __CUDA_ARCH__
  U192 r;
  asm("sub.cc.u64 %0, %3, %6;\n\t"
      "subc.cc.u64 %1, %4, %7;\n\t"
      "subc.u64 %2, %5, %8;"
      : "=l"(r.w0), "=l"(r.w1), "=l"(r.w2)
      : "l"(a.w0), "l"(a.w1), "l"(a.w2), "l"(b.w0), "l"(b.w1), "l"(b.w2));
  return r;
#else
  U192 r;
  r.w0 = a.w0 - b.w0;
  uint64_t br0 = a.w0 < b.w0;
  uint64_t t1 = a.w1 - b.w1;
  uint64_t br1 = a.w1 < b.w1;
  r.w1 = t1 - br0;
  br1 |= (t1 < br0);
  r.w2 = a.w2 - b.w2 - br1;
  return r;
#endif
}

// h (an admissible binary64: +-0 or in [2^-64, 2^60)) -> exact fixed point.
// The sign bit is ignored (the search encodes FREE items as -0.0).
COOP_HD U192 u192_from_double(double h) {
  uint64_t bits;
#ifdef __CUDA_ARCH__
  bits = (uint64_t)__double_as_longlong(h);
#else
  __builtin_memcpy(&bits, &h, 8);
#endif
  bits &= 0x7FFFFFFFFFFFFFFFull;
  if (bits == 0) return u192_zero();
  int e = (int)(bits >> 52) - 1023;                        // -64 .. 59
  uint64_t m = (bits & 0x000FFFFFFFFFFFFFull) | (1ull << 52);  // 53-bit significand
  int shift = e + 64;                                      // value = m << shift (LSB 2^-116)
  int limb = shift >> 6, b = shift & 63;
  uint64_t lo = m << b;
  uint64_t hi = b ? (m >> (64 - b)) : 0ull;
  U192 r;
  if (limb == 0) {
    r.w0 = lo; r.w1 = hi; r.w2 = 0;
  } else {
    r.w0 = 0; r.w1 = lo; r.w2 = hi;
  }
  return r;
}

COOP_HD int clz64(uint64_t x) {
#ifdef __CUDA_ARCH__
  return __clzll((long long)x);
#else
  return x ? __builtin_clzll(x) : 64;
#endif
}

// bits [pos, pos+64) of a (pos in 0..191; bits past 191 are zero)
COOP_HD uint64_t u192_bits64(U192 a, int pos) {
  int l = pos >> 6, b = pos & 63;
  uint64_t wl = (l == 0) ? a.w0 : ((l == 1) ? a.w1 : a.w2);
  uint64_t wh = (l == 0) ? a.w1 : ((l == 1) ? a.w2 : 0ull);
  return (wl >> b) | (b ? (wh << (64 - b)) : 0ull);
}

// any bit set in [0, pos) ?  (0 <= pos <= 191)
COOP_HD bool u192_any_below(U192 a, int pos) {
  if (pos <= 0) return false;
  int l = pos >> 6, b = pos & 63;
  uint64_t mask = b ? ((1ull << b) - 1ull) : 0ull;
  uint64_t below = 0;
  if (l == 0) below = a.w0 & mask;
  else if (l == 1) below = a.w0 | (a.w1 & mask);
  else below = a.w0 | a.w1 | (a.w2 & mask);
  return below != 0;
}

COOP_HD double scale2(double x, int e) {  // x * 2^e, exact for the ranges used here
#ifdef __CUDA_ARCH__
  // 2^e built from its encoding (e in [-1022, 1023]: every use here is a normal power of two),
  // one exact multiply instead of the library scalbn
  return x * __hiloint2double((e + 1023) << 20, 0);
#else
  return __builtin_scalbn(x, e);
#endif
}

// Correctly rounded (ties-to-even) binary64 value of a * 2^-116.
COOP_HD double u192_round_to_double(U192 a) {
  int p;  // index of the most significant set bit
  if (a.w2) p = 191 - clz64(a.w2);
  else if (a.w1) p = 127 - clz64(a.w1);
  else if (a.w0) p = 63 - clz64(a.w0);
  else return 0.0;
  if (p <= 52) return scale2((double)a.w0, -116);  // exact: fewer than 54 bits
  int sh = p - 52;                                   // drop sh low bits
  uint64_t mant = u192_bits64(a, sh) & ((1ull << 53) - 1ull);
  bool half = (u192_bits64(a, sh - 1) & 1ull) != 0;  // the first dropped bit
  bool sticky = u192_any_below(a, sh - 1);
  if (half && (sticky || (mant & 1ull))) {
    mant += 1;
    if (mant == (1ull << 53)) {
      mant >>= 1;
      sh += 1;
    }
  }
  return scale2((double)mant, sh - 116);
}

}  // namespace coop

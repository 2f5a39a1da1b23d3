// Word-level modular arithmetic for RNS limbs, primes p < 2^62.
//
// Every routine returns the canonical residue in [0, p) unless its name says
// "lazy" (then the documented wider range).  Because residues are canonical,
// results are bit-identical to any other correct implementation of the same
// modular function -- in particular to hear/ckks/ring.py:33-68 (Shoup for
// constant twiddles, Barrett for variable products), which computes the same
// residues through a different reduction.
#pragma once
#include <cstdint>

typedef unsigned long long u64;
typedef long long i64;

#define HB_DEV __device__ __forceinline__

// Per-prime constants, one entry per global prime index (chain primes then the
// special prime), resident in device global memory.
struct HbPrime {
  u64 p;        // the prime
  u64 two_p;    // 2p (lazy-range bound)
  u64 one_sh;   // floor(2^64 / p): Shoup companion of w = 1
  u64 r64;      // 2^64 mod p
  u64 r64_sh;   // Shoup companion of r64
  u64 ninv;     // N^-1 mod p
  u64 ninv_sh;  // Shoup companion of ninv
  u64 half;     // p >> 1, threshold of the centred lift
  // fp64-pipe arithmetic (used when every prime of the ring is < 2^42)
  double pd;    // p as a double (exact)
  double pinv;  // fl(1/p)
  double ninvd; // N^-1 mod p as a double
  double ninvq; // fl(ninv / p)
};

// ---------------------------------------------------------------------------
// fp64-pipe modular arithmetic for p < 2^42.
//
// Residues are integer-valued doubles in a balanced range; a product a*w is
// split error-free into hi + lo (hi = fl(aw), lo = fma(a, w, -hi)), the
// quotient q = rint(fl(a * fl(w/p))) (below), and
// r = fma(-q, p, hi) + lo is computed exactly (all intermediate integers are
// below 2^53), giving r = a*w mod p with |r| <= (1/2 + 2^-7) p for any
// |a| <= 2^45.  No integer multiplies: the fp64 pipe of B200 sustains ~3x
// the 64-bit-Shoup rate of the integer pipe (measured).
#define HB_RND_MAGIC 6755399441055744.0  // 1.5 * 2^52

// The quotient is rint(fl(a * wq)): one DMUL on the fp64 pipe plus one FRND
// (a separate, lower-rate pipe that is otherwise idle) instead of the
// fma-against-1.5*2^52 / subtract pair -- 5 fp64-pipe ops instead of 6
// (tools/microbench.cu: 3.36 vs 2.94 T modular products/s).  The rounded
// product moves q by at most 2^-8 relative to round(a*w/p) for |a| <= 2^45,
// so |r| stays within (1/2 + 2^-7) p and the remainder is still exact.
HB_DEV double fmod_mul(double a, double w, double wq, double p) {
  const double hi = a * w;
  const double lo = __fma_rn(a, w, -hi);
  const double q = rint(a * wq);
  return __fma_rn(-q, p, hi) + lo;
}

// |x| <= 2^51 -> x mod p in (-(1/2 + eps) p, (1/2 + eps) p)
HB_DEV double fmod_reduce(double x, double p, double pinv) {
  const double q = rint(x * pinv);
  return __fma_rn(-q, p, x);
}

// balanced residue -> canonical u64 in [0, p)
HB_DEV u64 fmod_canon(double x, double p, double pinv) {
  double r = fmod_reduce(x, p, pinv);
  if (r < 0.0) r += p;
  return (u64)__double_as_longlong(r + 4503599627370496.0) & 0xFFFFFFFFFFFFFull;
}

// canonical u64 (< 2^52) -> double, exact, without the conversion pipe
HB_DEV double u64_to_f(u64 x) {
  return __longlong_as_double((long long)(x | 0x4330000000000000ull)) - 4503599627370496.0;
}

HB_DEV u64 mulhi64(u64 a, u64 b) { return __umul64hi(a, b); }

// Harvey/Shoup product with a constant w < p, wsh = floor(w * 2^64 / p).
// Valid for ANY a < 2^64; result in [0, 2p).
HB_DEV u64 mul_shoup_lazy(u64 a, u64 w, u64 wsh, u64 p) {
  u64 q = mulhi64(a, wsh);
  return a * w - q * p;
}

HB_DEV u64 mul_shoup(u64 a, u64 w, u64 wsh, u64 p) {
  u64 r = mul_shoup_lazy(a, w, wsh, p);
  return r >= p ? r - p : r;
}

HB_DEV u64 csub(u64 x, u64 p) { return x >= p ? x - p : x; }

HB_DEV u64 add_mod(u64 a, u64 b, u64 p) { return csub(a + b, p); }
HB_DEV u64 sub_mod(u64 a, u64 b, u64 p) { return csub(a + p - b, p); }

// Any 64-bit word -> [0, p): Shoup with w = 1.
HB_DEV u64 reduce64(u64 x, const HbPrime& P) {
  return csub(x - mulhi64(x, P.one_sh) * P.p, P.p);
}

// 128-bit value (hi:lo), any hi < 2^64 -> [0, p).
//   hi*2^64 + lo == shoup(hi, r64) + shoup(lo, 1)   (mod p)
HB_DEV u64 reduce128(u64 hi, u64 lo, const HbPrime& P) {
  u64 a = mul_shoup_lazy(hi, P.r64, P.r64_sh, P.p);       // [0, 2p)
  u64 b = lo - mulhi64(lo, P.one_sh) * P.p;               // [0, 2p)
  u64 s = a + b;                                          // [0, 4p) < 2^64
  s = csub(s, P.two_p);
  return csub(s, P.p);
}

// Variable x variable product mod p (a, b < p).
HB_DEV u64 mul_mod(u64 a, u64 b, const HbPrime& P) {
  return reduce128(mulhi64(a, b), a * b, P);
}

// 128-bit accumulator for lazy multiply-accumulate chains.
struct Acc128 {
  u64 lo, hi;
  HB_DEV Acc128() : lo(0), hi(0) {}
  HB_DEV void mac(u64 a, u64 b) {
    u64 l = a * b, h = mulhi64(a, b);
    lo += l;
    hi += h + (lo < l ? 1ull : 0ull);
  }
  HB_DEV void add(u64 a) {
    lo += a;
    hi += (lo < a ? 1ull : 0ull);
  }
  // Fold to a residue and restart from it (keeps hi small between folds).
  HB_DEV u64 fold(const HbPrime& P) {
    u64 r = reduce128(hi, lo, P);
    lo = r;
    hi = 0;
    return r;
  }
};

// Centred lift of x mod ps into (-ps/2, ps/2], re-reduced mod target prime P.
// (hear/ckks/ring.py:186-207 lift_center + reduce_rows, fused.)
HB_DEV u64 lift_reduce(u64 x, u64 ps, u64 ps_half, const HbPrime& P) {
  if (x > ps_half) {                       // negative representative x - ps
    u64 m = reduce64(ps - x, P);           // |x - ps| mod p
    return m ? P.p - m : 0ull;
  }
  return reduce64(x, P);
}

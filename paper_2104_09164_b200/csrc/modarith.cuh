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
};

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

// Shared pieces of the NTT kernels (ntt.cu single-pass, ntt2.cu two-pass):
// fused-mode enum, the two arithmetic policies and the register butterfly
// groups.  See ntt.cu for the transform definition.
#pragma once
#include "ring.cuh"

namespace hb {

enum FwdMode : int {
  FWD_PLAIN = 0,     // src canonical mod dst prime
  FWD_LIFT = 1,      // src mod src_prime: centred lift then reduce (ModUp digit)
  FWD_MODDOWN = 2,   // FWD_LIFT, then dst = (aux - ntt) * scal (+ add[perm])
  FWD_I64 = 3,       // src holds signed int64 coefficients (encoder output)
  FWD_MODDOWN_SCATTER = 4,  // FWD_MODDOWN whose result lands at dst[perm[j]] and
                            // whose addend is read at j: a rotation computed on
                            // pre-permuted keys
  FWD_MODDOWN2 = 5,  // ModDown by P merged with the rescale by q_l that follows
                     // it (cluster NTT only): src = centred lift of the special
                     // row, perm REINTERPRETED as a second source row y (centred
                     // doubles, the ModDown'ed top row in the coefficient
                     // domain), scal_sh = P mod p_dst, scal = (P q_l)^-1:
                     //   dst = (aux - NTT(src + P*y)) * scal + add * s2,
                     // s2 = q_l^-1 mod p_dst passed by value in add2.  Equal bit
                     // for bit to FWD_MODDOWN followed by the rescale.
};

// ---------------------------------------------------------------------------
// Arithmetic policies.

struct PolU64 {
  typedef u64 T;
  typedef HbTw Tw;
  u64 p, two_p;
  HbPrime P;
  HB_DEV PolU64(const HbPrime& pr) : p(pr.p), two_p(pr.two_p), P(pr) {}
  static HB_DEV const Tw* fwd_table(const HbRing& R, int prime) {
    return R.tw_fwd + (size_t)prime * R.n;
  }
  static HB_DEV const Tw* inv_table(const HbRing& R, int prime) {
    return R.tw_inv + (size_t)prime * R.n;
  }
  HB_DEV T from_canon(u64 x) const { return x; }
  HB_DEV T from_signed(i64 v) const {
    if (v < 0) {
      u64 m = reduce64((u64)(-v), P);
      return m ? p - m : 0ull;
    }
    return reduce64((u64)v, P);
  }
  HB_DEV T from_lift(u64 x, u64 ps, u64 ps_half) const { return lift_reduce(x, ps, ps_half, P); }
  // values in [0, 4p)
  HB_DEV void fwd(T& x, T& y, const Tw& t) const {
    u64 X = csub(x, two_p);
    u64 Tv = mul_shoup_lazy(y, t.w, t.wsh, p);
    x = X + Tv;
    y = X - Tv + two_p;
  }
  // values in [0, 2p)
  HB_DEV void inv(T& x, T& y, const Tw& t) const {
    u64 X = x, Y = y;
    x = csub(X + Y, two_p);
    y = mul_shoup_lazy(X - Y + two_p, t.w, t.wsh, p);
  }
  HB_DEV T inv_round_end(T x) const { return x; }
  HB_DEV u64 fwd_final(T x) const { return csub(csub(x, two_p), p); }
  HB_DEV u64 inv_final(T x) const { return mul_shoup(x, P.ninv, P.ninv_sh, p); }
};

struct PolF64 {
  typedef double T;
  typedef HbTwD Tw;
  double p, pinv, ninv, ninvq;
  HB_DEV PolF64(const HbPrime& pr) : p(pr.pd), pinv(pr.pinv), ninv(pr.ninvd), ninvq(pr.ninvq) {}
  static HB_DEV const Tw* fwd_table(const HbRing& R, int prime) {
    return R.twd_fwd + (size_t)prime * R.n;
  }
  static HB_DEV const Tw* inv_table(const HbRing& R, int prime) {
    return R.twd_inv + (size_t)prime * R.n;
  }
  HB_DEV T from_canon(u64 x) const { return u64_to_f(x); }
  HB_DEV T from_signed(i64 v) const { return fmod_reduce((double)v, p, pinv); }
  HB_DEV T from_lift(u64 x, u64 ps, u64 ps_half) const {
    // centred lift of x mod ps (< 2^42): exact as a signed double
    const double c = x > ps_half ? -u64_to_f(ps - x) : u64_to_f(x);
    return fmod_reduce(c, p, pinv);
  }
  // |x| grows by <= 0.51p per stage, |y| reduced: stays < 9p over 14 stages
  HB_DEV void fwd(T& x, T& y, const Tw& t) const {
    const double Tv = fmod_mul(y, t.w, t.wq, p);
    const double X = x;
    x = X + Tv;
    y = X - Tv;
  }
  HB_DEV void inv(T& x, T& y, const Tw& t) const {
    const double X = x, Y = y;
    x = X + Y;
    y = fmod_mul(X - Y, t.w, t.wq, p);
  }
  // x doubles per GS stage: re-centre every round (4 stages -> |x| < 9p)
  HB_DEV T inv_round_end(T x) const { return fmod_reduce(x, p, pinv); }
  HB_DEV u64 fwd_final(T x) const { return fmod_canon(x, p, pinv); }
  HB_DEV u64 inv_final(T x) const { return fmod_canon(fmod_mul(x, ninv, ninvq, p), p, pinv); }
};

// Butterfly groups with a caller-supplied twiddle fetch (stage, group index)
// -> Pol::Tw; used by the block pass, which stages its twiddles in smem.
template <class Pol, int K, class F>
HB_DEV void fwd_group_f(typename Pol::T* x, int s0, int G, F fetch, const Pol& pol) {
#pragma unroll
  for (int st = 0; st < K; ++st) {
    const int h = 1 << (K - 1 - st);
#pragma unroll
    for (int u = 0; u < (1 << K); ++u) {
      if (u & h) continue;
      pol.fwd(x[u], x[u + h], fetch(s0 + st, G * ((1 << K) / (2 * h)) + u / (2 * h)));
    }
  }
}

template <class Pol, int K, class F>
HB_DEV void inv_group_f(typename Pol::T* x, int r0, int G, F fetch, const Pol& pol) {
#pragma unroll
  for (int st = 0; st < K; ++st) {
    const int r = r0 + st, hh = 1 << st;
#pragma unroll
    for (int u = 0; u < (1 << K); ++u) {
      if (u & hh) continue;
      pol.inv(x[u], x[u + hh], fetch(r, ((G << (r0 + K)) >> (r + 1)) + u / (2 * hh)));
    }
  }
}

// ---------------------------------------------------------------------------
// Butterfly groups.

template <class Pol, int K>
HB_DEV void fwd_group(typename Pol::T* x, int s0, int G, const typename Pol::Tw* tw,
                      const Pol& pol) {
#pragma unroll
  for (int st = 0; st < K; ++st) {
    const int s = s0 + st;
    const int h = 1 << (K - 1 - st);
#pragma unroll
    for (int u = 0; u < (1 << K); ++u) {
      if (u & h) continue;
      const int i = G * ((1 << K) / (2 * h)) + u / (2 * h);
      pol.fwd(x[u], x[u + h], tw[(1 << s) + i]);
    }
  }
}

template <class Pol, int K>
HB_DEV void inv_group(typename Pol::T* x, int r0, int G, int logn, const typename Pol::Tw* tw,
                      const Pol& pol) {
#pragma unroll
  for (int st = 0; st < K; ++st) {
    const int r = r0 + st;
    const int hh = 1 << st;
#pragma unroll
    for (int u = 0; u < (1 << K); ++u) {
      if (u & hh) continue;
      const int i = ((G << (r0 + K)) >> (r + 1)) + u / (2 * hh);
      pol.inv(x[u], x[u + hh], tw[((1 << logn) >> (r + 1)) + i]);
    }
  }
}

}  // namespace hb

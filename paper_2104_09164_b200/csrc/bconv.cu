// Fast RNS base conversion for hybrid (dnum < L+1) key switching.
//
// The reference switches keys with one special prime and per-prime digits
// (hear/ckks/engine.py:290-326): every digit is one residue and its ModUp is
// an exact centred lift.  BASELINE config 1 asks for dnum = 3 digits of
// alpha = (L+1)/dnum primes each, which needs the standard fast basis
// conversion between RNS bases B = {q_i} and C = {p_t}:
//
//   Conv_{B->C}(x)_t = sum_i [x_i * qhat_i^-1]_{q_i} * (qhat_i mod p_t)  (mod p_t),
//   qhat_i = prod_{i' != i} q_i'
//
// with every [.]_{q_i} taken as its CENTRED representative in (-q_i/2, q_i/2]
// (approximate: the integer it represents is x + u * Q_B, |u| <= |B|/2,
// zero-mean; with one source prime it is the reference's exact centred
// lift, so dnum = L+1 with one special prime reproduces its key switch).
// ModUp applies it from a digit's primes to every other prime of the
// extended basis; ModDown from the special primes to the chain
// (ckks/hybrid.py).  One thread per coefficient, one CTA row per task;
// the |B| scaled residues stay in registers / local memory and every target
// is one 128-bit multiply-accumulate chain with a single reduction (folded
// every 8 terms), exact for primes < 2^62 on the integer pipe.
#include "ring.cuh"

namespace hb {

constexpr int BCONV_MAXS = 32;
constexpr int BCONV_THREADS = 256;

struct HbBconvTask {
  const u64* src;            // source row 0 (coefficients); row i at src + i * src_stride
  u64* dst;                  // target row t at dst + dst_off[t]
  const long long* dst_off;  // [t] element offsets from dst
  const u64* tab;            // [s][2] (qhat_i^-1 mod q_i, its Shoup) then [s][t] qhat_i mod p_t
  const int* sprime;         // [s] global prime indices of the source basis
  const int* tprime;         // [t] global prime indices of the target basis
  long long src_stride;
  int s, t;
};

// SRC > 0: the source count is a compile-time constant (the scaled residues
// stay in registers); SRC = 0: any count up to BCONV_MAXS (local memory).
template <int SRC>
__global__ void __launch_bounds__(BCONV_THREADS)
k_bconv(const HbBconvTask* __restrict__ tasks, const HbPrime* __restrict__ primes, int n) {
  HB_PDL_ENTRY();
  const HbBconvTask tk = tasks[blockIdx.y];
  const int j = blockIdx.x * BCONV_THREADS + threadIdx.x;
  if (j >= n) return;
  const int s = SRC ? SRC : tk.s;
  u64 y[SRC ? SRC : BCONV_MAXS];
  unsigned neg = 0;   // bit i: term i uses the centred representative y_i - q_i
#pragma unroll
  for (int i = 0; i < (SRC ? SRC : BCONV_MAXS); ++i) {
    if (i >= s) break;
    const u64 q = primes[__ldg(tk.sprime + i)].p;
    u64 v = mul_shoup(__ldg(tk.src + i * tk.src_stride + j), __ldg(tk.tab + 2 * i),
                      __ldg(tk.tab + 2 * i + 1), q);
    if (v > (q >> 1)) {
      v = q - v;
      neg |= 1u << i;
    }
    y[i] = v;
  }
  const u64* m = tk.tab + 2 * s;
  for (int t = 0; t < tk.t; ++t) {
    const HbPrime P = primes[__ldg(tk.tprime + t)];
    Acc128 acc;   // a negative term -y * w enters as y * (p_t - w): one accumulator
#pragma unroll
    for (int i = 0; i < (SRC ? SRC : BCONV_MAXS); ++i) {
      if (i >= s) break;
      const u64 w = __ldg(m + i * tk.t + t);
      acc.mac(y[i], (neg >> i & 1) ? P.p - w : w);
      if ((i & 7) == 7) acc.fold(P);
    }
    tk.dst[__ldg(tk.dst_off + t) + j] = acc.fold(P);
  }
}

cudaError_t launch_bconv(const void* tasks, int ntasks, int nsrc, const HbPrime* primes, int n,
                         cudaStream_t st) {
  if (ntasks <= 0) return cudaSuccess;
  if (ntasks > 65535) return cudaErrorInvalidValue;
  const dim3 grid((n + BCONV_THREADS - 1) / BCONV_THREADS, ntasks);
  const HbBconvTask* t = reinterpret_cast<const HbBconvTask*>(tasks);
  // nsrc: the source count every task of the launch shares (a ModUp's
  // digit size, a ModDown's special-prime count), 0 when they differ
  switch (nsrc) {
#define HB_BCONV(S) \
  case S: (void)hb_launch(k_bconv<S>, grid, dim3(BCONV_THREADS), 0, st, t, primes, n); break;
    HB_BCONV(1) HB_BCONV(2) HB_BCONV(3) HB_BCONV(4) HB_BCONV(5) HB_BCONV(6) HB_BCONV(7)
    HB_BCONV(8)
#undef HB_BCONV
    default: (void)hb_launch(k_bconv<0>, grid, dim3(BCONV_THREADS), 0, st, t, primes, n);
  }
  return cudaGetLastError();
}

int bconv_task_size() { return (int)sizeof(HbBconvTask); }
int bconv_max_sources() { return BCONV_MAXS; }

}  // namespace hb

// Chunked exact modular dot products on the fp64 pipe.
//
//   sum_t a_t * b_t (mod p),  a_t, b_t < p < 2^B
//
// b_t is split into three w-bit limbs (w = ceil(B/3)); every a_t * limb is an
// integer below 2^(B+w) < 2^52, so a DFMA accumulates it EXACTLY, and F of them
// (F * 2^(B+w) + 2^B <= 2^53, ring.cuh chunk_fold) fit before one 3-op
// re-centring.  The three limb sums recombine once per output with the
// constants 2^w, 2^2w mod p.  That is 3 DFMAs per product instead of the
// 7-8 fp64 ops of a reduced product (modarith.cuh fmod_mul), and the result
// is the same canonical residue, so outputs are bit-identical to the
// reference's pw_mul + pw_add chains (hear/ckks/ring.py:127, 159) and its
// key-switch inner product (ring.py:136-156).
#include <cstdlib>
#include "ring.cuh"

namespace hb {

struct HbMacGroupC {
  const u64* const* cts;
  const u64* const* pts;
  u64* const* dsts;
  int nterms;
  int nout;
};

HB_DEV double limb(u64 x, int sh, u64 mask) { return u64_to_f((x >> sh) & mask); }

// recombine limb sums (each balanced after reduction) into a canonical residue
HB_DEV u64 recombine(double s0, double s1, double s2, const double* cc, double p, double pinv) {
  const double r0 = fmod_reduce(s0, p, pinv);
  const double r1 = fmod_mul(fmod_reduce(s1, p, pinv), cc[0], cc[1], p);
  const double r2 = fmod_mul(fmod_reduce(s2, p, pinv), cc[2], cc[3], p);
  return fmod_canon(r0 + r1 + r2, p, pinv);
}

// Shared-term MAC group (see ops.cu k_mac_gemm): lanes = 32 consecutive
// coefficients of row r; a thread keeps TO x TB outputs x 3 limb sums.
template <int TO, int TB, int WO, int WB>
__global__ void __launch_bounds__(256)
k_mac_gemm_c3(HbMacGroupC g, const HbPrime* __restrict__ primes, const double* __restrict__ cconst,
              int w, int fold, int n, int R, int BC) {
  HB_PDL_ENTRY();
  extern __shared__ const u64* ptrs[];
  const int T = g.nterms, O = g.nout;
  for (int i = threadIdx.x + threadIdx.y * 32; i < T + O * T + O; i += 256) {
    if (i < T) ptrs[i] = g.cts[i];
    else if (i < T + O * T) ptrs[i] = g.pts[i - T];
    else ptrs[i] = g.dsts[i - T - O * T];
  }
  __syncthreads();
  const u64* const* cts = ptrs;
  const u64* const* pts = ptrs + T;
  u64* const* dsts = const_cast<u64* const*>(ptrs + T + O * T);
  const int nchunk = n / 32;   // grid order as ops.cu k_mac_gemm (positions slowest)
  const int r = blockIdx.z / nchunk;
  const int j = (blockIdx.z % nchunk) * 32 + threadIdx.x;
  const int wi = threadIdx.y;
  const int o0 = (blockIdx.y * WO + wi / WB) * TO;
  const int b0 = (blockIdx.x * WB + wi % WB) * TB;
  if (o0 >= O || b0 >= BC) return;
  const HbPrime P = primes[r];
  const double p = P.pd, pinv = P.pinv;
  const u64 mask = (1ull << w) - 1;
  const size_t rj = (size_t)r * n + j;
  double acc[TO][TB][3];
#pragma unroll
  for (int o = 0; o < TO; ++o)
#pragma unroll
    for (int b = 0; b < TB; ++b) acc[o][b][0] = acc[o][b][1] = acc[o][b][2] = 0.0;
  int since = 0;
  // software pipeline as ops.cu k_mac_gemm_f64: term t+1 in flight
  u64 cn[TB], an[TO];
  auto fetch = [&](int t) {
#pragma unroll
    for (int b = 0; b < TB; ++b)
      cn[b] = (b0 + b < BC) ? __ldg(cts[t] + (size_t)(b0 + b) * R * n + rj) : 0ull;
#pragma unroll
    for (int o = 0; o < TO; ++o)
      an[o] = (o0 + o < O) ? __ldg(pts[(size_t)(o0 + o) * T + t] + rj) : 0ull;
  };
  fetch(0);
  for (int t = 0; t < T; ++t) {
    double c[TB][3], av[TO];
#pragma unroll
    for (int b = 0; b < TB; ++b) {
      const u64 v = cn[b];
      c[b][0] = limb(v, 0, mask);
      c[b][1] = limb(v, w, mask);
      c[b][2] = u64_to_f(v >> (2 * w));
    }
#pragma unroll
    for (int o = 0; o < TO; ++o) av[o] = u64_to_f(an[o]);
    if (t + 1 < T) fetch(t + 1);
#pragma unroll
    for (int o = 0; o < TO; ++o) {
      const double a = av[o];
#pragma unroll
      for (int b = 0; b < TB; ++b) {
        acc[o][b][0] = __fma_rn(a, c[b][0], acc[o][b][0]);
        acc[o][b][1] = __fma_rn(a, c[b][1], acc[o][b][1]);
        acc[o][b][2] = __fma_rn(a, c[b][2], acc[o][b][2]);
      }
    }
    if (++since == fold) {
      since = 0;
#pragma unroll
      for (int o = 0; o < TO; ++o)
#pragma unroll
        for (int b = 0; b < TB; ++b)
#pragma unroll
          for (int k = 0; k < 3; ++k) acc[o][b][k] = fmod_reduce(acc[o][b][k], p, pinv);
    }
  }
  const double* cc = cconst + 4 * r;
  double ccr[4] = {__ldg(cc), __ldg(cc + 1), __ldg(cc + 2), __ldg(cc + 3)};
#pragma unroll
  for (int o = 0; o < TO; ++o) {
    if (o0 + o >= O) continue;
#pragma unroll
    for (int b = 0; b < TB; ++b)
      if (b0 + b < BC)
        dsts[o0 + o][(size_t)(b0 + b) * R * n + rj] =
            recombine(acc[o][b][0], acc[o][b][1], acc[o][b][2], ccr, p, pinv);
  }
}

template <int TO, int TB, int WO, int WB>
static cudaError_t mac_c3_t(const HbMacGroupC& g, const HbPrime* primes, const double* cc, int w,
                            int fold, int n, int R, int BC, cudaStream_t st) {
  const size_t smem = sizeof(void*) * (size_t)(g.nterms + g.nout * g.nterms + g.nout);
  if (smem > 200 * 1024) {   // pointer tables too large for smem: split the outputs
    if (g.nout <= 1) return cudaErrorInvalidValue;
    HbMacGroupC a = g, b = g;
    a.nout = g.nout / 2;
    b.nout = g.nout - a.nout;
    b.pts = g.pts + (size_t)a.nout * g.nterms;
    b.dsts = g.dsts + a.nout;
    cudaError_t e = mac_c3_t<TO, TB, WO, WB>(a, primes, cc, w, fold, n, R, BC, st);
    return e != cudaSuccess ? e : mac_c3_t<TO, TB, WO, WB>(b, primes, cc, w, fold, n, R, BC, st);
  }
  static int smem_cur = 0;
  cudaError_t e = smem_attr_once((const void*)k_mac_gemm_c3<TO, TB, WO, WB>, (int)((int)smem), &smem_cur);
  if (e != cudaSuccess) return e;
  dim3 block(32, 8);
  dim3 grid((BC + TB * WB - 1) / (TB * WB), (g.nout + TO * WO - 1) / (TO * WO), R * (n / 32));
  (void)hb_launch(k_mac_gemm_c3<TO, TB, WO, WB>, dim3(grid), dim3(block), smem, st, g, primes, cc, w, fold, n, R, BC);
  return cudaGetLastError();
}

cudaError_t launch_mac_gemm_c3(const void* cts, const void* pts, const void* dsts, int nterms,
                               int nout, const HbRing& R, int rows, int BC, cudaStream_t st) {
  if (nout <= 0 || nterms <= 0) return cudaSuccess;
  HbMacGroupC g;
  g.cts = reinterpret_cast<const u64* const*>(cts);
  g.pts = reinterpret_cast<const u64* const*>(pts);
  g.dsts = reinterpret_cast<u64* const*>(dsts);
  g.nterms = nterms;
  g.nout = nout;
  const int w = R.chunk_w, f = R.chunk_fold;
  if (BC <= 2) return mac_c3_t<4, 2, 8, 1>(g, R.primes, R.chunk_consts, w, f, R.n, rows, BC, st);
  const char* v = getenv("HEAR_B200_MAC_TILE");
  if (v && v[0] == '2') return mac_c3_t<2, 4, 4, 2>(g, R.primes, R.chunk_consts, w, f, R.n, rows, BC, st);
  return mac_c3_t<4, 4, 4, 2>(g, R.primes, R.chunk_consts, w, f, R.n, rows, BC, st);
}

// Key-switch inner product (clip-blocked, see ops.cu k_ks_inner2): the digit
// residue de_i is split into limbs once and feeds both key components.
__global__ void __launch_bounds__(256)
k_ks_inner_c3(const HbKsTask2* __restrict__ tasks, const HbPrime* __restrict__ primes,
              const double* __restrict__ cconst, int w, int fold, int n, int nb) {
  HB_PDL_ENTRY();
  const HbKsTask2 tk = tasks[blockIdx.y];
  const int b = blockIdx.x * blockDim.y + threadIdx.y;    // grid order as ops.cu k_ks_inner2
  const int j = 2 * (blockIdx.z * 32 + threadIdx.x);
  if (j >= n || b >= nb) return;
  const HbPrime P = primes[tk.prime];
  const double p = P.pd, pinv = P.pinv;
  const u64 mask = (1ull << w) - 1;
  int s0 = j, s1 = j + 1;
  if (tk.perm) {
    const int2 pp = __ldg(reinterpret_cast<const int2*>(tk.perm + j));
    s0 = pp.x;
    s1 = pp.y;
  }
  const u64* de = tk.de + b * tk.de_bstride;
  double ab[2][3] = {{0, 0, 0}, {0, 0, 0}}, aa[2][3] = {{0, 0, 0}, {0, 0, 0}};
  int since = 0;
  for (int i = 0; i < tk.ndig; ++i) {
    const u64* d = de + i * tk.de_dstride;
    const u64 x[2] = {__ldg(d + s0), __ldg(d + s1)};
    const ulonglong2 kb = __ldg(reinterpret_cast<const ulonglong2*>(tk.kb + i * tk.key_stride + j));
    const ulonglong2 ka = __ldg(reinterpret_cast<const ulonglong2*>(tk.ka + i * tk.key_stride + j));
    const double kbv[2] = {u64_to_f(kb.x), u64_to_f(kb.y)};
    const double kav[2] = {u64_to_f(ka.x), u64_to_f(ka.y)};
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const double l0 = limb(x[e], 0, mask), l1 = limb(x[e], w, mask);
      const double l2 = u64_to_f(x[e] >> (2 * w));
      ab[e][0] = __fma_rn(kbv[e], l0, ab[e][0]);
      ab[e][1] = __fma_rn(kbv[e], l1, ab[e][1]);
      ab[e][2] = __fma_rn(kbv[e], l2, ab[e][2]);
      aa[e][0] = __fma_rn(kav[e], l0, aa[e][0]);
      aa[e][1] = __fma_rn(kav[e], l1, aa[e][1]);
      aa[e][2] = __fma_rn(kav[e], l2, aa[e][2]);
    }
    if (++since == fold) {
      since = 0;
#pragma unroll
      for (int e = 0; e < 2; ++e)
#pragma unroll
        for (int k = 0; k < 3; ++k) {
          ab[e][k] = fmod_reduce(ab[e][k], p, pinv);
          aa[e][k] = fmod_reduce(aa[e][k], p, pinv);
        }
    }
  }
  const double* cc = cconst + 4 * tk.prime;
  const double ccr[4] = {__ldg(cc), __ldg(cc + 1), __ldg(cc + 2), __ldg(cc + 3)};
  ulonglong2 rb, ra;
  rb.x = recombine(ab[0][0], ab[0][1], ab[0][2], ccr, p, pinv);
  rb.y = recombine(ab[1][0], ab[1][1], ab[1][2], ccr, p, pinv);
  ra.x = recombine(aa[0][0], aa[0][1], aa[0][2], ccr, p, pinv);
  ra.y = recombine(aa[1][0], aa[1][1], aa[1][2], ccr, p, pinv);
  *reinterpret_cast<ulonglong2*>(tk.out_b + b * tk.out_bstride + j) = rb;
  *reinterpret_cast<ulonglong2*>(tk.out_a + b * tk.out_bstride + j) = ra;
}

cudaError_t launch_ks_inner_c3(const void* tasks, int ntasks, int nb, const HbRing& R,
                               cudaStream_t st) {
  if (ntasks <= 0 || nb <= 0) return cudaSuccess;
  const int by = nb < 8 ? nb : 8;
  dim3 block(32, by);
  dim3 grid((nb + by - 1) / by, ntasks, (R.n / 2 + 31) / 32);
  (void)hb_launch(k_ks_inner_c3, dim3(grid), dim3(block), 0, st, reinterpret_cast<const HbKsTask2*>(tasks), R.primes,
                                        R.chunk_consts, R.chunk_w, R.chunk_fold, R.n, nb);
  return cudaGetLastError();
}

}  // namespace hb

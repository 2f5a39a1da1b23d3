// fp64 special FFT for the CKKS canonical embedding (hear/ckks/encoder.py).
//
// The reference evaluates a length-2N numpy FFT per polynomial
// (encoder.py:29-41).  Only the N/2 slot points zeta^(5^j) (zeta = e^{i pi/N},
// all = 1 mod 4) matter, and at those points x^(N/2) = i, so c(x) = w(x) with
// w_k = c_k + i c_{k+N/2} (k < N/2).  Writing x_m = zeta * (zeta^4)^m, slot
// evaluation becomes a length-n (n = N/2) complex DFT of the twisted sequence
// w_k zeta^k:
//   decode: slot_j = Re( DFT+[w_k zeta^k](m_j) ) / scale,   m_j = (5^j mod 2N - 1)/4
//   encode: w_k = zeta^-k * DFT-[W](k) / n with W[m_j] = v_j,
//           c_k = rint(Re w_k * scale), c_{k+n} = rint(Im w_k * scale)
// -- the same linear map as encoder.py:29-60 with a 4x shorter transform.
//
// The length-n DFT is a four-step FFT, n = R x C (R = 2^floor(log n / 2)),
// so any ring up to N = 2^17 runs with many CTAs per polynomial and a fixed
// shared-memory tile (no whole-polynomial smem buffer):
//   pass 1 (k_fft_cols): for each column j2 < C, the R-point DFT over
//          j1 of x[C j1 + j2], times the twiddle W_n^{j2 k1}; TJ columns per
//          CTA, written row-major to the workspace Y[k1][j2];
//   pass 2 (k_fft_rows): for each row k1 < R, the C-point DFT over j2 of
//          Y[k1][.], giving X[k1 + R k2]; TK rows per CTA.
// The codec's gather (encode: slot -> bin) is fused into pass 1's load, its
// scatter (decode: bin -> slot) and the rounding / overflow check (encode)
// into pass 2's store.  The workspace (n complex doubles per polynomial)
// stays in L2 between the passes.  Every twiddle is an exact table entry
// e^{2 pi i e / n} (host-computed in long double), never a product.
#include "ring.cuh"

namespace hb {

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ double2 cmulc(double2 a, double2 b) {  // a * conj(b)
  return make_double2(a.x * b.x + a.y * b.y, a.y * b.x - a.x * b.y);
}
__device__ __forceinline__ int brev(int x, int bits) { return bits ? (int)(__brev(x) >> (32 - bits)) : 0; }

// W_n^e for any e (mod n): root holds e^{+2 pi i k / n} for k < n/2.
__device__ __forceinline__ double2 wn(const HbFftTables& T, int e, bool conj) {
  e &= T.n2 - 1;
  double2 w = __ldg(T.root + (e & (T.n2 / 2 - 1)));
  if (e >= T.n2 / 2) w = make_double2(-w.x, -w.y);
  if (conj) w.y = -w.y;
  return w;
}

// `cnt` independent length-M (M = 2^logm) DFTs in shared memory, element i of
// sequence s at a[s * sstride + i * estride], input in bit-reversed order,
// output in natural order.  Radix-2 DIT; twiddles from the length-n table
// (stride n / M).  Ends with __syncthreads().
__device__ void fft_tile(double2* a, int logm, int cnt, int sstride, int estride,
                         const HbFftTables& T, bool conj) {
  const int m = 1 << logm;
  const int nb = (m >> 1) * cnt;   // butterflies per stage
  for (int s = 0; s < logm; ++s) {
    const int half = 1 << s;
    const int tstep = T.n2 >> (s + 1);   // W_{2 half} = W_n^{n / (2 half)}
    for (int b = threadIdx.x; b < nb; b += blockDim.x) {
      const int q = b % cnt;              // sequence fastest: consecutive lanes
      const int bb = b / cnt;             // hit consecutive columns (no conflicts)
      const int k = bb & (half - 1);
      const int i0 = ((bb >> s) << (s + 1)) + k, i1 = i0 + half;
      double2 w = __ldg(T.root + k * tstep);
      if (conj) w.y = -w.y;
      double2* p0 = a + q * sstride + i0 * estride;
      double2* p1 = a + q * sstride + i1 * estride;
      const double2 u = *p0;
      const double2 v = cmul(*p1, w);
      *p0 = make_double2(u.x + v.x, u.y + v.y);
      *p1 = make_double2(u.x - v.x, u.y - v.y);
    }
    __syncthreads();
  }
}

constexpr int FFT_TJ = 16;    // pass-1 columns per CTA
constexpr int FFT_TK = 8;     // pass-2 rows per CTA
constexpr int FFT_THREADS = 256;

struct FftGeom {
  int logr, logc, r, c;
};
static inline FftGeom geom(int logn2) {
  FftGeom g;
  g.logr = logn2 / 2;
  g.logc = logn2 - g.logr;
  g.r = 1 << g.logr;
  g.c = 1 << g.logc;
  return g;
}

// Pass 1.  ENC: x[bin] = slot value of that bin (W[m_j] = v_j);
// DEC: x[k] = (c_k + i c_{k+n}) zeta^k.  Grid (C / TJ, npoly).
template <bool ENC>
__global__ void __launch_bounds__(FFT_THREADS) k_fft_cols(const double* __restrict__ in,
                                                          double2* __restrict__ work,
                                                          HbFftTables T, int logr, int logc) {
  HB_PDL_ENTRY();
  extern __shared__ double2 sm[];   // [R][TJ]
  const int n = T.n2, r = 1 << logr, c = 1 << logc;
  const int j20 = blockIdx.x * FFT_TJ;
  const size_t poly = blockIdx.y;
  for (int idx = threadIdx.x; idx < r * FFT_TJ; idx += blockDim.x) {
    const int j1 = idx / FFT_TJ, jj = idx % FFT_TJ;
    const int g = c * j1 + j20 + jj;
    double2 x;
    if (ENC) {
      x = make_double2(__ldg(in + poly * n + __ldg(T.slot_of + g)), 0.0);
    } else {
      const double* cf = in + poly * 2 * n;
      x = cmul(make_double2(__ldg(cf + g), __ldg(cf + g + n)), __ldg(T.twist + g));
    }
    sm[brev(j1, logr) * FFT_TJ + jj] = x;
  }
  __syncthreads();
  fft_tile(sm, logr, FFT_TJ, 1, FFT_TJ, T, ENC);
  double2* y = work + poly * n;
  for (int idx = threadIdx.x; idx < r * FFT_TJ; idx += blockDim.x) {
    const int k1 = idx / FFT_TJ, jj = idx % FFT_TJ;
    const int j2 = j20 + jj;
    y[(size_t)k1 * c + j2] = cmul(sm[k1 * FFT_TJ + jj], wn(T, j2 * k1, ENC));
  }
}

// Pass 2.  Grid (R / TK, npoly).  ENC: coefficients c_k, c_{k+n} (rounded,
// overflow flagged past 2^52, encoder.py:50-55); DEC: slot values / scale.
template <bool ENC>
__global__ void __launch_bounds__(FFT_THREADS) k_fft_rows(const double2* __restrict__ work,
                                                          void* __restrict__ out, double scale,
                                                          HbFftTables T, int logr, int logc,
                                                          int* overflow) {
  HB_PDL_ENTRY();
  extern __shared__ double2 sm[];   // [C][TK]: butterflies of consecutive rows are adjacent
  const int n = T.n2, r = 1 << logr, c = 1 << logc;
  const int k10 = blockIdx.x * FFT_TK;
  const size_t poly = blockIdx.y;
  const double2* y = work + poly * n;
  for (int idx = threadIdx.x; idx < FFT_TK * c; idx += blockDim.x) {
    const int kk = idx / c, j2 = idx % c;
    sm[brev(j2, logc) * FFT_TK + kk] = y[(size_t)(k10 + kk) * c + j2];
  }
  __syncthreads();
  fft_tile(sm, logc, FFT_TK, 1, FFT_TK, T, ENC);
  bool of = false;
  const double inv = 1.0 / (double)n;
  for (int idx = threadIdx.x; idx < FFT_TK * c; idx += blockDim.x) {
    const int k2 = idx / FFT_TK, kk = idx % FFT_TK;   // consecutive lanes: consecutive bins
    const int k = k10 + kk + r * k2;
    const double2 x = sm[k2 * FFT_TK + kk];
    if (ENC) {
      const double2 w = cmulc(x, __ldg(T.twist + k));
      const double rr = rint(w.x * inv * scale), ri = rint(w.y * inv * scale);
      if (fabs(rr) >= 4503599627370496.0 || fabs(ri) >= 4503599627370496.0) of = true;
      long long* cf = (long long*)out + poly * 2 * n;
      cf[k] = (long long)rr;
      cf[k + n] = (long long)ri;
    } else {
      ((double*)out)[poly * n + __ldg(T.slot_of + k)] = x.x / scale;
    }
  }
  if (ENC && of) atomicExch(overflow, 1);
}

static cudaError_t run_fft(bool enc, const void* in, void* out, int npoly, double scale,
                           const HbFftTables& T, int* overflow, double2* work, int work_polys,
                           cudaStream_t st) {
  if (npoly <= 0) return cudaSuccess;
  if (T.logn2 < 8 || T.logn2 > 16 || work_polys <= 0) return cudaErrorInvalidValue;
  const FftGeom g = geom(T.logn2);
  const size_t sm1 = (size_t)g.r * FFT_TJ * sizeof(double2);
  const size_t sm2 = (size_t)FFT_TK * g.c * sizeof(double2);
  static int cur[4] = {0, 0, 0, 0};
  cudaError_t e;
  if ((e = smem_attr_once((const void*)k_fft_cols<true>, (int)sm1, &cur[0])) ||
      (e = smem_attr_once((const void*)k_fft_cols<false>, (int)sm1, &cur[1])) ||
      (e = smem_attr_once((const void*)k_fft_rows<true>, (int)sm2, &cur[2])) ||
      (e = smem_attr_once((const void*)k_fft_rows<false>, (int)sm2, &cur[3])))
    return e;
  const size_t n = T.n2;
  for (int p0 = 0; p0 < npoly; p0 += work_polys) {
    const int cnt = npoly - p0 < work_polys ? npoly - p0 : work_polys;
    const dim3 g1(g.c / FFT_TJ, cnt), g2(g.r / FFT_TK, cnt);
    if (enc) {
      const double* src = (const double*)in + (size_t)p0 * n;
      long long* dst = (long long*)out + (size_t)p0 * 2 * n;
      (void)hb_launch(k_fft_cols<true>, g1, dim3(FFT_THREADS), sm1, st, src, work, T, g.logr,
                      g.logc);
      (void)hb_launch(k_fft_rows<true>, g2, dim3(FFT_THREADS), sm2, st, (const double2*)work,
                      (void*)dst, scale, T, g.logr, g.logc, overflow);
    } else {
      const double* src = (const double*)in + (size_t)p0 * 2 * n;
      double* dst = (double*)out + (size_t)p0 * n;
      (void)hb_launch(k_fft_cols<false>, g1, dim3(FFT_THREADS), sm1, st, src, work, T, g.logr,
                      g.logc);
      (void)hb_launch(k_fft_rows<false>, g2, dim3(FFT_THREADS), sm2, st, (const double2*)work,
                      (void*)dst, scale, T, g.logr, g.logc, overflow);
    }
    if ((e = cudaGetLastError())) return e;
  }
  return cudaSuccess;
}

cudaError_t launch_encode(const double* slots, long long* coeffs, int npoly, double scale,
                          const HbFftTables& T, int* overflow, double2* work, int work_polys,
                          cudaStream_t st) {
  return run_fft(true, slots, coeffs, npoly, scale, T, overflow, work, work_polys, st);
}

cudaError_t launch_decode(const double* coeffs, double* slots, int npoly, double scale,
                          const HbFftTables& T, double2* work, int work_polys, cudaStream_t st) {
  return run_fft(false, coeffs, slots, npoly, scale, T, nullptr, work, work_polys, st);
}

}  // namespace hb

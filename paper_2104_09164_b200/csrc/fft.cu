// fp64 special FFT for the CKKS canonical embedding (hear/ckks/encoder.py).
//
// The reference evaluates a length-2N numpy FFT per polynomial.  Only the
// N/2 slot points zeta^(5^j) (zeta = e^{i pi/N}, all = 1 mod 4) matter, and at
// those points x^(N/2) = i, so c(x) = w(x) with w_k = c_k + i c_{k+N/2}
// (k < N/2).  Writing x_m = zeta * (zeta^4)^m, slot evaluation becomes a
// length-N/2 complex DFT of the twisted sequence w_k zeta^k:
//   decode: slot_j = Re( DFT+[w_k zeta^k](m_j) ) / scale,   m_j = (5^j mod 2N - 1)/4
//   encode: w_k = zeta^-k * DFT-[W](k) / (N/2) with W[m_j] = v_j,
//           c_k = rint(Re w_k * scale), c_{k+N/2} = rint(Im w_k * scale)
// which is the same linear map as encoder.py:29-41 evaluated with a 4x
// shorter transform.  One CTA per polynomial; the n2-point transform runs in
// shared memory (n2 <= 8192 complex doubles = 128 KB).
#include "ring.cuh"

namespace hb {

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ double2 cmulc(double2 a, double2 b) {  // a * conj(b)
  return make_double2(a.x * b.x + a.y * b.y, a.y * b.x - a.x * b.y);
}

__device__ __forceinline__ int brev(int x, int bits) { return __brev(x) >> (32 - bits); }

// In-place iterative radix-2 DIT on smem data already in bit-reversed order.
// sign > 0: exponent +2 pi i, sign < 0: exponent -2 pi i.
__device__ void fft_smem(double2* a, const HbFftTables& T, int sign) {
  const int n = T.n2;
  for (int len = 2; len <= n; len <<= 1) {
    const int half = len >> 1;
    const int step = n / len;
    for (int b = threadIdx.x; b < n / 2; b += blockDim.x) {
      const int grp = b / half, k = b % half;
      const int i0 = grp * len + k, i1 = i0 + half;
      double2 w = __ldg(T.root + k * step);
      if (sign < 0) w.y = -w.y;
      const double2 u = a[i0];
      const double2 v = cmul(a[i1], w);
      a[i0] = make_double2(u.x + v.x, u.y + v.y);
      a[i1] = make_double2(u.x - v.x, u.y - v.y);
    }
    __syncthreads();
  }
}

// Encode: real slot values (n2 per poly) -> signed int64 coefficients (N).
// Sets *overflow when any |coefficient| >= 2^52 (encoder.py:50-55).
__global__ void k_encode(const double* __restrict__ slots, long long* __restrict__ coeffs,
                         double scale, HbFftTables T, int* overflow) {
  HB_PDL_ENTRY();
  extern __shared__ double2 a[];
  const int n2 = T.n2;
  const double* v = slots + (size_t)blockIdx.x * n2;
  long long* c = coeffs + (size_t)blockIdx.x * 2 * n2;
  for (int j = threadIdx.x; j < n2; j += blockDim.x) {
    const int m = __ldg(T.slot_pos + j);
    a[brev(m, T.logn2)] = make_double2(__ldg(v + j), 0.0);
  }
  __syncthreads();
  fft_smem(a, T, -1);
  const double inv = 1.0 / (double)n2;
  bool of = false;
  for (int k = threadIdx.x; k < n2; k += blockDim.x) {
    double2 w = cmulc(a[k], __ldg(T.twist + k));
    const double re = w.x * inv * scale, im = w.y * inv * scale;
    const double rr = rint(re), ri = rint(im);
    if (fabs(rr) >= 4503599627370496.0 || fabs(ri) >= 4503599627370496.0) of = true;
    c[k] = (long long)rr;
    c[k + n2] = (long long)ri;
  }
  if (of) atomicExch(overflow, 1);
}

// Decode: double coefficients (N per poly) -> real slot values / scale.
__global__ void k_decode(const double* __restrict__ coeffs, double* __restrict__ slots,
                         double scale, HbFftTables T) {
  HB_PDL_ENTRY();
  extern __shared__ double2 a[];
  const int n2 = T.n2;
  const double* c = coeffs + (size_t)blockIdx.x * 2 * n2;
  double* v = slots + (size_t)blockIdx.x * n2;
  for (int k = threadIdx.x; k < n2; k += blockDim.x) {
    const double2 w = make_double2(__ldg(c + k), __ldg(c + k + n2));
    a[brev(k, T.logn2)] = cmul(w, __ldg(T.twist + k));
  }
  __syncthreads();
  fft_smem(a, T, +1);
  for (int j = threadIdx.x; j < n2; j += blockDim.x) v[j] = a[__ldg(T.slot_pos + j)].x / scale;
}

cudaError_t launch_encode(const double* slots, long long* coeffs, int npoly, double scale,
                          const HbFftTables& T, int* overflow, cudaStream_t st) {
  if (npoly <= 0) return cudaSuccess;
  const size_t smem = (size_t)T.n2 * sizeof(double2);
  static int smem_cur = 0;
  cudaError_t e = smem_attr_once((const void*)k_encode, (int)((int)smem), &smem_cur);
  if (e != cudaSuccess) return e;
  (void)hb_launch(k_encode, dim3(npoly), dim3(512), smem, st, slots, coeffs, scale, T, overflow);
  return cudaGetLastError();
}

cudaError_t launch_decode(const double* coeffs, double* slots, int npoly, double scale,
                          const HbFftTables& T, cudaStream_t st) {
  if (npoly <= 0) return cudaSuccess;
  const size_t smem = (size_t)T.n2 * sizeof(double2);
  static int smem_cur = 0;
  cudaError_t e = smem_attr_once((const void*)k_decode, (int)((int)smem), &smem_cur);
  if (e != cudaSuccess) return e;
  (void)hb_launch(k_decode, dim3(npoly), dim3(512), smem, st, coeffs, slots, scale, T);
  return cudaGetLastError();
}

}  // namespace hb

// Throughput probe: fp64 FMA vs 64-bit integer Shoup vs fp64 modular multiply.
#include <cstdio>
#include <cuda_runtime.h>
typedef unsigned long long u64;
__global__ void k_dfma(double* out, int iters) {
  double a[8]; for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3 + i;
  const double b = 1.0000001, c = 1e-9;
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = fma(a[i], b, c);
  double s = 0; for (int i = 0; i < 8; ++i) s += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_shoup(u64* out, int iters, u64 w, u64 wsh, u64 p) {
  u64 a[8]; for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 7919ull + i;
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) { u64 q = __umul64hi(a[i], wsh); a[i] = a[i] * w - q * p; }
  u64 s = 0; for (int i = 0; i < 8; ++i) s += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_fpmod(double* out, int iters, double w, double wp, double p) {
  double a[8]; for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 7919.0 + i;
  const double M = 6755399441055744.0;  // 1.5 * 2^52
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      double hi = a[i] * w; double lo = fma(a[i], w, -hi);
      double q = fma(a[i], wp, M) - M; double r = fma(-q, p, hi); a[i] = r + lo;
    }
  double s = 0; for (int i = 0; i < 8; ++i) s += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
// q = rint(a * w/p) with one rounding instruction instead of the magic-number pair
__global__ void k_fpmod_rint(double* out, int iters, double w, double wp, double p) {
  double a[8]; for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 7919.0 + i;
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      double hi = a[i] * w; double lo = fma(a[i], w, -hi);
      double q = rint(a[i] * wp); double r = fma(-q, p, hi); a[i] = r + lo;
    }
  double s = 0; for (int i = 0; i < 8; ++i) s += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_rint(double* out, int iters) {
  double a[8]; for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1.37 + i * 0.61;
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = rint(a[i]) + 0.75;
  double s = 0; for (int i = 0; i < 8; ++i) s += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
  const int blocks = 148 * 8, threads = 256, iters = 4096;
  double* dd; u64* du; cudaMalloc(&dd, blocks * threads * 8); cudaMalloc(&du, blocks * threads * 8);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b); float ms;
  const double ops = 8.0 * iters * blocks * threads;
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(a); k_dfma<<<blocks, threads>>>(dd, iters); cudaEventRecord(b); cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b); if (rep) printf("DFMA        %.2f T/s\n", ops / ms / 1e9);
    u64 p = 8590163969ull, w = 12345678901ull % p, wsh = (u64)(((unsigned __int128)w << 64) / p);
    cudaEventRecord(a); k_shoup<<<blocks, threads>>>(du, iters, w, wsh, p); cudaEventRecord(b); cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b); if (rep) printf("u64 shoup   %.2f T mulmod/s\n", ops / ms / 1e9);
    cudaEventRecord(a); k_fpmod<<<blocks, threads>>>(dd, iters, (double)w, (double)w / p, (double)p); cudaEventRecord(b); cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b); if (rep) printf("fp64 mulmod %.2f T mulmod/s\n", ops / ms / 1e9);
    cudaEventRecord(a); k_fpmod_rint<<<blocks, threads>>>(dd, iters, (double)w, (double)w / p, (double)p); cudaEventRecord(b); cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b); if (rep) printf("fp64 mulmod (rint q) %.2f T mulmod/s\n", ops / ms / 1e9);
    cudaEventRecord(a); k_rint<<<blocks, threads>>>(dd, iters); cudaEventRecord(b); cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b); if (rep) printf("rint+add    %.2f T pairs/s\n", ops / ms / 1e9);
  }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}

// Throughput probe: IMAD.WIDE.U32 (32 x 32 + 64 -> 64) alone, DFMA alone, and
// both interleaved in one thread (do the integer and fp64 pipes overlap?).
#include <cstdio>
#include <cuda_runtime.h>
typedef unsigned long long u64;
__device__ __forceinline__ u64 madw(unsigned a, unsigned b, u64 c) {
  u64 r; asm volatile("mad.wide.u32 %0, %1, %2, %3;" : "=l"(r) : "r"(a), "r"(b), "l"(c)); return r;
}
__global__ void k_imadw(u64* out, int iters, unsigned m) {
  u64 a[8]; for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 7919ull + i;
  unsigned x = threadIdx.x | 1;
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = madw(x, m + i, a[i]);
  u64 s = 0; for (int i = 0; i < 8; ++i) s += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_dfma(double* out, int iters) {
  double a[8]; for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3 + i;
  const double b = 1.0000001, c = 1e-9;
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = fma(a[i], b, c);
  double s = 0; for (int i = 0; i < 8; ++i) s += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_both(double* out, u64* out2, int iters, unsigned m) {
  double a[8]; u64 u[8];
  for (int i = 0; i < 8; ++i) { a[i] = threadIdx.x * 1e-3 + i; u[i] = threadIdx.x * 7919ull + i; }
  const double b = 1.0000001, c = 1e-9; unsigned x = threadIdx.x | 1;
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) { a[i] = fma(a[i], b, c); u[i] = madw(x, m + i, u[i]); }
  double s = 0; u64 t = 0; for (int i = 0; i < 8; ++i) { s += a[i]; t += u[i]; }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s; out2[blockIdx.x * blockDim.x + threadIdx.x] = t;
}
int main() {
  const int blocks = 148 * 8, threads = 256, iters = 4096;
  double* dd; u64* du; cudaMalloc(&dd, blocks * threads * 8); cudaMalloc(&du, blocks * threads * 8);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b); float ms;
  const double ops = 8.0 * iters * blocks * threads;
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(a); k_dfma<<<blocks, threads>>>(dd, iters); cudaEventRecord(b); cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b); if (rep) printf("DFMA            %.2f T/s\n", ops / ms / 1e9);
    cudaEventRecord(a); k_imadw<<<blocks, threads>>>(du, iters, 12345u); cudaEventRecord(b); cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b); if (rep) printf("IMAD.WIDE.U32   %.2f T/s\n", ops / ms / 1e9);
    cudaEventRecord(a); k_both<<<blocks, threads>>>(dd, du, iters, 12345u); cudaEventRecord(b); cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b); if (rep) printf("DFMA + IMAD.WIDE interleaved: %.2f T pairs/s\n", ops / ms / 1e9);
  }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}

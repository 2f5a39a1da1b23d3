#include <cstdint>
#include <cstdio>
__global__ void __launch_bounds__(256) k(double* out, int iters) {
  __shared__ uint32_t tbase_s;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"((uint32_t)__cvta_generic_to_shared(&tbase_s)) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tb = tbase_s;
  // this thread's 64 columns: lane quadrant of the warp, column half by warp / 4
  const uint32_t ta = tb + ((uint32_t)((warp & 3) * 32) << 16) + (warp >> 2) * 64;
  for (int i = 0; i < 8; ++i) {
    double a0 = threadIdx.x + 1000.0 * i, a1 = a0 + 0.25, a2 = a0 + 0.5, a3 = a0 + 0.75;
    unsigned long long u0 = __double_as_longlong(a0), u1 = __double_as_longlong(a1), u2 = __double_as_longlong(a2), u3 = __double_as_longlong(a3);
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(ta + 8 * i),
      "r"((uint32_t)u0), "r"((uint32_t)(u0 >> 32)), "r"((uint32_t)u1), "r"((uint32_t)(u1 >> 32)),
      "r"((uint32_t)u2), "r"((uint32_t)(u2 >> 32)), "r"((uint32_t)u3), "r"((uint32_t)(u3 >> 32)) : "memory");
  }
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  for (int it = 0; it < iters; ++it) {
    for (int i = 0; i < 8; ++i) {
      uint32_t r[8];
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];" : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]) : "r"(ta + 8 * i) : "memory");
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      double d[4];
      for (int k = 0; k < 4; ++k) d[k] = __longlong_as_double(((unsigned long long)r[2 * k + 1] << 32) | r[2 * k]) + 1.0;
      unsigned long long u[4];
      for (int k = 0; k < 4; ++k) u[k] = __double_as_longlong(d[k]);
      asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(ta + 8 * i),
        "r"((uint32_t)u[0]), "r"((uint32_t)(u[0] >> 32)), "r"((uint32_t)u[1]), "r"((uint32_t)(u[1] >> 32)),
        "r"((uint32_t)u[2]), "r"((uint32_t)(u[2] >> 32)), "r"((uint32_t)u[3]), "r"((uint32_t)(u[3] >> 32)) : "memory");
    }
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  for (int i = 0; i < 8; ++i) {
    uint32_t r[8];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];" : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]) : "r"(ta + 8 * i) : "memory");
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    for (int k = 0; k < 4; ++k)
      out[((size_t)blockIdx.x * 256 + threadIdx.x) * 32 + i * 4 + k] = __longlong_as_double(((unsigned long long)r[2 * k + 1] << 32) | r[2 * k]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" ::"r"(tb) : "memory");
}
int main() {
  const int nb = 148 * 8, iters = 5;
  double* d; cudaMalloc(&d, (size_t)nb * 256 * 32 * 8);
  k<<<nb, 256>>>(d, iters);
  cudaError_t e = cudaDeviceSynchronize();
  printf("err %s\n", cudaGetErrorString(e));
  double* h = (double*)malloc((size_t)nb * 256 * 32 * 8);
  cudaMemcpy(h, d, (size_t)nb * 256 * 32 * 8, cudaMemcpyDeviceToHost);
  long bad = 0;
  for (int b = 0; b < nb; ++b) for (int t = 0; t < 256; ++t) for (int i = 0; i < 8; ++i) for (int k = 0; k < 4; ++k) {
    double want = t + 1000.0 * i + 0.25 * k + iters;
    if (h[((size_t)b * 256 + t) * 32 + i * 4 + k] != want) { if (bad < 5) printf("bad b%d t%d i%d k%d got %f want %f\n", b, t, i, k, h[((size_t)b * 256 + t) * 32 + i * 4 + k], want); ++bad; }
  }
  printf("bad %ld\n", bad);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0); k<<<nb, 256>>>(d, 2000); cudaEventRecord(e1); cudaDeviceSynchronize();
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  printf("2000 iters x %d CTAs: %.3f ms -> %.1f GB/s TMEM rd+wr per SM-equivalent total %.2f TB/s\n", nb, ms, 0.0, (double)nb * 256 * 256 * 2 * 2000 / ms / 1e9);
  return 0;
}

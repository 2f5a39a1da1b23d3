// C-ABI of the B200 HEAR kernels (declared in include/hear_b200.h).
//
// Two families of entry points:
//   hb_*     device-pointer, task-table launches used by the Python engine
//            (paper_2104_09164_b200/ckks/engine.py); every call is
//            asynchronous on the given stream.
//   hear_*   reference-shaped, host-buffer entry points with the argument
//            meaning of hear/ckks/ring.py's numba kernels (rows x N uint64
//            arrays + per-row prime index), for a maintainer who binds them
//            from the reference via ctypes.  They copy in,
//            launch, copy out and synchronise.
#include <cuda_runtime.h>
#include <cstdio>
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "ring.cuh"

// programmatic dependent launch switch (ring.cuh); set only while a CUDA graph
// of the evaluation is captured (hb_set_pdl)
int g_hb_pdl = 0;

namespace hb {
cudaError_t launch_ntt_fwd(const HbNttTask*, int, const HbRing&, int, cudaStream_t);
cudaError_t launch_ntt_inv(const HbNttTask*, int, const HbRing&, cudaStream_t);
int ntt_kernels(const HbRing&, int);
bool ntt3_supported(const HbRing& R);
cudaError_t launch_ew(int, const HbEwTask*, int, const HbPrime*, int, cudaStream_t);
cudaError_t launch_tensor(const void*, int, const HbPrime*, int, bool, cudaStream_t);
cudaError_t launch_mac_strided(const void*, int, const HbMacTerm*, const HbPrime*, int, int, int,
                               bool, cudaStream_t);
cudaError_t launch_sum_rows(const HbMacTask*, int, const void*, const HbPrime*, int, cudaStream_t);
cudaError_t launch_mac_gemm(const void*, const void*, const void*, int, int, const HbPrime*, int,
                            int, int, cudaStream_t);
cudaError_t launch_mac_gemm_f64(const void*, const void*, const void*, int, int, const HbPrime*,
                                int, int, int, cudaStream_t);
cudaError_t launch_ks_inner2_f64(const void*, int, int, const HbPrime*, int, cudaStream_t);
cudaError_t launch_mac_pipe(const void*, const void*, const void*, int, int, const HbRing&, int,
                            int, cudaStream_t, const void* pts_last = nullptr, int prime_last = 0);
cudaError_t launch_ks_gemm(const void*, const void*, const void*, const void*, int, int,
                           const HbRing&, int, int, long long, long long, int, int,
                           cudaStream_t, const void* scat = nullptr, const void* c0s = nullptr,
                           const void* c0 = nullptr, long long c0_bstride = 0,
                           const void* pmod = nullptr);
cudaError_t launch_ks_inner2(const void*, int, int, const HbPrime*, int, cudaStream_t);
cudaError_t launch_ks3(const HbKsfTask*, int, const HbRing&, cudaStream_t);
cudaError_t launch_rot_sum(const void*, int, const void*, int, int, int, const HbPrime*, int,
                           cudaStream_t);
cudaError_t launch_bconv(const void*, int, int, const HbPrime*, int, cudaStream_t);
int bconv_task_size();
cudaError_t launch_lift_center(const u64*, u64, long long*, int, cudaStream_t);
cudaError_t launch_reduce_rows(const long long*, const int*, int, const HbPrime*, u64*, int,
                               cudaStream_t);
struct HbCrtTask;
cudaError_t launch_crt_double(const HbCrtTask*, int, const u64*, const HbPrime*, const int*, int,
                              int, int, cudaStream_t);
cudaError_t launch_encode(const double*, long long*, int, double, const HbFftTables&, int*, double2*, int,
                          cudaStream_t);
cudaError_t launch_decode(const double*, double*, int, double, const HbFftTables&, double2*, int,
                          cudaStream_t);
}  // namespace hb

using namespace hb;

struct hb_ring {
  HbRing dev;            // pointers into device memory
  HbPrime* primes_dev;
  HbTw* tw_fwd_dev;
  HbTw* tw_inv_dev;
  HbTwD* twd_fwd_dev;
  HbTwD* twd_inv_dev;
  double* tw1_fwd_dev;
  double* tw1_inv_dev;
  HbTwD* tw3_fwd_dev = nullptr;
  HbTwD* tw3_inv_dev = nullptr;
  std::vector<HbPrime> primes_host;
  int last_err;
};

struct hb_fft {
  HbFftTables t;
  double2* root_dev;
  double2* twist_dev;
  int* pos_dev;
  double2* work_dev = nullptr;   // four-step FFT intermediate, work_polys polynomials
  int work_polys = 0;
};

static thread_local char g_err[512];

static int fail(cudaError_t e, const char* where) {
  snprintf(g_err, sizeof(g_err), "%s: %s", where, cudaGetErrorString(e));
  return (int)e;
}

static unsigned long long shoup(unsigned long long w, unsigned long long p) {
  return (unsigned long long)(((unsigned __int128)w << 64) / p);
}

extern "C" {

const char* hb_last_error(void) { return g_err; }

int hb_version(void) { return 1; }

hb_ring* hb_ring_create(int logn, int nprimes, const unsigned long long* primes,
                        const unsigned long long* psi, const unsigned long long* ipsi) {
  const int n = 1 << logn;
  hb_ring* r = new hb_ring();
  memset(&r->dev, 0, sizeof(r->dev));
  r->primes_dev = nullptr;
  r->tw_fwd_dev = r->tw_inv_dev = nullptr;
  r->twd_fwd_dev = r->twd_inv_dev = nullptr;
  r->tw1_fwd_dev = r->tw1_inv_dev = nullptr;
  r->dev.logn = logn;
  r->dev.n = n;
  r->dev.nprimes = nprimes;
  r->primes_host.resize(nprimes);
  for (int i = 0; i < nprimes; ++i) {
    const unsigned long long p = primes[i];
    if (p >> 62) {
      snprintf(g_err, sizeof(g_err), "prime %llu exceeds 62 bits", p);
      delete r;
      return nullptr;
    }
    HbPrime& P = r->primes_host[i];
    P.p = p;
    P.two_p = 2 * p;
    P.one_sh = (unsigned long long)(((unsigned __int128)1 << 64) / p);
    P.r64 = (unsigned long long)(((unsigned __int128)1 << 64) % p);
    P.r64_sh = shoup(P.r64, p);
    // N^-1 mod p by Fermat
    unsigned __int128 acc = 1, base = (unsigned long long)n % p;
    unsigned long long e = p - 2;
    while (e) {
      if (e & 1) acc = acc * base % p;
      base = base * base % p;
      e >>= 1;
    }
    P.ninv = (unsigned long long)acc;
    P.ninv_sh = shoup(P.ninv, p);
    P.half = p >> 1;
    P.pd = (double)p;
    P.pinv = 1.0 / (double)p;
    P.ninvd = (double)P.ninv;
    P.ninvq = (double)P.ninv / (double)p;
  }
  bool f64 = true;
  for (int i = 0; i < nprimes; ++i) f64 = f64 && primes[i] < (1ull << 42);
  const char* force = getenv("HEAR_B200_INT_NTT");
  r->dev.use_f64 = (f64 && !(force && force[0] == '1')) ? 1 : 0;
  bool small = true;   // b <= 34 bits: products of a residue and a half-residue stay below 2^51
  for (int i = 0; i < nprimes; ++i) small = small && primes[i] < (1ull << 34);
  const char* nosplit = getenv("HEAR_B200_MAC_SPLIT");
  r->dev.split_ok = (small && !(nosplit && nosplit[0] == '0')) ? 1 : 0;
  std::vector<HbTw> tf((size_t)nprimes * n), ti((size_t)nprimes * n);
  std::vector<HbTwD> tfd((size_t)nprimes * n), tid((size_t)nprimes * n);
  std::vector<double> t1f((size_t)nprimes * n), t1i((size_t)nprimes * n);
  for (int i = 0; i < nprimes; ++i) {
    const double pd = (double)primes[i];
    for (int j = 0; j < n; ++j) {
      const size_t k = (size_t)i * n + j;
      tf[k].w = psi[k];
      tf[k].wsh = shoup(psi[k], primes[i]);
      ti[k].w = ipsi[k];
      ti[k].wsh = shoup(ipsi[k], primes[i]);
      tfd[k].w = (double)psi[k];
      tfd[k].wq = (double)psi[k] / pd;
      tid[k].w = (double)ipsi[k];
      tid[k].wq = (double)ipsi[k] / pd;
      t1f[k] = (double)psi[k];
      t1i[k] = (double)ipsi[k];
    }
  }
  // plane-major fine-stage tables (ring.cuh tw3_fwd / tw3_inv)
  std::vector<HbTwD> t3f((size_t)nprimes * n), t3i((size_t)nprimes * n);
  if (logn >= 6) {
    const int n8 = n / 8;
    const int off_inv[3] = {0, 4, 6};
    for (int i = 0; i < nprimes; ++i) {
      const size_t b = (size_t)i * n;
      for (int e = 0; e < 3; ++e)
        for (int ii = 0; ii < (1 << e); ++ii)
          for (int G = 0; G < n8; ++G)
            t3f[b + (size_t)((1 << e) - 1 + ii) * n8 + G] =
                tfd[b + ((size_t)1 << (logn - 3 + e)) + ((size_t)G << e) + ii];
      for (int rr = 0; rr < 3; ++rr)
        for (int ii = 0; ii < (1 << (2 - rr)); ++ii)
          for (int G = 0; G < n8; ++G)
            t3i[b + (size_t)(off_inv[rr] + ii) * n8 + G] =
                tid[b + (n >> (rr + 1)) + ((size_t)G << (2 - rr)) + ii];
    }
  }
  cudaError_t e;
  if ((e = cudaMalloc(&r->tw3_fwd_dev, sizeof(HbTwD) * t3f.size())) ||
      (e = cudaMalloc(&r->tw3_inv_dev, sizeof(HbTwD) * t3i.size())) ||
      (e = cudaMemcpy(r->tw3_fwd_dev, t3f.data(), sizeof(HbTwD) * t3f.size(), cudaMemcpyHostToDevice)) ||
      (e = cudaMemcpy(r->tw3_inv_dev, t3i.data(), sizeof(HbTwD) * t3i.size(), cudaMemcpyHostToDevice)) ||
      (e = cudaMalloc(&r->primes_dev, sizeof(HbPrime) * nprimes)) ||
      (e = cudaMalloc(&r->tw_fwd_dev, sizeof(HbTw) * tf.size())) ||
      (e = cudaMalloc(&r->tw_inv_dev, sizeof(HbTw) * ti.size())) ||
      (e = cudaMemcpy(r->primes_dev, r->primes_host.data(), sizeof(HbPrime) * nprimes,
                      cudaMemcpyHostToDevice)) ||
      (e = cudaMemcpy(r->tw_fwd_dev, tf.data(), sizeof(HbTw) * tf.size(), cudaMemcpyHostToDevice)) ||
      (e = cudaMemcpy(r->tw_inv_dev, ti.data(), sizeof(HbTw) * ti.size(), cudaMemcpyHostToDevice)) ||
      (e = cudaMalloc(&r->twd_fwd_dev, sizeof(HbTwD) * tfd.size())) ||
      (e = cudaMalloc(&r->twd_inv_dev, sizeof(HbTwD) * tid.size())) ||
      (e = cudaMemcpy(r->twd_fwd_dev, tfd.data(), sizeof(HbTwD) * tfd.size(), cudaMemcpyHostToDevice)) ||
      (e = cudaMemcpy(r->twd_inv_dev, tid.data(), sizeof(HbTwD) * tid.size(), cudaMemcpyHostToDevice)) ||
      (e = cudaMalloc(&r->tw1_fwd_dev, sizeof(double) * t1f.size())) ||
      (e = cudaMalloc(&r->tw1_inv_dev, sizeof(double) * t1i.size())) ||
      (e = cudaMemcpy(r->tw1_fwd_dev, t1f.data(), sizeof(double) * t1f.size(), cudaMemcpyHostToDevice)) ||
      (e = cudaMemcpy(r->tw1_inv_dev, t1i.data(), sizeof(double) * t1i.size(), cudaMemcpyHostToDevice))) {
    fail(e, "hb_ring_create");
    delete r;
    return nullptr;
  }
  r->dev.primes = r->primes_dev;
  r->dev.tw_fwd = r->tw_fwd_dev;
  r->dev.tw_inv = r->tw_inv_dev;
  r->dev.twd_fwd = r->twd_fwd_dev;
  r->dev.twd_inv = r->twd_inv_dev;
  r->dev.tw1_fwd = r->tw1_fwd_dev;
  r->dev.tw1_inv = r->tw1_inv_dev;
  r->dev.tw3_fwd = r->tw3_fwd_dev;
  r->dev.tw3_inv = r->tw3_inv_dev;
  return r;
}

void hb_ring_destroy(hb_ring* r) {
  if (!r) return;
  cudaFree(r->primes_dev);
  cudaFree(r->tw_fwd_dev);
  cudaFree(r->tw_inv_dev);
  cudaFree(r->twd_fwd_dev);
  cudaFree(r->twd_inv_dev);
  cudaFree(r->tw1_fwd_dev);
  cudaFree(r->tw1_inv_dev);
  cudaFree(r->tw3_fwd_dev);
  cudaFree(r->tw3_inv_dev);
  delete r;
}

// Per-prime constants as the kernels see them (host copy, for tests).
int hb_ring_prime_consts(const hb_ring* r, int i, unsigned long long* out8) {
  if (!r || i < 0 || i >= r->dev.nprimes) return -1;
  memcpy(out8, &r->primes_host[i], 8 * sizeof(unsigned long long));  // integer constants
  return 0;
}

int hb_sizeof_task(int kind) {
  switch (kind) {
    case 0: return (int)sizeof(HbNttTask);
    case 1: return (int)sizeof(HbEwTask);
    case 2: return (int)sizeof(HbMacTask);
    case 3: return (int)sizeof(HbMacTerm);
    case 5: return (int)sizeof(HbKsTask2);
    case 6: return bconv_task_size();
    case 7: return (int)sizeof(HbKsfTask);
    case 8: return (int)sizeof(HbRotSumTask);
    case 9: return (int)sizeof(HbRotSumRot);
    default: return -1;
  }
}

int hb_ntt_fwd(hb_ring* r, const void* tasks, int count, int mode, void* stream) {
  cudaError_t e = launch_ntt_fwd((const HbNttTask*)tasks, count, r->dev, mode, (cudaStream_t)stream);
  return e ? fail(e, "hb_ntt_fwd") : 0;
}

int hb_ntt_inv(hb_ring* r, const void* tasks, int count, void* stream) {
  cudaError_t e = launch_ntt_inv((const HbNttTask*)tasks, count, r->dev, (cudaStream_t)stream);
  return e ? fail(e, "hb_ntt_inv") : 0;
}

int hb_ntt_kernels(hb_ring* r, int count) { return ntt_kernels(r->dev, count); }

int hb_set_pdl(int on) {
  const int old = g_hb_pdl;
  g_hb_pdl = on ? 1 : 0;
  return old;
}

int hb_ring_uses_f64(const hb_ring* r) { return r && r->dev.use_f64 ? 1 : 0; }

int hb_ntt_fused_ks(const hb_ring* r) { return r && ntt3_supported(r->dev) ? 1 : 0; }

int hb_ew(hb_ring* r, int op, const void* tasks, int count, void* stream) {
  cudaError_t e = launch_ew(op, (const HbEwTask*)tasks, count, r->dev.primes, r->dev.n,
                            (cudaStream_t)stream);
  return e ? fail(e, "hb_ew") : 0;
}

int hb_mac_strided(hb_ring* r, const void* outs, int nout, const void* terms, int rows, int bc,
                   void* stream) {
  cudaError_t e = launch_mac_strided(outs, nout, (const HbMacTerm*)terms, r->dev.primes, r->dev.n,
                                     rows, bc, r->dev.use_f64 != 0, (cudaStream_t)stream);
  return e ? fail(e, "hb_mac_strided") : 0;
}

int hb_sum(hb_ring* r, const void* tasks, int count, const void* srcs, void* stream) {
  cudaError_t e = launch_sum_rows((const HbMacTask*)tasks, count, srcs, r->dev.primes, r->dev.n,
                                  (cudaStream_t)stream);
  return e ? fail(e, "hb_sum") : 0;
}

int hb_tensor(hb_ring* r, const void* tasks, int count, void* stream) {
  cudaError_t e = launch_tensor(tasks, count, r->dev.primes, r->dev.n, r->dev.use_f64 != 0,
                                (cudaStream_t)stream);
  return e ? fail(e, "hb_tensor") : 0;
}

int hb_mac_shared(hb_ring* r, const void* cts, const void* pts, const void* dsts, int nterms,
                  int nout, int rows, int bc, void* stream) {
  // fp64 rings: the cp.async-pipelined GEMM (mac.cu) at every batch size
  // (measured: also the lower latency at one clip); it declines term tables
  // larger than its shared memory, which take the register-tile GEMM
  cudaError_t e = cudaErrorNotSupported;
  if (r->dev.use_f64) {
    e = launch_mac_pipe(cts, pts, dsts, nterms, nout, r->dev, rows, bc, (cudaStream_t)stream);
    if (e == cudaErrorNotSupported) (void)cudaGetLastError();
  }
  if (e == cudaErrorNotSupported)
    e = r->dev.use_f64
      ? launch_mac_gemm_f64(cts, pts, dsts, nterms, nout, r->dev.primes, r->dev.n, rows, bc,
                            (cudaStream_t)stream)
      : launch_mac_gemm(cts, pts, dsts, nterms, nout, r->dev.primes, r->dev.n, rows, bc,
                        (cudaStream_t)stream);
  return e ? fail(e, "hb_mac_shared") : 0;
}

int hb_ks_gemm(hb_ring* r, const void* de, const void* keys, const void* keys_last,
               const void* dsts, int ndig, int nout, int rows, int bc, long long de_bstride,
               long long dst_bstride, int prime_last, int de_per_job, void* stream) {
  cudaError_t e = launch_ks_gemm(de, keys, keys_last, dsts, ndig, nout, r->dev, rows, bc,
                                 de_bstride, dst_bstride, prime_last, de_per_job,
                                 (cudaStream_t)stream);
  return e ? fail(e, "hb_ks_gemm") : 0;
}

// Extended-basis (Q*P) forms of the two GEMMs, for hoisted rotations whose
// ModDown is deferred past the plaintext products (lazy ModDown).
int hb_mac_shared_ext(hb_ring* r, const void* cts, const void* pts, const void* pts_last,
                      const void* dsts, int nterms, int nout, int rows, int bc, int prime_last,
                      void* stream) {
  if (!r->dev.use_f64) return fail(cudaErrorNotSupported, "hb_mac_shared_ext: fp64 rings only");
  cudaError_t e = launch_mac_pipe(cts, pts, dsts, nterms, nout, r->dev, rows, bc,
                                  (cudaStream_t)stream, pts_last, prime_last);
  return e ? fail(e, "hb_mac_shared_ext") : 0;
}

int hb_ks_gemm_rot(hb_ring* r, const void* de, const void* keys, const void* keys_last,
                   const void* dsts, const void* scat, const void* c0s, const void* c0,
                   const void* pmod, int ndig, int nout, int rows, int bc, long long de_bstride,
                   long long dst_bstride, long long c0_bstride, int prime_last, void* stream) {
  if (!scat || !c0s || !pmod) return fail(cudaErrorInvalidValue, "hb_ks_gemm_rot: null table");
  cudaError_t e = launch_ks_gemm(de, keys, keys_last, dsts, ndig, nout, r->dev, rows, bc,
                                 de_bstride, dst_bstride, prime_last, 0, (cudaStream_t)stream,
                                 scat, c0s, c0, c0_bstride, pmod);
  return e ? fail(e, "hb_ks_gemm_rot") : 0;
}

// Rotate-and-sum of hoisted rotations in the extended basis (ops.cu).
int hb_rot_sum(hb_ring* r, const void* tasks, int ntasks, const void* rots, int nrot, int ndig,
               int nb, void* stream) {
  if (!r->dev.use_f64) return fail(cudaErrorNotSupported, "hb_rot_sum: fp64 rings only");
  cudaError_t e = launch_rot_sum(tasks, ntasks, rots, nrot, ndig, nb, r->dev.primes, r->dev.n,
                                 (cudaStream_t)stream);
  return e ? fail(e, "hb_rot_sum") : 0;
}

// Fused ModUp + key-switch inner product (ntt3.cu k_ks3, TMEM accumulators).
int hb_ks_fused(hb_ring* r, const void* tasks, int count, void* stream) {
  cudaError_t e = launch_ks3((const HbKsfTask*)tasks, count, r->dev, (cudaStream_t)stream);
  return e ? fail(e, "hb_ks_fused") : 0;
}

int hb_ks_inner2(hb_ring* r, const void* tasks, int count, int nb, void* stream) {
  cudaError_t e = r->dev.use_f64
      ? launch_ks_inner2_f64(tasks, count, nb, r->dev.primes, r->dev.n, (cudaStream_t)stream)
      : launch_ks_inner2(tasks, count, nb, r->dev.primes, r->dev.n, (cudaStream_t)stream);
  return e ? fail(e, "hb_ks_inner2") : 0;
}

// Fast RNS base conversion (bconv.cu): hybrid key switching ModUp / ModDown.
int hb_bconv(hb_ring* r, const void* tasks, int count, int nsrc, void* stream) {
  if (nsrc < 0 || nsrc > 32) return fail(cudaErrorInvalidValue, "hb_bconv: source count");
  cudaError_t e = launch_bconv(tasks, count, nsrc, r->dev.primes, r->dev.n, (cudaStream_t)stream);
  return e ? fail(e, "hb_bconv") : 0;
}

int hb_crt_double(hb_ring* r, const void* tasks, int count, const unsigned long long* consts,
                  const int* prime_idx, int keep, int nl, void* stream) {
  cudaError_t e = launch_crt_double((const HbCrtTask*)tasks, count, consts, r->dev.primes, prime_idx,
                                    keep, nl, r->dev.n, (cudaStream_t)stream);
  return e ? fail(e, "hb_crt_double") : 0;
}

void hb_fft_destroy(hb_fft* f);

hb_fft* hb_fft_create(int logn2, const double* root_re_im, const double* twist_re_im,
                      const int* slot_pos) {
  const int n2 = 1 << logn2;
  if (logn2 < 8 || logn2 > 16) {
    fail(cudaErrorInvalidValue, "hb_fft_create: ring degree outside 2^9..2^17");
    return nullptr;
  }
  // the kernels index by DFT bin: invert slot j -> bin m_j (a permutation)
  std::vector<int> slot_of(n2, -1);
  for (int j = 0; j < n2; ++j) {
    if (slot_pos[j] < 0 || slot_pos[j] >= n2 || slot_of[slot_pos[j]] >= 0) {
      fail(cudaErrorInvalidValue, "hb_fft_create: slot_pos is not a permutation");
      return nullptr;
    }
    slot_of[slot_pos[j]] = j;
  }
  hb_fft* f = new hb_fft();
  f->t.logn2 = logn2;
  f->t.n2 = n2;
  // 64 MB of intermediate: 512 polynomials per launch pair at N = 2^14, 128 at 2^16
  f->work_polys = (int)((64ull << 20) / (sizeof(double2) * (size_t)n2));
  cudaError_t e;
  if ((e = cudaMalloc(&f->root_dev, sizeof(double2) * (n2 / 2))) ||
      (e = cudaMalloc(&f->twist_dev, sizeof(double2) * n2)) ||
      (e = cudaMalloc(&f->pos_dev, sizeof(int) * n2)) ||
      (e = cudaMalloc(&f->work_dev, sizeof(double2) * (size_t)n2 * f->work_polys)) ||
      (e = cudaMemcpy(f->root_dev, root_re_im, sizeof(double2) * (n2 / 2), cudaMemcpyHostToDevice)) ||
      (e = cudaMemcpy(f->twist_dev, twist_re_im, sizeof(double2) * n2, cudaMemcpyHostToDevice)) ||
      (e = cudaMemcpy(f->pos_dev, slot_of.data(), sizeof(int) * n2, cudaMemcpyHostToDevice))) {
    fail(e, "hb_fft_create");
    hb_fft_destroy(f);
    return nullptr;
  }
  f->t.root = f->root_dev;
  f->t.twist = f->twist_dev;
  f->t.slot_of = f->pos_dev;
  return f;
}

void hb_fft_destroy(hb_fft* f) {
  if (!f) return;
  cudaFree(f->root_dev);
  cudaFree(f->twist_dev);
  cudaFree(f->pos_dev);
  cudaFree(f->work_dev);
  delete f;
}

int hb_encode(hb_fft* f, const double* slots, long long* coeffs, int npoly, double scale,
              int* overflow, void* stream) {
  cudaError_t e = launch_encode(slots, coeffs, npoly, scale, f->t, overflow, f->work_dev,
                                f->work_polys, (cudaStream_t)stream);
  return e ? fail(e, "hb_encode") : 0;
}

int hb_decode(hb_fft* f, const double* coeffs, double* slots, int npoly, double scale,
              void* stream) {
  cudaError_t e = launch_decode(coeffs, slots, npoly, scale, f->t, f->work_dev, f->work_polys,
                                (cudaStream_t)stream);
  return e ? fail(e, "hb_decode") : 0;
}

// ---------------------------------------------------------------------------
// Reference-shaped host-buffer entry points (ring.py signatures).

static int host_rows_op(hb_ring* r, int nrows, const long long* gidx, int kind,
                        unsigned long long* inout, const unsigned long long* b,
                        unsigned long long* out) {
  const int n = r->dev.n;
  const size_t bytes = (size_t)nrows * n * sizeof(u64);
  u64 *d_a = nullptr, *d_b = nullptr, *d_o = nullptr;
  void* d_t = nullptr;
  cudaError_t e = cudaSuccess;
  if ((e = cudaMalloc(&d_a, bytes))) return fail(e, "hear host op");
  if (b && (e = cudaMalloc(&d_b, bytes))) goto done;
  if ((e = cudaMalloc(&d_o, bytes))) goto done;
  if ((e = cudaMemcpy(d_a, inout, bytes, cudaMemcpyHostToDevice))) goto done;
  if (b && (e = cudaMemcpy(d_b, b, bytes, cudaMemcpyHostToDevice))) goto done;
  if (kind <= 1) {
    std::vector<HbNttTask> t(nrows);
    for (int i = 0; i < nrows; ++i) {
      memset(&t[i], 0, sizeof(HbNttTask));
      t[i].src = d_a + (size_t)i * n;
      t[i].dst = d_o + (size_t)i * n;
      t[i].dst_prime = t[i].src_prime = (int)gidx[i];
    }
    if ((e = cudaMalloc(&d_t, sizeof(HbNttTask) * nrows))) goto done;
    if ((e = cudaMemcpy(d_t, t.data(), sizeof(HbNttTask) * nrows, cudaMemcpyHostToDevice))) goto done;
    e = kind == 0 ? launch_ntt_fwd((HbNttTask*)d_t, nrows, r->dev, 0, 0)
                  : launch_ntt_inv((HbNttTask*)d_t, nrows, r->dev, 0);
  } else {
    std::vector<HbEwTask> t(nrows);
    for (int i = 0; i < nrows; ++i) {
      memset(&t[i], 0, sizeof(HbEwTask));
      t[i].dst = d_o + (size_t)i * n;
      t[i].a = d_a + (size_t)i * n;
      t[i].b = d_b ? d_b + (size_t)i * n : nullptr;
      t[i].prime = (int)gidx[i];
    }
    if ((e = cudaMalloc(&d_t, sizeof(HbEwTask) * nrows))) goto done;
    if ((e = cudaMemcpy(d_t, t.data(), sizeof(HbEwTask) * nrows, cudaMemcpyHostToDevice))) goto done;
    e = launch_ew(kind - 2, (HbEwTask*)d_t, nrows, r->dev.primes, n, 0);
  }
  if (e) goto done;
  if ((e = cudaDeviceSynchronize())) goto done;
  e = cudaMemcpy(out ? out : inout, d_o, bytes, cudaMemcpyDeviceToHost);
done:
  cudaFree(d_a);
  cudaFree(d_b);
  cudaFree(d_o);
  cudaFree(d_t);
  return e ? fail(e, "hear host op") : 0;
}

// ring.py:113 ntt_fwd(a, gidx, ...) -- in place on a host (rows, N) array.
int hear_ntt_fwd(hb_ring* r, unsigned long long* a, int nrows, const long long* gidx) {
  return host_rows_op(r, nrows, gidx, 0, a, nullptr, nullptr);
}
// ring.py:120 ntt_inv(a, gidx, ...) -- in place.
int hear_ntt_inv(hb_ring* r, unsigned long long* a, int nrows, const long long* gidx) {
  return host_rows_op(r, nrows, gidx, 1, a, nullptr, nullptr);
}
// ring.py:127 pw_mul(out, a, b, gidx, ...)
int hear_pw_mul(hb_ring* r, unsigned long long* out, const unsigned long long* a,
                const unsigned long long* b, int nrows, const long long* gidx) {
  return host_rows_op(r, nrows, gidx, 2 + 2, const_cast<unsigned long long*>(a), b, out);
}
// ring.py:159 pw_add(out, a, b, gidx, p)
int hear_pw_add(hb_ring* r, unsigned long long* out, const unsigned long long* a,
                const unsigned long long* b, int nrows, const long long* gidx) {
  return host_rows_op(r, nrows, gidx, 2 + 0, const_cast<unsigned long long*>(a), b, out);
}
// ring.py:167 pw_sub(out, a, b, gidx, p)
int hear_pw_sub(hb_ring* r, unsigned long long* out, const unsigned long long* a,
                const unsigned long long* b, int nrows, const long long* gidx) {
  return host_rows_op(r, nrows, gidx, 2 + 1, const_cast<unsigned long long*>(a), b, out);
}

}  // extern "C"

// Device scratch of the remaining hear_* entry points: freed on every exit.
namespace {
struct DevBufs {
  std::vector<void*> p;
  ~DevBufs() {
    for (void* q : p) cudaFree(q);
  }
  template <typename T>
  cudaError_t get(T** out, size_t bytes, const void* host = nullptr) {
    void* q = nullptr;
    cudaError_t e = cudaMalloc(&q, bytes ? bytes : 1);
    if (e) return e;
    p.push_back(q);
    *out = (T*)q;
    return host ? cudaMemcpy(q, host, bytes, cudaMemcpyHostToDevice) : cudaSuccess;
  }
};

// EW launch over nrows host rows with per-row constants (scalar_mul /
// sub_scaled_inv): dst = op(a[, b]) with scal = c[r] mod p_{gidx[r]}.
int host_scaled_op(hb_ring* r, int op, unsigned long long* rows, const unsigned long long* corr,
                   const unsigned long long* c, int nrows, const long long* gidx,
                   const char* what) {
  if (nrows <= 0) return 0;
  const int n = r->dev.n;
  const size_t bytes = (size_t)nrows * n * sizeof(u64);
  DevBufs d;
  u64 *da = nullptr, *db = nullptr;
  HbEwTask* dt = nullptr;
  std::vector<HbEwTask> t(nrows);
  cudaError_t e;
  if ((e = d.get(&da, bytes, rows))) return fail(e, what);
  if (corr && (e = d.get(&db, bytes, corr))) return fail(e, what);
  for (int i = 0; i < nrows; ++i) {
    const int g = (int)gidx[i];
    if (g < 0 || g >= r->dev.nprimes) return fail(cudaErrorInvalidValue, what);
    const u64 p = r->primes_host[g].p;
    memset(&t[i], 0, sizeof(HbEwTask));
    t[i].dst = da + (size_t)i * n;
    t[i].a = da + (size_t)i * n;
    t[i].b = db ? db + (size_t)i * n : nullptr;
    t[i].scal = c[i] % p;
    t[i].scal_sh = shoup(t[i].scal, p);
    t[i].prime = g;
  }
  if ((e = d.get(&dt, sizeof(HbEwTask) * nrows, t.data()))) return fail(e, what);
  if ((e = launch_ew(op, dt, nrows, r->dev.primes, n, 0)) || (e = cudaDeviceSynchronize()) ||
      (e = cudaMemcpy(rows, da, bytes, cudaMemcpyDeviceToHost)))
    return fail(e, what);
  return 0;
}
}  // namespace

extern "C" {

// ring.py:175 scalar_mul(a, c, gidx, ...): a[r] *= c[r] in place.
int hear_scalar_mul(hb_ring* r, unsigned long long* a, const unsigned long long* c, int nrows,
                    const long long* gidx) {
  return host_scaled_op(r, EW_MUL_SCALAR, a, nullptr, c, nrows, gidx, "hear_scalar_mul");
}

// ring.py:210 sub_scaled_inv(rows, corr, pinv, gidx, ...):
// rows[r] = (rows[r] - corr[r]) * pinv[r] in place.
int hear_sub_scaled_inv(hb_ring* r, unsigned long long* rows, const unsigned long long* corr,
                        const unsigned long long* pinv, int nrows, const long long* gidx) {
  return host_scaled_op(r, EW_SUB_SCALED, rows, corr, pinv, nrows, gidx, "hear_sub_scaled_inv");
}

// ring.py:136 pw_mul_accum_perm(outb, outa, de, kb, ka, krow, perm, gidx, ...):
// outb/outa[r] += sum_i de[i][r][perm[n]] * kb/ka[i][krow[r]][n]  (mod p_{gidx[r]}).
// de: [ndig][nrows][N]; kb, ka: [ndig][krows][N]; perm: [N] (the reference's
// intp array); the inner product runs as the engine's per-job key-switch
// kernel (Galois gather on the digits), then one modular add into out.
int hear_pw_mul_accum_perm(hb_ring* r, unsigned long long* outb, unsigned long long* outa,
                           const unsigned long long* de, const unsigned long long* kb,
                           const unsigned long long* ka, const long long* krow,
                           const long long* perm, const long long* gidx, int ndig, int nrows,
                           int krows) {
  const char* what = "hear_pw_mul_accum_perm";
  if (nrows <= 0) return 0;
  const int n = r->dev.n;
  const size_t row = (size_t)n * sizeof(u64);
  DevBufs d;
  u64 *dde, *dkb, *dka, *dob, *doa, *dib, *dia;
  int* dperm;
  cudaError_t e;
  std::vector<int> p32(n);
  for (int j = 0; j < n; ++j) {
    if (perm[j] < 0 || perm[j] >= n) return fail(cudaErrorInvalidValue, what);
    p32[j] = (int)perm[j];
  }
  if ((e = d.get(&dde, row * ndig * nrows, de)) || (e = d.get(&dkb, row * ndig * krows, kb)) ||
      (e = d.get(&dka, row * ndig * krows, ka)) || (e = d.get(&dob, row * nrows, outb)) ||
      (e = d.get(&doa, row * nrows, outa)) || (e = d.get(&dib, row * nrows)) ||
      (e = d.get(&dia, row * nrows)) || (e = d.get(&dperm, sizeof(int) * n, p32.data())))
    return fail(e, what);
  std::vector<HbKsTask2> kt(nrows);
  std::vector<HbEwTask> at(2 * nrows);
  for (int i = 0; i < nrows; ++i) {
    if (krow[i] < 0 || krow[i] >= krows || gidx[i] < 0 || gidx[i] >= r->dev.nprimes)
      return fail(cudaErrorInvalidValue, what);
    memset(&kt[i], 0, sizeof(HbKsTask2));
    kt[i].de = dde + (size_t)i * n;
    kt[i].kb = dkb + (size_t)krow[i] * n;
    kt[i].ka = dka + (size_t)krow[i] * n;
    kt[i].out_b = dib + (size_t)i * n;
    kt[i].out_a = dia + (size_t)i * n;
    kt[i].perm = dperm;
    kt[i].de_dstride = (long long)nrows * n;
    kt[i].key_stride = (long long)krows * n;
    kt[i].ndig = ndig;
    kt[i].prime = (int)gidx[i];
    for (int c = 0; c < 2; ++c) {
      HbEwTask& t = at[2 * i + c];
      memset(&t, 0, sizeof(HbEwTask));
      t.dst = (c ? doa : dob) + (size_t)i * n;
      t.a = t.dst;
      t.b = (c ? dia : dib) + (size_t)i * n;
      t.prime = (int)gidx[i];
    }
  }
  HbKsTask2* dkt;
  HbEwTask* dat;
  if ((e = d.get(&dkt, sizeof(HbKsTask2) * nrows, kt.data())) ||
      (e = d.get(&dat, sizeof(HbEwTask) * 2 * nrows, at.data())))
    return fail(e, what);
  if (hb_ks_inner2(r, dkt, nrows, 1, nullptr)) return (int)cudaErrorLaunchFailure;
  if ((e = launch_ew(EW_ADD, dat, 2 * nrows, r->dev.primes, n, 0)) ||
      (e = cudaDeviceSynchronize()) ||
      (e = cudaMemcpy(outb, dob, row * nrows, cudaMemcpyDeviceToHost)) ||
      (e = cudaMemcpy(outa, doa, row * nrows, cudaMemcpyDeviceToHost)))
    return fail(e, what);
  return 0;
}

// ring.py:186 lift_center(x, p, out): one row of residues mod p -> centred int64.
int hear_lift_center(const unsigned long long* x, unsigned long long p, long long* out, int n) {
  if (n <= 0) return 0;
  DevBufs d;
  u64* dx;
  long long* dout;
  cudaError_t e;
  if ((e = d.get(&dx, sizeof(u64) * n, x)) || (e = d.get(&dout, sizeof(long long) * n)) ||
      (e = launch_lift_center(dx, p, dout, n, 0)) || (e = cudaDeviceSynchronize()) ||
      (e = cudaMemcpy(out, dout, sizeof(long long) * n, cudaMemcpyDeviceToHost)))
    return fail(e, "hear_lift_center");
  return 0;
}

// ring.py:198 reduce_rows(c, gidx, p, out): centred int64 coefficients [N] ->
// residues out[r] under prime gidx[r], out [nrows][N].
int hear_reduce_rows(hb_ring* r, const long long* c, const long long* gidx, int nrows,
                     unsigned long long* out) {
  if (nrows <= 0) return 0;
  const int n = r->dev.n;
  DevBufs d;
  long long* dc;
  int* dg;
  u64* dout;
  std::vector<int> g32(nrows);
  for (int i = 0; i < nrows; ++i) {
    if (gidx[i] < 0 || gidx[i] >= r->dev.nprimes)
      return fail(cudaErrorInvalidValue, "hear_reduce_rows");
    g32[i] = (int)gidx[i];
  }
  cudaError_t e;
  if ((e = d.get(&dc, sizeof(long long) * n, c)) || (e = d.get(&dg, sizeof(int) * nrows, g32.data())) ||
      (e = d.get(&dout, sizeof(u64) * n * nrows)) ||
      (e = launch_reduce_rows(dc, dg, nrows, r->dev.primes, dout, n, 0)) ||
      (e = cudaDeviceSynchronize()) ||
      (e = cudaMemcpy(out, dout, sizeof(u64) * n * nrows, cudaMemcpyDeviceToHost)))
    return fail(e, "hear_reduce_rows");
  return 0;
}

}  // extern "C"

// Negacyclic NTT over RNS limbs, one CTA per row polynomial, N <= 2^14.
//
// Computes exactly the transform of hear/ckks/ring.py:71-124 (Cooley-Tukey
// forward with bit-reversed psi powers, Gentleman-Sande inverse), so outputs
// are bit-identical canonical residues; the inverse uses the true inverse
// twiddles psi^-brv(j) (ring.py:282 has an off-by-one exponent).
//
// Schedule (B200): the whole row lives in shared memory (<= 128 KB), each of
// the N/16 threads owns 16 elements and runs 4 butterfly stages per round in
// registers, so a 2^14 transform is 4 register rounds with 3 shared-memory
// exchanges instead of 14 stage barriers.  The first forward round reads
// global memory directly (coalesced: lanes own consecutive columns); the last
// (contiguous) round goes through a swizzled shared-memory stage so the HBM
// store is coalesced too.  Swizzle sw(j) = j ^ ((j>>4)&15) makes both the
// strided (t >= 16) and the contiguous (16 per thread) phases conflict-free.
//
// Arithmetic policies (chosen per ring on the host):
//   F64  all primes < 2^42: butterflies on the fp64 pipe (modarith.cuh
//        fmod_mul: 6 fp64 ops, balanced residues, no integer multiplies);
//   U64  otherwise: Harvey lazy butterflies with 64-bit Shoup products.
// Both produce the same canonical residues.
#include <cstdlib>
#include "ntt_common.cuh"

namespace hb {

HB_DEV int sw(int j) { return j ^ ((j >> 4) & 15); }

// One strided forward round (t_last = N >> (s0+K) >= 16) on smem.
template <class Pol, int LOGN, int K>
HB_DEV void fwd_round_smem(typename Pol::T* sm, int s0, const typename Pol::Tw* tw,
                           const Pol& pol) {
  constexpr int N = 1 << LOGN, T = N / 16, GPT = 16 >> K;
  const int tl = N >> (s0 + K);
  typename Pol::T x[16];
#pragma unroll
  for (int q = 0; q < GPT; ++q) {
    const int gid = threadIdx.x + q * T;
    const int base = (gid / tl) * ((1 << K) * tl) + gid % tl;
#pragma unroll
    for (int u = 0; u < (1 << K); ++u) x[q * (1 << K) + u] = sm[sw(base + u * tl)];
  }
#pragma unroll
  for (int q = 0; q < GPT; ++q) {
    const int gid = threadIdx.x + q * T;
    fwd_group<Pol, K>(x + q * (1 << K), s0, gid / tl, tw, pol);
  }
#pragma unroll
  for (int q = 0; q < GPT; ++q) {
    const int gid = threadIdx.x + q * T;
    const int base = (gid / tl) * ((1 << K) * tl) + gid % tl;
#pragma unroll
    for (int u = 0; u < (1 << K); ++u) sm[sw(base + u * tl)] = x[q * (1 << K) + u];
  }
  __syncthreads();
}

template <class Pol, int MODE>
HB_DEV typename Pol::T fwd_load(const HbNttTask& tk, const Pol& pol, u64 ps, u64 ps_half, int j) {
  const u64 x = __ldg(tk.src + j);
  if (MODE == FWD_PLAIN) return pol.from_canon(x);
  if (MODE == FWD_I64) return pol.from_signed((i64)x);
  return pol.from_lift(x, ps, ps_half);
}

template <class Pol, int LOGN, int MODE>
HB_DEV void ntt_fwd_body(const HbNttTask& tk, const HbRing& R, const HbPrime& P) {
  constexpr int N = 1 << LOGN, T = N / 16;
  typedef typename Pol::T V;
  extern __shared__ u64 smraw[];
  V* sm = reinterpret_cast<V*>(smraw);
  const Pol pol(P);
  u64 ps = 0, ps_half = 0;
  if (MODE == FWD_LIFT || MODE == FWD_MODDOWN) {
    ps = R.primes[tk.src_prime].p;
    ps_half = ps >> 1;
  }
  const typename Pol::Tw* tw = Pol::fwd_table(R, tk.dst_prime);
  const int g = threadIdx.x;
  {  // round 0: stages 0..3 straight from global (G = 0, column g)
    V x[16];
#pragma unroll
    for (int u = 0; u < 16; ++u) x[u] = fwd_load<Pol, MODE>(tk, pol, ps, ps_half, u * T + g);
    fwd_group<Pol, 4>(x, 0, 0, tw, pol);
#pragma unroll
    for (int u = 0; u < 16; ++u) sm[sw(u * T + g)] = x[u];
    __syncthreads();
  }
  constexpr int MID = LOGN - 8;
  if (MID >= 4) fwd_round_smem<Pol, LOGN, 4>(sm, 4, tw, pol);
  if (MID >= 8) fwd_round_smem<Pol, LOGN, 4>(sm, 8, tw, pol);
  constexpr int REM = MID % 4, SREM = 4 + (MID / 4) * 4;
  if (REM == 1) fwd_round_smem<Pol, LOGN, 1>(sm, SREM, tw, pol);
  if (REM == 2) fwd_round_smem<Pol, LOGN, 2>(sm, SREM, tw, pol);
  if (REM == 3) fwd_round_smem<Pol, LOGN, 3>(sm, SREM, tw, pol);
  {  // final contiguous round; results canonical, staged for a coalesced store
    V x[16];
#pragma unroll
    for (int u = 0; u < 16; ++u) x[u] = sm[sw(16 * g + u)];
    fwd_group<Pol, 4>(x, LOGN - 4, g, tw, pol);
    u64* smu = smraw;
#pragma unroll
    for (int u = 0; u < 16; ++u) smu[sw(16 * g + u)] = pol.fwd_final(x[u]);
    __syncthreads();
  }
  const u64 p = P.p;
#pragma unroll 4
  for (int j = g; j < N; j += T) {
    u64 v = smraw[sw(j)];
    if (MODE == FWD_MODDOWN) {
      v = mul_shoup(sub_mod(__ldg(tk.aux + j), v, p), tk.scal, tk.scal_sh, p);
      if (tk.add) {
        const int src = tk.perm ? __ldg(tk.perm + j) : j;
        v = add_mod(v, __ldg(tk.add + src), p);
      }
      if (tk.add2) v = add_mod(v, __ldg(tk.add2 + j), p);
    }
    tk.dst[j] = v;
  }
}

template <int LOGN, int MODE, bool F64>
__global__ void __launch_bounds__((1 << LOGN) / 16)
k_ntt_fwd(const HbNttTask* __restrict__ tasks, HbRing R) {
  HB_PDL_ENTRY();
  const HbNttTask tk = tasks[blockIdx.x];
  const HbPrime P = R.primes[tk.dst_prime];
  if (F64)
    ntt_fwd_body<PolF64, LOGN, MODE>(tk, R, P);
  else
    ntt_fwd_body<PolU64, LOGN, MODE>(tk, R, P);
}

// Inverse: contiguous round first (after a coalesced global->smem stage),
// then strided rounds; the last round writes global directly (lanes = columns)
// with the N^-1 scaling fused.
template <class Pol, int LOGN, int K>
HB_DEV void inv_round_strided(typename Pol::T* sm, int r0, const typename Pol::Tw* tw,
                              const Pol& pol, bool last, u64* dst) {
  constexpr int N = 1 << LOGN, T = N / 16, GPT = 16 >> K;
  const int tl = 1 << r0;
  typename Pol::T x[16];
#pragma unroll
  for (int q = 0; q < GPT; ++q) {
    const int gid = threadIdx.x + q * T;
    const int base = (gid / tl) * ((1 << K) * tl) + gid % tl;
#pragma unroll
    for (int u = 0; u < (1 << K); ++u) x[q * (1 << K) + u] = sm[sw(base + u * tl)];
  }
#pragma unroll
  for (int q = 0; q < GPT; ++q) {
    const int gid = threadIdx.x + q * T;
    inv_group<Pol, K>(x + q * (1 << K), r0, gid / tl, LOGN, tw, pol);
  }
  if (last) {
#pragma unroll
    for (int q = 0; q < GPT; ++q) {
      const int gid = threadIdx.x + q * T;
      const int base = (gid / tl) * ((1 << K) * tl) + gid % tl;
#pragma unroll
      for (int u = 0; u < (1 << K); ++u) dst[base + u * tl] = pol.inv_final(x[q * (1 << K) + u]);
    }
    return;
  }
#pragma unroll
  for (int q = 0; q < GPT; ++q) {
    const int gid = threadIdx.x + q * T;
    const int base = (gid / tl) * ((1 << K) * tl) + gid % tl;
#pragma unroll
    for (int u = 0; u < (1 << K); ++u)
      sm[sw(base + u * tl)] = pol.inv_round_end(x[q * (1 << K) + u]);
  }
  __syncthreads();
}

template <class Pol, int LOGN>
HB_DEV void ntt_inv_body(const HbNttTask& tk, const HbRing& R, const HbPrime& P) {
  constexpr int N = 1 << LOGN, T = N / 16;
  typedef typename Pol::T V;
  extern __shared__ u64 smraw[];
  V* sm = reinterpret_cast<V*>(smraw);
  const Pol pol(P);
  const typename Pol::Tw* tw = Pol::inv_table(R, tk.dst_prime);
  const int g = threadIdx.x;
#pragma unroll 4
  for (int j = g; j < N; j += T) {
    const u64 v = __ldg(tk.src + j);
    if (tk.add2) const_cast<u64*>(tk.add2)[j] = v;   // inverse: verbatim copy of the input row
    sm[sw(j)] = pol.from_canon(v);
  }
  __syncthreads();
  {  // round 0: stages 0..3 on contiguous 16-element groups
    V x[16];
#pragma unroll
    for (int u = 0; u < 16; ++u) x[u] = sm[sw(16 * g + u)];
    inv_group<Pol, 4>(x, 0, g, LOGN, tw, pol);
#pragma unroll
    for (int u = 0; u < 16; ++u) sm[sw(16 * g + u)] = pol.inv_round_end(x[u]);
    __syncthreads();
  }
  constexpr int REST = LOGN - 4, NFULL = REST / 4, REM = REST % 4;
  if (REM == 0) {
    if (NFULL >= 1) inv_round_strided<Pol, LOGN, 4>(sm, 4, tw, pol, NFULL == 1, tk.dst);
    if (NFULL >= 2) inv_round_strided<Pol, LOGN, 4>(sm, 8, tw, pol, NFULL == 2, tk.dst);
    if (NFULL >= 3) inv_round_strided<Pol, LOGN, 4>(sm, 12, tw, pol, NFULL == 3, tk.dst);
  } else {
    if (NFULL >= 1) inv_round_strided<Pol, LOGN, 4>(sm, 4, tw, pol, false, tk.dst);
    if (NFULL >= 2) inv_round_strided<Pol, LOGN, 4>(sm, 8, tw, pol, false, tk.dst);
    constexpr int RR = 4 + NFULL * 4;
    if (REM == 1) inv_round_strided<Pol, LOGN, 1>(sm, RR, tw, pol, true, tk.dst);
    if (REM == 2) inv_round_strided<Pol, LOGN, 2>(sm, RR, tw, pol, true, tk.dst);
    if (REM == 3) inv_round_strided<Pol, LOGN, 3>(sm, RR, tw, pol, true, tk.dst);
  }
}

template <int LOGN, bool F64>
__global__ void __launch_bounds__((1 << LOGN) / 16)
k_ntt_inv(const HbNttTask* __restrict__ tasks, HbRing R) {
  HB_PDL_ENTRY();
  const HbNttTask tk = tasks[blockIdx.x];
  const HbPrime P = R.primes[tk.dst_prime];
  if (F64)
    ntt_inv_body<PolF64, LOGN>(tk, R, P);
  else
    ntt_inv_body<PolU64, LOGN>(tk, R, P);
}

// ---------------------------------------------------------------------------
// Host launchers.

template <int LOGN, int MODE, bool F64>
static cudaError_t fwd_one(const HbNttTask* tasks, int count, const HbRing& R, cudaStream_t st) {
  constexpr int N = 1 << LOGN, T = N / 16;
  const size_t smem = (size_t)N * sizeof(u64);
  static int smem_cur = 0;
  cudaError_t e = smem_attr_once((const void*)k_ntt_fwd<LOGN, MODE, F64>, (int)((int)smem), &smem_cur);
  if (e != cudaSuccess) return e;
  (void)hb_launch(k_ntt_fwd<LOGN, MODE, F64>, dim3(count), dim3(T), smem, st, tasks, R);
  return cudaGetLastError();
}

template <int LOGN, bool F64>
static cudaError_t fwd_mode(const HbNttTask* tasks, int count, const HbRing& R, int mode,
                            cudaStream_t st) {
  switch (mode) {
    case FWD_PLAIN: return fwd_one<LOGN, FWD_PLAIN, F64>(tasks, count, R, st);
    case FWD_LIFT: return fwd_one<LOGN, FWD_LIFT, F64>(tasks, count, R, st);
    case FWD_MODDOWN: return fwd_one<LOGN, FWD_MODDOWN, F64>(tasks, count, R, st);
    case FWD_I64: return fwd_one<LOGN, FWD_I64, F64>(tasks, count, R, st);
    default: return cudaErrorInvalidValue;
  }
}

template <int LOGN>
static cudaError_t launch_fwd_t(const HbNttTask* tasks, int count, const HbRing& R, int mode,
                                cudaStream_t st) {
  return R.use_f64 ? fwd_mode<LOGN, true>(tasks, count, R, mode, st)
                   : fwd_mode<LOGN, false>(tasks, count, R, mode, st);
}

template <int LOGN, bool F64>
static cudaError_t inv_one(const HbNttTask* tasks, int count, const HbRing& R, cudaStream_t st) {
  constexpr int N = 1 << LOGN, T = N / 16;
  const size_t smem = (size_t)N * sizeof(u64);
  static int smem_cur = 0;
  cudaError_t e = smem_attr_once((const void*)k_ntt_inv<LOGN, F64>, (int)((int)smem), &smem_cur);
  if (e != cudaSuccess) return e;
  (void)hb_launch(k_ntt_inv<LOGN, F64>, dim3(count), dim3(T), smem, st, tasks, R);
  return cudaGetLastError();
}

template <int LOGN>
static cudaError_t launch_inv_t(const HbNttTask* tasks, int count, const HbRing& R,
                                cudaStream_t st) {
  return R.use_f64 ? inv_one<LOGN, true>(tasks, count, R, st)
                   : inv_one<LOGN, false>(tasks, count, R, st);
}

bool ntt2_supported(int logn);
bool ntt3_supported(const HbRing& R);
cudaError_t launch_ntt3_fwd(const HbNttTask*, int, const HbRing&, int, cudaStream_t);
cudaError_t launch_ntt3_inv(const HbNttTask*, int, const HbRing&, cudaStream_t);
cudaError_t launch_ntt2_fwd(const HbNttTask*, int, const HbRing&, int, cudaStream_t);
cudaError_t launch_ntt2_inv(const HbNttTask*, int, const HbRing&, cudaStream_t);

// The cluster NTT (ntt3.cu) for fp64 rings at 2^13 / 2^14, the two-pass
// transform (ntt2.cu) for the other rings of 2^12..2^16; this file's
// one-row-per-CTA kernel for rings below 2^12.
static bool use_two_pass(int logn) { return ntt2_supported(logn); }

int ntt2_chunk();

int ntt_kernels(const HbRing& R, int count) {
  if (count <= 0) return 0;
  if (ntt3_supported(R)) return 1;
  if (use_two_pass(R.logn)) return 2 * ((count + ntt2_chunk() - 1) / ntt2_chunk());
  return 1;
}

cudaError_t launch_ntt_fwd(const HbNttTask* tasks, int count, const HbRing& R, int mode,
                           cudaStream_t st) {
  if (count <= 0) return cudaSuccess;
  if (ntt3_supported(R)) return launch_ntt3_fwd(tasks, count, R, mode, st);
  if (use_two_pass(R.logn)) return launch_ntt2_fwd(tasks, count, R, mode, st);
  switch (R.logn) {
    case 10: return launch_fwd_t<10>(tasks, count, R, mode, st);
    case 11: return launch_fwd_t<11>(tasks, count, R, mode, st);
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t launch_ntt_inv(const HbNttTask* tasks, int count, const HbRing& R, cudaStream_t st) {
  if (count <= 0) return cudaSuccess;
  if (ntt3_supported(R)) return launch_ntt3_inv(tasks, count, R, st);
  if (use_two_pass(R.logn)) return launch_ntt2_inv(tasks, count, R, st);
  switch (R.logn) {
    case 10: return launch_inv_t<10>(tasks, count, R, st);
    case 11: return launch_inv_t<11>(tasks, count, R, st);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace hb

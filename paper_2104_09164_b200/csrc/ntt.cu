// Negacyclic NTT over RNS limbs, one CTA per row polynomial, N <= 2^14.
//
// Computes exactly the transform of hear/ckks/ring.py:71-124 (Cooley-Tukey
// forward with bit-reversed psi powers, Gentleman-Sande inverse), so outputs
// are bit-identical residues; the inverse uses the true inverse twiddles
// psi^-brv(j) (ring.py:282 has an off-by-one exponent).
//
// Schedule (B200): the whole row lives in shared memory (<= 128 KB), each of
// the N/16 threads owns 16 elements and runs 4 butterfly stages per round in
// registers (Harvey lazy reduction, values in [0,4p)), so a 2^14 transform
// is 4 register rounds with 3 shared-memory exchanges instead of 14 stage
// barriers.  The first forward round reads global memory directly
// (coalesced: lanes own consecutive columns); the last (contiguous) round
// goes through a swizzled shared-memory stage so the store to HBM is
// coalesced too.  Swizzle sw(j) = j ^ ((j>>4)&15) makes both the strided
// (t >= 16) and the contiguous (16 per thread) access patterns conflict-free.
#include "ring.cuh"

namespace hb {

HB_DEV int sw(int j) { return j ^ ((j >> 4) & 15); }

// Fused input/epilogue modes of the forward transform.
enum FwdMode : int {
  FWD_PLAIN = 0,     // src canonical mod dst prime
  FWD_LIFT = 1,      // src mod src_prime: centred lift then reduce (ModUp digit)
  FWD_MODDOWN = 2,   // FWD_LIFT, then dst = (aux - ntt) * scal (+ add[perm])
  FWD_I64 = 3,       // src holds signed int64 coefficients (encoder output)
};

template <int MODE>
HB_DEV u64 fwd_load(const HbNttTask& tk, const HbPrime& P, u64 ps, u64 ps_half, int j) {
  u64 x = __ldg(tk.src + j);
  if (MODE == FWD_PLAIN) return x;
  if (MODE == FWD_I64) {
    i64 v = (i64)x;
    if (v < 0) {
      u64 m = reduce64((u64)(-v), P);
      return m ? P.p - m : 0ull;
    }
    return reduce64(x, P);
  }
  return lift_reduce(x, ps, ps_half, P);
}

// Forward CT butterflies for one group of 2^K elements (x[0..2^K)) covering
// stages s0..s0+K-1; G = group index along the outer axis.
template <int K>
HB_DEV void fwd_group(u64* x, int s0, int G, const HbTw* tw, u64 p, u64 two_p) {
#pragma unroll
  for (int st = 0; st < K; ++st) {
    const int s = s0 + st;
    const int h = 1 << (K - 1 - st);
#pragma unroll
    for (int u = 0; u < (1 << K); ++u) {
      if (u & h) continue;
      const int i = G * ((1 << K) / (2 * h)) + u / (2 * h);
      const HbTw t = tw[(1 << s) + i];
      u64 X = csub(x[u], two_p);
      u64 T = mul_shoup_lazy(x[u + h], t.w, t.wsh, p);
      x[u] = X + T;
      x[u + h] = X - T + two_p;
    }
  }
}

// Inverse GS butterflies for one group of 2^K elements, stages r0..r0+K-1.
template <int K>
HB_DEV void inv_group(u64* x, int r0, int G, int logn, const HbTw* tw, u64 p, u64 two_p) {
#pragma unroll
  for (int st = 0; st < K; ++st) {
    const int r = r0 + st;
    const int hh = 1 << st;
#pragma unroll
    for (int u = 0; u < (1 << K); ++u) {
      if (u & hh) continue;
      const int i = ((G << (r0 + K)) >> (r + 1)) + u / (2 * hh);
      const HbTw t = tw[((1 << logn) >> (r + 1)) + i];
      u64 X = x[u], Y = x[u + hh];
      x[u] = csub(X + Y, two_p);
      x[u + hh] = mul_shoup_lazy(X - Y + two_p, t.w, t.wsh, p);
    }
  }
}

// One strided forward round (t_last = N >> (s0+K) >= 16) from/to smem.
template <int LOGN, int K>
HB_DEV void fwd_round_smem(u64* sm, int s0, const HbTw* tw, u64 p, u64 two_p) {
  constexpr int N = 1 << LOGN, T = N / 16, GPT = 16 >> K;  // groups per thread
  const int tl = N >> (s0 + K);
  u64 x[16];
#pragma unroll
  for (int q = 0; q < GPT; ++q) {
    const int gid = threadIdx.x + q * T;
    const int c = gid % tl, G = gid / tl;
    const int base = G * ((1 << K) * tl) + c;
#pragma unroll
    for (int u = 0; u < (1 << K); ++u) x[q * (1 << K) + u] = sm[sw(base + u * tl)];
  }
#pragma unroll
  for (int q = 0; q < GPT; ++q) {
    const int gid = threadIdx.x + q * T;
    fwd_group<K>(x + q * (1 << K), s0, gid / tl, tw, p, two_p);
  }
  __syncthreads();
#pragma unroll
  for (int q = 0; q < GPT; ++q) {
    const int gid = threadIdx.x + q * T;
    const int c = gid % tl, G = gid / tl;
    const int base = G * ((1 << K) * tl) + c;
#pragma unroll
    for (int u = 0; u < (1 << K); ++u) sm[sw(base + u * tl)] = x[q * (1 << K) + u];
  }
  __syncthreads();
}

template <int LOGN, int MODE>
__global__ void __launch_bounds__((1 << LOGN) / 16)
k_ntt_fwd(const HbNttTask* __restrict__ tasks, HbRing R) {
  constexpr int N = 1 << LOGN, T = N / 16;
  extern __shared__ u64 sm[];
  const HbNttTask tk = tasks[blockIdx.x];
  const HbPrime P = R.primes[tk.dst_prime];
  const u64 p = P.p, two_p = P.two_p;
  u64 ps = 0, ps_half = 0;
  if (MODE == FWD_LIFT || MODE == FWD_MODDOWN) {
    ps = R.primes[tk.src_prime].p;
    ps_half = ps >> 1;
  }
  const HbTw* tw = R.tw_fwd + (size_t)tk.dst_prime * N;
  const int g = threadIdx.x;

  // Round 0: stages 0..3 straight from global (G = 0, column g).
  {
    u64 x[16];
#pragma unroll
    for (int u = 0; u < 16; ++u) x[u] = fwd_load<MODE>(tk, P, ps, ps_half, u * T + g);
    fwd_group<4>(x, 0, 0, tw, p, two_p);
#pragma unroll
    for (int u = 0; u < 16; ++u) sm[sw(u * T + g)] = x[u];
    __syncthreads();
  }
  // Middle strided rounds: stages 4 .. LOGN-5.
  constexpr int MID = LOGN - 8;  // stages left between round 0 and the final round
  if (MID >= 4) fwd_round_smem<LOGN, 4>(sm, 4, tw, p, two_p);
  if (MID >= 8) fwd_round_smem<LOGN, 4>(sm, 8, tw, p, two_p);
  constexpr int REM = MID % 4;
  constexpr int SREM = 4 + (MID / 4) * 4;
  if (REM == 1) fwd_round_smem<LOGN, 1>(sm, SREM, tw, p, two_p);
  if (REM == 2) fwd_round_smem<LOGN, 2>(sm, SREM, tw, p, two_p);
  if (REM == 3) fwd_round_smem<LOGN, 3>(sm, SREM, tw, p, two_p);
  // Final contiguous round: stages LOGN-4 .. LOGN-1, thread g owns [16g, 16g+16).
  {
    u64 x[16];
#pragma unroll
    for (int u = 0; u < 16; ++u) x[u] = sm[sw(16 * g + u)];
    fwd_group<4>(x, LOGN - 4, g, tw, p, two_p);
#pragma unroll
    for (int u = 0; u < 16; ++u) x[u] = csub(csub(x[u], two_p), p);
    __syncthreads();
#pragma unroll
    for (int u = 0; u < 16; ++u) sm[sw(16 * g + u)] = x[u];
    __syncthreads();
  }
  // Coalesced copy-out with the fused epilogue.
#pragma unroll 4
  for (int j = g; j < N; j += T) {
    u64 v = sm[sw(j)];
    if (MODE == FWD_MODDOWN) {
      v = mul_shoup(sub_mod(__ldg(tk.aux + j), v, p), tk.scal, tk.scal_sh, p);
      if (tk.add) {
        const int src = tk.perm ? __ldg(tk.perm + j) : j;
        v = add_mod(v, __ldg(tk.add + src), p);
      }
    }
    tk.dst[j] = v;
  }
}

// Inverse: contiguous round first (via a coalesced global->smem stage), then
// strided rounds; the last round writes global directly (lanes = columns)
// with the N^-1 scaling fused.
template <int LOGN, int K>
HB_DEV void inv_round_strided(u64* sm, int r0, const HbTw* tw, u64 p, u64 two_p,
                              bool last, const HbNttTask& tk, const HbPrime& P) {
  constexpr int N = 1 << LOGN, T = N / 16, GPT = 16 >> K;
  const int tl = 1 << r0;
  u64 x[16];
#pragma unroll
  for (int q = 0; q < GPT; ++q) {
    const int gid = threadIdx.x + q * T;
    const int c = gid % tl, G = gid / tl;
    const int base = G * ((1 << K) * tl) + c;
#pragma unroll
    for (int u = 0; u < (1 << K); ++u) x[q * (1 << K) + u] = sm[sw(base + u * tl)];
  }
#pragma unroll
  for (int q = 0; q < GPT; ++q) {
    const int gid = threadIdx.x + q * T;
    inv_group<K>(x + q * (1 << K), r0, gid / tl, LOGN, tw, p, two_p);
  }
  if (last) {
#pragma unroll
    for (int q = 0; q < GPT; ++q) {
      const int gid = threadIdx.x + q * T;
      const int c = gid % tl, G = gid / tl;
      const int base = G * ((1 << K) * tl) + c;
#pragma unroll
      for (int u = 0; u < (1 << K); ++u)
        tk.dst[base + u * tl] = mul_shoup(x[q * (1 << K) + u], P.ninv, P.ninv_sh, p);
    }
    return;
  }
  __syncthreads();
#pragma unroll
  for (int q = 0; q < GPT; ++q) {
    const int gid = threadIdx.x + q * T;
    const int c = gid % tl, G = gid / tl;
    const int base = G * ((1 << K) * tl) + c;
#pragma unroll
    for (int u = 0; u < (1 << K); ++u) sm[sw(base + u * tl)] = x[q * (1 << K) + u];
  }
  __syncthreads();
}

template <int LOGN>
__global__ void __launch_bounds__((1 << LOGN) / 16)
k_ntt_inv(const HbNttTask* __restrict__ tasks, HbRing R) {
  constexpr int N = 1 << LOGN, T = N / 16;
  extern __shared__ u64 sm[];
  const HbNttTask tk = tasks[blockIdx.x];
  const HbPrime P = R.primes[tk.dst_prime];
  const u64 p = P.p, two_p = P.two_p;
  const HbTw* tw = R.tw_inv + (size_t)tk.dst_prime * N;
  const int g = threadIdx.x;
  // Coalesced stage-in.
#pragma unroll 4
  for (int j = g; j < N; j += T) sm[sw(j)] = __ldg(tk.src + j);
  __syncthreads();
  // Round 0: stages 0..3 on contiguous 16-element groups.
  {
    u64 x[16];
#pragma unroll
    for (int u = 0; u < 16; ++u) x[u] = sm[sw(16 * g + u)];
    inv_group<4>(x, 0, g, LOGN, tw, p, two_p);
    __syncthreads();
#pragma unroll
    for (int u = 0; u < 16; ++u) sm[sw(16 * g + u)] = x[u];
    __syncthreads();
  }
  // Strided rounds r0 = 4, 8, ...; the last one stores to global.
  constexpr int REST = LOGN - 4;
  constexpr int NFULL = REST / 4, REM = REST % 4;
  if (REM == 0) {
    if (NFULL >= 1) inv_round_strided<LOGN, 4>(sm, 4, tw, p, two_p, NFULL == 1, tk, P);
    if (NFULL >= 2) inv_round_strided<LOGN, 4>(sm, 8, tw, p, two_p, NFULL == 2, tk, P);
    if (NFULL >= 3) inv_round_strided<LOGN, 4>(sm, 12, tw, p, two_p, NFULL == 3, tk, P);
  } else {
    if (NFULL >= 1) inv_round_strided<LOGN, 4>(sm, 4, tw, p, two_p, false, tk, P);
    if (NFULL >= 2) inv_round_strided<LOGN, 4>(sm, 8, tw, p, two_p, false, tk, P);
    constexpr int RR = 4 + NFULL * 4;
    if (REM == 1) inv_round_strided<LOGN, 1>(sm, RR, tw, p, two_p, true, tk, P);
    if (REM == 2) inv_round_strided<LOGN, 2>(sm, RR, tw, p, two_p, true, tk, P);
    if (REM == 3) inv_round_strided<LOGN, 3>(sm, RR, tw, p, two_p, true, tk, P);
  }
}

// ---------------------------------------------------------------------------
// Host launchers.

template <int LOGN>
static cudaError_t launch_fwd_t(const HbNttTask* tasks, int count, const HbRing& R, int mode,
                                cudaStream_t st) {
  constexpr int N = 1 << LOGN, T = N / 16;
  const size_t smem = (size_t)N * sizeof(u64);
  auto set = [&](const void* f) {
    return cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  };
  cudaError_t e = cudaSuccess;
  switch (mode) {
    case FWD_PLAIN:
      e = set((const void*)k_ntt_fwd<LOGN, FWD_PLAIN>);
      if (e == cudaSuccess) k_ntt_fwd<LOGN, FWD_PLAIN><<<count, T, smem, st>>>(tasks, R);
      break;
    case FWD_LIFT:
      e = set((const void*)k_ntt_fwd<LOGN, FWD_LIFT>);
      if (e == cudaSuccess) k_ntt_fwd<LOGN, FWD_LIFT><<<count, T, smem, st>>>(tasks, R);
      break;
    case FWD_MODDOWN:
      e = set((const void*)k_ntt_fwd<LOGN, FWD_MODDOWN>);
      if (e == cudaSuccess) k_ntt_fwd<LOGN, FWD_MODDOWN><<<count, T, smem, st>>>(tasks, R);
      break;
    case FWD_I64:
      e = set((const void*)k_ntt_fwd<LOGN, FWD_I64>);
      if (e == cudaSuccess) k_ntt_fwd<LOGN, FWD_I64><<<count, T, smem, st>>>(tasks, R);
      break;
    default:
      return cudaErrorInvalidValue;
  }
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

template <int LOGN>
static cudaError_t launch_inv_t(const HbNttTask* tasks, int count, const HbRing& R,
                                cudaStream_t st) {
  constexpr int N = 1 << LOGN, T = N / 16;
  const size_t smem = (size_t)N * sizeof(u64);
  cudaError_t e = cudaFuncSetAttribute((const void*)k_ntt_inv<LOGN>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  k_ntt_inv<LOGN><<<count, T, smem, st>>>(tasks, R);
  return cudaGetLastError();
}

cudaError_t launch_ntt_fwd(const HbNttTask* tasks, int count, const HbRing& R, int mode,
                           cudaStream_t st) {
  if (count <= 0) return cudaSuccess;
  switch (R.logn) {
    case 10: return launch_fwd_t<10>(tasks, count, R, mode, st);
    case 11: return launch_fwd_t<11>(tasks, count, R, mode, st);
    case 12: return launch_fwd_t<12>(tasks, count, R, mode, st);
    case 13: return launch_fwd_t<13>(tasks, count, R, mode, st);
    case 14: return launch_fwd_t<14>(tasks, count, R, mode, st);
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t launch_ntt_inv(const HbNttTask* tasks, int count, const HbRing& R, cudaStream_t st) {
  if (count <= 0) return cudaSuccess;
  switch (R.logn) {
    case 10: return launch_inv_t<10>(tasks, count, R, st);
    case 11: return launch_inv_t<11>(tasks, count, R, st);
    case 12: return launch_inv_t<12>(tasks, count, R, st);
    case 13: return launch_inv_t<13>(tasks, count, R, st);
    case 14: return launch_inv_t<14>(tasks, count, R, st);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace hb

// Two-pass negacyclic NTT for 2^12 <= N <= 2^16 (the default transform).
//
// Same function as ntt.cu (hear/ckks/ring.py:71-124, true inverse), split
// at stage S1 = log2(N) - 7 into a column pass and a block pass so that a CTA
// works on a 4096-element tile (32 KB of shared memory) instead of a whole
// row (128 KB at N = 2^14): 4+ CTAs per SM overlap their load, butterfly and
// store phases, which the one-row-per-SM kernel cannot (its profile is
// long-scoreboard bound with the fp64 pipe at 43 %).
//
//   forward  pass 1 "cols": stages 0..S1-1, for each column c < 128 the
//            M = N/128 elements {m*128 + c}; a tile = 4096/M adjacent columns.
//            Twiddles psi[1..M-1] (shared by every column, L1-resident).
//            pass 2 "blocks": stages S1..S1+6 inside each 128-element block;
//            a tile = 32 consecutive blocks; then the canonical store with the
//            fused ModDown epilogue.
//   inverse  pass A "blocks": stages 0..6 inside 128-element blocks;
//            pass B "cols": stages 7..log2(N)-1 over columns, N^-1 fused.
// The intermediate (lazy residues: u64 in [0,4p) or balanced doubles) goes
// through dst in place, so no scratch memory is needed (src may equal dst).
//
// Shared-memory layouts: the column tile is [m][c] (lanes = consecutive
// columns, conflict-free); the block tile swizzles 16-byte chunks with
// c ^ ((c>>3)&7) ^ (((c>>6)&1)<<2), conflict-free both for the stride-8
// 16-element groups (8-byte accesses, lanes span two blocks per half-warp)
// and for the contiguous 8-element groups (16-byte accesses).
#include <cstdlib>
#include <type_traits>
#include "ntt_common.cuh"

namespace hb {

constexpr int TILE = 4096;
constexpr int THREADS2 = 256;
#ifndef HB_NTT2_MINB
#define HB_NTT2_MINB 3
#endif
// rows per launch pair (keeps the intermediate L2-resident); env override
static int ntt_chunk() {
  static int c = -1;
  if (c < 0) {
    const char* v = getenv("HEAR_B200_NTT_CHUNK");
    c = v ? atoi(v) : 512;
    if (c <= 0) c = 1 << 30;
  }
  return c;
}

HB_DEV int swz_chunk(int c) { return c ^ ((c >> 3) & 7) ^ (((c >> 6) & 1) << 2); }
HB_DEV int swz(int j) { return (swz_chunk(j >> 1) << 1) | (j & 1); }

template <class Pol, int MODE>
HB_DEV typename Pol::T ld_in(const HbNttTask& tk, const Pol& pol, u64 ps, u64 ps_half, size_t j) {
  const u64 x = __ldg(tk.src + j);
  if (MODE == FWD_PLAIN) return pol.from_canon(x);
  if (MODE == FWD_I64) return pol.from_signed((i64)x);
  return pol.from_lift(x, ps, ps_half);
}

template <class Pol>
HB_DEV typename Pol::T as_val(u64 bits) {
  if constexpr (sizeof(typename Pol::T) == 8 && ((typename Pol::T)0.5) != 0)
    return __longlong_as_double((long long)bits);
  else
    return (typename Pol::T)bits;
}
template <class Pol>
HB_DEV u64 as_bits(typename Pol::T v) {
  if constexpr (((typename Pol::T)0.5) != 0)
    return (u64)__double_as_longlong(v);
  else
    return (u64)v;
}

// ---------------------------------------------------------------------------
// Column pass: stages [0, S1) forward, or [7, 7+S1) inverse.  M = 2^S1
// elements per column (stride 128), CW = TILE / M columns per CTA.
template <class Pol, int LOGN, int MODE, bool FWD>
__global__ void __launch_bounds__(THREADS2, HB_NTT2_MINB)
k_ntt2_cols(const HbNttTask* __restrict__ tasks, HbRing R) {
  HB_PDL_ENTRY();
  constexpr int S1 = LOGN - 7, M = 1 << S1, CW = TILE / M, NCH = 128 / CW;
  constexpr int GQ = M / 16;  // 16-element groups per column
  typedef typename Pol::T V;
  __shared__ V sm[TILE];
  const HbNttTask tk = tasks[blockIdx.x / NCH];
  const int c0 = (blockIdx.x % NCH) * CW;
  const HbPrime P = R.primes[tk.dst_prime];
  const Pol pol(P);
  const typename Pol::Tw* tw = FWD ? Pol::fwd_table(R, tk.dst_prime) : Pol::inv_table(R, tk.dst_prime);
  const int c = threadIdx.x % CW, gq = threadIdx.x / CW;
  u64 ps = 0, ps_half = 0;
  if (FWD && (MODE == FWD_LIFT || MODE == FWD_MODDOWN)) {
    ps = R.primes[tk.src_prime].p;
    ps_half = ps >> 1;
  }
  // round plan over the column: chunks of 4 stages, the last one shorter
  constexpr int NR = (S1 + 3) / 4;
  V x[16];
#pragma unroll
  for (int rd = 0; rd < NR; ++rd) {
    const int s0 = rd * 4;                       // local stage offset
    const int K = (rd == NR - 1) ? (S1 - s0) : 4;
    const int tl = FWD ? (M >> (s0 + K)) : (1 << s0);   // element stride of a group
    const int ng = M >> K;                        // groups per column
    const int gpt = 16 >> K;                      // groups per thread
    // gather this thread's groups (global memory on the first round)
#pragma unroll
    for (int q = 0; q < 16; ++q) {
      const int gsel = q >> K, u = q & ((1 << K) - 1);
      if (gsel >= gpt) break;
      const int gid = gq + gsel * GQ;
      const int m = (gid / tl) * (tl << K) + (gid % tl) + u * tl;
      if (rd == 0) {
        const size_t j = (size_t)m * 128 + c0 + c;
        if (FWD) x[q] = ld_in<Pol, MODE>(tk, pol, ps, ps_half, j);
        else x[q] = as_val<Pol>(__ldg(tk.dst + j));   // block pass's lazy output
      } else {
        x[q] = sm[m * CW + c];
      }
    }
    (void)ng;
    // butterflies
#pragma unroll
    for (int gsel = 0; gsel < 16; ++gsel) {
      if (gsel >= gpt) break;
      const int gid = gq + gsel * GQ;
      if (FWD) {
        if (K == 4) fwd_group<Pol, 4>(x + gsel * 16, s0, gid / tl, tw, pol);
        else if (K == 3) fwd_group<Pol, 3>(x + gsel * 8, s0, gid / tl, tw, pol);
        else if (K == 2) fwd_group<Pol, 2>(x + gsel * 4, s0, gid / tl, tw, pol);
        else fwd_group<Pol, 1>(x + gsel * 2, s0, gid / tl, tw, pol);
      } else {
        if (K == 4) inv_group<Pol, 4>(x + gsel * 16, s0 + 7, gid / tl, LOGN, tw, pol);
        else if (K == 3) inv_group<Pol, 3>(x + gsel * 8, s0 + 7, gid / tl, LOGN, tw, pol);
        else if (K == 2) inv_group<Pol, 2>(x + gsel * 4, s0 + 7, gid / tl, LOGN, tw, pol);
        else inv_group<Pol, 1>(x + gsel * 2, s0 + 7, gid / tl, LOGN, tw, pol);
      }
    }
    const bool last = rd == NR - 1;
#pragma unroll
    for (int q = 0; q < 16; ++q) {
      const int gsel = q >> K, u = q & ((1 << K) - 1);
      if (gsel >= gpt) break;
      const int gid = gq + gsel * GQ;
      const int m = (gid / tl) * (tl << K) + (gid % tl) + u * tl;
      if (last) {
        const size_t j = (size_t)m * 128 + c0 + c;
        if (FWD) tk.dst[j] = as_bits<Pol>(x[q]);          // lazy intermediate
        else tk.dst[j] = pol.inv_final(x[q]);             // canonical, N^-1 applied
      } else {
        sm[m * CW + c] = FWD ? x[q] : pol.inv_round_end(x[q]);
      }
    }
    if (!last) __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// Block pass: 7 stages inside each 128-element block; a CTA owns 32 blocks.
//   forward: stages S1..S1+3 on stride-8 groups of 16, then S1+4..S1+6 on
//            contiguous groups of 8, canonical store + fused epilogue;
//   inverse: stages 0..2 on contiguous groups of 8, then 3..6 on stride-8
//            groups of 16; lazy intermediate store.
template <class Pol, int LOGN, int MODE, bool FWD>
__global__ void __launch_bounds__(THREADS2, HB_NTT2_MINB)
k_ntt2_blocks(const HbNttTask* __restrict__ tasks, HbRing R) {
  HB_PDL_ENTRY();
  constexpr int N = 1 << LOGN, S1 = LOGN - 7, NT = N / TILE;
  typedef typename Pol::T V;
  __shared__ __align__(16) V sm[TILE];
  const HbNttTask tk = tasks[blockIdx.x / NT];
  const int tile = blockIdx.x % NT;
  const size_t base = (size_t)tile * TILE;
  const HbPrime P = R.primes[tk.dst_prime];
  const Pol pol(P);
  const typename Pol::Tw* tw = FWD ? Pol::fwd_table(R, tk.dst_prime) : Pol::inv_table(R, tk.dst_prime);
  const int t = threadIdx.x;
  const int blk = t >> 3, cc = t & 7;   // stride-8 groups: 8 per block, 32 blocks
  const int gblk = tile * 32 + blk;     // global 128-block index
  // fp64 policy: the tile's 32*127 twiddles (7 stages) are staged once in
  // smem with coalesced loads, so butterflies never wait on L2.
  constexpr bool SMTW = std::is_same<Pol, PolF64>::value;
  extern __shared__ double tws[];        // dynamic: 4064 doubles when SMTW
  const double pinv = P.pinv;
  if (SMTW) {
    const double* t1 = (FWD ? R.tw1_fwd : R.tw1_inv) + (size_t)tk.dst_prime * N;
#pragma unroll
    for (int e = 0; e < 7; ++e) {
      // forward stage S1+e: 32<<e entries from 2^(S1+e) + tile*(32<<e);
      // inverse stage e:    2048>>e entries from (N>>(e+1)) + tile*(2048>>e)
      const int len = FWD ? (32 << e) : (2048 >> e);
      const int off = FWD ? 32 * ((1 << e) - 1) : 4096 - (4096 >> e);
      const int src0 = FWD ? (1 << (S1 + e)) + tile * len : (N >> (e + 1)) + tile * len;
      for (int k = t; k < len; k += THREADS2) tws[off + k] = __ldg(t1 + src0 + k);
    }
    __syncthreads();
  }
  auto fetch_f = [&](int s, int i) {
    const int e = s - S1, len = 32 << e;
    const double w = tws[32 * ((1 << e) - 1) + i - tile * len];
    return HbTwD{w, w * pinv};
  };
  auto fetch_i = [&](int r, int i) {
    const int len = 2048 >> r;
    const double w = tws[4096 - (4096 >> r) + i - tile * len];
    return HbTwD{w, w * pinv};
  };
  const u64 p = P.p;
  if (FWD) {
    // round 1 (stages S1..S1+3): stride-8 groups straight from the column
    // pass's lazy intermediate in dst, result to smem
    {
      V x[16];
#pragma unroll
      for (int u = 0; u < 16; ++u) x[u] = as_val<Pol>(__ldg(tk.dst + base + blk * 128 + u * 8 + cc));
      if constexpr (SMTW) fwd_group_f<Pol, 4>(x, S1, gblk, fetch_f, pol);
      else fwd_group<Pol, 4>(x, S1, gblk, tw, pol);
#pragma unroll
      for (int u = 0; u < 16; ++u) sm[swz(blk * 128 + u * 8 + cc)] = x[u];
    }
    __syncthreads();
    // round 2 (stages S1+4..S1+6): contiguous groups of 8 from smem, canonical,
    // fused epilogue, 16-byte stores straight to dst
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const int g2 = t + q * THREADS2;          // 512 groups of 8
      const int b2 = g2 >> 4, G8 = g2 & 15;
      const int e0 = b2 * 128 + G8 * 8;
      // ModDown epilogue operands are issued before the butterflies so their
      // HBM latency overlaps the fp64 work (profiled: these loads were the
      // block pass's top stall)
      constexpr bool MD = MODE == FWD_MODDOWN;
      ulonglong2 ax[4];
      u64 ad[8];
      if (MODE == FWD_MODDOWN) {
#pragma unroll
        for (int v = 0; v < 4; ++v)
          ax[v] = __ldg(reinterpret_cast<const ulonglong2*>(tk.aux + base + e0 + 2 * v));
        if (tk.add) {
#pragma unroll
          for (int v = 0; v < 4; ++v) {
            const size_t j = base + e0 + 2 * v;
            int s0 = (int)j, s1 = (int)j + 1;
            if (tk.perm) {
              const int2 pp = __ldg(reinterpret_cast<const int2*>(tk.perm + j));
              s0 = pp.x;
              s1 = pp.y;
            }
            ad[2 * v] = __ldg(tk.add + s0);
            ad[2 * v + 1] = __ldg(tk.add + s1);
          }
        }
      }
      V x[8];
#pragma unroll
      for (int v = 0; v < 4; ++v) {
        const int pc = swz_chunk((e0 >> 1) + v);
        x[2 * v] = sm[2 * pc];
        x[2 * v + 1] = sm[2 * pc + 1];
      }
      const int G = (tile * 32 + b2) * 16 + G8;
      if constexpr (SMTW) fwd_group_f<Pol, 3>(x, S1 + 4, G, fetch_f, pol);
      else fwd_group<Pol, 3>(x, S1 + 4, G, tw, pol);
#pragma unroll
      for (int v = 0; v < 4; ++v) {
        const size_t j = base + e0 + 2 * v;
        ulonglong2 o;
        o.x = pol.fwd_final(x[2 * v]);
        o.y = pol.fwd_final(x[2 * v + 1]);
        if (MD) {
          o.x = mul_shoup(sub_mod(ax[v].x, o.x, p), tk.scal, tk.scal_sh, p);
          o.y = mul_shoup(sub_mod(ax[v].y, o.y, p), tk.scal, tk.scal_sh, p);
          if (tk.add) {
            o.x = add_mod(o.x, ad[2 * v], p);
            o.y = add_mod(o.y, ad[2 * v + 1], p);
          }
          if (tk.add2) {   // post-addend (the rotate-and-sum add)
            o.x = add_mod(o.x, __ldg(tk.add2 + j), p);
            o.y = add_mod(o.y, __ldg(tk.add2 + j + 1), p);
          }
        }
        *reinterpret_cast<ulonglong2*>(tk.dst + j) = o;
      }
    }
  } else {
    // round 1 (stages 0..2): contiguous groups of 8 straight from src
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const int g2 = t + q * THREADS2;
      const int b2 = g2 >> 4, G8 = g2 & 15;
      const int e0 = b2 * 128 + G8 * 8;
      V x[8];
#pragma unroll
      for (int v = 0; v < 4; ++v) {
        const ulonglong2 in = __ldg(reinterpret_cast<const ulonglong2*>(tk.src + base + e0) + v);
        if (tk.add2)   // inverse: verbatim copy of the input row
          reinterpret_cast<ulonglong2*>(const_cast<u64*>(tk.add2) + base + e0)[v] = in;
        x[2 * v] = pol.from_canon(in.x);
        x[2 * v + 1] = pol.from_canon(in.y);
      }
      const int G = (tile * 32 + b2) * 16 + G8;
      if constexpr (SMTW) inv_group_f<Pol, 3>(x, 0, G, fetch_i, pol);
      else inv_group<Pol, 3>(x, 0, G, LOGN, tw, pol);
#pragma unroll
      for (int v = 0; v < 4; ++v) {
        const int pc = swz_chunk((e0 >> 1) + v);
        sm[2 * pc] = pol.inv_round_end(x[2 * v]);
        sm[2 * pc + 1] = pol.inv_round_end(x[2 * v + 1]);
      }
    }
    __syncthreads();
    // round 2 (stages 3..6): stride-8 groups from smem, lazy result to dst
    V x[16];
#pragma unroll
    for (int u = 0; u < 16; ++u) x[u] = sm[swz(blk * 128 + u * 8 + cc)];
    if constexpr (SMTW) inv_group_f<Pol, 4>(x, 3, gblk, fetch_i, pol);
    else inv_group<Pol, 4>(x, 3, gblk, LOGN, tw, pol);
#pragma unroll
    for (int u = 0; u < 16; ++u)
      tk.dst[base + blk * 128 + u * 8 + cc] = as_bits<Pol>(pol.inv_round_end(x[u]));
  }
}

// ---------------------------------------------------------------------------
// Host launchers.

template <int LOGN, bool F64, int MODE>
static cudaError_t fwd2_t(const HbNttTask* tasks, int count, const HbRing& R, cudaStream_t st) {
  typedef typename std::conditional<F64, PolF64, PolU64>::type Pol;
  constexpr int S1 = LOGN - 7, M = 1 << S1, CW = TILE / M, NCH = 128 / CW;
  const size_t dyn = F64 ? 4064 * sizeof(double) : 0;
  static int smem_cur = 0;
  cudaError_t e = smem_attr_once((const void*)k_ntt2_blocks<Pol, LOGN, MODE, true>, (int)((int)dyn), &smem_cur);
  if (e != cudaSuccess) return e;
  const int CH = ntt_chunk();
  for (int c0 = 0; c0 < count; c0 += CH) {   // chunks keep the intermediate in L2
    const int c = count - c0 < CH ? count - c0 : CH;
    (void)hb_launch(k_ntt2_cols<Pol, LOGN, MODE, true>, dim3(c * NCH), dim3(THREADS2), 0, st, tasks + c0, R);
    (void)hb_launch(k_ntt2_blocks<Pol, LOGN, MODE, true>, dim3(c * ((1 << LOGN) / TILE)), dim3(THREADS2), dyn, st, tasks + c0, R);
  }
  return cudaGetLastError();
}

template <int LOGN, bool F64>
static cudaError_t inv2_t(const HbNttTask* tasks, int count, const HbRing& R, cudaStream_t st) {
  typedef typename std::conditional<F64, PolF64, PolU64>::type Pol;
  constexpr int S1 = LOGN - 7, M = 1 << S1, CW = TILE / M, NCH = 128 / CW;
  const size_t dyn = F64 ? 4064 * sizeof(double) : 0;
  static int smem_cur = 0;
  cudaError_t e = smem_attr_once((const void*)k_ntt2_blocks<Pol, LOGN, FWD_PLAIN, false>, (int)((int)dyn), &smem_cur);
  if (e != cudaSuccess) return e;
  const int CH = ntt_chunk();
  for (int c0 = 0; c0 < count; c0 += CH) {
    const int c = count - c0 < CH ? count - c0 : CH;
    (void)hb_launch(k_ntt2_blocks<Pol, LOGN, FWD_PLAIN, false>, dim3(c * ((1 << LOGN) / TILE)), dim3(THREADS2), dyn, st, tasks + c0, R);
    // the column pass reads the block pass's lazy output from dst
    (void)hb_launch(k_ntt2_cols<Pol, LOGN, FWD_PLAIN, false>, dim3(c * NCH), dim3(THREADS2), 0, st, tasks + c0, R);
  }
  return cudaGetLastError();
}

template <int LOGN, bool F64>
static cudaError_t fwd2_mode(const HbNttTask* tasks, int count, const HbRing& R, int mode,
                             cudaStream_t st) {
  switch (mode) {
    case FWD_PLAIN: return fwd2_t<LOGN, F64, FWD_PLAIN>(tasks, count, R, st);
    case FWD_LIFT: return fwd2_t<LOGN, F64, FWD_LIFT>(tasks, count, R, st);
    case FWD_MODDOWN: return fwd2_t<LOGN, F64, FWD_MODDOWN>(tasks, count, R, st);
    case FWD_I64: return fwd2_t<LOGN, F64, FWD_I64>(tasks, count, R, st);
    // the two-pass intermediate lives in dst, so a scatter through the
    // inverse Galois map would overwrite tiles other CTAs have not read yet:
    // scatter ModDowns run on the cluster NTT only (the engine gathers after
    // a plain ModDown on the two-pass rings)
    case FWD_MODDOWN_SCATTER: return cudaErrorNotSupported;
    default: return cudaErrorInvalidValue;
  }
}

int ntt2_chunk() { return ntt_chunk(); }

bool ntt2_supported(int logn) { return logn >= 12 && logn <= 16; }

cudaError_t launch_ntt2_fwd(const HbNttTask* tasks, int count, const HbRing& R, int mode,
                            cudaStream_t st) {
  if (count <= 0) return cudaSuccess;
  const bool f = R.use_f64 != 0;
  switch (R.logn) {
    case 12: return f ? fwd2_mode<12, true>(tasks, count, R, mode, st) : fwd2_mode<12, false>(tasks, count, R, mode, st);
    case 13: return f ? fwd2_mode<13, true>(tasks, count, R, mode, st) : fwd2_mode<13, false>(tasks, count, R, mode, st);
    case 14: return f ? fwd2_mode<14, true>(tasks, count, R, mode, st) : fwd2_mode<14, false>(tasks, count, R, mode, st);
    case 15: return f ? fwd2_mode<15, true>(tasks, count, R, mode, st) : fwd2_mode<15, false>(tasks, count, R, mode, st);
    case 16: return f ? fwd2_mode<16, true>(tasks, count, R, mode, st) : fwd2_mode<16, false>(tasks, count, R, mode, st);
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t launch_ntt2_inv(const HbNttTask* tasks, int count, const HbRing& R, cudaStream_t st) {
  if (count <= 0) return cudaSuccess;
  const bool f = R.use_f64 != 0;
  switch (R.logn) {
    case 12: return f ? inv2_t<12, true>(tasks, count, R, st) : inv2_t<12, false>(tasks, count, R, st);
    case 13: return f ? inv2_t<13, true>(tasks, count, R, st) : inv2_t<13, false>(tasks, count, R, st);
    case 14: return f ? inv2_t<14, true>(tasks, count, R, st) : inv2_t<14, false>(tasks, count, R, st);
    case 15: return f ? inv2_t<15, true>(tasks, count, R, st) : inv2_t<15, false>(tasks, count, R, st);
    case 16: return f ? inv2_t<16, true>(tasks, count, R, st) : inv2_t<16, false>(tasks, count, R, st);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace hb

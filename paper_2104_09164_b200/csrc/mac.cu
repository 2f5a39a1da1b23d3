// Layer MAC as a per-coefficient modular GEMM with a cp.async smem pipeline
// (default for fp64 rings).
//
//   dst[o][b] = sum_t pt[o][t] * ct[t][b]   (mod p_r)   at every (r, j)
//
// the mult_plain + add chains of one conv / FC layer (hear/convolution.py
// :276-312, fastpath.py:168-180; engine-side ring.py:127/159 pw_mul/pw_add),
// bit-identical canonical residues.  The rotated ciphertexts of a layer are
// GBs (read once from HBM), the plaintexts are shared by every clip (L2).
//
// B200 schedule: a CTA owns 32 coefficients of one RNS row, OB outputs and
// CB clip-components; every term's operand rows (CB ct rows + OB pt rows of
// 256 B) stream through an S-stage ring of shared-memory buffers with
// 16-byte cp.async copies, so S-1 terms are in flight while one is
// multiplied (the register-prefetch kernel in ops.cu stalled 47 % of its
// samples on the HBM latency of the ct loads, profiles/r01_*).  A warp owns
// TO x TB outputs per lane.
//
// Products WITHOUT a per-product reduction: the plaintext / key operand a
// (< p < 2^b) is split at s = ceil(b/2) bits, a = a1 * 2^s + a0, and the two
// partial sums  S0 = sum c*a0,  S1 = sum c*a1  are plain DFMA chains -- every
// product is an integer below 2^(b+s) <= 2^51 and the sums stay below 2^53,
// so they are EXACT in double.  They are reduced mod p every K terms (K = 3
// for a 34-bit prime, 31 at 32 bits, 63 at 31 bits) and combined once as
// S0 + 2^s * S1 mod p.  Two fp64-pipe ops per product instead of the six of
// fmod_mul + accumulate; same canonical residues.
#include <cstdint>
#include <cstdlib>
#include "ring.cuh"

#ifndef HB_MAC_STAGES
#define HB_MAC_STAGES 3   // cp.async pipeline depth of the GEMM (3 measured best: 2 % over 4)
#endif
#ifndef HB_MAC_T128
#define HB_MAC_T128 1   // 128-thread CTAs for the split-sum MAC (layer MAC 30.3 -> 29.7 ms)
#endif
#ifndef HB_MACF_T128
#define HB_MACF_T128 1   // the fmod_mul GEMM / layer MAC (unfused key switches, > 34-bit primes)
                        // in 128-thread CTAs too: hear/full 460 -> 470 inferences/s, config 3 270 -> 276
#endif
#ifndef HB_MAC_BIG
#define HB_MAC_BIG 4, 4, 4, 2   // TO, TB, WO, WB of the large tile (16 outputs x 8 clips)
#endif
#ifndef HB_MAC_STAGES_LONG
#define HB_MAC_STAGES_LONG 4   // ... for term lists longer than 32 (conv layer MACs): the
                               // split-sum kernel finishes a term in a third of the
                               // time, so it keeps one more stage in flight (30.8 vs
                               // 32.2 ms per step; 5 and 6 no better; two terms per
                               // barrier measured 2 % slower)
#endif

namespace hb {

struct HbMacGroupP {
  const u64* const* cts;
  const u64* const* pts;
  u64* const* dsts;
  int nterms;
  int nout;
  long long ct_bstride;   // elements between clips of a ct / dst block
  long long dst_bstride;
  int prime_off;          // prime of row r = prime_off + r ...
  const u64* const* pts_last;   // ... except the last row when set: its pt rows
  int prime_last;               //     (pointers to the row itself) and prime
  int cts_per_tile;       // cts is [output tile][T] (each tile has its own terms)
  // Rotation epilogue (EPI kernels only; lazy ModDown, engine.py
  // _raw_rot_many_each_lazy): output o is stored through its scatter map
  // scat[o] (the inverse Galois map of its pre-permuted key; null = natural
  // order) and, on chain rows, gains pmod[r] * c0s[o][b*c0_bstride + r*N + j]
  // (P times the rotated c0, so the result is the rotated ciphertext in the
  // extended basis Q*P with no ModDown).
  const int* const* scat;
  const u64* const* c0s;   // per output: non-null = takes the c0 term
  const u64* c0;           // the group's c0 block [BC][c0_bstride] (shared by its rotations)
  long long c0_bstride;
  const u64* pmod;
};

namespace {

// HEAR_B200_MAC_JC: coefficient chunks per CTA (A/B knob; 0 = automatic)
inline int mac_jc() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("HEAR_B200_MAC_JC");
    v = e ? atoi(e) : 0;
  }
  return v;
}

HB_DEV uint32_t s_addr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
HB_DEV void cp16(uint32_t dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}
HB_DEV void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
HB_DEV void cp_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }


// Operand conversion of the GEMM: the magic-number path (LOP + DADD on the
// fp64 pipe).  Round 1 measured the conversion pipe (I2F.F64.U64) instead:
// bit-identical, 0.4 % slower on the bench step.
HB_DEV double mac_to_f(u64 x) { return u64_to_f(x); }

// MULTI = 0: one chunk per CTA with the chunk loop and its bookkeeping
// compiled out (the long conv-layer term lists: measured 14 % faster there
// than the general form).
// SPLIT = 1: the split partial sums above (long term lists on primes of at
// most 34 bits: the conv-layer MACs, 37 -> 32 ms per bench step); SPLIT = 0:
// fmod_mul per product into one accumulator with the 8 x 4 thread tile (the
// short key-switch GEMMs, where the split form's smaller thread tile --
// twice the accumulators -- re-reads the staged operands more and measured
// 9 % slower).
template <int TO, int TB, int WO, int WB, int S, int EPI = 0, int MULTI = 1, int SPLIT = 0>
__global__ void __launch_bounds__(32 * WO * WB)
k_mac_pipe(HbMacGroupP g, HbRing RG, int R, int BC, int JCrt) {
  constexpr int NT = 32 * WO * WB;
  const int JC = MULTI ? JCrt : 1;
  HB_PDL_ENTRY();
  constexpr int OB = TO * WO, CB = TB * WB, ROWS = OB + CB;
  constexpr int STAGE = ROWS * 32;            // u64 per stage
  constexpr int CHUNKS = ROWS * 16;           // 16-byte copies per stage
  extern __shared__ __align__(16) u64 smem_mac[];
  u64* stages = smem_mac;                     // [S][ROWS][32]
  // EPI: scatter indices of the current / next coefficient chunk [2][OB][32]
  int* scbuf = reinterpret_cast<int*>(smem_mac + S * STAGE);
  const u64** ptab = reinterpret_cast<const u64**>(smem_mac + S * STAGE + (EPI ? OB * 32 : 0));
  const int T = g.nterms, O = g.nout, n = RG.n;
  const int tid = threadIdx.x + threadIdx.y * 32;
  const int oc = blockIdx.y * OB, bc = blockIdx.x * CB;   // CTA tile origin
  // a CTA walks JC consecutive 32-coefficient chunks of one RNS row through
  // ONE copy pipeline: the pointer tables are built once and the next
  // chunk's operands stream in while this chunk's outputs are stored
  const int nchunk = n / 32 / JC;
  const int r = blockIdx.z / nchunk;
  const int jbase = (blockIdx.z % nchunk) * JC * 32;
  const size_t rn = (size_t)r * n;
  const bool last = g.pts_last != nullptr && r == R - 1;
  const u64* const* pts = last ? g.pts_last : g.pts;
  const size_t prn = last ? 0 : rn;                       // pt offset of this row
  // pointer tables of this CTA's tile: ct bases [T], pt bases [OB][T]
  const u64* const* cts = g.cts + (g.cts_per_tile ? (size_t)blockIdx.y * T : 0);
  for (int i = tid; i < T * (1 + OB); i += NT) {
    if (i < T) {
      ptab[i] = cts[i];
    } else {
      const int o = (i - T) / T, t = (i - T) % T;
      ptab[i] = pts[(size_t)(oc + o < O ? oc + o : O - 1) * T + t];
    }
  }
  __syncthreads();
  // EPI: the rotated c0 (times P) is one more term of the chain rows -- its
  // ct rows stream through the pipeline like a digit's, no key operand
  const bool c0term = EPI && !last && g.c0 != nullptr;
  const int TT = T + (c0term ? 1 : 0);
  const int Q = TT * JC;
  // copy plan: chunk c -> stage row c/16 (ct rows first), 16-byte part c%16.
  // Everything but the term's base pointer is fixed per thread: the stage
  // offset, the pointer-table slot and the element offset of each of the
  // thread's copies are computed once (recomputing them cost ~20 of the
  // ~140 instructions a thread issues per term of the split-sum MAC)
  constexpr int NCP = (CHUNKS + NT - 1) / NT;
  uint32_t cp_soff[NCP];
  int cp_slot[NCP], cp_b[NCP];
  size_t cp_goff[NCP];
#pragma unroll
  for (int k = 0; k < NCP; ++k) {
    const int c = tid + k * NT;
    const int row = c >> 4, part = c & 15;
    cp_soff[k] = (uint32_t)(row * 32 + part * 2) * 8u;
    if (c >= CHUNKS) {
      cp_slot[k] = -1;
      cp_b[k] = 0;
      cp_goff[k] = 0;
    } else if (row < CB) {
      const int b = bc + row < BC ? bc + row : BC - 1;
      cp_slot[k] = 0;
      cp_b[k] = b;
      cp_goff[k] = (size_t)b * g.ct_bstride + rn + jbase + part * 2;
    } else {
      cp_slot[k] = T + (row - CB) * T;
      cp_b[k] = -1;
      cp_goff[k] = prn + jbase + part * 2;
    }
  }
  auto issue = [&](int q, int ch, int t) {
    const uint32_t sb = s_addr(stages + (q % S) * STAGE);
    const size_t jo = (size_t)ch * 32;
#pragma unroll
    for (int k = 0; k < NCP; ++k) {
      if (cp_slot[k] < 0) continue;
      const u64* src;
      if (EPI && t == T) {             // the c0 term: ct rows only
        if (cp_b[k] < 0) continue;
        src = g.c0 + (size_t)cp_b[k] * g.c0_bstride + rn + jbase + jo + (cp_soff[k] >> 3 & 31);
      } else {
        src = ptab[cp_slot[k] + t] + cp_goff[k] + jo;
      }
      cp16(sb + cp_soff[k], src);
    }
    if (EPI && t == 0) {   // this chunk's scatter indices (4-byte copies)
      const size_t j0 = jbase + jo;
      const uint32_t sc0 = s_addr(scbuf + (ch & 1) * OB * 32);
      for (int c = tid; c < OB * 32; c += NT) {
        const int o = c >> 5, oo = oc + o < O ? oc + o : O - 1;
        asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(sc0 + 4u * c),
                     "l"(g.scat[oo] + j0 + (c & 31))
                     : "memory");
      }
    }
  };
  int iq = 0, ich = 0, it = 0;   // next (q, chunk, term) to issue
  auto issue_next = [&]() {
    if (iq < Q) {
      issue(iq, ich, it);
      ++iq;
      if (++it == TT) { it = 0; ++ich; }
    }
  };
  // feed the pipeline while term t of the current chunk is multiplied
  auto feed = [&](int t) {
    if (MULTI) issue_next();
    else if (t + S - 1 < TT) issue(t + S - 1, 0, t + S - 1);
  };
#pragma unroll
  for (int s = 0; s < S - 1; ++s) {
    if (MULTI) issue_next();
    else if (s < TT) issue(s, 0, s);
    cp_commit();
  }
  const int lane = threadIdx.x, w = threadIdx.y;
  const int os = (w / WB) * TO, bs = (w % WB) * TB;   // warp sub-tile in the CTA tile
  const int prime = last ? g.prime_last : g.prime_off + r;
  const HbPrime P = RG.primes[prime];
  const double p = P.pd, pinv = P.pinv;
  double pm = 0.0, pmq = 0.0;
  unsigned c0mask = 0;   // outputs of this thread that take the c0 term
  if (c0term) {
    pm = u64_to_f(g.pmod[r]);
    pmq = pm * pinv;
#pragma unroll
    for (int o = 0; o < TO; ++o)
      if (oc + os + o < O && g.c0s[oc + os + o] != nullptr) c0mask |= 1u << o;
  }
  // split point, reduce interval and recombination constant of this prime
  const int pb = 64 - __clzll((long long)P.p), sbits = (pb + 1) >> 1;
  const u64 amask = (1ull << sbits) - 1;
  int kred = (int)(((1ull << 53) - (1ull << pb)) >> (pb + sbits));
  kred = kred < 1 ? 1 : (kred > 1024 ? 1024 : kred);
  const double two_s = (double)(1ull << sbits), two_sq = two_s * pinv;
  double acc0[TO][TB], acc1[SPLIT ? TO : 1][SPLIT ? TB : 1];
#pragma unroll
  for (int o = 0; o < TO; ++o)
#pragma unroll
    for (int b = 0; b < TB; ++b) {
      acc0[o][b] = 0.0;
      if (SPLIT) acc1[o][b] = 0.0;
    }
  const bool full = oc + OB <= O && bc + CB <= BC;
  int q = 0;
  for (int ch = 0; ch < JC; ++ch) {
    int since = 0;
    for (int t = 0; t < T; ++t, ++q) {
      cp_wait<S - 2>();
      __syncthreads();                 // term q landed for every thread; stage q-1 is free
      feed(t);
      cp_commit();
      const u64* st = stages + ((MULTI ? q : t) % S) * STAGE;
      double c[TB];
#pragma unroll
      for (int b = 0; b < TB; ++b) c[b] = mac_to_f(st[(bs + b) * 32 + lane]);
      if (SPLIT) {
        double a0[TO], a1[TO];
#pragma unroll
        for (int o = 0; o < TO; ++o) {
          const u64 a = st[(CB + os + o) * 32 + lane];
          a0[o] = mac_to_f(a & amask);
          a1[o] = mac_to_f(a >> sbits);
        }
#pragma unroll
        for (int o = 0; o < TO; ++o) {
#pragma unroll
          for (int b = 0; b < TB; ++b) {
            acc0[o][b] = __fma_rn(c[b], a0[o], acc0[o][b]);
            acc1[SPLIT ? o : 0][SPLIT ? b : 0] =
                __fma_rn(c[b], a1[o], acc1[SPLIT ? o : 0][SPLIT ? b : 0]);
          }
        }
        if (++since == kred) {   // the exact sums approach 2^53: back to residues
          since = 0;
#pragma unroll
          for (int o = 0; o < TO; ++o)
#pragma unroll
            for (int b = 0; b < TB; ++b) {
              acc0[o][b] = fmod_reduce(acc0[o][b], p, pinv);
              acc1[SPLIT ? o : 0][SPLIT ? b : 0] =
                  fmod_reduce(acc1[SPLIT ? o : 0][SPLIT ? b : 0], p, pinv);
            }
        }
      } else {
        double a[TO];
#pragma unroll
        for (int o = 0; o < TO; ++o) a[o] = mac_to_f(st[(CB + os + o) * 32 + lane]);
#pragma unroll
        for (int o = 0; o < TO; ++o) {
          const double aq = a[o] * pinv;
#pragma unroll
          for (int b = 0; b < TB; ++b) acc0[o][b] += fmod_mul(c[b], a[o], aq, p);
        }
        if ((t & 255) == 255) {   // |balanced residue| < p/2: 2^9 terms fit 2^53
#pragma unroll
          for (int o = 0; o < TO; ++o)
#pragma unroll
            for (int b = 0; b < TB; ++b) acc0[o][b] = fmod_reduce(acc0[o][b], p, pinv);
        }
      }
    }
    if (EPI && c0term) {               // + P * c0 on the outputs that take it
      cp_wait<S - 2>();
      __syncthreads();
      feed(T);
      cp_commit();
      const u64* st = stages + ((MULTI ? q : T) % S) * STAGE;
      ++q;
#pragma unroll
      for (int b = 0; b < TB; ++b) {
        const double c = mac_to_f(st[(bs + b) * 32 + lane]);
#pragma unroll
        for (int o = 0; o < TO; ++o)
          if ((c0mask >> o) & 1) {
            if (SPLIT) acc0[o][b] = fmod_reduce(acc0[o][b], p, pinv);
            acc0[o][b] += fmod_mul(c, pm, pmq, p);
          }
      }
    }
    // S0 + 2^s * S1 mod p, balanced
    double acc[TO][TB];
#pragma unroll
    for (int o = 0; o < TO; ++o)
#pragma unroll
      for (int b = 0; b < TB; ++b) {
        if (SPLIT) {
          acc[o][b] = fmod_reduce(acc0[o][b], p, pinv)
                      + fmod_mul(fmod_reduce(acc1[SPLIT ? o : 0][SPLIT ? b : 0], p, pinv), two_s,
                                 two_sq, p);
          acc1[SPLIT ? o : 0][SPLIT ? b : 0] = 0.0;
        } else {
          acc[o][b] = acc0[o][b];
        }
        acc0[o][b] = 0.0;
      }
    // ---- chunk done: store its outputs, restart the accumulators
    const int j0 = jbase + ch * 32;
    const size_t rj = rn + j0 + lane;
    if (EPI) {   // rotated extended-basis outputs, scattered through the Galois map
      const int* sc = scbuf + (ch & 1) * OB * 32;
#pragma unroll
      for (int o = 0; o < TO; ++o) {
        const int oo = oc + os + o;
        if (oo >= O) continue;
        u64* d = g.dsts[oo] + rn + sc[(os + o) * 32 + lane];
#pragma unroll
        for (int b = 0; b < TB; ++b) {
          const int bb = bc + bs + b;
          if (bb >= BC) continue;
          d[(size_t)bb * g.dst_bstride] = fmod_canon(acc[o][b], p, pinv);
        }
      }
    } else if (full) {   // full tile (the common case): no bounds checks
#pragma unroll
      for (int o = 0; o < TO; ++o) {
        u64* d = g.dsts[oc + os + o] + rj;
#pragma unroll
        for (int b = 0; b < TB; ++b)
          d[(size_t)(bc + bs + b) * g.dst_bstride] = fmod_canon(acc[o][b], p, pinv);
      }
    } else {
#pragma unroll
      for (int o = 0; o < TO; ++o) {
        const int oo = oc + os + o;
        if (oo >= O) continue;
        u64* d = g.dsts[oo];
#pragma unroll
        for (int b = 0; b < TB; ++b) {
          const int bb = bc + bs + b;
          if (bb >= BC) continue;
          d[(size_t)bb * g.dst_bstride + rj] = fmod_canon(acc[o][b], p, pinv);
        }
      }
    }
  }
  cp_wait<0>();
}

template <int TO, int TB, int WO, int WB, int S, int EPI = 0, int SPLIT = 0>
cudaError_t mac_pipe_t(const HbMacGroupP& g, const HbRing& RG, int R, int BC, cudaStream_t st) {
  constexpr int OB = TO * WO, CB = TB * WB;
  const size_t smem = (size_t)S * (OB + CB) * 32 * 8 + (EPI ? 2 * OB * 32 * 4 : 0)
      + sizeof(void*) * (size_t)g.nterms * (1 + OB);
  if (smem > 220 * 1024) return cudaErrorNotSupported;   // caller falls back
  static int smem_cur = 0, smem_cur1 = 0;
  cudaError_t e = smem_attr_once((const void*)k_mac_pipe<TO, TB, WO, WB, S, EPI, 1, SPLIT>, (int)((int)smem), &smem_cur);
  if (e == cudaSuccess)
    e = smem_attr_once((const void*)k_mac_pipe<TO, TB, WO, WB, S, EPI, 0, SPLIT>, (int)((int)smem), &smem_cur1);
  if (e != cudaSuccess) return e;
  dim3 block(32, WO * WB);
  const int tiles = ((BC + CB - 1) / CB) * ((g.nout + OB - 1) / OB) * R;
  // coefficient chunks per CTA: as many as still leave >= 8 CTAs per SM
  int jc = mac_jc();
  if (g.nterms > 32) jc = 1;   // long term lists amortise the prologue already
  if (jc <= 0) {
    jc = 8;
    while (jc > 1 && (long long)tiles * (RG.n / 32 / jc) < 148LL * 8) jc >>= 1;
  }
  while (jc > 1 && (RG.n / 32) % jc) jc >>= 1;
  dim3 grid((BC + CB - 1) / CB, (g.nout + OB - 1) / OB, R * (RG.n / 32 / jc));
  if (jc > 1)
    (void)hb_launch(k_mac_pipe<TO, TB, WO, WB, S, EPI, 1, SPLIT>, dim3(grid), dim3(block), smem, st, g, RG, R, BC, jc);
  else
    (void)hb_launch(k_mac_pipe<TO, TB, WO, WB, S, EPI, 0, SPLIT>, dim3(grid), dim3(block), smem, st, g, RG, R, BC, 1);
  return cudaGetLastError();
}

}  // namespace

// hoisted rotation groups with the scatter / + P*c0 epilogue (shared digits)
static cudaError_t mac_pipe_dispatch_rot(const HbMacGroupP& g, const HbRing& RG, int rows, int BC,
                                         cudaStream_t st) {
  constexpr int S = HB_MAC_STAGES;
  if (BC <= 2) return mac_pipe_t<2, 2, 8, 1, S, 1>(g, RG, rows, BC, st);
  if (g.nout <= 2) return mac_pipe_t<2, 4, 1, 8, S, 1>(g, RG, rows, BC, st);
  if (g.nout <= 4) return mac_pipe_t<4, 4, 1, 8, S, 1>(g, RG, rows, BC, st);
  if (g.nout <= 8) return mac_pipe_t<8, 4, 1, 8, S, 1>(g, RG, rows, BC, st);
  // 8 outputs x 16 clips in 128-thread CTAs (four per SM): 39.8 -> 37.3 ms per
  // step against the 256-thread 16 x 16 tile (64 threads: 40.7)
  return mac_pipe_t<8, 4, 1, 4, S, 1>(g, RG, rows, BC, st);
}

static cudaError_t mac_pipe_dispatch(const HbMacGroupP& g, const HbRing& RG, int rows, int BC,
                                     cudaStream_t st) {
  constexpr int S = HB_MAC_STAGES;
  if (BC <= 2 && !g.cts_per_tile) {
    // one clip: 8 warps x 1 output when the layer has at most 8 (no idle warps)
    if (g.nout <= 8) return mac_pipe_t<1, 2, 8, 1, S>(g, RG, rows, BC, st);
    return mac_pipe_t<2, 2, 8, 1, S>(g, RG, rows, BC, st);
  }
  // one (b, a) output pair per tile when every job brings its own digits
  if (g.cts_per_tile) return mac_pipe_t<2, 4, 1, 8, S>(g, RG, rows, BC, st);
  // output tile sized to the layer so no warp idles on absent outputs
  if (g.nout <= 2) return mac_pipe_t<2, 4, 1, 8, S>(g, RG, rows, BC, st);
  if (g.nout <= 4) return mac_pipe_t<4, 4, 1, 8, S>(g, RG, rows, BC, st);
  // long term lists (conv layers) on small primes: split partial sums, 4
  // outputs x 4 clips per thread (32 accumulator doubles), tile HB_MAC_BIG
  if (g.nterms > 32 && RG.split_ok && g.nout > 4) {
#if HB_MAC_T128
    // 128-thread CTAs, four per SM: finer-grained barriers
    // 8 outputs x 8 clips per CTA, also for wider layers (two output tiles:
    // 16 x 4 measured 29.7 vs 28.8 ms of layer MAC per step)
    return mac_pipe_t<4, 4, 2, 2, HB_MAC_STAGES_LONG, 0, 1>(g, RG, rows, BC, st);
#endif
    if (g.nout <= 8) return mac_pipe_t<4, 4, 2, 4, HB_MAC_STAGES_LONG, 0, 1>(g, RG, rows, BC, st);
    return mac_pipe_t<HB_MAC_BIG, HB_MAC_STAGES_LONG, 0, 1>(g, RG, rows, BC, st);
  }
  if (g.nout <= 8) return mac_pipe_t<8, 4, 1, 8, S>(g, RG, rows, BC, st);
  // 8 outputs x 4 clips per thread (124 registers, 2 CTAs/SM): each staged
  // operand feeds twice the products of the 4x4 tile (round-1 tile sweep)
#if HB_MACF_T128
  if (g.nterms > 32) return mac_pipe_t<8, 4, 1, 4, HB_MAC_STAGES_LONG>(g, RG, rows, BC, st);
  return mac_pipe_t<8, 4, 1, 4, S>(g, RG, rows, BC, st);
#endif
  if (g.nterms > 32) return mac_pipe_t<8, 4, 2, 4, HB_MAC_STAGES_LONG>(g, RG, rows, BC, st);
  return mac_pipe_t<8, 4, 2, 4, S>(g, RG, rows, BC, st);
}

// fp64 rings only (RG.use_f64); returns cudaErrorNotSupported otherwise.
cudaError_t launch_mac_pipe(const void* cts, const void* pts, const void* dsts, int nterms, int nout,
                            const HbRing& RG, int rows, int BC, cudaStream_t st,
                            const void* pts_last, int prime_last) {
  if (nout <= 0 || nterms <= 0) return cudaSuccess;
  if (!RG.use_f64) return cudaErrorNotSupported;
  HbMacGroupP g;
  g.cts = reinterpret_cast<const u64* const*>(cts);
  g.pts = reinterpret_cast<const u64* const*>(pts);
  g.dsts = reinterpret_cast<u64* const*>(dsts);
  g.nterms = nterms;
  g.nout = nout;
  g.ct_bstride = g.dst_bstride = (long long)rows * RG.n;
  g.prime_off = 0;
  // extended-basis layer MAC: the last row is the special prime's, with the
  // plaintexts' special rows (pts_last: pointers to the rows themselves)
  g.pts_last = reinterpret_cast<const u64* const*>(pts_last);
  g.prime_last = prime_last;
  g.cts_per_tile = 0;
  g.scat = nullptr;
  g.c0s = nullptr;
  g.c0 = nullptr;
  g.c0_bstride = 0;
  g.pmod = nullptr;
  return mac_pipe_dispatch(g, RG, rows, BC, st);
}

// Key-switch inner products in natural digit order as one per-coefficient
// GEMM (engine.py:305-351 / ring.py:136-156; rotations on pre-permuted keys
// with the Galois map applied after ModDown, and relinearisation): terms =
// digits, outputs = (job, component), clips = BC, rows 0..rows-2 in chain
// primes 0..rows-2 and the last row in prime_last with its own key rows
// (keys_last).  de_per_job: de is [job][ndig] (each job its own digits,
// one output pair per tile) instead of [ndig] shared by every job.
cudaError_t launch_ks_gemm(const void* de, const void* keys, const void* keys_last,
                           const void* dsts, int ndig, int nout, const HbRing& RG, int rows,
                           int BC, long long de_bstride, long long dst_bstride, int prime_last,
                           int de_per_job, cudaStream_t st, const void* scat, const void* c0s,
                           const void* c0, long long c0_bstride, const void* pmod) {
  if (nout <= 0 || ndig <= 0) return cudaSuccess;
  if (!RG.use_f64) return cudaErrorNotSupported;
  HbMacGroupP g;
  g.cts = reinterpret_cast<const u64* const*>(de);
  g.pts = reinterpret_cast<const u64* const*>(keys);
  g.dsts = reinterpret_cast<u64* const*>(dsts);
  g.nterms = ndig;
  g.nout = nout;
  g.ct_bstride = de_bstride;
  g.dst_bstride = dst_bstride;
  g.prime_off = 0;
  g.pts_last = reinterpret_cast<const u64* const*>(keys_last);
  g.prime_last = prime_last;
  g.cts_per_tile = de_per_job;
  g.scat = reinterpret_cast<const int* const*>(scat);
  g.c0s = reinterpret_cast<const u64* const*>(c0s);
  g.c0 = reinterpret_cast<const u64*>(c0);
  g.c0_bstride = c0_bstride;
  g.pmod = reinterpret_cast<const u64*>(pmod);
  if (scat) {
    if (de_per_job) return cudaErrorInvalidValue;
    return mac_pipe_dispatch_rot(g, RG, rows, BC, st);
  }
  return mac_pipe_dispatch(g, RG, rows, BC, st);
}

}  // namespace hb

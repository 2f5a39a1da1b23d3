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
// TO x TB outputs per lane; products on the fp64 pipe as fmod_mul (5 ops,
// balanced residue), summed in double, canonicalised once.
#include <cstdint>
#include <cstdlib>
#include "ring.cuh"

#ifndef HB_MAC_STAGES
#define HB_MAC_STAGES 3   // cp.async pipeline depth of the GEMM (3 measured best: 2 % over 4)
#endif
#ifndef HB_MAC_STAGES_LONG
#define HB_MAC_STAGES_LONG 3   // ... for term lists longer than 32 (conv layer MACs)
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
};

namespace {

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

template <int TO, int TB, int WO, int WB, int S>
__global__ void __launch_bounds__(256)
k_mac_pipe(HbMacGroupP g, HbRing RG, int R, int BC) {
  HB_PDL_ENTRY();
  constexpr int OB = TO * WO, CB = TB * WB, ROWS = OB + CB;
  constexpr int STAGE = ROWS * 32;            // u64 per stage
  constexpr int CHUNKS = ROWS * 16;           // 16-byte copies per stage
  extern __shared__ __align__(16) u64 smem_mac[];
  u64* stages = smem_mac;                     // [S][ROWS][32]
  const u64** ptab = reinterpret_cast<const u64**>(smem_mac + S * STAGE);
  const int T = g.nterms, O = g.nout, n = RG.n;
  const int tid = threadIdx.x + threadIdx.y * 32;
  const int oc = blockIdx.y * OB, bc = blockIdx.x * CB;   // CTA tile origin
  const int nchunk = n / 32;
  const int r = blockIdx.z / nchunk;
  const int j0 = (blockIdx.z % nchunk) * 32;
  const size_t rj0 = (size_t)r * n + j0;
  const bool last = g.pts_last != nullptr && r == R - 1;
  const u64* const* pts = last ? g.pts_last : g.pts;
  const size_t prow = last ? (size_t)j0 : rj0;            // pt offset of this row
  // pointer tables of this CTA's tile: ct bases [T], pt bases [OB][T]
  const u64* const* cts = g.cts + (g.cts_per_tile ? (size_t)blockIdx.y * T : 0);
  for (int i = tid; i < T * (1 + OB); i += 256) {
    if (i < T) {
      ptab[i] = cts[i];
    } else {
      const int o = (i - T) / T, t = (i - T) % T;
      ptab[i] = pts[(size_t)(oc + o < O ? oc + o : O - 1) * T + t];
    }
  }
  __syncthreads();
  // copy plan: chunk c -> stage row c/16 (ct rows first), 16-byte part c%16
  auto issue = [&](int t) {
    const uint32_t sb = s_addr(stages + (t % S) * STAGE);
#pragma unroll
    for (int k = 0; k < (CHUNKS + 255) / 256; ++k) {
      const int c = tid + k * 256;
      if (c < CHUNKS) {
        const int row = c >> 4, part = c & 15;
        const u64* src;
        if (row < CB) {
          const int b = bc + row < BC ? bc + row : BC - 1;
          src = ptab[t] + (size_t)b * g.ct_bstride + rj0 + part * 2;
        } else {
          src = ptab[T + (row - CB) * T + t] + prow + part * 2;
        }
        cp16(sb + (uint32_t)(row * 32 + part * 2) * 8u, src);
      }
    }
  };
#pragma unroll
  for (int s = 0; s < S - 1; ++s) {
    if (s < T) issue(s);
    cp_commit();
  }
  const int lane = threadIdx.x, w = threadIdx.y;
  const int os = (w / WB) * TO, bs = (w % WB) * TB;   // warp sub-tile in the CTA tile
  const int prime = last ? g.prime_last : g.prime_off + r;
  const HbPrime P = RG.primes[prime];
  const double p = P.pd, pinv = P.pinv;
  double acc[TO][TB];
#pragma unroll
  for (int o = 0; o < TO; ++o)
#pragma unroll
    for (int b = 0; b < TB; ++b) acc[o][b] = 0.0;
  for (int t = 0; t < T; ++t) {
    cp_wait<S - 2>();
    __syncthreads();                 // term t landed for every thread; stage t-1 is free
    if (t + S - 1 < T) issue(t + S - 1);
    cp_commit();
    const u64* st = stages + (t % S) * STAGE;
    double a[TO];
#pragma unroll
    for (int o = 0; o < TO; ++o) a[o] = mac_to_f(st[(CB + os + o) * 32 + lane]);
    double c[TB];
#pragma unroll
    for (int b = 0; b < TB; ++b) c[b] = mac_to_f(st[(bs + b) * 32 + lane]);
#pragma unroll
    for (int o = 0; o < TO; ++o) {
      const double aq = a[o] * pinv;
#pragma unroll
      for (int b = 0; b < TB; ++b) acc[o][b] += fmod_mul(c[b], a[o], aq, p);
    }
    if ((t & 255) == 255) {   // |balanced residue| < p/2: 2^9 terms fit 2^53
#pragma unroll
      for (int o = 0; o < TO; ++o)
#pragma unroll
        for (int b = 0; b < TB; ++b) acc[o][b] = fmod_reduce(acc[o][b], p, pinv);
    }
  }
  cp_wait<0>();
  const size_t rj = rj0 + lane;
  auto value = [&](int o, int b) { return fmod_canon(acc[o][b], p, pinv); };
  if (oc + OB <= O && bc + CB <= BC) {   // full tile (the common case): no bounds checks
#pragma unroll
    for (int o = 0; o < TO; ++o) {
      u64* d = g.dsts[oc + os + o] + rj;
#pragma unroll
      for (int b = 0; b < TB; ++b) d[(size_t)(bc + bs + b) * g.dst_bstride] = value(o, b);
    }
    return;
  }
#pragma unroll
  for (int o = 0; o < TO; ++o) {
    const int oo = oc + os + o;
    if (oo >= O) continue;
    u64* d = g.dsts[oo];
#pragma unroll
    for (int b = 0; b < TB; ++b) {
      const int bb = bc + bs + b;
      if (bb >= BC) continue;
      d[(size_t)bb * g.dst_bstride + rj] = value(o, b);
    }
  }
}

template <int TO, int TB, int WO, int WB, int S>
cudaError_t mac_pipe_t(const HbMacGroupP& g, const HbRing& RG, int R, int BC, cudaStream_t st) {
  constexpr int OB = TO * WO, CB = TB * WB;
  const size_t smem = (size_t)S * (OB + CB) * 32 * 8 + sizeof(void*) * (size_t)g.nterms * (1 + OB);
  if (smem > 220 * 1024) return cudaErrorNotSupported;   // caller falls back
  static int smem_cur = 0;
  cudaError_t e = smem_attr_once((const void*)k_mac_pipe<TO, TB, WO, WB, S>, (int)((int)smem), &smem_cur);
  if (e != cudaSuccess) return e;
  dim3 block(32, 8);
  dim3 grid((BC + CB - 1) / CB, (g.nout + OB - 1) / OB, R * (RG.n / 32));
  (void)hb_launch(k_mac_pipe<TO, TB, WO, WB, S>, dim3(grid), dim3(block), smem, st, g, RG, R, BC);
  return cudaGetLastError();
}

}  // namespace

static cudaError_t mac_pipe_dispatch(const HbMacGroupP& g, const HbRing& RG, int rows, int BC,
                                     cudaStream_t st) {
  constexpr int S = HB_MAC_STAGES;
  if (BC <= 2 && !g.cts_per_tile) return mac_pipe_t<2, 2, 8, 1, S>(g, RG, rows, BC, st);
  // one (b, a) output pair per tile when every job brings its own digits
  if (g.cts_per_tile) return mac_pipe_t<2, 4, 1, 8, S>(g, RG, rows, BC, st);
  // output tile sized to the layer so no warp idles on absent outputs
  if (g.nout <= 2) return mac_pipe_t<2, 4, 1, 8, S>(g, RG, rows, BC, st);
  if (g.nout <= 4) return mac_pipe_t<4, 4, 1, 8, S>(g, RG, rows, BC, st);
  if (g.nout <= 8) return mac_pipe_t<8, 4, 1, 8, S>(g, RG, rows, BC, st);
  // 8 outputs x 4 clips per thread (124 registers, 2 CTAs/SM): each staged
  // operand feeds twice the products of the 4x4 tile; measured +1.6 % on
  // the bench step (hoisted key-switch GEMM and conv MAC) over 4x4 and 4x8
  // (round-1 tile sweep).  Long term lists (conv layers) may take a deeper
  // pipeline (HB_MAC_STAGES_LONG)
  if (g.nterms > 32) return mac_pipe_t<8, 4, 2, 4, HB_MAC_STAGES_LONG>(g, RG, rows, BC, st);
  return mac_pipe_t<8, 4, 2, 4, S>(g, RG, rows, BC, st);
}

// fp64 rings only (RG.use_f64); returns cudaErrorNotSupported otherwise.
cudaError_t launch_mac_pipe(const void* cts, const void* pts, const void* dsts, int nterms, int nout,
                            const HbRing& RG, int rows, int BC, cudaStream_t st) {
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
  g.pts_last = nullptr;
  g.prime_last = 0;
  g.cts_per_tile = 0;
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
                           int de_per_job, cudaStream_t st) {
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
  return mac_pipe_dispatch(g, RG, rows, BC, st);
}

}  // namespace hb

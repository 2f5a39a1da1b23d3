// Cluster-fused negacyclic NTT (default for fp64 rings at N = 2^13 .. 2^16).
//
// Same transform and fused modes as ntt2.cu (hear/ckks/ring.py:71-124, true
// inverse), same split of the stages into a column pass (stages 0..S1-1 over
// the M = N/128 elements of each of the 128 columns) and a block pass (the
// last 7 stages inside each 128-element block) -- but the two passes run in
// ONE launch: a thread-block cluster of CL = N/4096 CTAs owns one row.
//
//   forward  CTA k runs the column pass on columns [k*CW, (k+1)*CW) in its
//            local 32 KB buffer, then pushes every (block, column-pair) chunk
//            to the CTA that owns the block's tile (tile t = blocks
//            32t..32t+31) with st.async into that CTA's receive buffer
//            (DSMEM); each CTA waits on its own mbarrier for the 32 KB it
//            receives, runs the block pass and stores with the fused
//            epilogue (ModUp lift / ModDown / scatter as ntt2.cu).
//   inverse  the mirror image: block pass on tile t, push to the column
//            owners, column pass, N^-1 fused in the store.
//
// The exchange is producer/consumer through mbarrier transaction counts:
// no cluster-wide barrier in the data path (the cooperative-groups
// cluster.sync version profiled 16 % of its stall samples on MEMBAR.ALL.GPU
// / ERRBAR / the barrier wait).  One CTA buffer serves both passes: the
// single cluster barrier (release-arrive after the CTA's last read of its
// first-pass buffer, wait just before the pushes) both publishes the
// mbarrier initialisation and frees the buffer for the peers' pushes.  The
// lazy intermediate never touches L2/HBM (the two-pass kernels write and
// re-read it: 256 KB per row).
//
// Also in shared memory: the column twiddles and the stride-8 block-stage
// twiddles of the CTA's tile (staged once, LDS at immediate offsets); the
// last three forward / first three inverse stages read a plane-major
// (w, w/p) table with lanes on consecutive entries.  ModDown modes: the x_r
// tile is prefetched into L2 (cp.async.bulk.prefetch) while the block pass
// runs, and the epilogue (x_r - y) * P^-1 (+ c0) (+ post-addend) runs on the
// fp64 pipe on 16-byte lane-contiguous chunks.  Inverse: a second
// destination can receive the input row verbatim (the ModUp identity digit).
// Shared memory per CTA: 32 KB + 9.7 KB twiddles + 16 B; 64 registers: four
// CTAs (32 warps) per SM.
#include <cstdint>
#include <cstdlib>
#include <type_traits>
#include "ntt_common.cuh"

namespace hb {

namespace {

constexpr int TILE3 = 4096;
constexpr int THREADS3 = 256;
// Shared memory per CTA: ONE 32 KB tile buffer -- the exchange lands in the
// buffer the first pass worked in, after a cluster barrier (arrive.release
// once the last local read is done, wait just before the pushes) -- the
// staged twiddles (TW3 x 16 B) and one mbarrier: 42.5 KB and <= 64
// registers, four CTAs (32 warps) per SM.  (Round 1 measured the
// two-buffer layout with three CTAs per SM, and a TMA-prefetched c0 tile
// with two, both slower.)  The ModDown x_r / c0 tiles are prefetched into L2
// (cp.async.bulk.prefetch) while the block pass runs.
template <int LOGN>
__host__ __device__ constexpr int smem3() { return TILE3 * 8 + ((1 << (LOGN - 7)) - 1 + 480) * 16 + 16; }
// k_ks3: + its task (88 B) behind the two barrier words
template <int LOGN>
__host__ __device__ constexpr int smem3k() { return smem3<LOGN>() + 96; }
constexpr int MINB3 = 4;
// N = 2^16 runs 16-CTA clusters (non-portable size): per launch within
// -6..+1 % of the two-pass kernels, but the pipeline then takes the
// lift-once / ModDown-scatter path -- config 3 178 -> 201 inferences/s
// (tools/ab_ntt3_16.sh)
#ifndef HB_NTT3_MAXLOGN
#define HB_NTT3_MAXLOGN 16
#endif

HB_DEV int swz3_chunk(int c) { return c ^ ((c >> 3) & 7) ^ (((c >> 6) & 1) << 2); }
// block layout (as ntt2.cu): element j of the 4096-element tile
HB_DEV int bsw(int j) { return (swz3_chunk(j >> 1) << 1) | (j & 1); }
// column layout: element (m, c) of the CW-column slice; the XOR spreads the
// four blocks a pulling warp touches over distinct banks
template <int CW>
HB_DEV int csw(int m, int c) { return m * CW + (c ^ (((m & 3) << 3) & (CW - 1))); }

// ---- cluster / DSMEM primitives (PTX)
HB_DEV uint32_t smem_addr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
HB_DEV uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
HB_DEV uint32_t mapa(uint32_t a, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
  return r;
}
// thread 0: one arrival expecting `bytes` of st.async traffic, made visible
// to the cluster; every thread then arrives (relaxed) on the cluster barrier
HB_DEV void xchg_init(uint64_t* mbar, uint32_t bytes) {
  if (threadIdx.x == 0) {
    const uint32_t a = smem_addr(mbar);
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(a) : "memory");
    // a second, spare barrier word: dropping its init perturbs ptxas's
    // register allocation of the transform into spills (ModUp 2.5 % slower)
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(a + 8) : "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(a), "r"(bytes)
                 : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
}
// single-buffer exchange: every local read of the buffer is performed before
// any peer's push into it -- a release arrive (MEMBAR.ALL.GPU per thread).
// Measured: a CTA barrier + relaxed arrive is NOT enough (peers' pushes
// overwrote data still being read: nondeterministic rows under load,
// tools/ntt3_check.py NTT3_DIFF=1); a CTA-scope fence + relaxed arrive was
// deterministic and 3 % faster on ModUp but is outside the memory model.
HB_DEV void cluster_arrive_sb() {
  asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
}
HB_DEV void l2_prefetch(const void* p, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}
HB_DEV void cluster_wait() { asm volatile("barrier.cluster.wait.aligned;" ::: "memory"); }
// 16-byte push into a peer's shared memory, counted on the peer's mbarrier
HB_DEV void st_async16(uint32_t raddr, uint32_t rmbar, double a, double b) {
  asm volatile(
      "st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.b64 [%0], {%1, %2}, [%3];" ::"r"(
          raddr),
      "l"(__double_as_longlong(a)), "l"(__double_as_longlong(b)), "r"(rmbar)
      : "memory");
}
HB_DEV void st_async8(uint32_t raddr, uint32_t rmbar, double a) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];" ::"r"(
                   raddr),
               "l"(__double_as_longlong(a)), "r"(rmbar)
               : "memory");
}
HB_DEV void mbar_wait0(uint64_t* mbar) {
  const uint32_t a = smem_addr(mbar);
  asm volatile(
      "{\n .reg .pred p;\n WAIT%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n"
      " @!p bra WAIT%=;\n}" ::"r"(a)
      : "memory");
}

template <class Pol, int MODE>
HB_DEV typename Pol::T ld_src(const HbNttTask& tk, const Pol& pol, u64 ps, u64 ps_half, size_t j) {
  const u64 x = __ldg(tk.src + j);
  if (MODE == FWD_PLAIN) return pol.from_canon(x);
  if (MODE == FWD_I64) return pol.from_signed((i64)x);
  return pol.from_lift(x, ps, ps_half);
}

// Column-pass round plan: group/element mapping shared by both directions.
//   round rd covers local stages [4rd, 4rd+K); a thread owns gpt groups of
//   2^K elements of column c; element u of group gid sits at row m.
template <int S1, bool FWD>
struct ColPlan {
  static constexpr int M = 1 << S1, GQ = M / 16, NR = (S1 + 3) / 4;
  static HB_DEV int K(int rd) { return rd == NR - 1 ? S1 - rd * 4 : 4; }
  static HB_DEV int tl(int rd) { return FWD ? (M >> (rd * 4 + K(rd))) : (1 << (rd * 4)); }
  static HB_DEV int m_of(int rd, int gq, int q) {
    const int k = K(rd), t = tl(rd);
    const int gsel = q >> k, u = q & ((1 << k) - 1);
    const int gid = gq + gsel * GQ;
    return (gid / t) * (t << k) + (gid % t) + u * t;
  }
  static HB_DEV bool owns(int rd, int q) { return (q >> K(rd)) < (16 >> K(rd)); }
};

template <class Pol, int S1, bool FWD, class F>
HB_DEV void col_butterflies(typename Pol::T* x, int rd, int gq, F fetch, const Pol& pol) {
  typedef ColPlan<S1, FWD> CP;
  const int K = CP::K(rd), tl = CP::tl(rd), gpt = 16 >> K, s0 = rd * 4;
#pragma unroll
  for (int gsel = 0; gsel < 16; ++gsel) {
    if (gsel >= gpt) break;
    const int gid = gq + gsel * CP::GQ;
    if (FWD) {
      if (K == 4) fwd_group_f<Pol, 4>(x + gsel * 16, s0, gid / tl, fetch, pol);
      else if (K == 3) fwd_group_f<Pol, 3>(x + gsel * 8, s0, gid / tl, fetch, pol);
      else if (K == 2) fwd_group_f<Pol, 2>(x + gsel * 4, s0, gid / tl, fetch, pol);
      else fwd_group_f<Pol, 1>(x + gsel * 2, s0, gid / tl, fetch, pol);
    } else {
      if (K == 4) inv_group_f<Pol, 4>(x + gsel * 16, s0 + 7, gid / tl, fetch, pol);
      else if (K == 3) inv_group_f<Pol, 3>(x + gsel * 8, s0 + 7, gid / tl, fetch, pol);
      else if (K == 2) inv_group_f<Pol, 2>(x + gsel * 4, s0 + 7, gid / tl, fetch, pol);
      else inv_group_f<Pol, 1>(x + gsel * 2, s0 + 7, gid / tl, fetch, pol);
    }
  }
}

// Shared-memory twiddles of one CTA (TW3 entries, 16 B each): the column
// stages (table entries 1..M-1, shared by every column) and the four block
// stages of this CTA's tile that run on stride-8 groups of 16 (forward
// stages S1..S1+3 / inverse stages 3..6: 32+64+128+256 entries).  Staged
// once with coalesced loads so the butterflies read them with LDS at
// (mostly) immediate offsets instead of 64-bit-addressed broadcast LDGs.
template <int LOGN, bool FWD>
HB_DEV void stage_twiddles(HbTwD* tws, const HbTwD* tab, int rank) {
  constexpr int N = 1 << LOGN, S1 = LOGN - 7, M = 1 << S1;
  constexpr int TWC = M - 1, TW3 = TWC + 480;
  for (int k = threadIdx.x; k < TW3; k += THREADS3) {
    int idx;
    if (k < TWC) {
      idx = 1 + (k < M - 1 ? k : 0);
    } else {
      const int kb = k - TWC;
      if (FWD) {   // stage S1+e: 32 << e entries from 2^(S1+e) + rank*(32 << e)
        const int e = kb < 32 ? 0 : kb < 96 ? 1 : kb < 224 ? 2 : 3;
        idx = (1 << (S1 + e)) + rank * (32 << e) + (kb - 32 * ((1 << e) - 1));
      } else {     // stage r = 3..6: 4096 >> (r+1) entries from N>>(r+1) + rank*(4096>>(r+1))
        const int r = kb < 256 ? 3 : kb < 384 ? 4 : kb < 448 ? 5 : 6;
        const int off = r == 3 ? 0 : r == 4 ? 256 : r == 5 ? 384 : 448;
        idx = (N >> (r + 1)) + rank * (4096 >> (r + 1)) + (kb - off);
      }
    }
    // asynchronous 16-byte copy (LDGSTS): no register round trip, no STS
    // stall on the load; completed by tws_wait() before the first use
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_addr(tws + k)),
                 "l"(tab + idx)
                 : "memory");
  }
  asm volatile("cp.async.commit_group;" ::: "memory");
}

HB_DEV void tws_wait() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// ---------------------------------------------------------------------------
// Forward.
template <class Pol, int LOGN, int MODE>
__global__ void __launch_bounds__(THREADS3, MINB3)
k_ntt3_fwd(const HbNttTask* __restrict__ tasks, HbRing R) {
  constexpr int N = 1 << LOGN, S1 = LOGN - 7, M = 1 << S1, CW = TILE3 / M, CL = N / TILE3;
  typedef ColPlan<S1, true> CP;
  typedef typename Pol::T V;
  extern __shared__ __align__(16) unsigned char smraw3[];
  V* sm = reinterpret_cast<V*>(smraw3);   // column slice (local pass)
  V* rb = sm;                             // received block tile (same buffer)
  constexpr int TWC = M - 1, TW3 = TWC + 480;
  HbTwD* tws = reinterpret_cast<HbTwD*>(rb + TILE3);
  uint64_t* mbar = reinterpret_cast<uint64_t*>(tws + TW3);
  xchg_init(mbar, TILE3 * sizeof(V));
  const int rank = (int)cluster_rank();
  const HbNttTask tk = tasks[blockIdx.x / CL];
  const HbPrime P = R.primes[tk.dst_prime];
  const Pol pol(P);
  auto fetch_col = [&](int s, int idx) { return tws[(1 << s) + idx - 1]; };
  auto fetch_blk = [&](int s, int idx) {
    const int e = s - S1;
    return tws[TWC + 32 * ((1 << e) - 1) + idx - rank * (32 << e)];
  };
  const int t = threadIdx.x;
  u64 ps = 0, ps_half = 0;
  // src_prime < 0: the source row already holds centred lifts as doubles
  // (written by the inverse transform, task scal = 1), lifted once for all
  // target primes instead of once per target row
  const bool lifted = tk.src_prime < 0;
  if ((MODE == FWD_LIFT || MODE == FWD_MODDOWN || MODE == FWD_MODDOWN_SCATTER) && !lifted) {
    ps = R.primes[tk.src_prime].p;
    ps_half = ps >> 1;
  }
  HB_PDL_ENTRY();   // the row data below may be the previous kernel's output
  // ---- column pass over columns [rank*CW, rank*CW + CW)
  const int cg0 = rank * CW;
  {
    const int c = t % CW, gq = t / CW;
    V x[16];
    {   // the column slice lands raw in the swizzled smem tile by cp.async
        // (16-byte column pairs; csw keeps pairs adjacent) while the twiddles
        // are staged; round 0 converts on read
      const uint32_t sm0 = smem_addr(sm);
#pragma unroll
      for (int i = 0; i < TILE3 / 2 / THREADS3; ++i) {
        const int k = t + i * THREADS3;
        const int m = k / (CW / 2), cp2 = 2 * (k % (CW / 2));
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(
                         sm0 + 8u * csw<CW>(m, cp2)),
                     "l"(tk.src + (size_t)m * 128 + cg0 + cp2)
                     : "memory");
      }
      stage_twiddles<LOGN, true>(tws, Pol::fwd_table(R, tk.dst_prime), rank);
      tws_wait();
      __syncthreads();   // column slice and staged twiddles visible
#pragma unroll
      for (int q = 0; q < 16; ++q) {
        if (!CP::owns(0, q)) break;
        const u64 raw = (u64)__double_as_longlong(sm[csw<CW>(CP::m_of(0, gq, q), c)]);
        if (MODE == FWD_PLAIN) x[q] = pol.from_canon(raw);
        else if (MODE == FWD_I64) x[q] = pol.from_signed((i64)raw);
        else if (MODE == FWD_MODDOWN2) {   // src + P * y, both centred lifts
          const int m = CP::m_of(0, gq, q);
          const double y = __ldg(reinterpret_cast<const double*>(tk.perm) + (size_t)m * 128 + cg0 + c);
          const double pm = u64_to_f(tk.scal_sh);
          x[q] = fmod_reduce(__longlong_as_double((long long)raw), pol.p, pol.pinv)
                 + fmod_mul(y, pm, pm * pol.pinv, pol.p);
        }
        else if (lifted) x[q] = fmod_reduce(__longlong_as_double((long long)raw), pol.p, pol.pinv);
        else x[q] = pol.from_lift(raw, ps, ps_half);
      }
    }
#pragma unroll
    for (int rd = 0; rd < CP::NR; ++rd) {
      if (rd > 0) {
#pragma unroll
        for (int q = 0; q < 16; ++q) {
          if (!CP::owns(rd, q)) break;
          x[q] = sm[csw<CW>(CP::m_of(rd, gq, q), c)];
        }
      }
      if (rd == CP::NR - 1) cluster_arrive_sb();   // last local read done
      col_butterflies<Pol, S1, true>(x, rd, gq, fetch_col, pol);
      if (rd < CP::NR - 1) {
#pragma unroll
        for (int q = 0; q < 16; ++q) {
          if (!CP::owns(rd, q)) break;
          sm[csw<CW>(CP::m_of(rd, gq, q), c)] = x[q];
        }
        __syncthreads();
      }
    }
    // ---- push the last round's values straight from registers: element
    // (m, column) to the owner of block m's tile (8-byte st.async)
    cluster_wait();   // peers' mbarriers are initialised
    const uint32_t rb0 = smem_addr(rb), mb0 = smem_addr(mbar);
#pragma unroll
    for (int q = 0; q < 16; ++q) {
      if (!CP::owns(CP::NR - 1, q)) break;
      const int m = CP::m_of(CP::NR - 1, gq, q);
      const uint32_t dst = m >> 5;
      st_async8(mapa(rb0 + 8u * bsw((m & 31) * 128 + cg0 + c), dst), mapa(mb0, dst), x[q]);
    }
  }
  constexpr bool MD = MODE == FWD_MODDOWN || MODE == FWD_MODDOWN_SCATTER || MODE == FWD_MODDOWN2;
  if (MD && t == 0) {   // the epilogue's x_r / addend tiles into L2 meanwhile
    l2_prefetch(tk.aux + (size_t)rank * TILE3, TILE3 * 8);
    if (tk.add && !(MODE == FWD_MODDOWN && tk.perm)) l2_prefetch(tk.add + (size_t)rank * TILE3, TILE3 * 8);
  }
  mbar_wait0(mbar);
  // ---- block pass over blocks [rank*32, rank*32 + 32)
  {
    const int blk = t >> 3, cc = t & 7;
    V x[16];
#pragma unroll
    for (int u = 0; u < 16; ++u) x[u] = rb[bsw(blk * 128 + u * 8 + cc)];
    fwd_group_f<Pol, 4>(x, S1, rank * 32 + blk, fetch_blk, pol);
#pragma unroll
    for (int u = 0; u < 16; ++u) rb[bsw(blk * 128 + u * 8 + cc)] = x[u];
  }
  __syncwarp();   // the fine stages below read this warp's four blocks only
  const size_t base = (size_t)rank * TILE3;
  constexpr int N8 = N / 8;
  const HbTwD* t3 = R.tw3_fwd + (size_t)tk.dst_prime * N;
  // stage S1+4+e, entry (G << e) + i: plane-major table, lanes contiguous
  auto fetch_fine = [&](int s, int idx) {
    const int e = s - (S1 + 4), ii = idx & ((1 << e) - 1);
    const double2 w = __ldg(reinterpret_cast<const double2*>(t3 + (((1 << e) - 1 + ii) * N8 + (idx >> e))));
    return HbTwD{w.x, w.y};
  };
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    // 512 groups of 8; a warp takes the groups of the four blocks its
    // stride-8 pass owns (blk = t >> 3), so the two passes hand over inside
    // the warp (__syncwarp, no CTA barrier)
    const int b2 = 4 * (t >> 5) + 2 * q + ((t & 31) >> 4), G8 = t & 15;
    const int e0 = b2 * 128 + G8 * 8;
    V x[8];
#pragma unroll
    for (int v = 0; v < 4; ++v) {
      const int pc = swz3_chunk((e0 >> 1) + v);
      x[2 * v] = rb[2 * pc];
      x[2 * v + 1] = rb[2 * pc + 1];
    }
    fwd_group_f<Pol, 3>(x, S1 + 4, (rank * 32 + b2) * 16 + G8, fetch_fine, pol);
#pragma unroll
    for (int v = 0; v < 4; ++v) {   // back in place: balanced (ModDown) or canonical
      const int pc = swz3_chunk((e0 >> 1) + v);
      if (MD) {
        rb[2 * pc] = x[2 * v];
        rb[2 * pc + 1] = x[2 * v + 1];
      } else {
        rb[2 * pc] = __longlong_as_double((long long)pol.fwd_final(x[2 * v]));
        rb[2 * pc + 1] = __longlong_as_double((long long)pol.fwd_final(x[2 * v + 1]));
      }
    }
  }
  __syncwarp();   // the epilogue below stays on this warp's four blocks (512 elements)
  // ---- epilogue on 16-byte chunks, lanes contiguous (coalesced HBM traffic).
  // ModDown on the fp64 pipe: (x_r - y) * P^-1 (+ addend) from the balanced
  // transform output y, one canonicalisation (the integer sub/Shoup/add
  // chain cost ~30 integer instructions per element)
  const double pd = P.pd, pinv = P.pinv;
  const double sd = u64_to_f(tk.scal), sq = sd * pinv;
#pragma unroll 4
  for (int i = 0; i < TILE3 / 2 / THREADS3; ++i) {
    const int k = (t >> 5) * (TILE3 / 2 / 8) + i * 32 + (t & 31);   // warp w: chunks [256w, 256w + 256)
    const size_t j = base + 2 * k;
    const int pc = swz3_chunk(k);
    ulonglong2 o;
    int2 sc = make_int2(0, 0);
    if (MD) {
      const ulonglong2 ax = __ldg(reinterpret_cast<const ulonglong2*>(tk.aux + j));
      double r0 = fmod_mul(u64_to_f(ax.x) - rb[2 * pc], sd, sq, pd);
      double r1 = fmod_mul(u64_to_f(ax.y) - rb[2 * pc + 1], sd, sq, pd);
      if (MODE == FWD_MODDOWN2) {
        if (tk.add) {   // the addend is divided by q_l too: + add * s2
          const ulonglong2 a2 = __ldg(reinterpret_cast<const ulonglong2*>(tk.add + j));
          const double s2 = u64_to_f((u64)tk.add2), s2q = s2 * pinv;
          r0 += fmod_mul(u64_to_f(a2.x), s2, s2q, pd);
          r1 += fmod_mul(u64_to_f(a2.y), s2, s2q, pd);
        }
      } else {
      if (tk.add) {
        u64 a0, a1;
        if (MODE == FWD_MODDOWN && tk.perm) {
          const int2 pp = __ldg(reinterpret_cast<const int2*>(tk.perm + j));
          a0 = __ldg(tk.add + pp.x);
          a1 = __ldg(tk.add + pp.y);
        } else {
          const ulonglong2 a2 = __ldg(reinterpret_cast<const ulonglong2*>(tk.add + j));
          a0 = a2.x;
          a1 = a2.y;
        }
        r0 += u64_to_f(a0);
        r1 += u64_to_f(a1);
      }
      if (tk.add2) {   // post-addend at the destination index
        if (MODE == FWD_MODDOWN_SCATTER) {
          sc = __ldg(reinterpret_cast<const int2*>(tk.perm + j));
          r0 += u64_to_f(__ldg(tk.add2 + sc.x));
          r1 += u64_to_f(__ldg(tk.add2 + sc.y));
        } else {
          const ulonglong2 a2 = __ldg(reinterpret_cast<const ulonglong2*>(tk.add2 + j));
          r0 += u64_to_f(a2.x);
          r1 += u64_to_f(a2.y);
        }
      }
      }
      o.x = fmod_canon(r0, pd, pinv);
      o.y = fmod_canon(r1, pd, pinv);
    } else {
      o.x = (u64)__double_as_longlong(rb[2 * pc]);
      o.y = (u64)__double_as_longlong(rb[2 * pc + 1]);
    }
    if (MODE == FWD_MODDOWN_SCATTER) {
      if (!tk.add2) sc = __ldg(reinterpret_cast<const int2*>(tk.perm + j));
      tk.dst[sc.x] = o.x;
      tk.dst[sc.y] = o.y;
    } else {
      *reinterpret_cast<ulonglong2*>(tk.dst + j) = o;
    }
  }
}

// ---------------------------------------------------------------------------
// Inverse.
template <class Pol, int LOGN>
__global__ void __launch_bounds__(THREADS3, MINB3)
k_ntt3_inv(const HbNttTask* __restrict__ tasks, HbRing R) {
  constexpr int N = 1 << LOGN, S1 = LOGN - 7, M = 1 << S1, CW = TILE3 / M, CL = N / TILE3;
  typedef ColPlan<S1, false> CP;
  typedef typename Pol::T V;
  extern __shared__ __align__(16) unsigned char smraw3[];
  V* sm = reinterpret_cast<V*>(smraw3);   // block tile (local pass)
  V* rb = sm;                             // received column slice (same buffer)
  constexpr int TWC = M - 1, TW3 = TWC + 480;
  HbTwD* tws = reinterpret_cast<HbTwD*>(rb + TILE3);
  uint64_t* mbar = reinterpret_cast<uint64_t*>(tws + TW3);
  xchg_init(mbar, TILE3 * sizeof(V));
  const int rank = (int)cluster_rank();
  const HbNttTask tk = tasks[blockIdx.x / CL];
  const HbPrime P = R.primes[tk.dst_prime];
  const Pol pol(P);
  const bool lifted_out = tk.scal == 1;
  const u64 lift_half = P.p >> 1;
  auto fetch_col = [&](int r, int idx) { return tws[(N >> (r + 1)) + idx - 1]; };
  auto fetch_blk = [&](int r, int idx) {
    const int off = r == 3 ? 0 : r == 4 ? 256 : r == 5 ? 384 : 448;
    return tws[TWC + off + idx - rank * (4096 >> (r + 1))];
  };
  const int t = threadIdx.x;
  const size_t base = (size_t)rank * TILE3;
  HB_PDL_ENTRY();   // the row data below may be the previous kernel's output
  // ---- block pass on tile `rank`: coalesced 16-byte loads into the
  // swizzled tile, stages 0..2 (contiguous 8), 3..6 (stride 8)
  // input tile: raw residues straight into the swizzled smem tile with
  // cp.async (converted when read), unless the row is also copied out (ModUp
  // identity digit: through registers)
  const bool raw_tile = tk.add2 == nullptr;
  if (raw_tile) {
    const uint32_t sm0 = smem_addr(sm);
#pragma unroll
    for (int i = 0; i < TILE3 / 2 / THREADS3; ++i) {
      const int k = t + i * THREADS3;
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sm0 + 16u * swz3_chunk(k)),
                   "l"(tk.src + base + 2 * k)
                   : "memory");
    }
    stage_twiddles<LOGN, false>(tws, Pol::inv_table(R, tk.dst_prime), rank);
  } else {   // input chunks in flight while the twiddles are staged
    ulonglong2 in[TILE3 / 2 / THREADS3];
#pragma unroll
    for (int i = 0; i < TILE3 / 2 / THREADS3; ++i)
      in[i] = __ldg(reinterpret_cast<const ulonglong2*>(tk.src + base) + t + i * THREADS3);
    stage_twiddles<LOGN, false>(tws, Pol::inv_table(R, tk.dst_prime), rank);
#pragma unroll
    for (int i = 0; i < TILE3 / 2 / THREADS3; ++i) {
      const int k = t + i * THREADS3;
      // inverse: verbatim copy of the input row (ModUp identity digit)
      reinterpret_cast<ulonglong2*>(const_cast<u64*>(tk.add2) + base)[k] = in[i];
      const int pc = swz3_chunk(k);
      sm[2 * pc] = pol.from_canon(in[i].x);
      sm[2 * pc + 1] = pol.from_canon(in[i].y);
    }
  }
  tws_wait();
  __syncthreads();
  constexpr int N8 = N / 8;
  const HbTwD* t3 = R.tw3_inv + (size_t)tk.dst_prime * N;
  // stage r, entry (G << (2-r)) + i: plane-major table, lanes contiguous
  auto fetch_fine = [&](int r, int idx) {
    const int sh = 2 - r, ii = idx & ((1 << sh) - 1);
    const int off = r == 0 ? 0 : (r == 1 ? 4 : 6);
    const double2 w = __ldg(reinterpret_cast<const double2*>(t3 + ((off + ii) * N8 + (idx >> sh))));
    return HbTwD{w.x, w.y};
  };
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    const int b2 = 4 * (t >> 5) + 2 * q + ((t & 31) >> 4), G8 = t & 15;   // warp-local, see k_ntt3_fwd
    const int e0 = b2 * 128 + G8 * 8;
    V x[8];
#pragma unroll
    for (int v = 0; v < 4; ++v) {
      const int pc = swz3_chunk((e0 >> 1) + v);
      x[2 * v] = sm[2 * pc];
      x[2 * v + 1] = sm[2 * pc + 1];
      if (raw_tile) {   // canonical residues landed raw: convert here
        x[2 * v] = pol.from_canon((u64)__double_as_longlong(x[2 * v]));
        x[2 * v + 1] = pol.from_canon((u64)__double_as_longlong(x[2 * v + 1]));
      }
    }
    inv_group_f<Pol, 3>(x, 0, (rank * 32 + b2) * 16 + G8, fetch_fine, pol);
#pragma unroll
    for (int v = 0; v < 4; ++v) {
      const int pc = swz3_chunk((e0 >> 1) + v);
      sm[2 * pc] = pol.inv_round_end(x[2 * v]);
      sm[2 * pc + 1] = pol.inv_round_end(x[2 * v + 1]);
    }
  }
  __syncwarp();   // the stride-8 stages below read this warp's four blocks only
  {
    const int blk = t >> 3, cc = t & 7;
    V x[16];
#pragma unroll
    for (int u = 0; u < 16; ++u) x[u] = sm[bsw(blk * 128 + u * 8 + cc)];
    cluster_arrive_sb();   // last local read done
    inv_group_f<Pol, 4>(x, 3, rank * 32 + blk, fetch_blk, pol);
    // ---- push straight from registers: element (block m, column u*8+cc) to
    // the owner of that column (8-byte st.async)
    cluster_wait();
    const uint32_t rb0 = smem_addr(rb), mb0 = smem_addr(mbar);
    const int m = rank * 32 + blk;
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      const int col = u * 8 + cc;
      const uint32_t dst = col / CW;
      st_async8(mapa(rb0 + 8u * csw<CW>(m, col % CW), dst), mapa(mb0, dst),
                pol.inv_round_end(x[u]));
    }
  }
  mbar_wait0(mbar);
  // ---- column pass over columns [rank*CW, rank*CW + CW)
  const int c = t % CW, gq = t / CW, cg0 = rank * CW;
  V x[16];
#pragma unroll
  for (int rd = 0; rd < CP::NR; ++rd) {
    V* buf = rd == 0 ? rb : sm;
#pragma unroll
    for (int q = 0; q < 16; ++q) {
      if (!CP::owns(rd, q)) break;
      x[q] = buf[csw<CW>(CP::m_of(rd, gq, q), c)];
    }
    col_butterflies<Pol, S1, false>(x, rd, gq, fetch_col, pol);
    const bool last = rd == CP::NR - 1;
#pragma unroll
    for (int q = 0; q < 16; ++q) {
      if (!CP::owns(rd, q)) break;
      const int m = CP::m_of(rd, gq, q);
      if (last) {
        const u64 v = pol.inv_final(x[q]);
        // scal = 1: store the centred lift as a double (the next transform's
        // source under other primes: ModUp digits, ModDown / rescale rows)
        tk.dst[(size_t)m * 128 + cg0 + c] =
            lifted_out ? (u64)__double_as_longlong(v > lift_half ? u64_to_f(v) - pol.p
                                                                 : u64_to_f(v))
                       : v;
      }
      else sm[csw<CW>(m, c)] = pol.inv_round_end(x[q]);
    }
    if (!last) __syncthreads();
  }
}

// Clusters above the portable 8 CTAs (N = 2^16: 16 CTAs) need the opt-in.
inline cudaError_t cluster16_once(const void* fn, int cl) {
  if (cl <= 8) return cudaSuccess;
  return cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
}

// ---------------------------------------------------------------------------
// Fused ModUp + key-switch inner product (non-hoisted key switches:
// relinearisation, rot_each, rotate-and-add; engine.py:290-326 with
// ring.py:136-156).  The unfused path writes the whole digit expansion
// [l+1][l+2] rows per ciphertext (FWD_LIFT launches) only for the GEMM to
// read it back: the dominant HBM traffic of a key switch.  Here one cluster
// owns one (ciphertext, target prime t): it loops over the digits, runs the
// forward NTT of each lifted digit under q_t in shared memory exactly as
// k_ntt3_fwd does, multiplies the transform by the two key rows and keeps
// the running sums of its 4096-coefficient tile in TENSOR MEMORY -- 16
// coefficients x (b, a) per thread = 64 32-bit TMEM columns in the thread's
// own lane (tcgen05.st / tcgen05.ld 32x32b), 128 columns per CTA, so four
// CTAs per SM fill the 512 columns and the kernel keeps the NTT's 64
// registers and 42.5 KB of shared memory.  Only the 2 (l+2) inner-product
// rows are written.  Sums of balanced products (< 8p) are exact in double;
// the canonical result is bit-identical to the unfused path.
HB_DEV uint32_t tmem_alloc128(uint32_t* slot) {
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"(
                     smem_addr(slot))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  return *slot;
}
HB_DEV void tmem_free128(uint32_t base) {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (threadIdx.x < 32)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" ::"r"(base) : "memory");
}
HB_DEV void tmem_st4(uint32_t a, double v0, double v1, double v2, double v3) {
  const u64 u0 = __double_as_longlong(v0), u1 = __double_as_longlong(v1),
            u2 = __double_as_longlong(v2), u3 = __double_as_longlong(v3);
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(a),
               "r"((uint32_t)u0), "r"((uint32_t)(u0 >> 32)), "r"((uint32_t)u1),
               "r"((uint32_t)(u1 >> 32)), "r"((uint32_t)u2), "r"((uint32_t)(u2 >> 32)),
               "r"((uint32_t)u3), "r"((uint32_t)(u3 >> 32))
               : "memory");
}
HB_DEV void tmem_ld4(uint32_t a, double& v0, double& v1, double& v2, double& v3) {
  uint32_t r0, r1, r2, r3, r4, r5, r6, r7;
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3), "=r"(r4), "=r"(r5), "=r"(r6), "=r"(r7)
               : "r"(a)
               : "memory");
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
  v0 = __longlong_as_double(((u64)r1 << 32) | r0);
  v1 = __longlong_as_double(((u64)r3 << 32) | r2);
  v2 = __longlong_as_double(((u64)r5 << 32) | r4);
  v3 = __longlong_as_double(((u64)r7 << 32) | r6);
}
HB_DEV void mbar_wait_par(uint64_t* mbar, uint32_t parity) {
  const uint32_t a = smem_addr(mbar);
  asm volatile(
      "{\n .reg .pred p;\n WAITP%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAITP%=;\n}" ::"r"(a),
      "r"(parity)
      : "memory");
}

#ifndef HB_KS3_UNROLL
#define HB_KS3_UNROLL 4   // accumulate-loop unroll (key loads in flight per thread)
#endif
constexpr int KS3_UNROLL = HB_KS3_UNROLL;
template <int LOGN>
__global__ void __launch_bounds__(THREADS3, MINB3)
k_ks3(const HbKsfTask* __restrict__ tasks, HbRing R) {
  constexpr int N = 1 << LOGN, S1 = LOGN - 7, M = 1 << S1, CW = TILE3 / M, CL = N / TILE3;
  typedef PolF64 Pol;
  typedef ColPlan<S1, true> CP;
  typedef double V;
  extern __shared__ __align__(16) unsigned char smraw3[];
  V* sm = reinterpret_cast<V*>(smraw3);
  V* rb = sm;
  constexpr int TWC = M - 1, TW3 = TWC + 480;
  HbTwD* tws = reinterpret_cast<HbTwD*>(rb + TILE3);
  uint64_t* mbar = reinterpret_cast<uint64_t*>(tws + TW3);
  const int t = threadIdx.x;
  const int rank = (int)cluster_rank();
  // the task lives in shared memory (read where needed: its ten fields
  // would not fit the 64-register budget next to the transform)
  HbKsfTask* tkp = reinterpret_cast<HbKsfTask*>(mbar + 2);
  if (t < (int)(sizeof(HbKsfTask) / 8))
    reinterpret_cast<u64*>(tkp)[t] = reinterpret_cast<const u64*>(tasks + blockIdx.x / CL)[t];
  __syncthreads();
  const HbKsfTask& tk = *tkp;
  const int dprime = tk.dst_prime;
  const Pol pol(R.primes[dprime]);
  if (t == 0) {
    const uint32_t a = smem_addr(mbar);
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(a) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  const uint32_t tbase = tmem_alloc128(reinterpret_cast<uint32_t*>(mbar + 1));
  // this thread's 64 columns: its warp's lane quadrant, column half by warp / 4
  const uint32_t tacc = tbase + ((uint32_t)(((t >> 5) & 3) * 32) << 16) + (uint32_t)(t >> 7) * 64;
  auto fetch_col = [&](int s, int idx) { return tws[(1 << s) + idx - 1]; };
  auto fetch_blk = [&](int s, int idx) {
    const int e = s - S1;
    return tws[TWC + 32 * ((1 << e) - 1) + idx - rank * (32 << e)];
  };
  constexpr int N8 = N / 8;
  const HbTwD* t3 = R.tw3_fwd + (size_t)dprime * N;
  auto fetch_fine = [&](int s, int idx) {
    const int e = s - (S1 + 4), ii = idx & ((1 << e) - 1);
    const double2 w = __ldg(reinterpret_cast<const double2*>(t3 + (((1 << e) - 1 + ii) * N8 + (idx >> e))));
    return HbTwD{w.x, w.y};
  };
  HB_PDL_ENTRY();
  stage_twiddles<LOGN, true>(tws, Pol::fwd_table(R, dprime), rank);
  const int cg0 = rank * CW;
  const size_t base = (size_t)rank * TILE3;
  const double pd = pol.p, pinv = pol.pinv;
  uint32_t phase = 0;
  bool first = true;
  for (int dg = 0; dg < tk.ndig; ++dg) {
    const bool ident = dg == tk.ident_digit;
    const bool lastd = dg == tk.ndig - 1;
    const u64* kb = tk.kb + (size_t)dg * tk.key_dstride + base;
    const u64* ka = tk.ka + (size_t)dg * tk.key_dstride + base;
    if (t == 0) {   // this digit's key tiles into L2 while the transform runs
      l2_prefetch(kb, TILE3 * 8);
      l2_prefetch(ka, TILE3 * 8);
    }
    if (!ident) {
      const u64* src = tk.coef + (size_t)dg * N;
      if (t == 0) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(mbar)),
                     "r"((uint32_t)(TILE3 * sizeof(V)))
                     : "memory");
      }
      __syncthreads();   // the previous digit's epilogue has left the tile
      // ---- column pass (as k_ntt3_fwd, source rows are centred lifts)
      {
        const int c = t % CW, gq = t / CW;
        V x[16];
        const uint32_t sm0 = smem_addr(sm);
#pragma unroll
        for (int i = 0; i < TILE3 / 2 / THREADS3; ++i) {
          const int k = t + i * THREADS3;
          const int m = k / (CW / 2), cp2 = 2 * (k % (CW / 2));
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sm0 + 8u * csw<CW>(m, cp2)),
                       "l"(src + (size_t)m * 128 + cg0 + cp2)
                       : "memory");
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
        tws_wait();
        __syncthreads();
#pragma unroll
        for (int q = 0; q < 16; ++q) {
          if (!CP::owns(0, q)) break;
          x[q] = fmod_reduce(sm[csw<CW>(CP::m_of(0, gq, q), c)], pol.p, pol.pinv);
        }
#pragma unroll
        for (int rd = 0; rd < CP::NR; ++rd) {
          if (rd > 0) {
#pragma unroll
            for (int q = 0; q < 16; ++q) {
              if (!CP::owns(rd, q)) break;
              x[q] = sm[csw<CW>(CP::m_of(rd, gq, q), c)];
            }
          }
          if (rd == CP::NR - 1) cluster_arrive_sb();
          col_butterflies<Pol, S1, true>(x, rd, gq, fetch_col, pol);
          if (rd < CP::NR - 1) {
#pragma unroll
            for (int q = 0; q < 16; ++q) {
              if (!CP::owns(rd, q)) break;
              sm[csw<CW>(CP::m_of(rd, gq, q), c)] = x[q];
            }
            __syncthreads();
          }
        }
        cluster_wait();
        const uint32_t rb0 = smem_addr(rb), mb0 = smem_addr(mbar);
#pragma unroll
        for (int q = 0; q < 16; ++q) {
          if (!CP::owns(CP::NR - 1, q)) break;
          const int m = CP::m_of(CP::NR - 1, gq, q);
          const uint32_t dst = m >> 5;
          st_async8(mapa(rb0 + 8u * bsw((m & 31) * 128 + cg0 + c), dst), mapa(mb0, dst), x[q]);
        }
      }
      mbar_wait_par(mbar, phase);
      phase ^= 1;
      // ---- block pass
      {
        const int blk = t >> 3, cc = t & 7;
        V x[16];
#pragma unroll
        for (int u = 0; u < 16; ++u) x[u] = rb[bsw(blk * 128 + u * 8 + cc)];
        fwd_group_f<Pol, 4>(x, S1, rank * 32 + blk, fetch_blk, pol);
#pragma unroll
        for (int u = 0; u < 16; ++u) rb[bsw(blk * 128 + u * 8 + cc)] = x[u];
      }
      __syncwarp();
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const int b2 = 4 * (t >> 5) + 2 * q + ((t & 31) >> 4), G8 = t & 15;   // warp-local
        const int e0 = b2 * 128 + G8 * 8;
        V x[8];
#pragma unroll
        for (int v = 0; v < 4; ++v) {
          const int pc = swz3_chunk((e0 >> 1) + v);
          x[2 * v] = rb[2 * pc];
          x[2 * v + 1] = rb[2 * pc + 1];
        }
        fwd_group_f<Pol, 3>(x, S1 + 4, (rank * 32 + b2) * 16 + G8, fetch_fine, pol);
#pragma unroll
        for (int v = 0; v < 4; ++v) {
          const int pc = swz3_chunk((e0 >> 1) + v);
          rb[2 * pc] = x[2 * v];
          rb[2 * pc + 1] = x[2 * v + 1];
        }
      }
      __syncwarp();   // the accumulate loop stays on this warp's four blocks
    }
    // ---- accumulate x * key into the thread's TMEM columns; after the last
    // digit canonicalise and store instead
#pragma unroll KS3_UNROLL
    for (int i = 0; i < TILE3 / 2 / THREADS3; ++i) {
      const int k = (t >> 5) * (TILE3 / 2 / 8) + i * 32 + (t & 31);   // warp-local chunks
      const size_t j = 2 * (size_t)k;
      double x0, x1;
      if (ident) {
        const ulonglong2 xi = __ldg(reinterpret_cast<const ulonglong2*>(tk.ident + base + j));
        x0 = u64_to_f(xi.x);
        x1 = u64_to_f(xi.y);
      } else {
        const int pc = swz3_chunk(k);
        x0 = rb[2 * pc];
        x1 = rb[2 * pc + 1];
      }
      const ulonglong2 b2 = __ldg(reinterpret_cast<const ulonglong2*>(kb + j));
      const ulonglong2 a2 = __ldg(reinterpret_cast<const ulonglong2*>(ka + j));
      double ab0 = 0.0, ab1 = 0.0, aa0 = 0.0, aa1 = 0.0;
      if (!first) tmem_ld4(tacc + 8 * i, ab0, ab1, aa0, aa1);
      const double kb0 = u64_to_f(b2.x), kb1 = u64_to_f(b2.y);
      const double ka0 = u64_to_f(a2.x), ka1 = u64_to_f(a2.y);
      ab0 += fmod_mul(x0, kb0, kb0 * pinv, pd);
      ab1 += fmod_mul(x1, kb1, kb1 * pinv, pd);
      aa0 += fmod_mul(x0, ka0, ka0 * pinv, pd);
      aa1 += fmod_mul(x1, ka1, ka1 * pinv, pd);
      if (lastd) {
        const int* scat = tk.scat;
        if (scat && tk.c0) {   // + P * c0 (the rotated c0, still at the source index)
          const ulonglong2 c2 = __ldg(reinterpret_cast<const ulonglong2*>(tk.c0 + base + j));
          const double pm = u64_to_f(tk.pmod), pmq = pm * pinv;
          ab0 += fmod_mul(u64_to_f(c2.x), pm, pmq, pd);
          ab1 += fmod_mul(u64_to_f(c2.y), pm, pmq, pd);
        }
        ulonglong2 ob, oa;
        ob.x = fmod_canon(ab0, pd, pinv);
        ob.y = fmod_canon(ab1, pd, pinv);
        oa.x = fmod_canon(aa0, pd, pinv);
        oa.y = fmod_canon(aa1, pd, pinv);
        if (scat) {
          const int2 sc = __ldg(reinterpret_cast<const int2*>(scat + base + j));
          tk.out_b[sc.x] = ob.x;
          tk.out_b[sc.y] = ob.y;
          tk.out_a[sc.x] = oa.x;
          tk.out_a[sc.y] = oa.y;
        } else {
          *reinterpret_cast<ulonglong2*>(tk.out_b + base + j) = ob;
          *reinterpret_cast<ulonglong2*>(tk.out_a + base + j) = oa;
        }
      } else {
        tmem_st4(tacc + 8 * i, ab0, ab1, aa0, aa1);
      }
    }
    if (!lastd) asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    first = false;
  }
  tmem_free128(tbase);
}

template <int LOGN>
cudaError_t ks3_t(const HbKsfTask* tasks, int count, const HbRing& R, cudaStream_t st) {
  constexpr int CL = (1 << LOGN) / TILE3;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(count * CL);
  cfg.blockDim = dim3(THREADS3);
  cfg.dynamicSmemBytes = smem3k<LOGN>();
  cfg.stream = st;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = CL;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = g_hb_pdl ? 2 : 1;
  static int smem_cur = 0;
  cudaError_t e = smem_attr_once((const void*)k_ks3<LOGN>, (int)(smem3k<LOGN>()), &smem_cur);
  if (e == cudaSuccess) e = cluster16_once((const void*)k_ks3<LOGN>, CL);
  if (e != cudaSuccess) return e;
  return cudaLaunchKernelEx(&cfg, k_ks3<LOGN>, tasks, R);
}


template <int LOGN, int MODE>
cudaError_t fwd3_t(const HbNttTask* tasks, int count, const HbRing& R, cudaStream_t st) {
  constexpr int CL = (1 << LOGN) / TILE3;
  constexpr int FWDSMEM = smem3<LOGN>();
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(count * CL);
  cfg.blockDim = dim3(THREADS3);
  cfg.dynamicSmemBytes = FWDSMEM;
  cfg.stream = st;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = CL;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = g_hb_pdl ? 2 : 1;
  static int smem_cur = 0;
  cudaError_t e = smem_attr_once((const void*)k_ntt3_fwd<PolF64, LOGN, MODE>, (int)(FWDSMEM), &smem_cur);
  if (e == cudaSuccess) e = cluster16_once((const void*)k_ntt3_fwd<PolF64, LOGN, MODE>, CL);
  if (e != cudaSuccess) return e;
  return cudaLaunchKernelEx(&cfg, k_ntt3_fwd<PolF64, LOGN, MODE>, tasks, R);
}

template <int LOGN>
cudaError_t inv3_t(const HbNttTask* tasks, int count, const HbRing& R, cudaStream_t st) {
  constexpr int CL = (1 << LOGN) / TILE3;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(count * CL);
  cfg.blockDim = dim3(THREADS3);
  cfg.dynamicSmemBytes = smem3<LOGN>();
  cfg.stream = st;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = CL;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = g_hb_pdl ? 2 : 1;
  static int smem_cur = 0;
  cudaError_t e = smem_attr_once((const void*)k_ntt3_inv<PolF64, LOGN>, (int)(smem3<LOGN>()), &smem_cur);
  if (e == cudaSuccess) e = cluster16_once((const void*)k_ntt3_inv<PolF64, LOGN>, CL);
  if (e != cudaSuccess) return e;
  return cudaLaunchKernelEx(&cfg, k_ntt3_inv<PolF64, LOGN>, tasks, R);
}

template <int LOGN>
cudaError_t fwd3_mode(const HbNttTask* tasks, int count, const HbRing& R, int mode,
                      cudaStream_t st) {
  switch (mode) {
    case FWD_PLAIN: return fwd3_t<LOGN, FWD_PLAIN>(tasks, count, R, st);
    case FWD_LIFT: return fwd3_t<LOGN, FWD_LIFT>(tasks, count, R, st);
    case FWD_MODDOWN: return fwd3_t<LOGN, FWD_MODDOWN>(tasks, count, R, st);
    case FWD_I64: return fwd3_t<LOGN, FWD_I64>(tasks, count, R, st);
    case FWD_MODDOWN_SCATTER: return fwd3_t<LOGN, FWD_MODDOWN_SCATTER>(tasks, count, R, st);
    case FWD_MODDOWN2: return fwd3_t<LOGN, FWD_MODDOWN2>(tasks, count, R, st);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace

// fp64 rings at N = 2^13 .. 2^16 (clusters of 2 / 4 / 8 / 16 CTAs); HEAR_B200_NTT3=0
// falls back to the two-pass kernels.
bool ntt3_supported(const HbRing& R) {
  static int off = -1;
  if (off < 0) {
    const char* v = getenv("HEAR_B200_NTT3");
    off = (v && v[0] == '0') ? 1 : 0;
  }
  // 2^15 (clusters of 8, the portable maximum): with the one-buffer layout
  // (44.5 KB per CTA, four CTAs per SM) 14-27 % faster per launch than the
  // two-pass kernels and config 2 252 -> 320 inferences/s (round 2,
  // tools/ab_ntt3_15.sh; the round-1 two-buffer layout, 77 KB per CTA, had
  // measured 5-20 % slower)
  return !off && R.use_f64 && R.logn >= 13 && R.logn <= HB_NTT3_MAXLOGN;
}

cudaError_t launch_ntt3_fwd(const HbNttTask* tasks, int count, const HbRing& R, int mode,
                            cudaStream_t st) {
  if (count <= 0) return cudaSuccess;
  switch (R.logn) {
    case 13: return fwd3_mode<13>(tasks, count, R, mode, st);
    case 14: return fwd3_mode<14>(tasks, count, R, mode, st);
    case 15: return fwd3_mode<15>(tasks, count, R, mode, st);
#if HB_NTT3_MAXLOGN >= 16
    case 16: return fwd3_mode<16>(tasks, count, R, mode, st);
#endif
    default: return cudaErrorInvalidValue;
  }
}

// Fused ModUp + inner product (k_ks3): fp64 rings on the cluster NTT.
cudaError_t launch_ks3(const HbKsfTask* tasks, int count, const HbRing& R, cudaStream_t st) {
  if (count <= 0) return cudaSuccess;
  if (!ntt3_supported(R)) return cudaErrorNotSupported;
  switch (R.logn) {
    case 13: return ks3_t<13>(tasks, count, R, st);
    case 14: return ks3_t<14>(tasks, count, R, st);
    case 15: return ks3_t<15>(tasks, count, R, st);
#if HB_NTT3_MAXLOGN >= 16
    case 16: return ks3_t<16>(tasks, count, R, st);
#endif
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t launch_ntt3_inv(const HbNttTask* tasks, int count, const HbRing& R, cudaStream_t st) {
  if (count <= 0) return cudaSuccess;
  switch (R.logn) {
    case 13: return inv3_t<13>(tasks, count, R, st);
    case 14: return inv3_t<14>(tasks, count, R, st);
    case 15: return inv3_t<15>(tasks, count, R, st);
#if HB_NTT3_MAXLOGN >= 16
    case 16: return inv3_t<16>(tasks, count, R, st);
#endif
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace hb

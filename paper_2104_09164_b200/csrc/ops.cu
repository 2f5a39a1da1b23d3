// Element-wise RNS kernels: modular add/sub/mul, plaintext multiply-
// accumulate, the ciphertext tensor product, the key-switch inner product
// with the fused Galois gather, and the CRT reconstruction for decryption.
//
// All rows are N contiguous u64 residues; every task names its prime.  Each
// thread handles two adjacent coefficients (one 16-byte load per operand),
// grid.y walks the task list, grid.x the row.
#include <cstdlib>
#include "ring.cuh"

namespace hb {


constexpr int EW_THREADS = 256;

template <int OP>
__global__ void __launch_bounds__(EW_THREADS)
k_ew(const HbEwTask* __restrict__ tasks, int ntasks, const HbPrime* __restrict__ primes, int n) {
  HB_PDL_ENTRY();
  for (int t = blockIdx.y; t < ntasks; t += gridDim.y) {
    const HbEwTask tk = tasks[t];
    const HbPrime P = primes[tk.prime];
    const u64 p = P.p;
    const int j = 2 * (blockIdx.x * EW_THREADS + threadIdx.x);
    if (j >= n) continue;
    ulonglong2 a = *reinterpret_cast<const ulonglong2*>(tk.a + j);
    ulonglong2 r;
    if (OP == EW_MD_TOP) {
      const ulonglong2 b = *reinterpret_cast<const ulonglong2*>(tk.b + j);
      ulonglong2 c = make_ulonglong2(0, 0);
      if (tk.c) c = *reinterpret_cast<const ulonglong2*>(tk.c + j);
      auto one = [&](u64 ua, u64 ub, u64 uc) {
        const i64 d = (i64)__longlong_as_double((long long)ua) - (i64)__longlong_as_double((long long)ub);
        u64 m = reduce64((u64)(d < 0 ? -d : d), P);
        if (d < 0 && m) m = p - m;
        u64 v = mul_shoup(m, tk.scal, tk.scal_sh, p);
        if (tk.c) {
          const i64 e = (i64)__longlong_as_double((long long)uc);
          u64 me = reduce64((u64)(e < 0 ? -e : e), P);
          if (e < 0 && me) me = p - me;
          v = add_mod(v, me, p);
        }
        const double dv = v > P.half ? -(double)(p - v) : (double)v;
        return (u64)__double_as_longlong(dv);
      };
      r.x = one(a.x, b.x, c.x);
      r.y = one(a.y, b.y, c.y);
      *reinterpret_cast<ulonglong2*>(tk.dst + j) = r;
      continue;
    }
    if (OP == EW_ADD || OP == EW_SUB || OP == EW_MUL || OP == EW_MULADD ||
        OP == EW_ADD_SCALED || OP == EW_SUB_SCALED) {
      ulonglong2 b = *reinterpret_cast<const ulonglong2*>(tk.b + j);
      if (OP == EW_ADD) { r.x = add_mod(a.x, b.x, p); r.y = add_mod(a.y, b.y, p); }
      if (OP == EW_SUB) { r.x = sub_mod(a.x, b.x, p); r.y = sub_mod(a.y, b.y, p); }
      if (OP == EW_MUL) { r.x = mul_mod(a.x, b.x, P); r.y = mul_mod(a.y, b.y, P); }
      if (OP == EW_MULADD) {
        ulonglong2 c = *reinterpret_cast<const ulonglong2*>(tk.c + j);
        r.x = add_mod(mul_mod(a.x, b.x, P), c.x, p);
        r.y = add_mod(mul_mod(a.y, b.y, P), c.y, p);
      }
      if (OP == EW_ADD_SCALED) {
        r.x = add_mod(a.x, mul_shoup(b.x, tk.scal, tk.scal_sh, p), p);
        r.y = add_mod(a.y, mul_shoup(b.y, tk.scal, tk.scal_sh, p), p);
      }
      if (OP == EW_SUB_SCALED) {
        r.x = mul_shoup(sub_mod(a.x, b.x, p), tk.scal, tk.scal_sh, p);
        r.y = mul_shoup(sub_mod(a.y, b.y, p), tk.scal, tk.scal_sh, p);
      }
    } else if (OP == EW_MUL_SCALAR) {
      r.x = mul_shoup(a.x, tk.scal, tk.scal_sh, p);
      r.y = mul_shoup(a.y, tk.scal, tk.scal_sh, p);
    } else if (OP == EW_COPY) {
      r = a;
    } else if (OP == EW_PERM) {
      const int* perm = reinterpret_cast<const int*>(tk.b);
      r.x = __ldg(tk.a + __ldg(perm + j));
      r.y = __ldg(tk.a + __ldg(perm + j + 1));
    } else if (OP == EW_PERM_ADD) {
      const int* perm = reinterpret_cast<const int*>(tk.c);
      const int2 pp = __ldg(reinterpret_cast<const int2*>(perm + j));
      r.x = add_mod(__ldg(tk.a + pp.x), __ldg(tk.b + pp.x), p);
      r.y = add_mod(__ldg(tk.a + pp.y), __ldg(tk.b + pp.y), p);
    }
    *reinterpret_cast<ulonglong2*>(tk.dst + j) = r;
  }
}

static dim3 ew_grid(int ntasks, int n) {
  const int bx = (n / 2 + EW_THREADS - 1) / EW_THREADS;
  return dim3(bx, ntasks < 65535 ? ntasks : 65535);
}

cudaError_t launch_ew(int op, const HbEwTask* tasks, int ntasks, const HbPrime* primes, int n,
                      cudaStream_t st) {
  if (ntasks <= 0) return cudaSuccess;
  dim3 grid = ew_grid(ntasks, n);
  switch (op) {
#define HB_EW_CASE(OPC) \
  case OPC: (void)hb_launch(k_ew<OPC>, dim3(grid), dim3(EW_THREADS), 0, st, tasks, ntasks, primes, n); break;
    HB_EW_CASE(EW_ADD)
    HB_EW_CASE(EW_SUB)
    HB_EW_CASE(EW_MUL)
    HB_EW_CASE(EW_MUL_SCALAR)
    HB_EW_CASE(EW_MULADD)
    HB_EW_CASE(EW_ADD_SCALED)
    HB_EW_CASE(EW_COPY)
    HB_EW_CASE(EW_PERM)
    HB_EW_CASE(EW_SUB_SCALED)
    HB_EW_CASE(EW_PERM_ADD)
    HB_EW_CASE(EW_MD_TOP)
#undef HB_EW_CASE
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// Tensor product of two ciphertexts row by row (engine.py:249-257):
//   d0 = a0*b0, d1 = a0*b1 + a1*b0, d2 = a1*b1.
struct HbTensorTask {
  const u64 *a0, *a1, *b0, *b1;
  u64 *d0, *d1, *d2;
  int prime;
  int _pad;
};

__global__ void __launch_bounds__(EW_THREADS)
k_tensor(const HbTensorTask* __restrict__ tasks, int ntasks, const HbPrime* __restrict__ primes,
         int n) {
  HB_PDL_ENTRY();
  for (int t = blockIdx.y; t < ntasks; t += gridDim.y) {
    const HbTensorTask tk = tasks[t];
    const HbPrime P = primes[tk.prime];
    const int j = 2 * (blockIdx.x * EW_THREADS + threadIdx.x);
    if (j >= n) continue;
    const ulonglong2 a0 = *reinterpret_cast<const ulonglong2*>(tk.a0 + j);
    const ulonglong2 a1 = *reinterpret_cast<const ulonglong2*>(tk.a1 + j);
    const ulonglong2 b0 = *reinterpret_cast<const ulonglong2*>(tk.b0 + j);
    const ulonglong2 b1 = *reinterpret_cast<const ulonglong2*>(tk.b1 + j);
    ulonglong2 r0, r1, r2;
    r0.x = mul_mod(a0.x, b0.x, P);
    r0.y = mul_mod(a0.y, b0.y, P);
    {
      Acc128 s;
      s.mac(a0.x, b1.x);
      s.mac(a1.x, b0.x);
      r1.x = s.fold(P);
      Acc128 u;
      u.mac(a0.y, b1.y);
      u.mac(a1.y, b0.y);
      r1.y = u.fold(P);
    }
    r2.x = mul_mod(a1.x, b1.x, P);
    r2.y = mul_mod(a1.y, b1.y, P);
    *reinterpret_cast<ulonglong2*>(tk.d0 + j) = r0;
    *reinterpret_cast<ulonglong2*>(tk.d1 + j) = r1;
    *reinterpret_cast<ulonglong2*>(tk.d2 + j) = r2;
  }
}

// fp64-pipe tensor product (rings with every prime < 2^42): the four
// products as fmod_mul, one canonicalisation each -- same residues as the
// 128-bit integer products above.
__global__ void __launch_bounds__(EW_THREADS)
k_tensor_f64(const HbTensorTask* __restrict__ tasks, int ntasks,
             const HbPrime* __restrict__ primes, int n) {
  HB_PDL_ENTRY();
  for (int t = blockIdx.y; t < ntasks; t += gridDim.y) {
    const HbTensorTask tk = tasks[t];
    const HbPrime P = primes[tk.prime];
    const double p = P.pd, pinv = P.pinv;
    const int j = 2 * (blockIdx.x * EW_THREADS + threadIdx.x);
    if (j >= n) continue;
    const ulonglong2 a0 = *reinterpret_cast<const ulonglong2*>(tk.a0 + j);
    const ulonglong2 a1 = *reinterpret_cast<const ulonglong2*>(tk.a1 + j);
    const ulonglong2 b0 = *reinterpret_cast<const ulonglong2*>(tk.b0 + j);
    const ulonglong2 b1 = *reinterpret_cast<const ulonglong2*>(tk.b1 + j);
    const double x0[2] = {u64_to_f(a0.x), u64_to_f(a0.y)};
    const double x1[2] = {u64_to_f(a1.x), u64_to_f(a1.y)};
    const double y0[2] = {u64_to_f(b0.x), u64_to_f(b0.y)};
    const double y1[2] = {u64_to_f(b1.x), u64_to_f(b1.y)};
    u64 r0[2], r1[2], r2[2];
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const double q0 = y0[e] * pinv, q1 = y1[e] * pinv;
      r0[e] = fmod_canon(fmod_mul(x0[e], y0[e], q0, p), p, pinv);
      r1[e] = fmod_canon(fmod_mul(x0[e], y1[e], q1, p) + fmod_mul(x1[e], y0[e], q0, p), p, pinv);
      r2[e] = fmod_canon(fmod_mul(x1[e], y1[e], q1, p), p, pinv);
    }
    *reinterpret_cast<ulonglong2*>(tk.d0 + j) = make_ulonglong2(r0[0], r0[1]);
    *reinterpret_cast<ulonglong2*>(tk.d1 + j) = make_ulonglong2(r1[0], r1[1]);
    *reinterpret_cast<ulonglong2*>(tk.d2 + j) = make_ulonglong2(r2[0], r2[1]);
  }
}

cudaError_t launch_tensor(const void* tasks, int ntasks, const HbPrime* primes, int n, bool f64,
                          cudaStream_t st) {
  if (ntasks <= 0) return cudaSuccess;
  if (f64)
    (void)hb_launch(k_tensor_f64, dim3(ew_grid(ntasks, n)), dim3(EW_THREADS), 0, st,
                    reinterpret_cast<const HbTensorTask*>(tasks), ntasks, primes, n);
  else
    (void)hb_launch(k_tensor, dim3(ew_grid(ntasks, n)), dim3(EW_THREADS), 0, st,
                    reinterpret_cast<const HbTensorTask*>(tasks), ntasks, primes, n);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// Exact CRT reconstruction of `keep` coefficient rows into a centred integer,
// correctly rounded to double (engine.py:156-175).  Constants (little-endian
// 64-bit limbs, NL limbs each): Q, floor(Q/2), and per prime the residue
// coefficient qhat_inv_i and the multiword qhat_i = Q/q_i.
//   v = sum_i [x_i * qhat_inv_i]_{q_i} * qhat_i  mod Q;  v > Q/2 => v - Q.
constexpr int CRT_MAXL = 8;

struct HbCrtTask {
  const u64* rows;   // keep rows of n coefficients (row stride n)
  double* out;       // n doubles
};

HB_DEV double mw_to_double(const u64* m, int nl, bool neg) {
  int top = nl - 1;
  while (top > 0 && m[top] == 0) --top;
  if (top == 0 && m[0] == 0) return 0.0;
  const int lz = __clzll(m[top]);
  const int msb = top * 64 + (63 - lz);  // bit index of the leading 1
  // Extract 64 bits [msb-63, msb], OR-ing everything below into a sticky bit.
  const int lo_bit = msb - 63;
  if (lo_bit <= 0) {  // value < 2^64: one correctly rounded conversion
    const double d = __ull2double_rn(m[0]);
    return neg ? -d : d;
  }
  bool sticky = false;
  const int wi = lo_bit >> 6, bi = lo_bit & 63;
  u64 w = m[wi] >> bi;
  if (bi) w |= m[wi + 1] << (64 - bi);
  if (bi && (m[wi] & ((1ull << bi) - 1))) sticky = true;
  for (int k = 0; k < wi && !sticky; ++k)
    if (m[k]) sticky = true;
  if (sticky) w |= 1ull;  // bit 0 is below the 53-bit mantissa: acts as sticky
  double d = ldexp(__ull2double_rn(w), lo_bit);
  return neg ? -d : d;
}

__global__ void k_crt_double(const HbCrtTask* __restrict__ tasks, int ntasks, const u64* __restrict__ consts,
                             const HbPrime* __restrict__ primes, const int* __restrict__ prime_idx,
                             int keep, int nl, int n) {
  HB_PDL_ENTRY();
  // consts layout: Q[nl], Qhalf[nl], qhat_inv[keep], qhat[keep][nl]
  const u64* Q = consts;
  const u64* Qh = consts + nl;
  const u64* qinv = consts + 2 * nl;
  const u64* qhat = consts + 2 * nl + keep;
  for (int t = blockIdx.y; t < ntasks; t += gridDim.y) {
    const HbCrtTask tk = tasks[t];
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= n) continue;
    u64 acc[CRT_MAXL + 1];
    for (int l = 0; l <= nl; ++l) acc[l] = 0;
    for (int i = 0; i < keep; ++i) {
      const HbPrime P = primes[prime_idx[i]];
      const u64 y = mul_mod(tk.rows[(size_t)i * n + j], qinv[i], P);
      // acc += y * qhat_i (multiword)
      u64 carry = 0;
      for (int l = 0; l < nl; ++l) {
        const u64 m = qhat[i * nl + l];
        u64 lo = y * m, hi = __umul64hi(y, m);
        lo += carry;
        hi += (lo < carry);
        const u64 s = acc[l] + lo;
        hi += (s < lo);
        acc[l] = s;
        carry = hi;
      }
      acc[nl] += carry;
    }
    // reduce mod Q: acc < keep * Q, subtract Q while acc >= Q
    for (int rep = 0; rep < keep; ++rep) {
      bool ge = acc[nl] != 0;
      if (!ge) {
        ge = true;
        for (int l = nl - 1; l >= 0; --l) {
          if (acc[l] != Q[l]) { ge = acc[l] > Q[l]; break; }
        }
      }
      if (!ge) break;
      u64 borrow = 0;
      for (int l = 0; l < nl; ++l) {
        const u64 q = Q[l] + borrow;
        const u64 nb = (q < borrow) || (acc[l] < q);
        acc[l] -= q;
        borrow = nb;
      }
      acc[nl] -= borrow;
    }
    // centre: v > Q/2 -> v - Q (negative, magnitude Q - v)
    bool gt = false;
    for (int l = nl - 1; l >= 0; --l) {
      if (acc[l] != Qh[l]) { gt = acc[l] > Qh[l]; break; }
    }
    u64 mag[CRT_MAXL];
    if (gt) {
      u64 borrow = 0;
      for (int l = 0; l < nl; ++l) {
        const u64 a = acc[l] + borrow;
        const u64 nb = (a < borrow) || (Q[l] < a);
        mag[l] = Q[l] - a;
        borrow = nb;
      }
    } else {
      for (int l = 0; l < nl; ++l) mag[l] = acc[l];
    }
    tk.out[j] = mw_to_double(mag, nl, gt);
  }
}

cudaError_t launch_crt_double(const HbCrtTask* tasks, int ntasks, const u64* consts,
                              const HbPrime* primes, const int* prime_idx, int keep, int nl, int n,
                              cudaStream_t st) {
  if (ntasks <= 0) return cudaSuccess;
  if (nl > CRT_MAXL) return cudaErrorInvalidValue;
  dim3 grid((n + 255) / 256, ntasks < 65535 ? ntasks : 65535);
  (void)hb_launch(k_crt_double, dim3(grid), dim3(256), 0, st, tasks, ntasks, consts, primes, prime_idx, keep, nl, n);
  return cudaGetLastError();
}

}  // namespace hb

namespace hb {

// ---------------------------------------------------------------------------
// Strided plaintext multiply-accumulate for a whole layer in one launch.
// Every output o is a [BC, R, N] block (BC = batch x 2 components) at
// outs[o].dst; its terms reference plaintext bases (rows r at +r*N) and
// ciphertext bases with the same [BC, R, N] geometry.  grid.y walks
// (o, bc, r); the row index is the chain-prime index.
struct HbMacOut {
  u64* dst;
  int nterms;
  int term_off;
};

__global__ void __launch_bounds__(EW_THREADS)
k_mac_strided(const HbMacOut* __restrict__ outs, int nout, const HbMacTerm* __restrict__ terms,
              const HbPrime* __restrict__ primes, int n, int R, int BC) {
  HB_PDL_ENTRY();
  const long long total = (long long)nout * BC * R;
  for (long long y = blockIdx.y; y < total; y += gridDim.y) {
    const int o = (int)(y / ((long long)BC * R));
    const int rem = (int)(y % ((long long)BC * R));
    const int bc = rem / R, r = rem % R;
    const HbMacOut ou = outs[o];
    const HbPrime P = primes[r];
    const int j = 2 * (blockIdx.x * EW_THREADS + threadIdx.x);
    if (j >= n) continue;
    const size_t ct_off = ((size_t)bc * R + r) * n + j;
    const size_t pt_off = (size_t)r * n + j;
    Acc128 s0, s1;
    for (int k = 0; k < ou.nterms; ++k) {
      const HbMacTerm tm = terms[ou.term_off + k];
      const ulonglong2 a = __ldg(reinterpret_cast<const ulonglong2*>(tm.pt + pt_off));
      const ulonglong2 b = __ldg(reinterpret_cast<const ulonglong2*>(tm.ct + ct_off));
      s0.mac(a.x, b.x);
      s1.mac(a.y, b.y);
      if ((k & 7) == 7) { s0.fold(P); s1.fold(P); }
    }
    ulonglong2 v;
    v.x = s0.fold(P);
    v.y = s1.fold(P);
    *reinterpret_cast<ulonglong2*>(ou.dst + ct_off) = v;
  }
}

// fp64-pipe variant (rings with every prime < 2^42): products as fmod_mul
// (5 fp64 ops + one rounding) summed as balanced doubles, one
// canonicalisation -- instead of 64x64->128-bit integer products and
// 128-bit folds on the integer pipe; same canonical residues.
__global__ void __launch_bounds__(256)
k_mac_strided_f64(const HbMacOut* __restrict__ outs, int nout, const HbMacTerm* __restrict__ terms,
                  const HbPrime* __restrict__ primes, int n, int R, int BC) {
  HB_PDL_ENTRY();
  const long long total = (long long)nout * BC * R;
  for (long long y = blockIdx.y; y < total; y += gridDim.y) {
    const int o = (int)(y / ((long long)BC * R));
    const int rem = (int)(y % ((long long)BC * R));
    const int bc = rem / R, r = rem % R;
    const HbMacOut ou = outs[o];
    const HbPrime P = primes[r];
    const double p = P.pd, pinv = P.pinv;
    const int j = 2 * (blockIdx.x * EW_THREADS + threadIdx.x);
    if (j >= n) continue;
    const size_t ct_off = ((size_t)bc * R + r) * n + j;
    const size_t pt_off = (size_t)r * n + j;
    double s0 = 0.0, s1 = 0.0;
    for (int k = 0; k < ou.nterms; ++k) {
      const HbMacTerm tm = terms[ou.term_off + k];
      const ulonglong2 a = __ldg(reinterpret_cast<const ulonglong2*>(tm.pt + pt_off));
      const ulonglong2 b = __ldg(reinterpret_cast<const ulonglong2*>(tm.ct + ct_off));
      const double a0 = u64_to_f(a.x), a1 = u64_to_f(a.y);
      s0 += fmod_mul(u64_to_f(b.x), a0, a0 * pinv, p);
      s1 += fmod_mul(u64_to_f(b.y), a1, a1 * pinv, p);
      if ((k & 255) == 255) { s0 = fmod_reduce(s0, p, pinv); s1 = fmod_reduce(s1, p, pinv); }
    }
    ulonglong2 v;
    v.x = fmod_canon(s0, p, pinv);
    v.y = fmod_canon(s1, p, pinv);
    *reinterpret_cast<ulonglong2*>(ou.dst + ct_off) = v;
  }
}

cudaError_t launch_mac_strided(const void* outs, int nout, const HbMacTerm* terms,
                               const HbPrime* primes, int n, int R, int BC, bool f64,
                               cudaStream_t st) {
  if (nout <= 0) return cudaSuccess;
  const long long total = (long long)nout * BC * R;
  dim3 grid((n / 2 + EW_THREADS - 1) / EW_THREADS, total < 65535 ? (int)total : 65535);
  if (f64)
    (void)hb_launch(k_mac_strided_f64, dim3(grid), dim3(EW_THREADS), 0, st, reinterpret_cast<const HbMacOut*>(outs), nout,
                                                   terms, primes, n, R, BC);
  else
    (void)hb_launch(k_mac_strided, dim3(grid), dim3(EW_THREADS), 0, st, reinterpret_cast<const HbMacOut*>(outs), nout,
                                               terms, primes, n, R, BC);
  return cudaGetLastError();
}

}  // namespace hb

namespace hb {

// ---------------------------------------------------------------------------
// Shared-term multiply-accumulate group: outputs that sum products with the
// SAME ciphertext term list (hconv's giant/baby partial sums, the FC
// diagonals): out_o = sum_t pt[o][t] * ct[t] (mac.cu k_mac_pipe, and the
// k_mac_gemm fallbacks below).
struct HbMacGroup {
  const u64* const* cts;   // [nterms] ciphertext bases ([BC, R, N] blocks)
  const u64* const* pts;   // [nout][nterms] plaintext bases (rows at +r*N)
  u64* const* dsts;        // [nout] output bases ([BC, R, N])
  int nterms;
  int nout;
};

// ---------------------------------------------------------------------------
// Key-switch inner product, clip-blocked: one task per (job, output row r);
// block = 32 coefficient pairs x up to 8 clips, so the key rows (shared by
// every clip) are fetched once per block and broadcast through L1.


__global__ void __launch_bounds__(256)
k_ks_inner2(const HbKsTask2* __restrict__ tasks, const HbPrime* __restrict__ primes, int n,
            int nb) {
  HB_PDL_ENTRY();
  const HbKsTask2 tk = tasks[blockIdx.y];
  // grid: x = clip group (fastest), y = task, z = coefficient chunk (slowest):
  // the clips of one key row run back to back, so the key is read from HBM once
  const int b = blockIdx.x * blockDim.y + threadIdx.y;
  const int j = 2 * (blockIdx.z * 32 + threadIdx.x);
  if (j >= n || b >= nb) return;
  const HbPrime P = primes[tk.prime];
  int s0 = j, s1 = j + 1;
  if (tk.perm) {
    const int2 pp = __ldg(reinterpret_cast<const int2*>(tk.perm + j));
    s0 = pp.x;
    s1 = pp.y;
  }
  const u64* de = tk.de + b * tk.de_bstride;
  Acc128 b0, b1, a0, a1;
  for (int i = 0; i < tk.ndig; ++i) {
    const u64* d = de + i * tk.de_dstride;
    const u64 x0 = __ldg(d + s0), x1 = __ldg(d + s1);
    const ulonglong2 kb = __ldg(reinterpret_cast<const ulonglong2*>(tk.kb + i * tk.key_stride + j));
    const ulonglong2 ka = __ldg(reinterpret_cast<const ulonglong2*>(tk.ka + i * tk.key_stride + j));
    b0.mac(x0, kb.x);
    b1.mac(x1, kb.y);
    a0.mac(x0, ka.x);
    a1.mac(x1, ka.y);
    if ((i & 7) == 7) { b0.fold(P); b1.fold(P); a0.fold(P); a1.fold(P); }
  }
  ulonglong2 rb, ra;
  rb.x = b0.fold(P);
  rb.y = b1.fold(P);
  ra.x = a0.fold(P);
  ra.y = a1.fold(P);
  *reinterpret_cast<ulonglong2*>(tk.out_b + b * tk.out_bstride + j) = rb;
  *reinterpret_cast<ulonglong2*>(tk.out_a + b * tk.out_bstride + j) = ra;
}

// ring.py:186 lift_center: residues mod p -> centred int64 in (-p/2, p/2].
__global__ void k_lift_center(const u64* __restrict__ x, u64 p, long long* __restrict__ out,
                              int n) {
  HB_PDL_ENTRY();
  const u64 half = p >> 1;
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x) {
    const u64 v = x[j];
    out[j] = v > half ? (long long)v - (long long)p : (long long)v;
  }
}

// ring.py:198 reduce_rows: one centred int64 coefficient vector -> residues
// under the prime of every output row (grid.y = row).
__global__ void k_reduce_rows(const long long* __restrict__ c, const int* __restrict__ gidx,
                              const HbPrime* __restrict__ primes, u64* __restrict__ out, int n) {
  HB_PDL_ENTRY();
  const long long p = (long long)primes[gidx[blockIdx.y]].p;
  u64* o = out + (size_t)blockIdx.y * n;
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x) {
    long long v = c[j] % p;
    o[j] = (u64)(v < 0 ? v + p : v);
  }
}

cudaError_t launch_lift_center(const u64* x, u64 p, long long* out, int n, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  (void)hb_launch(k_lift_center, dim3((n + 255) / 256), dim3(256), 0, st, x, p, out, n);
  return cudaGetLastError();
}

cudaError_t launch_reduce_rows(const long long* c, const int* gidx, int nrows,
                               const HbPrime* primes, u64* out, int n, cudaStream_t st) {
  if (n <= 0 || nrows <= 0) return cudaSuccess;
  (void)hb_launch(k_reduce_rows, dim3((n + 255) / 256, nrows), dim3(256), 0, st, c, gidx, primes,
                  out, n);
  return cudaGetLastError();
}

cudaError_t launch_ks_inner2(const void* tasks, int ntasks, int nb, const HbPrime* primes, int n,
                             cudaStream_t st) {
  if (ntasks <= 0 || nb <= 0) return cudaSuccess;
  const int by = nb < 8 ? nb : 8;
  dim3 block(32, by);
  dim3 grid((nb + by - 1) / by, ntasks, (n / 2 + 31) / 32);
  (void)hb_launch(k_ks_inner2, dim3(grid), dim3(block), 0, st, reinterpret_cast<const HbKsTask2*>(tasks), primes, n, nb);
  return cudaGetLastError();
}

}  // namespace hb

namespace hb {

// ---------------------------------------------------------------------------
// Shared-term MAC as a per-coefficient modular GEMM:
//   out[o][bc][r][j] = sum_t pt[o][t][r][j] * ct[t][bc][r][j]   (mod p_r)
// for a group of outputs sharing one ciphertext term list (hconv partial
// sums, FC diagonals).  Lanes own 32 consecutive coefficients (coalesced 8 B
// loads of both operands); each thread keeps a TO x TB register tile of
// 128-bit accumulators, so every loaded plaintext value feeds TB products
// and every ciphertext value TO products.  The 8 warps of a block tile
// (WO x WB) over outputs x clip-components; pointer tables live in smem.
template <int TO, int TB, int WO, int WB>
__global__ void __launch_bounds__(256, (TO * TB > 16 ? 1 : 2))
k_mac_gemm(HbMacGroup g, const HbPrime* __restrict__ primes, int n, int R, int BC) {
  HB_PDL_ENTRY();
  extern __shared__ const u64* ptrs[];   // cts[T] | pts[O*T] | dsts[O]
  const int T = g.nterms, O = g.nout;
  for (int i = threadIdx.x + threadIdx.y * 32; i < T + O * T + O; i += 256) {
    if (i < T) ptrs[i] = g.cts[i];
    else if (i < T + O * T) ptrs[i] = g.pts[i - T];
    else ptrs[i] = g.dsts[i - T - O * T];
  }
  __syncthreads();
  const u64* const* cts = ptrs;
  const u64* const* pts = ptrs + T;
  u64* const* dsts = const_cast<u64* const*>(ptrs + T + O * T);

  // grid: x = clip-component tile (fastest), y = output tile, z = coefficient
  // chunk (slowest) -> CTAs that share a plaintext/ciphertext chunk run
  // back to back and hit it in L2 instead of re-reading HBM
  const int nchunk = n / 32;
  const int r = blockIdx.z / nchunk;
  const int j = (blockIdx.z % nchunk) * 32 + threadIdx.x;
  const int w = threadIdx.y;
  const int o0 = (blockIdx.y * WO + w / WB) * TO;
  const int b0 = (blockIdx.x * WB + w % WB) * TB;
  if (o0 >= O || b0 >= BC) return;
  const HbPrime P = primes[r];
  const size_t rj = (size_t)r * n + j;
  Acc128 acc[TO][TB];
  for (int t = 0; t < T; ++t) {
    u64 c[TB];
#pragma unroll
    for (int b = 0; b < TB; ++b)
      c[b] = (b0 + b < BC) ? __ldg(cts[t] + (size_t)(b0 + b) * R * n + rj) : 0ull;
#pragma unroll
    for (int o = 0; o < TO; ++o) {
      const u64 a = (o0 + o < O) ? __ldg(pts[(size_t)(o0 + o) * T + t] + rj) : 0ull;
#pragma unroll
      for (int b = 0; b < TB; ++b) acc[o][b].mac(a, c[b]);
    }
    if ((t & 7) == 7) {
#pragma unroll
      for (int o = 0; o < TO; ++o)
#pragma unroll
        for (int b = 0; b < TB; ++b) acc[o][b].fold(P);
    }
  }
#pragma unroll
  for (int o = 0; o < TO; ++o) {
    if (o0 + o >= O) continue;
#pragma unroll
    for (int b = 0; b < TB; ++b)
      if (b0 + b < BC) dsts[o0 + o][(size_t)(b0 + b) * R * n + rj] = acc[o][b].fold(P);
  }
}

template <int TO, int TB, int WO, int WB>
static cudaError_t mac_gemm_t(const HbMacGroup& g, const HbPrime* primes, int n, int R, int BC,
                              cudaStream_t st) {
  const size_t smem = sizeof(void*) * (size_t)(g.nterms + g.nout * g.nterms + g.nout);
  if (smem > 200 * 1024) {   // pointer tables too large for smem: split the outputs
    if (g.nout <= 1) return cudaErrorInvalidValue;
    HbMacGroup a = g, b = g;
    a.nout = g.nout / 2;
    b.nout = g.nout - a.nout;
    b.pts = g.pts + (size_t)a.nout * g.nterms;
    b.dsts = g.dsts + a.nout;
    cudaError_t e = mac_gemm_t<TO, TB, WO, WB>(a, primes, n, R, BC, st);
    return e != cudaSuccess ? e : mac_gemm_t<TO, TB, WO, WB>(b, primes, n, R, BC, st);
  }
  static int smem_cur = 0;
  cudaError_t e = smem_attr_once((const void*)k_mac_gemm<TO, TB, WO, WB>, (int)((int)smem), &smem_cur);
  if (e != cudaSuccess) return e;
  dim3 block(32, 8);
  dim3 grid((BC + TB * WB - 1) / (TB * WB), (g.nout + TO * WO - 1) / (TO * WO), R * (n / 32));
  (void)hb_launch(k_mac_gemm<TO, TB, WO, WB>, dim3(grid), dim3(block), smem, st, g, primes, n, R, BC);
  return cudaGetLastError();
}

cudaError_t launch_mac_gemm(const void* cts, const void* pts, const void* dsts, int nterms,
                            int nout, const HbPrime* primes, int n, int R, int BC,
                            cudaStream_t st) {
  if (nout <= 0 || nterms <= 0) return cudaSuccess;
  HbMacGroup g;
  g.cts = reinterpret_cast<const u64* const*>(cts);
  g.pts = reinterpret_cast<const u64* const*>(pts);
  g.dsts = reinterpret_cast<u64* const*>(dsts);
  g.nterms = nterms;
  g.nout = nout;
  if (BC <= 2) return mac_gemm_t<4, 2, 8, 1>(g, primes, n, R, BC, st);
  return mac_gemm_t<4, 4, 4, 2>(g, primes, n, R, BC, st);
}

}  // namespace hb

namespace hb {

// fp64-pipe variant of k_mac_gemm for rings whose primes are all < 2^42:
// each product a*c is reduced exactly to a balanced residue with 6 fp64 ops
// (modarith.cuh fmod_mul with q = round(a * (c/p)) from a*pinv), summed in
// double (|sum| < 2^53 for < 2^9 terms), canonicalised once at the end.
template <int TO, int TB, int WO, int WB>
__global__ void __launch_bounds__(256)
k_mac_gemm_f64(HbMacGroup g, const HbPrime* __restrict__ primes, int n, int R, int BC) {
  HB_PDL_ENTRY();
  extern __shared__ const u64* ptrs[];
  const int T = g.nterms, O = g.nout;
  for (int i = threadIdx.x + threadIdx.y * 32; i < T + O * T + O; i += 256) {
    if (i < T) ptrs[i] = g.cts[i];
    else if (i < T + O * T) ptrs[i] = g.pts[i - T];
    else ptrs[i] = g.dsts[i - T - O * T];
  }
  __syncthreads();
  const u64* const* cts = ptrs;
  const u64* const* pts = ptrs + T;
  u64* const* dsts = const_cast<u64* const*>(ptrs + T + O * T);
  // grid: x = clip-component tile (fastest), y = output tile, z = coefficient
  // chunk (slowest) -> CTAs that share a plaintext/ciphertext chunk run
  // back to back and hit it in L2 instead of re-reading HBM
  const int nchunk = n / 32;
  const int r = blockIdx.z / nchunk;
  const int j = (blockIdx.z % nchunk) * 32 + threadIdx.x;
  const int w = threadIdx.y;
  const int o0 = (blockIdx.y * WO + w / WB) * TO;
  const int b0 = (blockIdx.x * WB + w % WB) * TB;
  if (o0 >= O || b0 >= BC) return;
  const HbPrime P = primes[r];
  const double p = P.pd, pinv = P.pinv;
  const size_t rj = (size_t)r * n + j;
  double acc[TO][TB];
#pragma unroll
  for (int o = 0; o < TO; ++o)
#pragma unroll
    for (int b = 0; b < TB; ++b) acc[o][b] = 0.0;
  // software pipeline: term t+1's operands are in flight while term t's
  // products run (the loads are two-level: smem pointer, then L2)
  u64 cn[TB], an[TO];
  auto fetch = [&](int t) {
#pragma unroll
    for (int b = 0; b < TB; ++b)
      cn[b] = (b0 + b < BC) ? __ldg(cts[t] + (size_t)(b0 + b) * R * n + rj) : 0ull;
#pragma unroll
    for (int o = 0; o < TO; ++o)
      an[o] = (o0 + o < O) ? __ldg(pts[(size_t)(o0 + o) * T + t] + rj) : 0ull;
  };
  fetch(0);
  for (int t = 0; t < T; ++t) {
    double c[TB], a[TO];
#pragma unroll
    for (int b = 0; b < TB; ++b) c[b] = u64_to_f(cn[b]);
#pragma unroll
    for (int o = 0; o < TO; ++o) a[o] = u64_to_f(an[o]);
    if (t + 1 < T) fetch(t + 1);
#pragma unroll
    for (int o = 0; o < TO; ++o) {
      const double aq = a[o] * pinv;
#pragma unroll
      for (int b = 0; b < TB; ++b) acc[o][b] += fmod_mul(c[b], a[o], aq, p);
    }
    if ((t & 255) == 255) {
#pragma unroll
      for (int o = 0; o < TO; ++o)
#pragma unroll
        for (int b = 0; b < TB; ++b) acc[o][b] = fmod_reduce(acc[o][b], p, pinv);
    }
  }
#pragma unroll
  for (int o = 0; o < TO; ++o) {
    if (o0 + o >= O) continue;
#pragma unroll
    for (int b = 0; b < TB; ++b)
      if (b0 + b < BC) dsts[o0 + o][(size_t)(b0 + b) * R * n + rj] = fmod_canon(acc[o][b], p, pinv);
  }
}

template <int TO, int TB, int WO, int WB>
static cudaError_t mac_gemm_f64_t(const HbMacGroup& g, const HbPrime* primes, int n, int R, int BC,
                                  cudaStream_t st) {
  const size_t smem = sizeof(void*) * (size_t)(g.nterms + g.nout * g.nterms + g.nout);
  if (smem > 200 * 1024) {   // pointer tables too large for smem: split the outputs
    if (g.nout <= 1) return cudaErrorInvalidValue;
    HbMacGroup a = g, b = g;
    a.nout = g.nout / 2;
    b.nout = g.nout - a.nout;
    b.pts = g.pts + (size_t)a.nout * g.nterms;
    b.dsts = g.dsts + a.nout;
    cudaError_t e = mac_gemm_f64_t<TO, TB, WO, WB>(a, primes, n, R, BC, st);
    return e != cudaSuccess ? e : mac_gemm_f64_t<TO, TB, WO, WB>(b, primes, n, R, BC, st);
  }
  static int smem_cur = 0;
  cudaError_t e = smem_attr_once((const void*)k_mac_gemm_f64<TO, TB, WO, WB>, (int)((int)smem), &smem_cur);
  if (e != cudaSuccess) return e;
  dim3 block(32, 8);
  dim3 grid((BC + TB * WB - 1) / (TB * WB), (g.nout + TO * WO - 1) / (TO * WO), R * (n / 32));
  (void)hb_launch(k_mac_gemm_f64<TO, TB, WO, WB>, dim3(grid), dim3(block), smem, st, g, primes, n, R, BC);
  return cudaGetLastError();
}

cudaError_t launch_mac_gemm_f64(const void* cts, const void* pts, const void* dsts, int nterms,
                                int nout, const HbPrime* primes, int n, int R, int BC,
                                cudaStream_t st) {
  if (nout <= 0 || nterms <= 0) return cudaSuccess;
  HbMacGroup g;
  g.cts = reinterpret_cast<const u64* const*>(cts);
  g.pts = reinterpret_cast<const u64* const*>(pts);
  g.dsts = reinterpret_cast<u64* const*>(dsts);
  g.nterms = nterms;
  g.nout = nout;
  if (BC <= 2) return mac_gemm_f64_t<4, 2, 8, 1>(g, primes, n, R, BC, st);
  // 4x4 tiles measured fastest on the conv shapes (round-1 tile sweep): 4x8
  // needs ~156 registers (one CTA per SM), too few warps to cover load latency
  return mac_gemm_f64_t<4, 4, 4, 2>(g, primes, n, R, BC, st);
}

// fp64 variant of the clip-blocked key-switch inner product.
__global__ void __launch_bounds__(256)
k_ks_inner2_f64(const HbKsTask2* __restrict__ tasks, const HbPrime* __restrict__ primes, int n,
                int nb, int by) {
  HB_PDL_ENTRY();
  const HbKsTask2 tk = tasks[blockIdx.y];
  // grid: x = clip group (fastest), y = task, z = coefficient chunk (slowest):
  // the clips of one key row run back to back, so the key is read from HBM once.
  // blockDim.y = by clips x (blockDim.y / by) coefficient chunks: at one or two
  // clips a CTA still has 8 warps (one-warp CTAs streamed the keys at half
  // the HBM rate)
  const int b = blockIdx.x * by + threadIdx.y % by;
  const int j = 2 * ((blockIdx.z * (blockDim.y / by) + threadIdx.y / by) * 32 + threadIdx.x);
  if (j >= n || b >= nb) return;
  const HbPrime P = primes[tk.prime];
  const double p = P.pd, pinv = P.pinv;
  int s0 = j, s1 = j + 1;
  if (tk.perm) {
    const int2 pp = __ldg(reinterpret_cast<const int2*>(tk.perm + j));
    s0 = pp.x;
    s1 = pp.y;
  }
  const u64* de = tk.de + b * tk.de_bstride;
  double b0 = 0, b1 = 0, a0 = 0, a1 = 0;
  // two-deep software pipeline over the digits: digit i+1's operands (L2)
  // are in flight while digit i multiplies
  u64 xd0, xd1;
  ulonglong2 kb, ka;
  auto fetch = [&](int i) {
    const u64* d = de + i * tk.de_dstride;
    xd0 = __ldg(d + s0);
    xd1 = __ldg(d + s1);
    kb = __ldg(reinterpret_cast<const ulonglong2*>(tk.kb + i * tk.key_stride + j));
    ka = __ldg(reinterpret_cast<const ulonglong2*>(tk.ka + i * tk.key_stride + j));
  };
  fetch(0);
  for (int i = 0; i < tk.ndig; ++i) {
    const double x0 = u64_to_f(xd0), x1 = u64_to_f(xd1);
    const double kb0 = u64_to_f(kb.x), kb1 = u64_to_f(kb.y);
    const double ka0 = u64_to_f(ka.x), ka1 = u64_to_f(ka.y);
    if (i + 1 < tk.ndig) fetch(i + 1);
    const double q0 = x0 * pinv, q1 = x1 * pinv;
    b0 += fmod_mul(kb0, x0, q0, p);
    b1 += fmod_mul(kb1, x1, q1, p);
    a0 += fmod_mul(ka0, x0, q0, p);
    a1 += fmod_mul(ka1, x1, q1, p);
  }
  if (tk.scat && tk.c0) {   // + P * c0 (the rotated c0, still at the source index)
    const ulonglong2 c2 = __ldg(reinterpret_cast<const ulonglong2*>(tk.c0 + b * tk.c0_bstride + j));
    const double pm = u64_to_f(tk.pmod), pmq = pm * pinv;
    b0 += fmod_mul(u64_to_f(c2.x), pm, pmq, p);
    b1 += fmod_mul(u64_to_f(c2.y), pm, pmq, p);
  }
  ulonglong2 rb, ra;
  rb.x = fmod_canon(b0, p, pinv);
  rb.y = fmod_canon(b1, p, pinv);
  ra.x = fmod_canon(a0, p, pinv);
  ra.y = fmod_canon(a1, p, pinv);
  if (tk.scat) {   // rotated ciphertext rows in the extended basis
    const int2 sc = __ldg(reinterpret_cast<const int2*>(tk.scat + j));
    u64* ob = tk.out_b + b * tk.out_bstride;
    u64* oa = tk.out_a + b * tk.out_bstride;
    ob[sc.x] = rb.x;
    ob[sc.y] = rb.y;
    oa[sc.x] = ra.x;
    oa[sc.y] = ra.y;
    return;
  }
  *reinterpret_cast<ulonglong2*>(tk.out_b + b * tk.out_bstride + j) = rb;
  *reinterpret_cast<ulonglong2*>(tk.out_a + b * tk.out_bstride + j) = ra;
}

cudaError_t launch_ks_inner2_f64(const void* tasks, int ntasks, int nb, const HbPrime* primes,
                                 int n, cudaStream_t st) {
  if (ntasks <= 0 || nb <= 0) return cudaSuccess;
  const int by = nb < 8 ? nb : 8;
  const int cy = 8 / by;   // coefficient chunks per CTA
  dim3 block(32, by * cy);
  dim3 grid((nb + by - 1) / by, ntasks, (n / 2 / 32 + cy - 1) / cy);
  (void)hb_launch(k_ks_inner2_f64, dim3(grid), dim3(block), 0, st, reinterpret_cast<const HbKsTask2*>(tasks), primes, n, nb, by);
  return cudaGetLastError();
}

// Rotate-and-sum of hoisted rotations in the extended basis Q*P
// (hear/fastpath.py:141-154 rotate_sum_each's odd part: ct + sum_j rot_j(ct),
// each rotation engine.py:328-351) WITHOUT materialising the rotations:
//   out_b[m] = P*(c0[m] + sum_j c0[pi_j(m)]) + sum_j sum_i d_i[pi_j(m)] * Kb_ij[m]
//   out_a[m] = P* c1[m]                      + sum_j sum_i d_i[pi_j(m)] * Ka_ij[m]
// on every chain row and (without the P terms) the special row; the caller
// divides P out once.  The digits are gathered through the Galois map (it
// permutes aligned 32-element blocks onto aligned blocks, so the gathers are
// sector-exact), the keys are read in place (shared by the 8 clips of a CTA
// through L1).  The unfused form wrote one extended rotation per amount and
// re-read them all for the sum.
#ifndef HB_RS_MINB
#define HB_RS_MINB 4   // <= 64 registers: the gather chain is latency-bound, 4 CTAs per SM (8.8 -> 6.2 ms per step)
#endif
__global__ void __launch_bounds__(256, HB_RS_MINB)
k_rot_sum_f64(const HbRotSumTask* __restrict__ tasks, const HbRotSumRot* __restrict__ rots,
              int nrot, int ndig, const HbPrime* __restrict__ primes, int n, int nb) {
  HB_PDL_ENTRY();
  const HbRotSumTask tk = tasks[blockIdx.y];
  const int b = blockIdx.x * blockDim.y + threadIdx.y;
  const int j = 2 * (blockIdx.z * 32 + threadIdx.x);
  if (j >= n || b >= nb) return;
  const HbPrime P = primes[tk.prime];
  const double p = P.pd, pinv = P.pinv;
  const u64* de = tk.de + b * tk.de_bstride;
  const bool chain = tk.row >= 0;
  double b0 = 0, b1 = 0, a0 = 0, a1 = 0;
  u64 s0 = 0, s1 = 0, t0 = 0, t1 = 0;   // sums of c0 terms / the identity's c1
  if (chain) {
    const ulonglong2 v0 = __ldg(reinterpret_cast<const ulonglong2*>(tk.c0 + b * tk.c_bstride + j));
    const ulonglong2 v1 = __ldg(reinterpret_cast<const ulonglong2*>(tk.c1 + b * tk.c_bstride + j));
    s0 = v0.x; s1 = v0.y; t0 = v1.x; t1 = v1.y;
  }
  for (int q = 0; q < nrot; ++q) {
    const HbRotSumRot rt = rots[q];
    const int2 pp = __ldg(reinterpret_cast<const int2*>(rt.perm + j));
    if (chain) {
      s0 += __ldg(tk.c0 + b * tk.c_bstride + pp.x);
      s1 += __ldg(tk.c0 + b * tk.c_bstride + pp.y);
    }
    const size_t krow = (size_t)(chain ? tk.row : rt.special_row) * n + j;
    const u64* kbp = rt.kb + krow;
    const u64* kap = rt.ka + krow;
#pragma unroll 2
    for (int i = 0; i < ndig; ++i) {
      const u64* d = de + i * tk.de_dstride;
      const double x0 = u64_to_f(__ldg(d + pp.x)), x1 = u64_to_f(__ldg(d + pp.y));
      const ulonglong2 kb = __ldg(reinterpret_cast<const ulonglong2*>(kbp + i * rt.key_dstride));
      const ulonglong2 ka = __ldg(reinterpret_cast<const ulonglong2*>(kap + i * rt.key_dstride));
      const double q0 = x0 * pinv, q1 = x1 * pinv;
      b0 += fmod_mul(u64_to_f(kb.x), x0, q0, p);
      b1 += fmod_mul(u64_to_f(kb.y), x1, q1, p);
      a0 += fmod_mul(u64_to_f(ka.x), x0, q0, p);
      a1 += fmod_mul(u64_to_f(ka.y), x1, q1, p);
    }
    if ((q & 63) == 63) {   // balanced sums stay far below 2^53
      b0 = fmod_reduce(b0, p, pinv); b1 = fmod_reduce(b1, p, pinv);
      a0 = fmod_reduce(a0, p, pinv); a1 = fmod_reduce(a1, p, pinv);
    }
  }
  if (chain) {   // + P * (sums of c0 / the identity's c1); sums < 2^45
    const double pm = u64_to_f(tk.pmod), pmq = pm * pinv;
    b0 += fmod_mul(u64_to_f(s0), pm, pmq, p);
    b1 += fmod_mul(u64_to_f(s1), pm, pmq, p);
    a0 += fmod_mul(u64_to_f(t0), pm, pmq, p);
    a1 += fmod_mul(u64_to_f(t1), pm, pmq, p);
  }
  ulonglong2 rb, ra;
  rb.x = fmod_canon(b0, p, pinv);
  rb.y = fmod_canon(b1, p, pinv);
  ra.x = fmod_canon(a0, p, pinv);
  ra.y = fmod_canon(a1, p, pinv);
  *reinterpret_cast<ulonglong2*>(tk.out_b + b * tk.out_bstride + j) = rb;
  *reinterpret_cast<ulonglong2*>(tk.out_a + b * tk.out_bstride + j) = ra;
}

cudaError_t launch_rot_sum(const void* tasks, int ntasks, const void* rots, int nrot, int ndig,
                           int nb, const HbPrime* primes, int n, cudaStream_t st) {
  if (ntasks <= 0 || nb <= 0) return cudaSuccess;
  if (nrot > 1024) return cudaErrorInvalidValue;   // c0 sums must stay below 2^45
  const int by = nb < 8 ? nb : 8;
  dim3 block(32, by);
  dim3 grid((nb + by - 1) / by, ntasks, (n / 2 + 31) / 32);
  (void)hb_launch(k_rot_sum_f64, dim3(grid), dim3(block), 0, st,
                  reinterpret_cast<const HbRotSumTask*>(tasks),
                  reinterpret_cast<const HbRotSumRot*>(rots), nrot, ndig, primes, n, nb);
  return cudaGetLastError();
}

// Many-term modular sums: dst = sum_k srcs[term_off + k] (mod p) per row task
// (HbMacTask layout, pt unused) -- the left-to-right add chains of sum_each
// (hear/fastpath.py rotate-and-sum / FC partial sums, ring.py:159 pw_add) in
// one pass: each source row is read once and the result written once,
// instead of a read-read-write per pairwise add.  Residues < p < 2^62 summed
// in 64 bits (fewer than 4 terms per 2^63 headroom is never reached: the
// caller bounds nterms so nterms * p < 2^64), one reduction at the end.
__global__ void __launch_bounds__(256)
k_sum_rows(const HbMacTask* __restrict__ tasks, const u64* const* __restrict__ srcs,
           const HbPrime* __restrict__ primes, int n) {
  HB_PDL_ENTRY();
  const HbMacTask tk = tasks[blockIdx.y];
  const int j = 2 * (blockIdx.x * blockDim.x + threadIdx.x);
  if (j >= n) return;
  const HbPrime P = primes[tk.prime];
  u64 a0 = 0, a1 = 0;
  const u64* const* s = srcs + tk.term_off;
  for (int k = 0; k < tk.nterms; ++k) {
    const ulonglong2 v = __ldg(reinterpret_cast<const ulonglong2*>(s[k] + j));
    a0 += v.x;
    a1 += v.y;
  }
  ulonglong2 o;
  o.x = reduce64(a0, P);
  o.y = reduce64(a1, P);
  *reinterpret_cast<ulonglong2*>(tk.dst + j) = o;
}

cudaError_t launch_sum_rows(const HbMacTask* tasks, int count, const void* srcs,
                            const HbPrime* primes, int n, cudaStream_t st) {
  if (count <= 0) return cudaSuccess;
  dim3 grid((n / 2 + 255) / 256, count);
  (void)hb_launch(k_sum_rows, dim3(grid), dim3(256), 0, st, tasks, reinterpret_cast<const u64* const*>(srcs), primes, n);
  return cudaGetLastError();
}

}  // namespace hb

/*
 * CPU oracle of the HEAR CKKS ring kernels -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain-C restatement of hear/ckks/ring.py's numba kernels (one function per
 * kernel, same argument meaning: (rows, N) uint64 arrays, a per-row global
 * prime index `gidx`, per-prime constant tables), parallelised over rows with
 * OpenMP exactly like the reference's prange loops.  Used by tests/ as the
 * checker, by bench.py's cpu_baseline and by `bench.py --impl reference`;
 * never linked into the product library.
 *
 * Two corrections relative to the shipped reference tables:
 * the inverse NTT expects the true inverse twiddles psi^-brv(j) (ring.py:282
 * uses exponent brv(j)+1), and the Barrett constant mu = floor(2^(63+k)/p) is
 * computed in exact integer arithmetic (ring.py:264-268 overflows it to 0).
 */
#include <stdint.h>
#include <stddef.h>

typedef uint64_t u64;
typedef int64_t i64;
typedef unsigned __int128 u128;

static inline u64 mulhi(u64 a, u64 b) { return (u64)(((u128)a * b) >> 64); }

/* ring.py:33-39 */
static inline u64 mul_shoup(u64 a, u64 w, u64 wsh, u64 p) {
  u64 q = mulhi(a, wsh);
  u64 r = a * w - q * p;
  return r >= p ? r - p : r;
}

/* ring.py:42-52, with the exact mu = floor(2^(63+k)/p), sh = k-1 */
static inline u64 mul_barrett(u64 a, u64 b, u64 p, u64 mu, u64 sh) {
  u128 x = (u128)a * b;
  u64 lo = (u64)x, hi = (u64)(x >> 64);
  u64 t = (hi << (64 - sh)) | (lo >> sh);
  u64 q = mulhi(t, mu);
  u64 r = lo - q * p;
  while (r >= p) r -= p;
  return r;
}

static inline u64 addmod(u64 a, u64 b, u64 p) { u64 r = a + b; return r >= p ? r - p : r; }
static inline u64 submod(u64 a, u64 b, u64 p) { u64 r = a + p - b; return r >= p ? r - p : r; }

/* ring.py:71-87 */
static void ntt_fwd_row(u64* a, int n, const u64* psi, const u64* psish, u64 p) {
  int t = n;
  for (int m = 1; m < n; m <<= 1) {
    t >>= 1;
    for (int i = 0; i < m; ++i) {
      const u64 w = psi[m + i], ws = psish[m + i];
      const int j1 = 2 * i * t;
      for (int j = j1; j < j1 + t; ++j) {
        u64 u = a[j];
        u64 v = mul_shoup(a[j + t], w, ws, p);
        a[j] = addmod(u, v, p);
        a[j + t] = submod(u, v, p);
      }
    }
  }
}

/* ring.py:90-110 */
static void ntt_inv_row(u64* a, int n, const u64* ipsi, const u64* ipsish, u64 p, u64 ninv,
                        u64 ninvsh) {
  int t = 1;
  for (int m = n; m > 1; m >>= 1) {
    int j1 = 0;
    const int h = m >> 1;
    for (int i = 0; i < h; ++i) {
      const u64 w = ipsi[h + i], ws = ipsish[h + i];
      for (int j = j1; j < j1 + t; ++j) {
        u64 u = a[j], v = a[j + t];
        a[j] = addmod(u, v, p);
        a[j + t] = mul_shoup(submod(u, v, p), w, ws, p);
      }
      j1 += 2 * t;
    }
    t <<= 1;
  }
  for (int j = 0; j < n; ++j) a[j] = mul_shoup(a[j], ninv, ninvsh, p);
}

/* ring.py:113-117 ntt_fwd */
void or_ntt_fwd(u64* a, int rows, int n, const i64* gidx, const u64* psi, const u64* psish,
                const u64* p) {
#pragma omp parallel for schedule(static)
  for (int r = 0; r < rows; ++r) {
    const i64 g = gidx[r];
    ntt_fwd_row(a + (size_t)r * n, n, psi + (size_t)g * n, psish + (size_t)g * n, p[g]);
  }
}

/* ring.py:120-124 ntt_inv */
void or_ntt_inv(u64* a, int rows, int n, const i64* gidx, const u64* ipsi, const u64* ipsish,
                const u64* p, const u64* ninv, const u64* ninvsh) {
#pragma omp parallel for schedule(static)
  for (int r = 0; r < rows; ++r) {
    const i64 g = gidx[r];
    ntt_inv_row(a + (size_t)r * n, n, ipsi + (size_t)g * n, ipsish + (size_t)g * n, p[g],
                ninv[g], ninvsh[g]);
  }
}

/* ring.py:127-133 pw_mul */
void or_pw_mul(u64* out, const u64* a, const u64* b, int rows, int n, const i64* gidx,
               const u64* p, const u64* mu, const u64* sh) {
#pragma omp parallel for schedule(static)
  for (int r = 0; r < rows; ++r) {
    const i64 g = gidx[r];
    const size_t o = (size_t)r * n;
    for (int j = 0; j < n; ++j) out[o + j] = mul_barrett(a[o + j], b[o + j], p[g], mu[g], sh[g]);
  }
}

/* ring.py:159-172 pw_add / pw_sub (op 0 / 1) */
void or_pw_addsub(u64* out, const u64* a, const u64* b, int rows, int n, const i64* gidx,
                  const u64* p, int sub) {
#pragma omp parallel for schedule(static)
  for (int r = 0; r < rows; ++r) {
    const u64 pp = p[gidx[r]];
    const size_t o = (size_t)r * n;
    if (sub)
      for (int j = 0; j < n; ++j) out[o + j] = submod(a[o + j], b[o + j], pp);
    else
      for (int j = 0; j < n; ++j) out[o + j] = addmod(a[o + j], b[o + j], pp);
  }
}

/* ring.py:175-183 scalar_mul (in place, per-row constants) */
void or_scalar_mul(u64* a, const u64* c, int rows, int n, const i64* gidx, const u64* p,
                   const u64* mu, const u64* sh) {
#pragma omp parallel for schedule(static)
  for (int r = 0; r < rows; ++r) {
    const i64 g = gidx[r];
    u64* row = a + (size_t)r * n;
    for (int j = 0; j < n; ++j) row[j] = mul_barrett(row[j], c[r], p[g], mu[g], sh[g]);
  }
}

/* ring.py:136-156 pw_mul_accum_perm: outb/outa[r] += perm(de[i][r]) * kb/ka[i][krow[r]]
 * de: (ndig, rows, n); kb, ka: (ndig, krows, n) */
void or_pw_mul_accum_perm(u64* outb, u64* outa, const u64* de, const u64* kb, const u64* ka,
                          const i64* krow, const i64* perm, const i64* gidx, int ndig, int rows,
                          int krows, int n, const u64* p, const u64* mu, const u64* sh) {
#pragma omp parallel for schedule(static)
  for (int r = 0; r < rows; ++r) {
    const i64 g = gidx[r];
    const u64 pp = p[g], mm = mu[g], ss = sh[g];
    const size_t kr = (size_t)krow[r];
    for (int j = 0; j < n; ++j) {
      u64 sb = outb[(size_t)r * n + j], sa = outa[(size_t)r * n + j];
      const i64 dn = perm[j];
      for (int i = 0; i < ndig; ++i) {
        const u64 x = de[((size_t)i * rows + r) * n + dn];
        sb = addmod(sb, mul_barrett(x, kb[((size_t)i * krows + kr) * n + j], pp, mm, ss), pp);
        sa = addmod(sa, mul_barrett(x, ka[((size_t)i * krows + kr) * n + j], pp, mm, ss), pp);
      }
      outb[(size_t)r * n + j] = sb;
      outa[(size_t)r * n + j] = sa;
    }
  }
}

/* ring.py:186-195 lift_center */
void or_lift_center(const u64* x, int n, u64 p, i64* out) {
  const u64 half = p >> 1;
  for (int j = 0; j < n; ++j) out[j] = x[j] > half ? (i64)x[j] - (i64)p : (i64)x[j];
}

/* ring.py:198-207 reduce_rows: centred int64 coefficients -> residues per row */
void or_reduce_rows(const i64* c, int n, const i64* gidx, int rows, const u64* p, u64* out) {
#pragma omp parallel for schedule(static)
  for (int r = 0; r < rows; ++r) {
    const i64 pp = (i64)p[gidx[r]];
    for (int j = 0; j < n; ++j) {
      i64 v = c[j] % pp;
      if (v < 0) v += pp;
      out[(size_t)r * n + j] = (u64)v;
    }
  }
}

/* ring.py:210-219 sub_scaled_inv: rows[r] = (rows[r] - corr[r]) * pinv[r] */
void or_sub_scaled_inv(u64* rowsv, const u64* corr, const u64* pinv, int rows, int n,
                       const i64* gidx, const u64* p, const u64* mu, const u64* sh) {
#pragma omp parallel for schedule(static)
  for (int r = 0; r < rows; ++r) {
    const i64 g = gidx[r];
    const size_t o = (size_t)r * n;
    for (int j = 0; j < n; ++j)
      rowsv[o + j] = mul_barrett(submod(rowsv[o + j], corr[o + j], p[g]), pinv[r], p[g], mu[g], sh[g]);
  }
}

/* Fast RNS base conversion (the standard hybrid key-switching ModUp /
 * ModDown; no reference counterpart -- the reference uses per-prime digits):
 * out[t][j] = sum_i [x_i[j] * qhat_inv[i]]_{q_i} * qhat_mod[i][t]  mod p_t,
 * with the centred representative of every [.]_{q_i} (in (-q_i/2, q_i/2]):
 * the converted integer is x + u Q, |u| <= s/2 (one source: the exact
 * centred lift of the reference's per-prime ModUp / ModDown),
 * source row i at src + i*src_stride, target row t at dst + dst_off[t].
 * Plain 128-bit remainders (an independent reduction from the GPU's). */
void or_bconv(const u64* src, int s, i64 src_stride, const i64* sprime, u64* dst, int t,
              const i64* dst_off, const i64* tprime, int n, const u64* p, const u64* qhat_inv,
              const u64* qhat_mod) {
#pragma omp parallel for schedule(static)
  for (int j = 0; j < n; ++j) {
    u64 y[64];
    int neg[64];
    for (int i = 0; i < s; ++i) {
      const u64 q = p[sprime[i]];
      y[i] = (u64)(((u128)src[(size_t)i * src_stride + j] * qhat_inv[i]) % q);
      neg[i] = y[i] > q / 2;            /* centred representative y - q */
      if (neg[i]) y[i] = q - y[i];
    }
    for (int k = 0; k < t; ++k) {
      const u64 pt = p[tprime[k]];
      u64 acc = 0;
      for (int i = 0; i < s; ++i) {
        const u64 term = (u64)(((u128)y[i] * qhat_mod[(size_t)i * t + k]) % pt);
        acc = neg[i] ? (acc + pt - term) % pt : (acc + term) % pt;
      }
      dst[dst_off[k] + j] = acc;
    }
  }
}

int or_num_threads(void) {
#ifdef _OPENMP
  extern int omp_get_max_threads(void);
  return omp_get_max_threads();
#else
  return 1;
#endif
}

/*
 * hear_b200.h -- C ABI of the B200 kernels behind HEAR's RNS-CKKS hot path.
 *
 * Library: paper_2104_09164_b200/lib/libhear_b200.so (sm_100a).  Plain
 * pointers and sizes only.  Two families:
 *
 *  hear_*  reference-shaped, HOST-buffer entry points.  Same argument meaning
 *          as the numba kernels of hear/ckks/ring.py that they replace: an
 *          (nrows, N) uint64 row-major array plus a per-row global prime index
 *          (chain primes 0..L, then the special prime).  Each call copies in,
 *          runs on the GPU, copies out, synchronises; returns 0 on success.
 *          Binding recipe for the reference: INTEGRATION.md.
 *
 *  hb_*    device-pointer entry points used by the Python engine
 *          (paper_2104_09164_b200/ckks/engine.py).  Work is described by task
 *          tables resident in device memory (layouts: csrc/ring.cuh) and is
 *          enqueued asynchronously on `stream` (a cudaStream_t, may be 0).
 *          Return 0 or a cudaError_t code; hb_last_error() has the text.
 *
 * Residues are canonical (in [0, p)), so every kernel's output is
 * bit-identical to the reference's integer arithmetic on the same inputs
 * (after the two ring-table corrections documented in DESIGN.md §2).
 */
#ifndef HEAR_B200_H
#define HEAR_B200_H

#ifdef __cplusplus
extern "C" {
#endif

typedef struct hb_ring hb_ring; /* per-parameter-set tables on the GPU   */
typedef struct hb_fft hb_fft;   /* canonical-embedding FFT tables        */

/* ---- library / context -------------------------------------------------- */
const char* hb_last_error(void);
int hb_version(void);

/* Replaces hear/ckks/ring.py:253-292 RingContext table construction.
 * primes[nprimes] (< 2^62, = 1 mod 2N); psi/ipsi: [nprimes][N] bit-reversed
 * powers of the primitive 2N-th root and of its inverse. NULL on failure. */
hb_ring* hb_ring_create(int logn, int nprimes, const unsigned long long* primes,
                        const unsigned long long* psi, const unsigned long long* ipsi);
void hb_ring_destroy(hb_ring* ring);
int hb_ring_prime_consts(const hb_ring* ring, int prime_index, unsigned long long* out8);
int hb_sizeof_task(int kind); /* 0 ntt, 1 ew, 2 mac/sum, 3 mac-term, 5 ks2, 6 bconv */

/* ---- reference-shaped host-buffer kernels (hear/ckks/ring.py) ------------ */
/* ring.py:113 ntt_fwd(a, gidx, psi, psish, p) -- in place                     */
int hear_ntt_fwd(hb_ring* ring, unsigned long long* a, int nrows, const long long* gidx);
/* ring.py:120 ntt_inv(a, gidx, ipsi, ipsish, p, ninv, ninvsh) -- in place     */
int hear_ntt_inv(hb_ring* ring, unsigned long long* a, int nrows, const long long* gidx);
/* ring.py:127 pw_mul(out, a, b, gidx, p, mu, sh)                              */
int hear_pw_mul(hb_ring* ring, unsigned long long* out, const unsigned long long* a,
                const unsigned long long* b, int nrows, const long long* gidx);
/* ring.py:159 pw_add(out, a, b, gidx, p)                                      */
int hear_pw_add(hb_ring* ring, unsigned long long* out, const unsigned long long* a,
                const unsigned long long* b, int nrows, const long long* gidx);
/* ring.py:167 pw_sub(out, a, b, gidx, p)                                      */
int hear_pw_sub(hb_ring* ring, unsigned long long* out, const unsigned long long* a,
                const unsigned long long* b, int nrows, const long long* gidx);

/* ring.py:136 pw_mul_accum_perm(outb, outa, de, kb, ka, krow, perm, gidx, p, mu, sh):
 * outb/outa[r] += sum_i de[i][r][perm[n]] * kb/ka[i][krow[r]][n] (mod p_gidx[r]);
 * de [ndig][nrows][N], kb/ka [ndig][krows][N], perm [N] (intp), in place      */
int hear_pw_mul_accum_perm(hb_ring* ring, unsigned long long* outb, unsigned long long* outa,
                           const unsigned long long* de, const unsigned long long* kb,
                           const unsigned long long* ka, const long long* krow,
                           const long long* perm, const long long* gidx, int ndig, int nrows,
                           int krows);
/* ring.py:175 scalar_mul(a, c, gidx, p, mu, sh): a[r] *= c[r], in place       */
int hear_scalar_mul(hb_ring* ring, unsigned long long* a, const unsigned long long* c, int nrows,
                    const long long* gidx);
/* ring.py:186 lift_center(x, p, out): residues -> centred int64 (one row)     */
int hear_lift_center(const unsigned long long* x, unsigned long long p, long long* out, int n);
/* ring.py:198 reduce_rows(c, gidx, p, out): centred int64 [N] -> [nrows][N]   */
int hear_reduce_rows(hb_ring* ring, const long long* c, const long long* gidx, int nrows,
                     unsigned long long* out);
/* ring.py:210 sub_scaled_inv(rows, corr, pinv, gidx, p, mu, sh):
 * rows[r] = (rows[r] - corr[r]) * pinv[r], in place                         */
int hear_sub_scaled_inv(hb_ring* ring, unsigned long long* rows, const unsigned long long* corr,
                        const unsigned long long* pinv, int nrows, const long long* gidx);

/* ---- device task-table kernels --------------------------------------------- */
/* Forward NTT over `count` row tasks (HbNttTask, csrc/ring.cuh).  mode 0:
 * plain (ring.py:113); 1: fused centred lift + reduce of a digit row, the
 * ModUp of engine.py:290-303 (ring.py:186-207 + 113); 2: ModUp +
 * sub_scaled_inv + optional Galois-gathered addend, the ModDown / rescale of
 * engine.py:213-227, 263-281, 350; 3: signed int64 coefficients
 * (engine.py:84-88 _coeffs_to_ntt); 4: mode 2 for a rotation computed on
 * pre-permuted keys, the result scattered through the inverse Galois map
 * (perm) and the addend read in natural order.  Modes 2/4 add the optional
 * post-addend `add2` at the destination index (the add of rotate-and-sum,
 * fastpath.py rot-add, fused).  5 (cluster NTT only): the ModDown of mode 2
 * merged with the rescale that follows it (engine.py:213-227 then 263-281):
 * src = centred special-prime row, `perm` REINTERPRETED as a second source
 * row y (centred doubles: the ModDown'ed top row in the coefficient domain,
 * hb_ew op 10), scal_sh = P mod p_dst, scal = (P q_l)^-1, add2 = q_l^-1 by
 * value:  dst = (aux - NTT(src + P*y)) * scal + add * add2 -- one transform
 * per target row instead of two, same residues as the two steps.  Clusters
 * of N/4096 CTAs on fp64 rings at N = 2^13 .. 2^16 (csrc/ntt3.cu), else
 * two-pass (csrc/ntt2.cu). */
int hb_ntt_fwd(hb_ring* ring, const void* tasks, int count, int mode, void* stream);
/* Inverse NTT over row tasks (ring.py:120, true inverse twiddles).            */
int hb_ntt_inv(hb_ring* ring, const void* tasks, int count, void* stream);
/* Kernel launches one hb_ntt_fwd / hb_ntt_inv call of `count` rows enqueues
 * (launch accounting; no reference counterpart).                             */
int hb_ntt_kernels(hb_ring* ring, int count);
/* 1 when the ring's modular arithmetic runs on the fp64 pipe (every prime
 * < 2^42 and HEAR_B200_INT_NTT unset), else 0.                              */
int hb_ring_uses_f64(const hb_ring* ring);
/* 1 when the ring runs the cluster-fused NTT (fp64 rings, N = 2^13 .. 2^16):
 * hb_ntt_inv then stores centred lifts as doubles for tasks with scal = 1
 * (read back by forward tasks with src_prime = -1), hb_ntt_fwd accepts
 * mode 5 and hb_ks_fused is available.                                       */
int hb_ntt_fused_ks(const hb_ring* ring);
/* Launch every library kernel with programmatic dependent launch (PDL:
 * the next kernel's CTAs are scheduled while the previous grid drains; each
 * kernel waits on griddepcontrol before touching its inputs) while `on`.
 * For CUDA-graph capture, where task tables are static device data.  Returns
 * the previous setting.                                                     */
int hb_set_pdl(int on);
/* Element-wise op `op` over HbEwTask rows: 0 add (ring.py:159), 1 sub
 * (ring.py:167), 2 mul (ring.py:127), 3 scalar mul (ring.py:175), 4 a*b+c
 * (engine.py:202-203), 5 a+b*c (engine.py:204-208), 6 copy, 7 gather,
 * 8 (a-b)*c (ring.py:210), 9 gathered a+b, 10 centre(((a-b)*scal + c) mod p)
 * on centred-double rows (the top row of a merged ModDown + rescale).        */
int hb_ew(hb_ring* ring, int op, const void* tasks, int count, void* stream);
/* Many-term sums dst = sum_k srcs[term_off + k] (mod p) over HbMacTask rows
 * (the add chains of sum_each: hear/fastpath.py rotate-and-sum and FC
 * partial sums, ring.py:159 pw_add), srcs a device array of row pointers;
 * nterms * p < 2^64.                                                        */
int hb_sum(hb_ring* ring, const void* tasks, int count, const void* srcs, void* stream);
/* Same, one launch per layer over [B*2, rows, N] ciphertext blocks.          */
int hb_mac_strided(hb_ring* ring, const void* outs, int nout, const void* terms, int rows,
                   int bc, void* stream);
/* Shared-term MAC for a group of outputs over one ciphertext term list:
 * dsts[o] = sum_t pts[o*nterms + t] * cts[t]; device arrays of row-block
 * base pointers ([bc, rows, N] ciphertext blocks, [rows, N] plaintexts).     */
int hb_mac_shared(hb_ring* ring, const void* cts, const void* pts, const void* dsts, int nterms,
                  int nout, int rows, int bc, void* stream);
/* Key-switch inner products in natural digit order (rotations on pre-permuted
 * keys, relinearisation) as one per-coefficient modular GEMM (engine.py:
 * 305-351, ring.py:136-156): for o < nout (job x component), b < bc,
 * r < rows:  dsts[o][b*dst_bstride + r*N + j] =
 *   sum_i de[i][b*de_bstride + r*N + j] * K[o*ndig + i][j]   (mod q_r)
 * with K = keys[..] + r*N for r < rows-1 and K = keys_last[..] (the key's
 * special row) and the special prime prime_last for r = rows-1.  de is
 * [ndig] row-block base pointers shared by every job, or [nout/2][ndig]
 * (each job its own digits) when de_per_job.  Pointer tables live in device
 * memory.  fp64 rings only.                                                  */
int hb_ks_gemm(hb_ring* ring, const void* de, const void* keys, const void* keys_last,
               const void* dsts, int ndig, int nout, int rows, int bc, long long de_bstride,
               long long dst_bstride, int prime_last, int de_per_job, void* stream);
/* Hoisted rotations left in the extended basis Q*P (ModDown deferred past the
 * plaintext products, Σ_j pt_j * rot_j(ct) with ONE ModDown per output; the
 * reference divides P out after every rotation, engine.py:305-351): the
 * hb_ks_gemm inner product on pre-permuted keys with output o (job x
 * component) stored through its scatter map scat[o] (int32 [N], the inverse
 * Galois map) and, on chain rows r < rows-1 for the outputs with c0s[o] != 0
 * (the b components), plus pmod[r] * c0[b*c0_bstride + r*N + j]  (c0: the
 * rotated handle's c0 block, pmod[r] = P mod q_r):
 *   dsts[o][b*dst_bstride + r*N + scat[o][j]] = <digits, key>[j] + P*c0[j].   */
int hb_ks_gemm_rot(hb_ring* ring, const void* de, const void* keys, const void* keys_last,
                   const void* dsts, const void* scat, const void* c0s, const void* c0,
                   const void* pmod, int ndig, int nout, int rows, int bc, long long de_bstride,
                   long long dst_bstride, long long c0_bstride, int prime_last, void* stream);
/* hb_mac_shared over extended-basis blocks [bc, rows, N] whose last row is
 * the special prime prime_last: plaintext special rows come from pts_last
 * (pointers to the rows themselves, [nout*nterms]).                          */
int hb_mac_shared_ext(hb_ring* ring, const void* cts, const void* pts, const void* pts_last,
                      const void* dsts, int nterms, int nout, int rows, int bc, int prime_last,
                      void* stream);
/* Rotate-and-sum ct + sum_j rot_j(ct) of one hoisted group, in the extended
 * basis and without materialising the rotations (hear/fastpath.py:141-154
 * rotate_sum_each's odd part; each rotation engine.py:328-351): HbRotSumTask
 * per (handle, output row), HbRotSumRot per amount (Galois gather map,
 * reference-layout key components); nb clips per task, ndig digits:
 *   out_b[m] = P (c0[m] + sum_j c0[pi_j m]) + sum_j sum_i de_i[pi_j m] kb_ij[m]
 *   out_a[m] = P  c1[m]                     + sum_j sum_i de_i[pi_j m] ka_ij[m]
 * (no P terms on the special row).  The caller divides P out once.           */
int hb_rot_sum(hb_ring* ring, const void* tasks, int ntasks, const void* rots, int nrot,
               int ndig, int nb, void* stream);
/* Fused ModUp + key-switch inner product for non-hoisted key switches
 * (relinearisation, rot_each, rotate-and-add; engine.py:290-326 digit
 * expansion + ring.py:136-156 inner product in ONE kernel): one HbKsfTask per
 * (ciphertext, target row) = {coef, ident, kb, ka, out_b, out_a, key_dstride,
 * ndig, dst_prime, ident_digit, scat, c0, pmod}:
 *   out_{b,a}[j] = sum_i NTT_dst(lift(coef_i))[j] * k{b,a}[i*key_dstride + j]
 * where coef_i = coef + i*N holds digit i's centred lift as doubles
 * (coefficient domain, written by hb_ntt_inv with scal = 1) and digit
 * ident_digit is taken from the NTT-form row `ident` instead of transformed.
 * The digit expansion is never written: the transforms run in shared memory
 * of a thread-block cluster and the running sums live in tensor memory
 * (csrc/ntt3.cu k_ks3).  With scat != 0 the outputs are stored through that
 * scatter map (the inverse Galois map of a pre-permuted rotation key) and
 * out_b gains pmod * c0[j]: out_b / out_a are rows of the ROTATED ciphertext
 * in the extended basis (lazy ModDown).  fp64 rings with hb_ntt_fused_ks()
 * == 1 only.                                                                 */
int hb_ks_fused(hb_ring* ring, const void* tasks, int count, void* stream);
/* Key-switch inner product, one task per (job, output row), nb clips per task
 * (ring.py:136-156 pw_mul_accum_perm, key rows shared across clips).  fp64
 * rings: a task with scat != 0 stores its sums through that scatter map and
 * adds pmod * c0 to the b component -- the rotation left in the extended
 * basis (lazy ModDown at batches below the GEMM's).                          */
int hb_ks_inner2(hb_ring* ring, const void* tasks, int count, int nb, void* stream);
/* Fast RNS base conversion, one task per (polynomial, source basis):
 * dst_t = sum_i [src_i * qhat_i^-1]_{q_i} * (qhat_i mod p_t) mod p_t
 * (csrc/bconv.cu; the ModUp / ModDown of hybrid dnum-digit key switching,
 * BASELINE config 1; the reference's per-prime digits need none).  nsrc:
 * the source count shared by every task (selects a register-resident
 * kernel), 0 when the tasks differ.                                           */
int hb_bconv(hb_ring* ring, const void* tasks, int count, int nsrc, void* stream);
/* Ciphertext tensor product d0, d1, d2 (engine.py:249-257).                  */
int hb_tensor(hb_ring* ring, const void* tasks, int count, void* stream);
/* Exact CRT of `keep` coefficient rows to centred doubles (engine.py:156-175). */
int hb_crt_double(hb_ring* ring, const void* tasks, int count, const unsigned long long* consts,
                  const int* prime_idx, int keep, int nl, void* stream);

/* ---- canonical-embedding codec (hear/ckks/encoder.py) ------------------------ */
hb_fft* hb_fft_create(int logn2, const double* root_re_im, const double* twist_re_im,
                      const int* slot_pos);
void hb_fft_destroy(hb_fft* fft);
/* encoder.py:48-56 encode_coeffs: slots [npoly][N/2] -> rint(coeffs*scale)
 * [npoly][N] int64; *overflow set when |coeff| >= 2^52.                      */
int hb_encode(hb_fft* fft, const double* slots, long long* coeffs, int npoly, double scale,
              int* overflow, void* stream);
/* encoder.py:59-60 decode_coeffs: coeffs [npoly][N] -> real slots / scale.    */
int hb_decode(hb_fft* fft, const double* coeffs, double* slots, int npoly, double scale,
              void* stream);

#ifdef __cplusplus
}
#endif
#endif /* HEAR_B200_H */

// Device-side ring context and task descriptors shared by all kernels.
#pragma once
#include <cuda_runtime.h>
#include <utility>
#include "modarith.cuh"

// ---- programmatic dependent launch (PDL) ------------------------------------
// When g_hb_pdl is set (CUDA-graph capture of the evaluation, where task
// tables are static device data), every library kernel is launched with
// programmatic stream serialisation: the next kernel's CTAs may be scheduled
// while this one drains.  Every kernel starts with HB_PDL_ENTRY() -- wait for
// the previous grid's completion and memory, then allow the next grid to
// launch -- so results are unchanged; without the attribute both are no-ops.
extern int g_hb_pdl;
#define HB_PDL_WAIT() asm volatile("griddepcontrol.wait;" ::: "memory")
#define HB_PDL_LAUNCH() asm volatile("griddepcontrol.launch_dependents;" ::: "memory")
#define HB_PDL_ENTRY() \
  do {                 \
    HB_PDL_WAIT();     \
    HB_PDL_LAUNCH();   \
  } while (0)

template <typename... KArgs, typename... Args>
inline cudaError_t hb_launch(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                             cudaStream_t st, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = g_hb_pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

// Twiddle entry: power of the 2N-th root plus its Shoup companion, stored
// together so one 16-byte load fetches both.
struct __align__(16) HbTw {
  u64 w, wsh;
};

// fp64 twiddle entry: w as an exact double and fl(w / p).
struct __align__(16) HbTwD {
  double w, wq;
};

struct HbRing {
  int logn;
  int n;
  int nprimes;
  int use_f64;            // every prime < 2^42: transforms run on the fp64 pipe
  int split_ok;           // every prime < 2^34: mac.cu may sum split products exactly
  const HbPrime* primes;  // [nprimes]
  const HbTw* tw_fwd;     // [nprimes][n]  psi^brv(j)            (ring.py:281)
  const HbTw* tw_inv;     // [nprimes][n]  psi^-brv(j)  (true inverse)
  const HbTwD* twd_fwd;   // fp64 copies of the two tables
  const HbTwD* twd_inv;
  const double* tw1_fwd;  // fp64 powers only (8 B entries, staged in smem by ntt2.cu)
  const double* tw1_inv;
  // fine-stage twiddles of the cluster NTT (ntt3.cu), plane-major so that a
  // warp's lanes (consecutive groups G) read consecutive entries:
  //   fwd stage logn-3+e, entry (G << e) + i  at  ((2^e - 1) + i) * n/8 + G
  //   inv stage r,        entry (G << (2-r)) + i  at  (off[r] + i) * n/8 + G,
  //   off = {0, 4, 6}
  const HbTwD* tw3_fwd;   // [nprimes][n] (7n/8 used)
  const HbTwD* tw3_inv;
};

// Raise a kernel's dynamic shared-memory limit only when a launch needs more
// than already granted (cudaFuncSetAttribute on every launch costs host time
// in eager, launch-bound phases).  `cur` is a per-instantiation static.
inline cudaError_t smem_attr_once(const void* fn, int bytes, int* cur) {
  if (bytes <= *cur) return cudaSuccess;
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e == cudaSuccess) *cur = bytes;
  return e;
}

// One row-polynomial transform.  Field meaning depends on the kernel mode;
// see ntt.cu.
struct HbNttTask {
  const u64* src;
  u64* dst;
  const u64* aux;   // ModDown/rescale: extended-basis row x_r
  const u64* add;   // optional addend row (gathered through perm if set)
  const int* perm;  // optional automorphism gather for `add`
  u64 scal;         // epilogue constant (P^-1 / q_l^-1 mod p_dst)
  u64 scal_sh;
  const u64* add2;  // forward ModDown: optional post-addend, read at the
                    // destination index (after the Galois gather / scatter):
                    // fuses the "ct + rot(ct)" add of rotate-and-sum.
                    // inverse: optional second destination receiving the
                    // input row verbatim (the ModUp identity digit row)
  int src_prime;    // prime of src when it differs from dst_prime (lift)
  int dst_prime;    // prime the transform runs in
};

// One (ciphertext, target row) of the fused ModUp + key-switch inner product
// (ntt3.cu k_ks3): out_b / out_a = sum_i NTT_t(lift(digit i)) * key_{b,a}[i].
struct HbKsfTask {
  const u64* coef;     // digit i's centred lift as doubles, coefficient domain, at coef + i*N
  const u64* ident;    // NTT-form row of the digit whose prime IS the target (else null)
  const u64* kb;       // key rows of the target prime: digit i at kb + i*key_dstride
  const u64* ka;
  u64* out_b;          // the two inner-product rows of this target prime
  u64* out_a;
  long long key_dstride;
  int ndig;
  int dst_prime;
  int ident_digit;     // the digit served by `ident` (-1: none, the special row)
  int _pad;
  // rotation left in the extended basis (lazy ModDown): outputs stored through
  // the scatter map (the inverse Galois map of the pre-permuted key), out_b
  // plus pmod * c0 on chain rows -- out_b / out_a are then rows of the rotated
  // ciphertext in basis Q*P.  scat = null: plain inner-product rows.
  const int* scat;
  const u64* c0;       // this target row of the rotated handle's c0 (null: special row)
  u64 pmod;            // P mod p_dst
};

// One output row of a plaintext multiply-accumulate:
//   dst = sum_t pt_t * ct_t  (mod p)   over terms [term_off, term_off + nterms)
struct HbMacTask {
  u64* dst;
  int prime;
  int nterms;
  int term_off;
  int _pad;
};

struct HbMacTerm {
  const u64* pt;
  const u64* ct;
};


// Generic element-wise row op.
struct HbEwTask {
  u64* dst;
  const u64* a;
  const u64* b;
  const u64* c;
  u64 scal;
  u64 scal_sh;
  int prime;
  int _pad;
};

// Element-wise ops of ops.cu k_ew (launch_ew / hb_ew).
enum EwOp : int {
  EW_ADD = 0,       // dst = a + b                       (ring.py:159 pw_add)
  EW_SUB = 1,       // dst = a - b                       (ring.py:167 pw_sub)
  EW_MUL = 2,       // dst = a * b                       (ring.py:127 pw_mul)
  EW_MUL_SCALAR = 3,// dst = a * scal                    (ring.py:175 scalar_mul)
  EW_MULADD = 4,    // dst = a * b + c                   (engine.py:202-203)
  EW_ADD_SCALED = 5,// dst = a + b * scal                (engine.py:204-208)
  EW_COPY = 6,      // dst = a
  EW_PERM = 7,      // dst = a[perm]  (b reinterpreted as int32 perm)
  EW_SUB_SCALED = 8,// dst = (a - b) * scal              (ring.py:210 sub_scaled_inv)
  EW_PERM_ADD = 9,  // dst = a[perm] + b[perm]  (c reinterpreted as int32 perm): the
                    // Galois gather of a rotation applied after ModDown (engine.py:350)
  EW_MD_TOP = 10,   // a, b, c, dst hold centred lifts as doubles (coefficient domain):
                    // dst = centre(((a - b) * scal + c) mod p), c optional -- the top
                    // row after ModDown (+ addend), input of the merged rescale
};

// Special-FFT tables of the canonical embedding (fft.cu).
struct HbFftTables {
  int logn2;            // log2(N/2)
  int n2;
  const double2* root;  // [n2/2]: e^{+2 pi i k / n2}
  const double2* twist; // [n2]:   zeta^k = e^{i pi k / N}
  const int* slot_of;   // [n2]:   DFT bin m -> slot j with m_j = m (inverse of m_j)
};

// Rotate-and-sum in the extended basis (ops.cu k_rot_sum_f64): one output row
// of one handle, and one entry per rotation amount of the group.
struct HbRotSumTask {
  const u64* de;     // clip 0, digit 0, this row of the digit expansion
  const u64* c0;     // clip 0, this row of c0 / c1 (null on the special row)
  const u64* c1;
  u64* out_b;        // clip 0, this row of the two output components
  u64* out_a;
  long long de_bstride, de_dstride, c_bstride, out_bstride;
  u64 pmod;          // P mod p_row
  int prime;
  int row;           // chain row index, or -1 for the special row
};
struct HbRotSumRot {
  const int* perm;   // rotated[m] = in[perm[m]]
  const u64* kb;     // digit 0, row 0 of the (reference-layout) key components
  const u64* ka;
  long long key_dstride;
  int special_row;   // row index of the key's special row
  int _pad;
};

// Clip-blocked key-switch inner product task (ops.cu k_ks_inner2).
struct HbKsTask2 {
  const u64* de;      // clip 0, digit 0, row r
  const u64* kb;      // digit 0 key row (krow[r])
  const u64* ka;
  u64* out_b;         // clip 0
  u64* out_a;
  const int* perm;
  long long de_bstride, de_dstride, key_stride, out_bstride;
  int ndig;
  int prime;
  // rotation left in the extended basis (fp64 kernel only; lazy ModDown at
  // small batches): outputs stored through the scatter map, out_b plus
  // pmod * c0[b*c0_bstride + j] when c0 is set.  scat = null: as before.
  const int* scat;
  const u64* c0;
  long long c0_bstride;
  u64 pmod;
};

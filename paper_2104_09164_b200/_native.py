"""ctypes binding of lib/libhear_b200.so (declared in include/hear_b200.h).

There is no fallback: importing the engine without the built library, or
without a CUDA device, raises.  Task tables are numpy structured arrays whose
layout mirrors the C structs in csrc/ring.cuh; `upload` copies one to the
device on the current torch stream.
"""

from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("HEAR_B200_LIB") or os.path.join(_HERE, "lib", "libhear_b200.so")

_lib = None


class NativeError(RuntimeError):
    """A kernel launch or the library itself failed."""


def lib():
    """Load the kernel library (once).  Raises if it is missing."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise NativeError(
                f"{LIB_PATH} is missing: build it with `python -m paper_2104_09164_b200.build` "
                "(or __graft_entry__.build()); there is no CPU fallback")
        L = ctypes.CDLL(LIB_PATH)
        vp, i32, u64p = ctypes.c_void_p, ctypes.c_int, ctypes.POINTER(ctypes.c_uint64)
        L.hb_last_error.restype = ctypes.c_char_p
        L.hb_version.restype = i32
        L.hb_ring_create.restype = vp
        L.hb_ring_create.argtypes = [i32, i32, vp, vp, vp]
        L.hb_ring_destroy.argtypes = [vp]
        L.hb_ring_prime_consts.argtypes = [vp, i32, vp]
        L.hb_sizeof_task.argtypes = [i32]
        L.hb_ntt_fwd.argtypes = [vp, vp, i32, i32, vp]
        L.hb_ntt_inv.argtypes = [vp, vp, i32, vp]
        L.hb_ntt_kernels.argtypes = [vp, i32]
        L.hb_ring_uses_f64.argtypes = [vp]
        L.hb_ntt_fused_ks.argtypes = [vp]
        L.hb_set_pdl.argtypes = [i32]
        L.hb_ks_gemm.argtypes = [vp, vp, vp, vp, vp, i32, i32, i32, i32, ctypes.c_longlong,
                                 ctypes.c_longlong, i32, i32, vp]
        L.hb_ks_gemm_rot.argtypes = [vp] * 9 + [i32] * 4 + [ctypes.c_longlong] * 3 + [i32, vp]
        L.hb_mac_shared_ext.argtypes = [vp] * 5 + [i32] * 5 + [vp]
        L.hb_ks_fused.argtypes = [vp, vp, i32, vp]
        L.hb_rot_sum.argtypes = [vp, vp, i32, vp, i32, i32, i32, vp]
        L.hb_ew.argtypes = [vp, i32, vp, i32, vp]
        L.hb_tensor.argtypes = [vp, vp, i32, vp]
        L.hb_mac_strided.argtypes = [vp, vp, i32, vp, i32, i32, vp]
        L.hb_sum.argtypes = [vp, vp, i32, vp, vp]
        L.hb_ks_inner2.argtypes = [vp, vp, i32, i32, vp]
        L.hb_bconv.argtypes = [vp, vp, i32, i32, vp]
        L.hb_mac_shared.argtypes = [vp, vp, vp, vp, i32, i32, i32, i32, vp]
        L.hb_crt_double.argtypes = [vp, vp, i32, vp, vp, i32, i32, vp]
        L.hb_fft_create.restype = vp
        L.hb_fft_create.argtypes = [i32, vp, vp, vp]
        L.hb_fft_destroy.argtypes = [vp]
        L.hb_encode.argtypes = [vp, vp, vp, i32, ctypes.c_double, vp, vp]
        L.hb_decode.argtypes = [vp, vp, vp, i32, ctypes.c_double, vp]
        for name in ("hear_ntt_fwd", "hear_ntt_inv"):
            getattr(L, name).argtypes = [vp, vp, i32, vp]
        for name in ("hear_pw_mul", "hear_pw_add", "hear_pw_sub"):
            getattr(L, name).argtypes = [vp, vp, vp, vp, i32, vp]
        L.hear_pw_mul_accum_perm.argtypes = [vp] * 9 + [i32] * 3
        L.hear_scalar_mul.argtypes = [vp, vp, vp, i32, vp]
        L.hear_lift_center.argtypes = [vp, ctypes.c_uint64, vp, i32]
        L.hear_reduce_rows.argtypes = [vp, vp, vp, i32, vp]
        L.hear_sub_scaled_inv.argtypes = [vp, vp, vp, vp, i32, vp]
        _lib = L
        _check_layouts()
    return _lib


launch_count = 0   # hb_* launch calls issued through this binding
_kernels = 0       # CUDA kernels those calls enqueued


def kernel_launches() -> int:
    return _kernels


def check(rc: int, what: str, kernels: int = 1):
    """Verify one hb_* launch call and count the kernels it enqueued."""
    global launch_count, _kernels
    launch_count += 1
    _kernels += kernels
    if rc != 0:
        msg = _lib.hb_last_error().decode() if _lib is not None else "?"
        raise NativeError(f"{what} failed ({rc}): {msg}")


# ---- task-table layouts (csrc/ring.cuh) -------------------------------------

NTT_TASK = np.dtype([("src", "<u8"), ("dst", "<u8"), ("aux", "<u8"), ("add", "<u8"),
                     ("perm", "<u8"), ("scal", "<u8"), ("scal_sh", "<u8"), ("add2", "<u8"),
                     ("src_prime", "<i4"), ("dst_prime", "<i4")])
EW_TASK = np.dtype([("dst", "<u8"), ("a", "<u8"), ("b", "<u8"), ("c", "<u8"),
                    ("scal", "<u8"), ("scal_sh", "<u8"), ("prime", "<i4"), ("_pad", "<i4")])
MAC_TASK = np.dtype([("dst", "<u8"), ("prime", "<i4"), ("nterms", "<i4"),
                     ("term_off", "<i4"), ("_pad", "<i4")])
MAC_TERM = np.dtype([("pt", "<u8"), ("ct", "<u8")])
MAC_OUT = np.dtype([("dst", "<u8"), ("nterms", "<i4"), ("term_off", "<i4")])
KS_TASK2 = np.dtype([("de", "<u8"), ("kb", "<u8"), ("ka", "<u8"), ("out_b", "<u8"),
                     ("out_a", "<u8"), ("perm", "<u8"), ("de_bstride", "<i8"),
                     ("de_dstride", "<i8"), ("key_stride", "<i8"), ("out_bstride", "<i8"),
                     ("ndig", "<i4"), ("prime", "<i4"), ("scat", "<u8"), ("c0", "<u8"),
                     ("c0_bstride", "<i8"), ("pmod", "<u8")])
TENSOR_TASK = np.dtype([("a0", "<u8"), ("a1", "<u8"), ("b0", "<u8"), ("b1", "<u8"),
                        ("d0", "<u8"), ("d1", "<u8"), ("d2", "<u8"),
                        ("prime", "<i4"), ("_pad", "<i4")])
CRT_TASK = np.dtype([("rows", "<u8"), ("out", "<u8")])
BCONV_TASK = np.dtype([("src", "<u8"), ("dst", "<u8"), ("dst_off", "<u8"), ("tab", "<u8"),
                       ("sprime", "<u8"), ("tprime", "<u8"), ("src_stride", "<i8"),
                       ("s", "<i4"), ("t", "<i4")])

KSF_TASK = np.dtype([("coef", "<u8"), ("ident", "<u8"), ("kb", "<u8"), ("ka", "<u8"),
                     ("out_b", "<u8"), ("out_a", "<u8"), ("key_dstride", "<i8"),
                     ("ndig", "<i4"), ("dst_prime", "<i4"), ("ident_digit", "<i4"),
                     ("_pad", "<i4"), ("scat", "<u8"), ("c0", "<u8"), ("pmod", "<u8")])

ROTSUM_TASK = np.dtype([("de", "<u8"), ("c0", "<u8"), ("c1", "<u8"), ("out_b", "<u8"),
                        ("out_a", "<u8"), ("de_bstride", "<i8"), ("de_dstride", "<i8"),
                        ("c_bstride", "<i8"), ("out_bstride", "<i8"), ("pmod", "<u8"),
                        ("prime", "<i4"), ("row", "<i4")])
ROTSUM_ROT = np.dtype([("perm", "<u8"), ("kb", "<u8"), ("ka", "<u8"), ("key_dstride", "<i8"),
                       ("special_row", "<i4"), ("_pad", "<i4")])

# NTT fused modes (csrc/ntt.cu FwdMode)
FWD_PLAIN, FWD_LIFT, FWD_MODDOWN, FWD_I64, FWD_MODDOWN_SCATTER, FWD_MODDOWN2 = 0, 1, 2, 3, 4, 5
# element-wise ops (csrc/ops.cu EwOp)
EW_ADD, EW_SUB, EW_MUL, EW_MUL_SCALAR, EW_MULADD, EW_ADD_SCALED, EW_COPY, EW_PERM, \
    EW_SUB_SCALED, EW_PERM_ADD, EW_MD_TOP = range(11)


def _check_layouts():
    L = _lib
    for kind, dt in enumerate((NTT_TASK, EW_TASK, MAC_TASK, MAC_TERM, None, KS_TASK2,
                               BCONV_TASK, KSF_TASK, ROTSUM_TASK, ROTSUM_ROT)):
        if dt is not None and L.hb_sizeof_task(kind) != dt.itemsize:
            raise NativeError(f"task layout {kind} mismatch: C {L.hb_sizeof_task(kind)} "
                              f"vs numpy {dt.itemsize}")


def shoup(w, p):
    """Shoup companion floor(w * 2^64 / p) for integer or array w."""
    if isinstance(w, np.ndarray):
        return np.array([(int(x) << 64) // int(pp) for x, pp in
                         zip(w.tolist(), np.broadcast_to(p, w.shape).tolist())], dtype=np.uint64)
    return (int(w) << 64) // int(p)

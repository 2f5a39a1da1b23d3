"""Kernel-level binding stub a maintainer adds to the reference package
(as hear/ckks/ring_b200.py) to run its ring kernels on the B200 library.

It binds the `hear_*` host-buffer entry points of include/hear_b200.h with
ctypes and wraps a reference `hear.ckks.ring.RingContext`'s tables
(ring.py:253-292).  Every method has the name, argument meaning and in-place
behaviour of the numba kernel or RingContext wrapper it replaces
(ring.py:113-219, 296-313).  INTEGRATION.md §2 shows this file;
tests/test_gpu_boundary.py runs it as written.
"""

from __future__ import annotations

import ctypes
import os

import numpy as np

LIB = os.environ.get("HEAR_B200_LIB") or os.path.join(
    os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
    "paper_2104_09164_b200", "lib", "libhear_b200.so")
_L = ctypes.CDLL(LIB)
vp, i32 = ctypes.c_void_p, ctypes.c_int
_L.hb_last_error.restype = ctypes.c_char_p
_L.hb_ring_create.restype = vp
_L.hb_ring_create.argtypes = [i32, i32, vp, vp, vp]
_L.hb_ring_destroy.argtypes = [vp]
for f in ("hear_ntt_fwd", "hear_ntt_inv"):
    getattr(_L, f).argtypes = [vp, vp, i32, vp]
for f in ("hear_pw_mul", "hear_pw_add", "hear_pw_sub"):
    getattr(_L, f).argtypes = [vp, vp, vp, vp, i32, vp]
_L.hear_pw_mul_accum_perm.argtypes = [vp] * 9 + [i32] * 3
_L.hear_scalar_mul.argtypes = [vp, vp, vp, i32, vp]
_L.hear_lift_center.argtypes = [vp, ctypes.c_uint64, vp, i32]
_L.hear_reduce_rows.argtypes = [vp, vp, vp, i32, vp]
_L.hear_sub_scaled_inv.argtypes = [vp, vp, vp, vp, i32, vp]


def _ok(rc, what):
    if rc != 0:
        raise RuntimeError(f"{what}: {_L.hb_last_error().decode()}")


def _u64(a):
    assert a.dtype == np.uint64 and a.flags.c_contiguous
    return a.ctypes.data


def _g(gidx):
    return np.ascontiguousarray(gidx, dtype=np.int64)


class B200Ring:
    """Device ring over a reference RingContext's primes and forward table.

    The inverse table is rebuilt as the entrywise inverse of psi
    (psi^-brv(j)): the reference's own ipsi (ring.py:282, exponent brv(j)+1)
    is not the inverse transform."""

    def __init__(self, rc):
        self.n, self.logn = rc.n, rc.logn
        self.primes = [int(q) for q in rc.primes]
        p = np.array(self.primes, dtype=np.uint64)
        psi = np.ascontiguousarray(rc.psi, dtype=np.uint64)
        ipsi = np.array([[pow(int(w), -1, q) for w in row] for row, q in zip(psi, self.primes)],
                        dtype=np.uint64)
        self.h = _L.hb_ring_create(self.logn, len(p), p.ctypes.data, psi.ctypes.data,
                                   ipsi.ctypes.data)
        if not self.h:
            raise RuntimeError(_L.hb_last_error().decode())

    def __del__(self):
        if getattr(self, "h", None):
            _L.hb_ring_destroy(self.h)

    # RingContext wrappers (ring.py:296-313)
    def fwd(self, rows, gidx):                       # ntt_fwd, in place
        g = _g(gidx)
        _ok(_L.hear_ntt_fwd(self.h, _u64(rows), rows.shape[0], g.ctypes.data), "ntt_fwd")

    def inv(self, rows, gidx):                       # ntt_inv, in place
        g = _g(gidx)
        _ok(_L.hear_ntt_inv(self.h, _u64(rows), rows.shape[0], g.ctypes.data), "ntt_inv")

    def _binop(self, fn, a, b, gidx, out):
        out = np.empty_like(a) if out is None else out
        g = _g(gidx)
        _ok(fn(self.h, _u64(out), _u64(a), _u64(b), a.shape[0], g.ctypes.data), fn.__name__)
        return out

    def mul(self, a, b, gidx, out=None):             # pw_mul
        return self._binop(_L.hear_pw_mul, a, b, gidx, out)

    def add(self, a, b, gidx, out=None):             # pw_add
        return self._binop(_L.hear_pw_add, a, b, gidx, out)

    def sub(self, a, b, gidx, out=None):             # pw_sub
        return self._binop(_L.hear_pw_sub, a, b, gidx, out)

    # module-level kernels of ring.py, same argument order minus the tables
    def pw_mul_accum_perm(self, outb, outa, de, kb, ka, krow, perm, gidx):   # ring.py:136
        krow, perm, g = _g(krow), _g(perm), _g(gidx)
        _ok(_L.hear_pw_mul_accum_perm(self.h, _u64(outb), _u64(outa), _u64(de), _u64(kb),
                                      _u64(ka), krow.ctypes.data, perm.ctypes.data,
                                      g.ctypes.data, de.shape[0], outb.shape[0], kb.shape[1]),
            "pw_mul_accum_perm")

    def scalar_mul(self, a, c, gidx):                # ring.py:175, in place
        c, g = np.ascontiguousarray(c, dtype=np.uint64), _g(gidx)
        _ok(_L.hear_scalar_mul(self.h, _u64(a), c.ctypes.data, a.shape[0], g.ctypes.data),
            "scalar_mul")

    @staticmethod
    def lift_center(x, p, out):                      # ring.py:186
        _ok(_L.hear_lift_center(_u64(x), int(p), out.ctypes.data, x.shape[0]), "lift_center")

    def reduce_rows(self, c, gidx, out):             # ring.py:198
        c, g = np.ascontiguousarray(c, dtype=np.int64), _g(gidx)
        _ok(_L.hear_reduce_rows(self.h, c.ctypes.data, g.ctypes.data, out.shape[0], _u64(out)),
            "reduce_rows")

    def sub_scaled_inv(self, rows, corr, pinv, gidx):   # ring.py:210, in place
        pinv, g = np.ascontiguousarray(pinv, dtype=np.uint64), _g(gidx)
        _ok(_L.hear_sub_scaled_inv(self.h, _u64(rows), _u64(corr), pinv.ctypes.data,
                                   rows.shape[0], g.ctypes.data), "sub_scaled_inv")

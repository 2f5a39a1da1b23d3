"""Canonical-embedding codec on the GPU (restates hear/ckks/encoder.py).

Slot j is the evaluation of the coefficient polynomial at zeta^(5^j),
zeta = e^{i pi/N}; conjugate points carry the mirrored values so the
coefficients stay real.  The transform itself is the length-N/2 special FFT
of csrc/fft.cu (one CTA per polynomial, fp64).
"""

from __future__ import annotations

import ctypes

import numpy as np
import torch

from .. import _native as nat

MAX_ENCODE_COEFF = float(1 << 52)


class EncodeOverflow(ValueError):
    """Scaled coefficients exceed exact float64 integer range (encoder.py:44)."""


class Embedding:
    """Slot-index tables and the device FFT handle for ring degree n."""

    def __init__(self, n: int, device=None):
        self.n = n
        self.n2 = n // 2
        two_n = 2 * n
        g = np.empty(self.n2, dtype=np.int64)
        cur = 1
        for j in range(self.n2):
            g[j] = cur
            cur = cur * 5 % two_n
        self.rot_group = g
        self.conj_group = (two_n - g) % two_n
        self.slot_pos = ((g - 1) // 4).astype(np.int32)   # DFT bin of slot j
        k = np.arange(self.n2, dtype=np.longdouble)
        pi = np.longdouble("3.14159265358979323846264338327950288")
        ang_root = 2 * pi * k[: self.n2 // 2] / self.n2
        ang_tw = pi * k / n
        self.root = np.stack([np.cos(ang_root), np.sin(ang_root)], -1).astype(np.float64)
        self.twist = np.stack([np.cos(ang_tw), np.sin(ang_tw)], -1).astype(np.float64)
        self.device = torch.device(device or "cuda")
        L = nat.lib()
        h = L.hb_fft_create(self.n2.bit_length() - 1, np.ascontiguousarray(self.root).ctypes.data,
                            np.ascontiguousarray(self.twist).ctypes.data,
                            self.slot_pos.ctypes.data)
        if not h:
            raise nat.NativeError(L.hb_last_error().decode())
        self.handle = ctypes.c_void_p(h)
        self._lib = L
        self._flag = torch.zeros(1, dtype=torch.int32, device=self.device)

    def __del__(self):
        try:
            if getattr(self, "handle", None):
                self._lib.hb_fft_destroy(self.handle)
        except Exception:
            pass

    def encode_coeffs(self, slots: torch.Tensor, scale: float, check: bool = True) -> torch.Tensor:
        """(M, N/2) float64 slot values -> (M, N) int64 rounded coefficients
        (encoder.py:48-56).  Raises EncodeOverflow past 2^52."""
        slots = slots.to(self.device, torch.float64).contiguous()
        m = slots.shape[0]
        out = torch.empty(m, self.n, dtype=torch.int64, device=self.device)
        if check:
            self._flag.zero_()
        st = torch.cuda.current_stream(self.device).cuda_stream
        nat.check(self._lib.hb_encode(self.handle, slots.data_ptr(), out.data_ptr(), m,
                                      float(scale), self._flag.data_ptr(), st), "encode")
        if check and int(self._flag.item()):
            raise EncodeOverflow("encoded coefficient magnitude exceeds 2^52; "
                                 "scale too large for these values")
        return out

    def decode_coeffs(self, coeffs: torch.Tensor, scale: float) -> torch.Tensor:
        """(M, N) float64 coefficients -> (M, N/2) real slot values / scale."""
        coeffs = coeffs.to(self.device, torch.float64).contiguous()
        m = coeffs.shape[0]
        out = torch.empty(m, self.n2, dtype=torch.float64, device=self.device)
        st = torch.cuda.current_stream(self.device).cuda_stream
        nat.check(self._lib.hb_decode(self.handle, coeffs.data_ptr(), out.data_ptr(), m,
                                      float(scale), st), "decode")
        return out

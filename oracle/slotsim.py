"""Exact slot simulator -- TEST INFRASTRUCTURE ONLY (oracle/).

Restates hear/backend.py:222-266 (SimBackend): float64 slot vectors with the
(level, scale) ledger; every op is the plain slot operation.  It realises
the same contract as the GPU engine (paper_2104_09164_b200.backend) so the
network schedule can be checked on the CPU against the cleartext network and
the reference's operation counters.  Never imported by the product path.
Handles may hold a batch (payload shape (B, n2)).
"""

from __future__ import annotations

import numpy as np

from paper_2104_09164_b200.backend import BackendBase, Ct, Pt


class SimBackend(BackendBase):
    exact = True

    def _raw_encode(self, values, level, scale):
        return Pt(values.copy(), level, scale, self.n2)

    def encode_many(self, values, level, scale):
        from fractions import Fraction
        return [Pt(v.copy(), level, Fraction(scale), self.n2) for v in np.asarray(values)]

    def _raw_enc(self, values, level, scale):
        return Ct(np.array(values, dtype=np.float64), level, scale, self.n2)

    def _raw_dec(self, ct):
        return ct.payload.copy()

    def _raw_add(self, a, b):
        return Ct(a.payload + b.payload, a.level, a.scale, self.n2)

    def _raw_add_plain(self, a, p):
        return Ct(a.payload + p.payload, a.level, a.scale, self.n2)

    def _raw_mult(self, a, b):
        return Ct(a.payload * b.payload, a.level, a.scale * b.scale, self.n2)

    def _raw_mult_plain(self, a, p):
        return Ct(a.payload * p.payload, a.level, a.scale * p.scale, self.n2)

    def _raw_rot(self, a, k):
        return Ct(np.roll(a.payload, -k, axis=-1), a.level, a.scale, self.n2)

    def _raw_rot_many(self, a, ks):
        return {k: self._raw_rot(a, k) for k in ks}

    def _raw_rescale(self, a):
        return Ct(a.payload.copy(), a.level - 1, a.scale / self.prime_at(a.level), self.n2)

    def _raw_mod_down(self, a, to_level):
        return Ct(a.payload.copy(), to_level, a.scale, self.n2)

    def poison(self, ct, mask, value: float = 1e30):
        vals = ct.payload.copy()
        vals[..., np.asarray(mask, dtype=bool)] = value
        return Ct(vals, ct.level, ct.scale, self.n2)

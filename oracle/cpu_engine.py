"""CPU oracle of the reference CKKS engine -- TEST INFRASTRUCTURE ONLY.

Restates hear/ckks/engine.py (keygen, raised-modulus encryption, decrypt
with exact CRT, tensor product + relinearisation, Galois rotations with
per-prime digits and one special prime, hoisting, exact RNS rescale) on top
of the C kernels of oracle/ckks_ref.c, with the reference's numpy codec
(hear/ckks/encoder.py) and its numpy random draws in the same order.
Ring tables use the corrected inverse twiddles and Barrett constants.

Used only as the checker in tests/, for bench.py's cpu_baseline leg and
for `bench.py --impl reference`.  Payloads are (c0, c1) uint64 numpy pairs
of shape (level+1, N), exactly the reference's format.
"""

from __future__ import annotations

import ctypes
import os

import numpy as np

from paper_2104_09164_b200.backend import BackendBase, Ct, LevelScaleError, Pt
from paper_2104_09164_b200.ckks.ntheory import bit_reverse_table, root_2n

from .build import build

_LIB = None


def lib():
    global _LIB
    if _LIB is None:
        _LIB = ctypes.CDLL(build())
        vp, i32 = ctypes.c_void_p, ctypes.c_int
        _LIB.or_ntt_fwd.argtypes = [vp, i32, i32, vp, vp, vp, vp]
        _LIB.or_ntt_inv.argtypes = [vp, i32, i32, vp, vp, vp, vp, vp, vp]
        _LIB.or_pw_mul.argtypes = [vp, vp, vp, i32, i32, vp, vp, vp, vp]
        _LIB.or_pw_addsub.argtypes = [vp, vp, vp, i32, i32, vp, vp, i32]
        _LIB.or_scalar_mul.argtypes = [vp, vp, i32, i32, vp, vp, vp, vp]
        _LIB.or_pw_mul_accum_perm.argtypes = [vp] * 8 + [i32] * 4 + [vp] * 3
        _LIB.or_lift_center.argtypes = [vp, i32, ctypes.c_uint64, vp]
        _LIB.or_reduce_rows.argtypes = [vp, i32, vp, i32, vp, vp]
        _LIB.or_sub_scaled_inv.argtypes = [vp, vp, vp, i32, i32, vp, vp, vp, vp]
        _LIB.or_bconv.argtypes = [vp, i32, ctypes.c_int64, vp, vp, i32, vp, vp, i32, vp, vp, vp]
    return _LIB


def _p(a: np.ndarray) -> int:
    return a.ctypes.data


def _shoup(w, q):
    return np.array([(int(x) << 64) // q for x in w], dtype=np.uint64)


class OracleRing:
    """Tables of hear/ckks/ring.py:253-292 (corrected) + C kernel wrappers."""

    def __init__(self, params):
        self.params = params
        self.n = params.n
        self.logn = self.n.bit_length() - 1
        self.primes = list(params.chain_primes) + [params.special_prime]
        self.special_idx = len(self.primes) - 1
        k = len(self.primes)
        self.p = np.array(self.primes, dtype=np.uint64)
        bits = [q.bit_length() for q in self.primes]
        self.sh = np.array([b - 1 for b in bits], dtype=np.uint64)
        self.mu = np.array([(1 << (63 + b)) // q for q, b in zip(self.primes, bits)],
                           dtype=np.uint64)
        brv = bit_reverse_table(self.logn)
        self.psi = np.zeros((k, self.n), dtype=np.uint64)
        self.psish = np.zeros_like(self.psi)
        self.ipsi = np.zeros_like(self.psi)
        self.ipsish = np.zeros_like(self.psi)
        self.ninv = np.zeros(k, dtype=np.uint64)
        self.ninvsh = np.zeros(k, dtype=np.uint64)
        for i, q in enumerate(self.primes):
            root = root_2n(q, 2 * self.n)
            rinv = pow(root, -1, q)
            pw = [pow(root, int(e), q) for e in brv]
            ipw = [pow(rinv, int(e), q) for e in brv]
            self.psi[i], self.ipsi[i] = pw, ipw
            self.psish[i], self.ipsish[i] = _shoup(pw, q), _shoup(ipw, q)
            ni = pow(self.n, -1, q)
            self.ninv[i], self.ninvsh[i] = ni, (ni << 64) // q
        self.exp_map = 2 * brv + 1
        self._perm: dict = {}

    @staticmethod
    def _g(gidx):
        return np.ascontiguousarray(gidx, dtype=np.int64)

    def fwd(self, rows, gidx):
        g = self._g(gidx)
        lib().or_ntt_fwd(_p(rows), rows.shape[0], self.n, _p(g), _p(self.psi), _p(self.psish),
                         _p(self.p))

    def inv(self, rows, gidx):
        g = self._g(gidx)
        lib().or_ntt_inv(_p(rows), rows.shape[0], self.n, _p(g), _p(self.ipsi), _p(self.ipsish),
                         _p(self.p), _p(self.ninv), _p(self.ninvsh))

    def mul(self, a, b, gidx):
        a, b = np.ascontiguousarray(a), np.ascontiguousarray(b)
        out = np.empty_like(a)
        g = self._g(gidx)
        lib().or_pw_mul(_p(out), _p(a), _p(b), a.shape[0], self.n, _p(g), _p(self.p),
                        _p(self.mu), _p(self.sh))
        return out

    def _addsub(self, a, b, gidx, sub):
        a, b = np.ascontiguousarray(a), np.ascontiguousarray(b)
        out = np.empty_like(a)
        g = self._g(gidx)
        lib().or_pw_addsub(_p(out), _p(a), _p(b), a.shape[0], self.n, _p(g), _p(self.p), sub)
        return out

    def add(self, a, b, gidx):
        return self._addsub(a, b, gidx, 0)

    def sub(self, a, b, gidx):
        return self._addsub(a, b, gidx, 1)

    def scalar_mul(self, a, c, gidx):
        c = np.ascontiguousarray(c, dtype=np.uint64)
        g = self._g(gidx)
        lib().or_scalar_mul(_p(a), _p(c), a.shape[0], self.n, _p(g), _p(self.p), _p(self.mu),
                            _p(self.sh))

    def reduce_rows(self, coeffs, gidx):
        c = np.ascontiguousarray(coeffs, dtype=np.int64)
        g = self._g(gidx)
        out = np.empty((len(g), self.n), dtype=np.uint64)
        lib().or_reduce_rows(_p(c), self.n, _p(g), len(g), _p(self.p), _p(out))
        return out

    def lift_center(self, x, q):
        x = np.ascontiguousarray(x)
        out = np.empty(self.n, dtype=np.int64)
        lib().or_lift_center(_p(x), self.n, q, _p(out))
        return out

    def galois_element(self, r):
        return pow(5, r % (self.n // 2), 2 * self.n)

    def ntt_perm(self, g):
        if g not in self._perm:
            two_n = 2 * self.n
            pos = np.full(two_n, -1, dtype=np.int64)
            pos[self.exp_map] = np.arange(self.n)
            self._perm[g] = pos[(self.exp_map * g) % two_n].astype(np.int64)
        return self._perm[g]

    def coeff_automorphism(self, coeffs, g):
        k = np.arange(self.n, dtype=np.int64)
        e = (k * g) % (2 * self.n)
        out = np.zeros_like(coeffs)
        out[e % self.n] = np.where(e >= self.n, -coeffs, coeffs)
        return out


class _Ksk:
    def __init__(self, b, a, lmax):
        self.b, self.a, self.lmax = b, a, lmax


class OracleKeys:
    def __init__(self):
        self.s_coeffs = self.s_ntt = self.pk_b = self.pk_a = self.relin = None
        self.rot: dict = {}


class OracleCkks(BackendBase):
    """CPU port of hear/ckks/engine.py:48-361."""

    exact = False

    def __init__(self, params, seed: int = 0):
        super().__init__(params)
        self.ring = OracleRing(params)
        self.rng = np.random.default_rng(seed)
        self.n = params.n
        self.L = params.max_level
        self.S = self.ring.special_idx
        self.P = params.special_prime
        chain = params.chain_primes
        self._pmod = np.array([self.P % q for q in chain], dtype=np.uint64)
        self._pinv = np.array([pow(self.P, -1, q) for q in chain], dtype=np.uint64)
        self._resc_inv = [np.array([pow(chain[l], -1, chain[j]) for j in range(l)], dtype=np.uint64)
                          for l in range(self.L + 1)]
        two_n = 2 * self.n
        g = np.empty(self.n // 2, dtype=np.int64)
        cur = 1
        for j in range(self.n // 2):
            g[j] = cur
            cur = cur * 5 % two_n
        self._rot_group, self._conj_group = g, (two_n - g) % two_n
        self.keys = OracleKeys()
        self._keygen()

    # ---- sampling (engine.py:77-99) ----
    def _ternary(self):
        return self.rng.integers(-1, 2, self.n).astype(np.int64)

    def _gauss(self):
        return np.rint(self.rng.normal(0.0, self.params.error_std, self.n)).astype(np.int64)

    def _uniform_rows(self, gidx):
        out = np.empty((len(gidx), self.n), dtype=np.uint64)
        for r, g in enumerate(gidx):
            out[r] = self.rng.integers(0, self.ring.primes[g], self.n, dtype=np.uint64)
        return out

    def _full_gidx(self, lmax=None):
        return list(range((self.L if lmax is None else lmax) + 1)) + [self.S]

    def _coeffs_to_ntt(self, coeffs, gidx):
        out = self.ring.reduce_rows(coeffs, gidx)
        self.ring.fwd(out, gidx)
        return out

    # ---- keygen (engine.py:101-147) ----
    def _keygen(self):
        k = self.keys
        gidx = self._full_gidx()
        k.s_coeffs = self._ternary()
        k.s_ntt = self._coeffs_to_ntt(k.s_coeffs, gidx)
        k.pk_a = self._uniform_rows(gidx)
        e = self._coeffs_to_ntt(self._gauss(), gidx)
        k.pk_b = self.ring.sub(e, self.ring.mul(k.pk_a, k.s_ntt, gidx), gidx)
        k.relin = self._make_ksk(self.ring.mul(k.s_ntt, k.s_ntt, gidx), self.L)

    def _make_ksk(self, target, lmax):
        gidx = self._full_gidx(lmax)
        ndig = lmax + 1
        kb = np.empty((ndig, len(gidx), self.n), dtype=np.uint64)
        ka = np.empty_like(kb)
        s = self.keys.s_ntt[[*range(lmax + 1), -1]]
        for i in range(ndig):
            a = self._uniform_rows(gidx)
            e = self._coeffs_to_ntt(self._gauss(), gidx)
            b = self.ring.sub(e, self.ring.mul(a, s, gidx), gidx)
            prod = target[i:i + 1].copy()
            self.ring.scalar_mul(prod, self._pmod[i:i + 1], [i])
            b[i] = self.ring.add(b[i:i + 1], prod, [i])[0]
            kb[i], ka[i] = b, a
        return _Ksk(kb, ka, lmax)

    def ensure_rotation_keys(self, rot_levels):
        for amount, lmax in sorted(rot_levels.items()):
            amount %= self.n2
            if amount == 0:
                continue
            have = self.keys.rot.get(amount)
            if have is not None and have.lmax >= lmax:
                continue
            g = self.ring.galois_element(amount)
            target = self._coeffs_to_ntt(self.ring.coeff_automorphism(self.keys.s_coeffs, g),
                                         self._full_gidx(lmax))
            self.keys.rot[amount] = self._make_ksk(target, lmax)

    # ---- codec (encoder.py) ----
    def _encode_coeffs(self, values, scale):
        spec = np.zeros(2 * self.n, dtype=np.complex128)
        spec[self._rot_group] = values
        spec[self._conj_group] = np.conj(values)
        coeffs = np.fft.fft(spec)[:self.n].real / self.n * float(scale)
        if np.abs(coeffs).max() >= float(1 << 52):
            raise ValueError("encoded coefficient magnitude exceeds 2^52")
        return np.rint(coeffs).astype(np.int64)

    def _raw_encode(self, values, level, scale):
        rows = self._coeffs_to_ntt(self._encode_coeffs(values, scale), list(range(level + 1)))
        return Pt(rows, level, scale, self.n2)

    def _decrypt_coeffs(self, ct, keep):
        c0, c1 = ct.payload
        gidx = list(range(keep))
        m = self.ring.add(self.ring.mul(c1[:keep], self.keys.s_ntt[:keep], gidx), c0[:keep], gidx)
        self.ring.inv(m, gidx)
        primes = [self.params.chain_primes[j] for j in range(keep)]
        q = 1
        for p in primes:
            q *= p
        recon = np.zeros(self.n, dtype=object)
        for j, p in enumerate(primes):
            qi = q // p
            recon += m[j].astype(object) * (qi * pow(qi, -1, p))
        recon %= q
        return np.array([float(v - q) if v > q // 2 else float(v) for v in recon])

    def _rows_needed(self, scale):
        need = max(np.log2(float(scale)), 0.0) + 40
        bits = 0.0
        for k, p in enumerate(self.params.chain_primes):
            bits += np.log2(p)
            if bits >= need:
                return k + 1
        return self.L + 1

    def _raw_dec(self, ct):
        keep = min(ct.level + 1, self._rows_needed(ct.scale))
        coeffs = self._decrypt_coeffs(ct, keep)
        buf = np.zeros(2 * self.n)
        buf[:self.n] = coeffs
        return (np.fft.ifft(buf) * (2 * self.n))[self._rot_group].real / float(ct.scale)

    # ---- encryption (engine.py:194-227) ----
    def _raw_enc(self, values, level, scale):
        if np.ndim(values) != 1:
            raise ValueError("the CPU oracle encrypts one clip per call")
        rows = list(range(level + 1))
        gidx = rows + [self.S]
        m = self._raw_encode(values, level, scale).payload
        u = self._coeffs_to_ntt(self._ternary(), gidx)
        e0 = self._coeffs_to_ntt(self._gauss(), gidx)
        e1 = self._coeffs_to_ntt(self._gauss(), gidx)
        sel = rows + [self.L + 1]
        c0 = self.ring.add(self.ring.mul(u, self.keys.pk_b[sel], gidx), e0, gidx)
        c1 = self.ring.add(self.ring.mul(u, self.keys.pk_a[sel], gidx), e1, gidx)
        pm = m.copy()
        self.ring.scalar_mul(pm, self._pmod[:level + 1], rows)
        c0[:level + 1] = self.ring.add(c0[:level + 1], pm, rows)
        return Ct((self._drop_special(c0, level), self._drop_special(c1, level)), level, scale,
                  self.n2)

    def _scaled_drop(self, rows_in, src_row, src_prime_idx, targets, inv):
        """(rows - [x]_src lifted) * inv over `targets` (ModDown / rescale core)."""
        xs = src_row[None].copy()
        self.ring.inv(xs, [src_prime_idx])
        lifted = self.ring.lift_center(xs[0], self.ring.primes[src_prime_idx])
        corr = self.ring.reduce_rows(lifted, targets)
        self.ring.fwd(corr, targets)
        out = np.ascontiguousarray(rows_in).copy()
        g = np.asarray(targets, dtype=np.int64)
        lib().or_sub_scaled_inv(_p(out), _p(corr), _p(np.ascontiguousarray(inv)), len(g), self.n,
                                _p(g), _p(self.ring.p), _p(self.ring.mu), _p(self.ring.sh))
        return out

    def _drop_special(self, rows_sp, level):
        return self._scaled_drop(rows_sp[:level + 1], rows_sp[-1], self.S,
                                 list(range(level + 1)), self._pinv[:level + 1])

    # ---- arithmetic (engine.py:231-286) ----
    def _raw_add(self, a, b):
        g = list(range(a.level + 1))
        return Ct((self.ring.add(a.payload[0], b.payload[0], g),
                   self.ring.add(a.payload[1], b.payload[1], g)), a.level, a.scale, self.n2)

    def _raw_add_plain(self, a, p):
        g = list(range(a.level + 1))
        return Ct((self.ring.add(a.payload[0], p.payload[:a.level + 1], g), a.payload[1].copy()),
                  a.level, a.scale, self.n2)

    def _raw_mult_plain(self, a, p):
        g = list(range(a.level + 1))
        rows = p.payload[:a.level + 1]
        return Ct((self.ring.mul(a.payload[0], rows, g), self.ring.mul(a.payload[1], rows, g)),
                  a.level, a.scale * p.scale, self.n2)

    def _raw_mult(self, a, b):
        lvl = a.level
        g = list(range(lvl + 1))
        a0, a1 = a.payload
        b0, b1 = b.payload
        d0 = self.ring.mul(a0, b0, g)
        d1 = self.ring.add(self.ring.mul(a0, b1, g), self.ring.mul(a1, b0, g), g)
        d2 = self.ring.mul(a1, b1, g)
        ks0, ks1 = self._ks_apply(self._decompose(d2, lvl), self.keys.relin, lvl, None)
        return Ct((self.ring.add(d0, ks0, g), self.ring.add(d1, ks1, g)), lvl,
                  a.scale * b.scale, self.n2)

    def _raw_rescale(self, a):
        lvl = a.level
        out = [self._scaled_drop(poly[:lvl], poly[lvl], lvl, list(range(lvl)), self._resc_inv[lvl])
               for poly in a.payload]
        return Ct((out[0], out[1]), lvl - 1, a.scale / self.params.chain_primes[lvl], self.n2)

    def _raw_mod_down(self, a, to_level):
        return Ct((a.payload[0][:to_level + 1].copy(), a.payload[1][:to_level + 1].copy()),
                  to_level, a.scale, self.n2)

    # ---- key switching (engine.py:290-361) ----
    def _decompose(self, d, lvl):
        ndig, rows = lvl + 1, lvl + 2
        gidx = list(range(lvl + 1)) + [self.S]
        coeffs = np.ascontiguousarray(d).copy()
        self.ring.inv(coeffs, list(range(lvl + 1)))
        de = np.empty((ndig, rows, self.n), dtype=np.uint64)
        for i in range(ndig):
            lifted = self.ring.lift_center(coeffs[i], self.params.chain_primes[i])
            de[i] = self._coeffs_to_ntt(lifted, gidx)
        return de

    def _ks_apply(self, de, key, lvl, perm):
        ndig, rows = lvl + 1, lvl + 2
        if key.lmax < lvl:
            raise LevelScaleError(f"key switching key trimmed to level {key.lmax}, need {lvl}")
        gidx = np.array(list(range(lvl + 1)) + [self.S], dtype=np.int64)
        perm = np.arange(self.n, dtype=np.int64) if perm is None else perm
        outb = np.zeros((rows, self.n), dtype=np.uint64)
        outa = np.zeros_like(outb)
        krow = np.array(list(range(lvl + 1)) + [key.lmax + 1], dtype=np.int64)
        kb, ka = np.ascontiguousarray(key.b[:ndig]), np.ascontiguousarray(key.a[:ndig])
        de = np.ascontiguousarray(de)
        lib().or_pw_mul_accum_perm(_p(outb), _p(outa), _p(de), _p(kb), _p(ka), _p(krow), _p(perm),
                                   _p(gidx), ndig, rows, key.b.shape[1], self.n, _p(self.ring.p),
                                   _p(self.ring.mu), _p(self.ring.sh))
        return self._drop_special(outb, lvl), self._drop_special(outa, lvl)

    def _rot_key(self, amount):
        key = self.keys.rot.get(amount % self.n2)
        if key is None:
            raise KeyError(f"no rotation key for amount {amount % self.n2}")
        return key

    def _apply_rot(self, a, k, de=None):
        lvl = a.level
        perm = self.ring.ntt_perm(self.ring.galois_element(k))
        if de is None:
            de = self._decompose(a.payload[1], lvl)
        ks0, ks1 = self._ks_apply(de, self._rot_key(k), lvl, perm)
        c0 = self.ring.add(np.ascontiguousarray(a.payload[0][:, perm]), ks0, list(range(lvl + 1)))
        return Ct((c0, ks1), lvl, a.scale, self.n2)

    def _raw_rot(self, a, k):
        return self._apply_rot(a, k)

    def _raw_rot_many(self, a, ks):
        if not ks:
            return {}
        de = self._decompose(a.payload[1], a.level)
        return {k: self._apply_rot(a, k, de=de) for k in ks}

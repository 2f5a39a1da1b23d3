"""Hybrid (dnum-digit) RNS key switching -- TEST INFRASTRUCTURE ONLY.

CPU restatement of the standard hybrid key-switching algorithm used for
BASELINE config 1 (dnum = 3): the reference package has no counterpart (it
switches keys with per-prime digits and one special prime,
hear/ckks/engine.py:290-326), so parity is pinned on this restatement of
the published algorithm:

  * the chain q_0..q_L is split into dnum digits of alpha = ceil((L+1)/dnum)
    consecutive primes; k special primes P = p_0..p_{k-1} extend the basis;
  * key for target s': per digit j, b_j = -a_j s + e_j + P * [Q/Q_j]
    * [(Q/Q_j)^-1]_{Q_j} * s'  -- in RNS: P mod q_i on the rows of digit j's
    primes, 0 on every other row;
  * ModUp of digit j: fast base conversion of its residues (coefficient
    form) to every other prime of Q_l + P, then forward NTT;
  * inner product over the digits, Galois permutation applied to the
    extended digits for rotations (hoisting);
  * ModDown: fast base conversion of the special rows to Q_l,
    out = (x - conv) * P^-1 mod q_i.

All arithmetic is the C oracle's (oracle/ckks_ref.c: NTTs, Barrett
products, or_bconv).  Never imported by the product path.
"""

from __future__ import annotations

import numpy as np

from .cpu_engine import OracleRing, _p, lib


class _Shim:
    """Parameter view whose prime list is chain + special primes."""

    def __init__(self, n, chain, specials):
        self.n = n
        self.chain_primes = tuple(chain) + tuple(specials[:-1])
        self.special_prime = specials[-1]


def bconv_tables(primes, src, dst):
    """(qhat_inv [s], qhat_mod [s][t]) of the conversion src -> dst (global
    prime indices), in Python integers."""
    qs = [primes[i] for i in src]
    inv, mod = [], []
    for a, q in enumerate(qs):
        qhat = 1
        for b, q2 in enumerate(qs):
            if b != a:
                qhat *= q2
        inv.append(pow(qhat % q, -1, q))
        mod.append([qhat % primes[t] for t in dst])
    return np.array(inv, dtype=np.uint64), np.array(mod, dtype=np.uint64).reshape(len(src), len(dst))


class HybridOracle:
    def __init__(self, params, s_coeffs, dnum: int, special_primes, seed: int = 0):
        self.n = params.n
        self.chain = list(params.chain_primes)
        self.L = len(self.chain) - 1
        self.sp = [int(p) for p in special_primes]
        self.k = len(self.sp)
        self.primes = self.chain + self.sp
        self.ring = OracleRing(_Shim(self.n, self.chain, self.sp))
        self.alpha = -(-(self.L + 1) // dnum)
        self.digits = [list(range(j * self.alpha, min((j + 1) * self.alpha, self.L + 1)))
                       for j in range(dnum)]
        self.P = 1
        for p in self.sp:
            self.P *= p
        self.rng = np.random.default_rng(seed)
        self.s_coeffs = np.asarray(s_coeffs, dtype=np.int64)
        self.all_rows = list(range(len(self.primes)))
        self.s_ntt = self._to_ntt(self.s_coeffs, self.all_rows)
        self.relin = self.make_key(self.ring.mul(self.s_ntt, self.s_ntt, self.all_rows))
        self.rot_keys: dict = {}

    def _to_ntt(self, coeffs, gidx):
        out = self.ring.reduce_rows(coeffs, gidx)
        self.ring.fwd(out, gidx)
        return out

    def specials(self):
        return list(range(self.L + 1, self.L + 1 + self.k))

    def make_key(self, target):
        """[dnum] (b, a) over all L+1+k primes; target in NTT form."""
        rows = self.all_rows
        kb = np.empty((len(self.digits), len(rows), self.n), dtype=np.uint64)
        ka = np.empty_like(kb)
        for j, dig in enumerate(self.digits):
            a = np.stack([self.rng.integers(0, self.primes[g], self.n, dtype=np.uint64)
                          for g in rows])
            e = self._to_ntt(np.rint(self.rng.normal(0.0, 3.2, self.n)).astype(np.int64), rows)
            b = self.ring.sub(e, self.ring.mul(a, self.s_ntt, rows), rows)
            pm = np.array([self.P % self.primes[i] for i in dig], dtype=np.uint64)
            gadget = target[dig].copy()
            self.ring.scalar_mul(gadget, pm, dig)
            b[dig] = self.ring.add(b[dig], gadget, dig)
            kb[j], ka[j] = b, a
        return kb, ka

    def ensure_rotation_key(self, amount: int):
        amount %= self.n // 2
        if amount and amount not in self.rot_keys:
            g = self.ring.galois_element(amount)
            tgt = self._to_ntt(self.ring.coeff_automorphism(self.s_coeffs, g), self.all_rows)
            self.rot_keys[amount] = self.make_key(tgt)

    def _bconv(self, src_rows, src, dst):
        """src_rows [s, N] coefficient residues -> [t, N]."""
        inv, mod = bconv_tables(self.primes, src, dst)
        src_rows = np.ascontiguousarray(src_rows)
        out = np.empty((len(dst), self.n), dtype=np.uint64)
        sp, tp = np.array(src, dtype=np.int64), np.array(dst, dtype=np.int64)
        off = np.arange(len(dst), dtype=np.int64) * self.n
        lib().or_bconv(_p(src_rows), len(src), self.n, _p(sp), _p(out), len(dst), _p(off),
                       _p(tp), self.n, _p(self.ring.p), _p(inv), _p(np.ascontiguousarray(mod)))
        return out

    def ext_rows(self, lvl):
        return list(range(lvl + 1)) + self.specials()

    def modup(self, d, lvl):
        """d [l+1, N] NTT form -> [nd, l+1+k, N] extended digits (NTT form)."""
        rows = self.ext_rows(lvl)
        coef = d.copy()
        self.ring.inv(coef, list(range(lvl + 1)))
        out = []
        for dig in self.digits:
            dig = [i for i in dig if i <= lvl]
            if not dig:
                continue
            ext = np.empty((len(rows), self.n), dtype=np.uint64)
            tgt = [g for g in rows if g not in dig]
            conv = self._bconv(coef[dig], dig, tgt)
            self.ring.fwd(conv, tgt)
            for r, g in enumerate(rows):
                ext[r] = d[g] if g in dig else conv[tgt.index(g)]
            out.append(ext)
        return np.stack(out)

    def inner(self, ext, key, lvl, perm=None):
        """sum_j perm(ext_j) * key_j over the rows of Q_l + P -> (b, a)."""
        rows = self.ext_rows(lvl)
        kb, ka = key
        krow = rows   # keys hold every prime: global index == key row
        ob = np.zeros((len(rows), self.n), dtype=np.uint64)
        oa = np.zeros_like(ob)
        de = np.ascontiguousarray(ext)
        idx = np.arange(self.n, dtype=np.int64) if perm is None else np.asarray(perm, np.int64)
        lib().or_pw_mul_accum_perm(_p(ob), _p(oa), _p(de), _p(np.ascontiguousarray(kb)),
                                   _p(np.ascontiguousarray(ka)), _p(np.array(krow, np.int64)),
                                   _p(idx), _p(np.array(rows, np.int64)), de.shape[0], len(rows),
                                   kb.shape[1], self.n, _p(self.ring.p), _p(self.ring.mu),
                                   _p(self.ring.sh))
        return ob, oa

    def moddown(self, x, lvl):
        """x [l+1+k, N] NTT form over Q_l + P -> [l+1, N] = (x - conv(x_P)) / P."""
        chain = list(range(lvl + 1))
        sp = self.specials()
        xs = x[lvl + 1:].copy()
        self.ring.inv(xs, sp)
        conv = self._bconv(xs, sp, chain)
        self.ring.fwd(conv, chain)
        out = x[:lvl + 1].copy()
        pinv = np.array([pow(self.P % q, -1, q) for q in self.chain[:lvl + 1]], dtype=np.uint64)
        g = np.array(chain, dtype=np.int64)
        lib().or_sub_scaled_inv(_p(out), _p(conv), _p(pinv), len(chain), self.n, _p(g),
                                _p(self.ring.p), _p(self.ring.mu), _p(self.ring.sh))
        return out

    def mult(self, a, b, lvl):
        """Tensor product + hybrid relinearisation of (c0, c1) x (d0, d1)."""
        rows = list(range(lvl + 1))
        m = self.ring.mul
        d0 = m(a[0], b[0], rows)
        d1 = self.ring.add(m(a[0], b[1], rows), m(a[1], b[0], rows), rows)
        d2 = m(a[1], b[1], rows)
        ib, ia = self.inner(self.modup(d2, lvl), self.relin, lvl)
        return (self.ring.add(d0, self.moddown(ib, lvl), rows),
                self.ring.add(d1, self.moddown(ia, lvl), rows))

    def rot(self, a, lvl, amount):
        self.ensure_rotation_key(amount)
        g = self.ring.galois_element(amount)
        perm = self.ring.ntt_perm(g)
        rows = list(range(lvl + 1))
        ib, ia = self.inner(self.modup(a[1], lvl), self.rot_keys[amount % (self.n // 2)], lvl, perm)
        return (self.ring.add(a[0][:, perm], self.moddown(ib, lvl), rows), self.moddown(ia, lvl))

"""Hybrid key switching with dnum digits and k special primes (BASELINE
config 1: N = 2^16, 24 x 50-bit chain primes, dnum = 3).

The reference switches keys with per-prime digits and one special prime
(hear/ckks/engine.py:290-326; this package's CkksBackend reproduces it
bit-exactly).  The hybrid generalisation groups the chain into dnum digits
of alpha = ceil((L+1)/dnum) consecutive primes and extends the basis by k
special primes P = p_0..p_{k-1}:

  key (target s')   per digit j: b_j = -a_j s + e_j + [P on digit j's rows] s'
  ModUp             INTT -> centred fast base conversion of the digit's
                    residues to every other prime of Q_l + P (csrc/bconv.cu)
                    -> NTT; the digit's own rows are the input rows
  inner product     sum_j perm(ext_j) * key_j on every row of Q_l + P
                    (ks_inner2 kernel: Galois gather on the digits = hoisting)
  ModDown           INTT of the k special rows -> base conversion to Q_l ->
                    NTT -> (x - conv) * P^-1 (one element-wise launch)

Shared by relinearisation and rotation exactly like the engine's own key
switch; results are ordinary chain ciphertexts of the engine (CtData), so
rescale / add / decrypt are the engine's.  With dnum = L+1 and one special
prime the centred conversions are the reference's exact centred lifts.
The CPU restatement it is pinned to is oracle/hybrid_ref.py.

Keys are drawn from this object's own generator (never the engine's
reference-order stream): per digit, one uniform row per prime of the full
basis (chain then special primes), then one Gaussian error polynomial.
"""

from __future__ import annotations

import numpy as np
import torch

from .. import _native as nat
from ..backend import Ct
from .engine import CtData, _tasks
from .ring import RingContext, _upload, shoup_np


class _BasisView:
    """Parameter view for RingContext whose prime list is chain + specials."""

    def __init__(self, n, chain, specials):
        self.n = n
        self.chain_primes = tuple(chain) + tuple(specials[:-1])
        self.special_prime = specials[-1]


class HybridKeySwitch:
    def __init__(self, backend, dnum: int, special_primes, seed: int = 0):
        be = backend
        self.be = be
        self.n = be.n
        self.chain = list(be.params.chain_primes)
        self.L = len(self.chain) - 1
        self.sp = [int(p) for p in special_primes]
        self.k = len(self.sp)
        if not 1 <= dnum <= self.L + 1:
            raise ValueError(f"dnum must be in 1..{self.L + 1}")
        self.primes = self.chain + self.sp
        self.alpha = -(-(self.L + 1) // dnum)
        self.digits = [list(range(j * self.alpha, min((j + 1) * self.alpha, self.L + 1)))
                       for j in range(dnum)]
        self.digits = [d for d in self.digits if d]
        self.dnum = len(self.digits)
        if self.alpha > 32 or self.k > 32:
            raise ValueError("a base conversion source basis holds at most 32 primes")
        self.ring = RingContext(_BasisView(self.n, self.chain, self.sp), be.dev)
        self.dev = be.dev
        self.P = 1
        for p in self.sp:
            self.P *= p
        self.rng = np.random.default_rng(seed)
        self._tab: dict = {}
        pinv = np.array([pow(self.P % q, -1, q) for q in self.chain], dtype=np.uint64)
        self._pinv = pinv
        self._pinv_sh = shoup_np(pinv, np.array(self.chain, dtype=np.uint64))
        self.rot_keys: dict = {}
        self.relin = None
        if be.keys.s_coeffs is not None:
            self.s_ntt = self._to_ntt(be.keys.s_coeffs, self.all_rows)
            sq = self.ring.empty(len(self.all_rows))
            rp = self.ring.row_ptrs
            self._ew(nat.EW_MUL, rp(sq), rp(self.s_ntt), self.all_rows, b=rp(self.s_ntt))
            self.relin = self.make_key(sq)

    # ---- helpers ---------------------------------------------------------------

    @property
    def all_rows(self) -> list:
        return list(range(len(self.primes)))

    def specials(self) -> list:
        return list(range(self.L + 1, self.L + 1 + self.k))

    def ext_rows(self, lvl: int) -> list:
        return list(range(lvl + 1)) + self.specials()

    def digits_at(self, lvl: int) -> list:
        return [[i for i in d if i <= lvl] for d in self.digits if d[0] <= lvl]

    def _ew(self, op, dst, a, primes, b=None, scal=None, scal_sh=None):
        f = dict(dst=dst, a=a, prime=np.asarray(primes))
        if b is not None:
            f["b"] = b
        if scal is not None:
            f["scal"], f["scal_sh"] = scal, scal_sh
        self.ring.ew(op, _tasks(nat.EW_TASK, len(dst), **f))

    def _to_ntt(self, coeffs: np.ndarray, gidx) -> torch.Tensor:
        c = torch.from_numpy(np.ascontiguousarray(coeffs, dtype=np.int64)).to(self.dev)[None]
        r = len(gidx)
        out = self.ring.empty(r)
        src = np.repeat(self.ring.row_ptrs(c), r)
        self.ring.ntt_fwd(_tasks(nat.NTT_TASK, r, src=src, dst=self.ring.row_ptrs(out),
                                 dst_prime=np.asarray(gidx), src_prime=np.asarray(gidx)),
                          nat.FWD_I64)
        return out

    def _table(self, src: tuple, dst: tuple) -> tuple:
        """Device conversion table + index arrays for src -> dst (global primes)."""
        key = (src, dst)
        if key not in self._tab:
            qs = [self.primes[i] for i in src]
            words = []
            mods = []
            for a, q in enumerate(qs):
                qhat = 1
                for b, q2 in enumerate(qs):
                    if b != a:
                        qhat *= q2
                inv = pow(qhat % q, -1, q)
                words += [inv, (inv << 64) // q]
                mods.append([qhat % self.primes[t] for t in dst])
            words += [m for row in mods for m in row]
            tab = torch.from_numpy(np.array(words, dtype=np.uint64).view(np.int64)).to(self.dev)
            sp = torch.tensor(src, dtype=torch.int32, device=self.dev)
            tp = torch.tensor(dst, dtype=torch.int32, device=self.dev)
            self._tab[key] = (tab, sp, tp)
        return self._tab[key]

    def _bconv(self, jobs):
        """jobs: [(src_row0_ptr, src tuple, dst_base_ptr, dst offsets (rows), dst tuple)]."""
        if not jobs:
            return
        t = np.zeros(len(jobs), dtype=nat.BCONV_TASK)
        for q, (src_ptr, src, dst_ptr, rows, dst) in enumerate(jobs):
            tab, sp, tp = self._table(tuple(src), tuple(dst))
            off = self._offsets(tuple(rows))
            t[q] = (src_ptr, dst_ptr, off.data_ptr(), tab.data_ptr(), sp.data_ptr(),
                    tp.data_ptr(), self.n, len(src), len(dst))
        # one launch per source count (the register-resident kernel variant)
        for ns in np.unique(t["s"]):
            sub = t[t["s"] == ns]
            for c0 in range(0, len(sub), 65535):
                d = _upload(sub[c0:c0 + 65535], self.dev)
                nat.check(nat.lib().hb_bconv(self.ring.handle, d.data_ptr(),
                                             len(sub[c0:c0 + 65535]), int(ns), self.ring.stream),
                          "bconv")

    def _offsets(self, rows: tuple) -> torch.Tensor:
        key = ("off", rows)
        if key not in self._tab:
            self._tab[key] = torch.tensor(np.asarray(rows, dtype=np.int64) * self.n,
                                          device=self.dev)
        return self._tab[key]

    # ---- keys ------------------------------------------------------------------

    def make_key(self, target: torch.Tensor):
        """(b, a) [dnum, L+1+k, N] encrypting P * target on each digit's rows."""
        rows = self.all_rows
        nd = len(self.digits)
        kb = self.ring.empty(nd, len(rows))
        ka = self.ring.empty(nd, len(rows))
        rp = self.ring.row_ptrs
        pmod = np.array([self.P % q for q in self.chain], dtype=np.uint64)
        pmod_sh = shoup_np(pmod, np.array(self.chain, dtype=np.uint64))
        for j, dig in enumerate(self.digits):
            a = np.stack([self.rng.integers(0, self.primes[g], self.n, dtype=np.uint64)
                          for g in rows])
            e = self._to_ntt(np.rint(self.rng.normal(0.0, 3.2, self.n)).astype(np.int64), rows)
            ka[j].copy_(torch.from_numpy(a.view(np.int64)).to(self.dev))
            t = self.ring.empty(len(rows))
            self._ew(nat.EW_MUL, rp(t), rp(ka[j]), rows, b=rp(self.s_ntt))
            self._ew(nat.EW_SUB, rp(kb[j]), rp(e), rows, b=rp(t))
            dr = rp(kb[j])[dig]
            self._ew(nat.EW_ADD_SCALED, dr, dr, dig, b=rp(target)[dig],
                     scal=pmod[dig], scal_sh=pmod_sh[dig])
        return kb, ka

    def ensure_rotation_keys(self, amounts):
        for amount in sorted({int(a) % (self.n // 2) for a in amounts}):
            if amount == 0 or amount in self.rot_keys:
                continue
            g = self.ring.galois_element(amount)
            sg = self.ring.coeff_automorphism(self.be.keys.s_coeffs, g)
            self.rot_keys[amount] = self.make_key(self._to_ntt(sg, self.all_rows))

    # ---- ModUp / inner product / ModDown ------------------------------------------

    def modup(self, ptrs: np.ndarray, lvl: int) -> torch.Tensor:
        """Input rows [B, l+1] (uint64 row pointers, NTT form) -> extended
        digits [B, nd, l+1+k, N] (NTT form)."""
        ptrs = np.asarray(ptrs, dtype=np.uint64)
        bsz = ptrs.shape[0]
        rows = self.ext_rows(lvl)
        digs = self.digits_at(lvl)
        nd, nr = len(digs), len(rows)
        rp = self.ring.row_ptrs
        coef = self.ring.empty(bsz, lvl + 1)
        prim = np.tile(np.arange(lvl + 1), bsz)
        self.ring.ntt_inv(_tasks(nat.NTT_TASK, bsz * (lvl + 1), src=ptrs.ravel(), dst=rp(coef),
                                 dst_prime=prim, src_prime=prim))
        ext = self.ring.empty(bsz, nd, nr)
        er = rp(ext).reshape(bsz, nd, nr)
        cr = rp(coef).reshape(bsz, lvl + 1)
        cp_dst, cp_src, cp_pr = [], [], []
        jobs = []
        fwd_dst, fwd_pr = [], []
        for b in range(bsz):
            for j, dig in enumerate(digs):
                tgt = [g for g in rows if g not in dig]
                tpos = [rows.index(g) for g in tgt]
                for i in dig:
                    cp_dst.append(er[b, j, rows.index(i)])
                    cp_src.append(ptrs[b, i])
                    cp_pr.append(i)
                jobs.append((cr[b, dig[0]], dig, er[b, j, 0], tpos, tgt))
                fwd_dst += [er[b, j, p] for p in tpos]
                fwd_pr += tgt
        self._ew(nat.EW_COPY, np.array(cp_dst, dtype=np.uint64),
                 np.array(cp_src, dtype=np.uint64), cp_pr)
        self._bconv(jobs)
        fd = np.array(fwd_dst, dtype=np.uint64)
        self.ring.ntt_fwd(_tasks(nat.NTT_TASK, len(fd), src=fd, dst=fd,
                                 dst_prime=np.array(fwd_pr), src_prime=np.array(fwd_pr)))
        return ext

    def inner(self, ext: torch.Tensor, keys, lvl: int, perms=None) -> torch.Tensor:
        """[J, B, 2, l+1+k, N]: per job j, sum_d perm_j(ext_d) * key_j[d] on
        every extended row (perms[j]: int32 device perm or None)."""
        bsz, nd, nr = ext.shape[0], ext.shape[1], ext.shape[2]
        rows = self.ext_rows(lvl)
        out = self.ring.empty(len(keys), bsz, 2, nr)
        rp = self.ring.row_ptrs
        orr = rp(out).reshape(len(keys), bsz, 2, nr)
        de0 = rp(ext).reshape(bsz, nd, nr)[0, 0]
        tasks = []
        for j, (kb, ka) in enumerate(keys):
            kbr = rp(kb).reshape(kb.shape[0], kb.shape[1])[0]
            kar = rp(ka).reshape(ka.shape[0], ka.shape[1])[0]
            perm = 0 if perms is None or perms[j] is None else perms[j].data_ptr()
            tasks.append(_tasks(nat.KS_TASK2, nr, de=de0, kb=kbr[rows], ka=kar[rows],
                                out_b=orr[j, 0, 0], out_a=orr[j, 0, 1], perm=perm,
                                de_bstride=nd * nr * self.n, de_dstride=nr * self.n,
                                key_stride=kb.shape[1] * self.n, out_bstride=2 * nr * self.n,
                                ndig=nd, prime=np.array(rows)))
        self.ring.ks_inner2(np.concatenate(tasks), bsz)
        return out

    def moddown(self, x: torch.Tensor, lvl: int) -> torch.Tensor:
        """x [M, l+1+k, N] (NTT form over Q_l + P) -> [M, l+1, N] = (x - conv(x_P)) / P."""
        m, nr = x.shape[0], x.shape[1]
        rp = self.ring.row_ptrs
        xr = rp(x).reshape(m, nr)
        sp = self.specials()
        chain = list(range(lvl + 1))
        spc = self.ring.empty(m, self.k)
        spr = np.tile(np.array(sp), m)
        self.ring.ntt_inv(_tasks(nat.NTT_TASK, m * self.k, src=xr[:, lvl + 1:].ravel(),
                                 dst=rp(spc), dst_prime=spr, src_prime=spr))
        conv = self.ring.empty(m, lvl + 1)
        cr = rp(conv).reshape(m, lvl + 1)
        sr = rp(spc).reshape(m, self.k)
        self._bconv([(sr[q, 0], sp, cr[q, 0], chain, chain) for q in range(m)])
        cpr = np.tile(np.array(chain), m)
        self.ring.ntt_fwd(_tasks(nat.NTT_TASK, m * (lvl + 1), src=rp(conv), dst=rp(conv),
                                 dst_prime=cpr, src_prime=cpr))
        out = self.ring.empty(m, lvl + 1)
        self._ew(nat.EW_SUB_SCALED, rp(out), xr[:, :lvl + 1].ravel(), cpr, b=rp(conv),
                 scal=np.tile(self._pinv[:lvl + 1], m), scal_sh=np.tile(self._pinv_sh[:lvl + 1], m))
        return out

    # ---- ciphertext operations -------------------------------------------------

    def mult(self, a: Ct, b: Ct) -> Ct:
        """Tensor product (engine kernel) + hybrid relinearisation."""
        lvl = a.level
        if b.level != lvl:
            raise ValueError("mult level mismatch")
        x, y = a.payload.data, b.payload.data
        bsz, r = x.shape[0], lvl + 1
        rp = self.be.ring.row_ptrs
        d = self.ring.empty(bsz, 3, r)
        xr, yr, dr = rp(x).reshape(bsz, 2, r), rp(y).reshape(bsz, 2, r), rp(d).reshape(bsz, 3, r)
        self.ring.tensor(_tasks(nat.TENSOR_TASK, bsz * r, a0=xr[:, 0].ravel(),
                                a1=xr[:, 1].ravel(), b0=yr[:, 0].ravel(), b1=yr[:, 1].ravel(),
                                d0=dr[:, 0].ravel(), d1=dr[:, 1].ravel(), d2=dr[:, 2].ravel(),
                                prime=np.tile(np.arange(r), bsz)))
        ip = self.inner(self.modup(dr[:, 2], lvl), [self.relin], lvl)[0]
        md = self.moddown(ip.reshape(bsz * 2, -1, self.n), lvl).reshape(bsz, 2, r, self.n)
        out = self.ring.empty(bsz, 2, r)
        self._ew(nat.EW_ADD, rp(out), rp(md), np.tile(np.arange(r), 2 * bsz),
                 b=dr[:, :2].ravel())
        return Ct(CtData(out), lvl, a.scale * b.scale, self.be.n2)

    def rot_many(self, a: Ct, amounts) -> dict:
        """Hoisted rotations: one ModUp, one inner product per amount."""
        lvl = a.level
        amounts = sorted({int(k) % (self.n // 2) for k in amounts} - {0})
        x = a.payload.data
        bsz, r = x.shape[0], lvl + 1
        rp = self.be.ring.row_ptrs
        xr = rp(x).reshape(bsz, 2, r)
        ext = self.modup(xr[:, 1], lvl)
        keys, perms = [], []
        for k in amounts:
            if k not in self.rot_keys:
                raise KeyError(f"no hybrid rotation key for amount {k}")
            keys.append(self.rot_keys[k])
            perms.append(self.ring.perm_dev(self.ring.galois_element(k)))
        ip = self.inner(ext, keys, lvl, perms)
        nj = len(amounts)
        md = self.moddown(ip.reshape(nj * bsz * 2, -1, self.n), lvl)
        md = md.reshape(nj, bsz, 2, r, self.n)
        out = {0: a}
        for j, k in enumerate(amounts):
            res = self.ring.empty(bsz, 2, r)
            rr = rp(res).reshape(bsz, 2, r)
            mr = rp(md[j]).reshape(bsz, 2, r)
            pp = np.full(bsz * r, perms[j].data_ptr(), dtype=np.uint64)
            # c0' = perm(c0) + ModDown(b), c1' = ModDown(a)
            self._ew(nat.EW_PERM, rr[:, 0].ravel(), xr[:, 0].ravel(), np.tile(np.arange(r), bsz),
                     b=pp)
            self._ew(nat.EW_ADD, rr[:, 0].ravel(), rr[:, 0].ravel(), np.tile(np.arange(r), bsz),
                     b=mr[:, 0].ravel())
            self._ew(nat.EW_COPY, rr[:, 1].ravel(), mr[:, 1].ravel(), np.tile(np.arange(r), bsz))
            out[k] = Ct(CtData(res), lvl, a.scale, self.be.n2)
        return out

    def rot(self, a: Ct, amount: int) -> Ct:
        k = int(amount) % (self.n // 2)
        return self.rot_many(a, [k])[k]

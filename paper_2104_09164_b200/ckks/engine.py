"""Leveled RNS-CKKS engine on the B200 -- drop-in for hear/ckks/engine.py.

Same parameter objects, same keygen / enc / evaluate / dec contract, same
randomness: every random polynomial is drawn from the host numpy generator in
exactly the reference's call order (engine.py:77-147, 194-211), so with equal
seeds the secret, public, relinearisation and rotation keys and every fresh
ciphertext are bit-identical to the reference's.  All arithmetic after the
draw runs in the CUDA kernels of csrc/ (NTT, ModUp/ModDown base conversion,
key-switch inner product with the Galois gather, rescale, codec).

Ciphertext payloads are `CtData`: one int64 tensor [B, 2, level+1, N] holding
B independent clips (rows ascending from q0, NTT form).  B = 1 reproduces the
reference exactly; B > 1 evaluates B clips with the same schedule and the
same key material in one set of kernel launches.

Key switching follows the reference design (engine.py:288-326): one special
prime P, per-prime digits (dnum = level+1); ModUp of a digit is the centred
lift of its residue re-reduced under every target prime, ModDown divides P
out with the centred special residue.  These are exact integer maps, so the
GPU results are the same residues the (fixed) reference computes.
"""

from __future__ import annotations

import os
from fractions import Fraction

import numpy as np
import torch

from .. import _native as nat
from ..backend import BackendBase, Ct, LevelScaleError, Pt
from .encoder import Embedding
from .params import ParameterSet
from .ring import RingContext, shoup_np


class MissingRotationKey(RuntimeError):
    pass


class CtData:
    """Device payload of a (batched) ciphertext: [B, 2, rows, N] int64."""

    __slots__ = ("data",)

    def __init__(self, data: torch.Tensor):
        self.data = data

    @property
    def batch(self) -> int:
        return self.data.shape[0]

    @property
    def rows(self) -> int:
        return self.data.shape[2]

    def __getitem__(self, i):
        """payload[0] / payload[1]: c0 / c1 rows (reference tuple access)."""
        t = self.data[:, i]
        return t[0] if self.batch == 1 else t

    def to_host(self):
        """(c0, c1) uint64 numpy arrays shaped like the reference payload."""
        h = self.data.cpu().numpy().view(np.uint64)
        if self.batch == 1:
            return h[0, 0].copy(), h[0, 1].copy()
        return h[:, 0].copy(), h[:, 1].copy()


class CtExt:
    """Rotated ciphertext left in the extended basis Q*P (ModDown deferred):
    [B, 2, level+2, N], special row last.  Produced by
    rot_many_each(lazy=True) and consumed only by mac_many, which divides P
    out once per accumulated output; it has no `.data`, so every other op
    fails loudly."""

    __slots__ = ("xdata",)

    def __init__(self, xdata: torch.Tensor):
        self.xdata = xdata

    @property
    def batch(self) -> int:
        return self.xdata.shape[0]


class _Digits:
    """Digits of a batch of polynomials before their expansion: the centred
    lifts in the coefficient domain (doubles, [nb, ndig, N]) and the NTT-form
    input rows they came from (pointers [nb, ndig]).  The fused key switch
    (csrc/ntt3.cu k_ks3) consumes this directly; `expand` materialises the
    [nb, ndig, ndig+1, N] expansion of the unfused path."""

    __slots__ = ("coef", "src", "lvl")

    def __init__(self, coef, src, lvl):
        self.coef, self.src, self.lvl = coef, src, lvl

    @property
    def shape(self):
        return (self.coef.shape[0],)


class _Ksk:
    __slots__ = ("b", "a", "lmax", "bp", "ap")

    def __init__(self, b, a, lmax):
        self.b = b          # [ndig, lmax+2, N] device (reference layout)
        self.a = a
        self.lmax = lmax
        # rotation keys only: columns pre-permuted by the inverse Galois
        # permutation, so the inner product needs no gather (see _ks_apply_many)
        self.bp = None
        self.ap = None


class KeyMaterial:
    def __init__(self):
        self.s_coeffs = None
        self.s_ntt = None   # [L+2, N] device, special row last
        self.pk_b = None
        self.pk_a = None
        self.relin = None
        self.rot: dict = {}


def key_layout(params: ParameterSet, manifest) -> list:
    """[(name, shape)] of the public evaluation material in key_tensors order
    (the reference's KeyMaterial, engine.py:27-36): public key rows, the
    relinearisation key and one key per rotation amount of the manifest
    [(amount, lmax)], digit-major [ndig, rows, N] with the special row last.
    Pure function of the parameters: receivers allocate from it."""
    n, L = params.n, params.max_level
    out = [("pk_b", (L + 2, n)), ("pk_a", (L + 2, n)),
           ("relin_b", (L + 1, L + 2, n)), ("relin_a", (L + 1, L + 2, n))]
    for amt, lmax in sorted(manifest):
        out += [(f"rot{amt}_b", (lmax + 1, lmax + 2, n)), (f"rot{amt}_a", (lmax + 1, lmax + 2, n))]
    return out


def _tasks(dtype, n, **fields) -> np.ndarray:
    t = np.zeros(n, dtype=dtype)
    for k, v in fields.items():
        t[k] = v
    return t


class CkksBackend(BackendBase):
    """GPU realisation of the backend contract (hear/ckks/engine.py:48)."""

    exact = False

    def __init__(self, params: ParameterSet, seed: int = 0, device=None, keygen: bool = True,
                 enc_seed=None):
        super().__init__(params)
        self.ring = RingContext(params, device)
        self.dev = self.ring.device
        self.emb = Embedding(params.n, self.dev)
        # keygen=True: one generator for keys then encryptions, in the
        # reference's draw order (bit-exact keys and ciphertexts).  A receiver
        # (keygen=False, keys replicated from another rank) must NOT replay
        # that stream -- its first ternary draw would be the sender's secret
        # key -- so it encrypts from its own stream: `enc_seed` (e.g. a
        # SeedSequence spawned per rank) or fresh OS entropy.
        if keygen:
            self.rng = np.random.default_rng(seed)
        else:
            self.rng = np.random.default_rng(enc_seed)
        self.n = params.n
        self.L = params.max_level
        self.S = self.ring.special_idx
        self.P = params.special_prime
        chain = params.chain_primes
        self._pmod = np.array([self.P % q for q in chain], dtype=np.uint64)
        self._pinv = np.array([pow(self.P, -1, q) for q in chain], dtype=np.uint64)
        self._pmod_sh = shoup_np(self._pmod, np.array(chain, dtype=np.uint64))
        self._pinv_sh = shoup_np(self._pinv, np.array(chain, dtype=np.uint64))
        # rescale constants: inv[l][j] = q_l^-1 mod q_j (engine.py:67-71)
        self._resc = []
        for lvl in range(self.L + 1):
            inv = np.array([pow(chain[lvl], -1, chain[j]) for j in range(lvl)], dtype=np.uint64)
            ps = np.array(chain[:lvl], dtype=np.uint64)
            self._resc.append((inv, shoup_np(inv, ps) if lvl else inv))
        self._crt_cache: dict = {}
        self._mdr: dict = {}   # level -> (P q_l)^-1 mod q_t, the merged ModDown + rescale
        # rotation inner products on pre-permuted keys (default; HEAR_B200_PREPERM=0
        # disables): the digits are read in natural order, so a hoisted group
        # is one GEMM over digits x (rotation, component) and the Galois map is
        # applied by the ModDown scatter; bit-identical, 2x rotation-key memory
        self.preperm = os.environ.get("HEAR_B200_PREPERM", "1") == "1"
        # batched key switches of at least this many clips take the GEMM inner
        # product (ks_gemm); smaller ones the per-job kernel (ks_inner2), which
        # has the lower latency at one or two clips
        self.ks_gemm_min = int(os.environ.get("HEAR_B200_KS_GEMM_MIN", "8"))
        # hoisted rotations of several handles share one ModUp / ModDown launch
        # when each handle carries at most `batch_hoist_max` clips: at one clip
        # per handle the merged launches fill the GPU (B=1 latency 4.77 -> 4.15
        # ms); at 128 clips they are throughput-neutral inside the CUDA graph.
        # HEAR_B200_BATCH_HOIST=1 / 0 forces it on / off for every batch size.
        self.batch_hoist_max = {"1": 1 << 30, "0": 0}.get(
            os.environ.get("HEAR_B200_BATCH_HOIST", ""), 16)
        # cluster NTT: inverse transforms whose rows feed ModUp / ModDown /
        # rescale write centred lifts as doubles (task scal = 1) and the
        # forward transforms read them with src_prime = -1: one lift per row
        self.lift_once = bool(nat.lib().hb_ntt_fused_ks(self.ring.handle))
        # lazy ModDown ("double hoisting"): hoisted rotations that only feed
        # plaintext accumulations (conv layers, strategy "full") stay in the
        # extended basis Q*P -- the inner-product GEMM scatters them through
        # the Galois map and adds P*c0 -- the layer MAC runs over level+2 rows
        # (plaintexts carry their special-prime row) and P is divided out once
        # per output: conv2/conv3 of 1d-w64 need 8/16 ModDowns instead of 94.
        # Primitives stay bit-exact; a lazy layer differs from the reference's
        # ciphertext by rounding noise only (one ModDown rounding instead of
        # one per rotation).  HEAR_B200_LAZY_MODDOWN=0 restores the eager path.
        self.lazy = (os.environ.get("HEAR_B200_LAZY_MODDOWN", "1") == "1" and self.ring.use_f64
                     and self.preperm and self.lift_once)
        # smallest batch that takes the lazy forms (below ks_gemm_min the
        # extended-basis rotations come from the per-job inner-product kernel:
        # B=1 latency 4.06 -> 3.49 ms)
        self.lazy_min = int(os.environ.get("HEAR_B200_LAZY_MIN", "1"))
        self._pmod_dev = self._dev(self._pmod)
        # non-hoisted key switches (relinearisation, rot_each, rotate-and-add)
        # run ModUp and the inner product in ONE kernel (k_ks3: transforms in
        # cluster shared memory, sums in tensor memory) once the launch fills
        # the GPU: the digit expansion is never written.  Bit-identical.
        # HEAR_B200_KS_FUSED=0 disables; HEAR_B200_KS_FUSED_MIN = smallest
        # number of (ciphertext, row) tasks that takes the fused kernel.
        self.fuse_ks = (os.environ.get("HEAR_B200_KS_FUSED", "1") == "1" and self.ring.use_f64
                        and self.preperm and self.lift_once)
        self.fuse_ks_min = int(os.environ.get("HEAR_B200_KS_FUSED_MIN", "600"))
        self.keys = KeyMaterial()
        if keygen:
            self._keygen()

    # ------------------------------------------------------------------ key transport

    def key_tensors(self) -> list:
        """Ordered (name, tensor) list of the public evaluation material, for
        replication to other ranks (bench.py broadcasts it over NCCL)."""
        k = self.keys
        out = [("pk_b", k.pk_b), ("pk_a", k.pk_a), ("relin_b", k.relin.b),
               ("relin_a", k.relin.a)]
        for amt in sorted(k.rot):
            out += [(f"rot{amt}_b", k.rot[amt].b), (f"rot{amt}_a", k.rot[amt].a)]
        return out

    def key_manifest(self) -> list:
        """[(amount, lmax)] of the rotation keys (shapes follow from it)."""
        return [(a, self.keys.rot[a].lmax) for a in sorted(self.keys.rot)]

    def alloc_keys(self, manifest):
        """Allocate empty evaluation keys of the given layout (receiver side),
        in the order and shapes of key_layout / key_tensors."""
        k = self.keys
        t = {name: torch.empty(shape, dtype=torch.int64, device=self.dev)
             for name, shape in key_layout(self.params, manifest)}
        k.pk_b, k.pk_a = t["pk_b"], t["pk_a"]
        k.relin = _Ksk(t["relin_b"], t["relin_a"], self.L)
        for amt, lmax in manifest:
            k.rot[amt] = _Ksk(t[f"rot{amt}_b"], t[f"rot{amt}_a"], lmax)

    # ------------------------------------------------------------------ sampling

    def _ternary(self) -> np.ndarray:
        return self.rng.integers(-1, 2, self.n).astype(np.int64)

    def _gauss(self) -> np.ndarray:
        return np.rint(self.rng.normal(0.0, self.params.error_std, self.n)).astype(np.int64)

    def _uniform_rows(self, gidx) -> np.ndarray:
        out = np.empty((len(gidx), self.n), dtype=np.uint64)
        for r, g in enumerate(gidx):
            out[r] = self.rng.integers(0, self.ring.primes[g], self.n, dtype=np.uint64)
        return out

    def _full_gidx(self, lmax=None) -> list:
        lmax = self.L if lmax is None else lmax
        return list(range(lmax + 1)) + [self.S]

    def _dev(self, arr: np.ndarray) -> torch.Tensor:
        a = np.ascontiguousarray(arr)
        if a.dtype == np.uint64:
            a = a.view(np.int64)
        return torch.from_numpy(a).to(self.dev)

    # ------------------------------------------------------------------ kernels

    def _coeffs_to_ntt(self, coeffs: torch.Tensor, gidx) -> torch.Tensor:
        """Signed int64 coefficients [M, N] -> NTT rows [M, len(gidx), N]."""
        coeffs = coeffs.contiguous()
        m, r = coeffs.shape[0], len(gidx)
        out = self.ring.empty(m, r)
        src = np.repeat(self.ring.row_ptrs(coeffs), r)
        self.ring.ntt_fwd(_tasks(nat.NTT_TASK, m * r, src=src, dst=self.ring.row_ptrs(out),
                                 dst_prime=np.tile(np.asarray(gidx), m),
                                 src_prime=np.tile(np.asarray(gidx), m)), nat.FWD_I64)
        return out

    def _ew(self, op, dst, a, b=None, c=None, primes=None, scal=None, scal_sh=None):
        """Element-wise op over matching row lists (pointer arrays)."""
        n = len(dst)
        f = dict(dst=dst, a=a, prime=primes)
        if b is not None:
            f["b"] = b
        if c is not None:
            f["c"] = c
        if scal is not None:
            f["scal"], f["scal_sh"] = scal, scal_sh
        self.ring.ew(op, _tasks(nat.EW_TASK, n, **f))

    def _row_primes(self, batch_shape: int, rows: int, gidx=None) -> np.ndarray:
        g = np.arange(rows) if gidx is None else np.asarray(gidx)
        return np.tile(g, batch_shape)

    def _intt_rows(self, src: torch.Tensor, primes: np.ndarray) -> torch.Tensor:
        out = torch.empty_like(src)
        n = src.numel() // self.n
        self.ring.ntt_inv(_tasks(nat.NTT_TASK, n, src=self.ring.row_ptrs(src),
                                 dst=self.ring.row_ptrs(out), dst_prime=primes, src_prime=primes))
        return out

    # ------------------------------------------------------------------ keygen

    def _keygen(self):
        k = self.keys
        gidx = self._full_gidx()
        k.s_coeffs = self._ternary()
        k.s_ntt = self._coeffs_to_ntt(self._dev(k.s_coeffs)[None], gidx)[0]
        k.pk_a = self._dev(self._uniform_rows(gidx))
        e = self._coeffs_to_ntt(self._dev(self._gauss())[None], gidx)[0]
        k.pk_b = self._sub_prod(e, k.pk_a, k.s_ntt, gidx)
        s2 = self.ring.empty(len(gidx))
        rp = self.ring.row_ptrs
        self._ew(nat.EW_MUL, rp(s2), rp(k.s_ntt), rp(k.s_ntt), primes=np.array(gidx))
        k.relin = self._make_ksk(s2, self.L)

    def _sub_prod(self, e, a, s, gidx):
        """e - a*s over rows (keygen b-component)."""
        rp = self.ring.row_ptrs
        t = torch.empty_like(a)
        self._ew(nat.EW_MUL, rp(t), rp(a), rp(s), primes=np.array(gidx))
        out = torch.empty_like(a)
        self._ew(nat.EW_SUB, rp(out), rp(e), rp(t), primes=np.array(gidx))
        return out

    def _make_ksk(self, target_ntt: torch.Tensor, lmax: int) -> _Ksk:
        """Key encrypting P*target under s, one component per digit prime
        (engine.py:112-132)."""
        gidx = self._full_gidx(lmax)
        rows, ndig = len(gidx), lmax + 1
        s = self.keys.s_ntt[list(range(lmax + 1)) + [self.L + 1]].contiguous()
        kb = self.ring.empty(ndig, rows)
        ka = self.ring.empty(ndig, rows)
        rp = self.ring.row_ptrs
        for i in range(ndig):
            a = self._dev(self._uniform_rows(gidx))
            e = self._coeffs_to_ntt(self._dev(self._gauss())[None], gidx)[0]
            ka[i].copy_(a)
            kb[i].copy_(self._sub_prod(e, a, s, gidx))
            # digit i's component carries P*target on its own prime row only
            self._ew(nat.EW_ADD_SCALED, rp(kb[i, i:i + 1]), rp(kb[i, i:i + 1]),
                     rp(target_ntt[i:i + 1]), primes=np.array([i]),
                     scal=self._pmod[i:i + 1], scal_sh=self._pmod_sh[i:i + 1])
        return _Ksk(kb, ka, lmax)

    def ensure_rotation_keys(self, rot_levels: dict):
        """Keys for {amount: max evaluation level} (engine.py:134-147)."""
        for amount, lmax in sorted(rot_levels.items()):
            amount %= self.n2
            if amount == 0:
                continue
            have = self.keys.rot.get(amount)
            if have is not None and have.lmax >= lmax:
                continue
            g = self.ring.galois_element(amount)
            sg = self.ring.coeff_automorphism(self.keys.s_coeffs, g)
            target = self._coeffs_to_ntt(self._dev(sg)[None], self._full_gidx(lmax))[0]
            self.keys.rot[amount] = self._make_ksk(target, lmax)
            if self.preperm:
                self._permute_key(amount)

    def _permute_key(self, amount: int):
        """K'[m] = K[pi^-1(m)] for every key row: with it the rotation's inner
        product reads the digits in natural order and the Galois gather moves
        to one pass after ModDown (ModDown commutes with the automorphism)."""
        key = self.keys.rot[amount]
        perm = self.ring.ntt_perm(self.ring.galois_element(amount))
        inv = np.empty_like(perm)
        inv[perm] = np.arange(len(perm), dtype=perm.dtype)
        pinv = torch.from_numpy(inv).to(self.dev)
        rp = self.ring.row_ptrs
        key.bp, key.ap = torch.empty_like(key.b), torch.empty_like(key.a)
        for src, dst in ((key.b, key.bp), (key.a, key.ap)):
            rows = src.numel() // self.n
            self._ew(nat.EW_PERM, rp(dst), rp(src), np.full(rows, pinv.data_ptr(), dtype=np.uint64),
                     primes=np.zeros(rows, dtype=np.int64))

    def finish_keys(self):
        """Derive the permuted rotation keys after keys were received from
        another rank (parallel.replicate_keys)."""
        for amount, key in self.keys.rot.items():
            if self.preperm and key.bp is None:
                self._permute_key(amount)

    # ------------------------------------------------------------------ codec

    def _encode_rows(self, values: torch.Tensor, level: int, scale) -> torch.Tensor:
        """[M, level+1, N] plaintext rows; with lazy ModDown one more row, the
        residues under the special prime (extended-basis accumulations)."""
        coeffs = self.emb.encode_coeffs(values, float(scale))
        return self._coeffs_to_ntt(coeffs, list(range(level + 1)) + ([self.S] if self.lazy else []))

    def _raw_encode(self, values, level, scale) -> Pt:
        rows = self._encode_rows(torch.as_tensor(values, dtype=torch.float64)[None], level, scale)
        return Pt(rows[0], level, scale, self.n2)

    def encode_many(self, values: np.ndarray, level: int, scale) -> list:
        """Encode M plaintext vectors (M, N/2) at one (level, scale) in one
        launch sequence.  Same values as M encode() calls."""
        values = np.asarray(values, dtype=np.float64)
        if values.ndim != 2 or values.shape[1] != self.n2:
            raise ValueError(f"plaintexts must have {self.n2} slots")
        scale = Fraction(scale)
        rows = self._encode_rows(torch.from_numpy(values), level, scale)
        return [Pt(rows[i], level, scale, self.n2) for i in range(rows.shape[0])]

    def _rows_needed(self, scale) -> int:
        """Chain prefix that holds value*scale + noise (engine.py:177-185)."""
        need = max(np.log2(float(scale)), 0.0) + 40
        bits = 0.0
        for k, p in enumerate(self.params.chain_primes):
            bits += np.log2(p)
            if bits >= need:
                return k + 1
        return self.L + 1

    def _crt_consts(self, keep: int):
        if keep not in self._crt_cache:
            primes = list(self.params.chain_primes[:keep])
            Q = 1
            for p in primes:
                Q *= p
            nl = (Q.bit_length() + 63) // 64

            def limbs(x):
                return [(x >> (64 * i)) & ((1 << 64) - 1) for i in range(nl)]

            qhat = [Q // p for p in primes]
            words = limbs(Q) + limbs(Q // 2) + [pow(h, -1, p) for h, p in zip(qhat, primes)]
            for h in qhat:
                words += limbs(h)
            c = torch.from_numpy(np.array(words, dtype=np.uint64).view(np.int64)).to(self.dev)
            idx = torch.arange(keep, dtype=torch.int32, device=self.dev)
            self._crt_cache[keep] = (c, idx, nl)
        return self._crt_cache[keep]

    def _decrypt_coeffs(self, ct: Ct, keep: int) -> torch.Tensor:
        """Centred coefficients of <ct, s> as float64 [B, N] (engine.py:156-175)."""
        d = ct.payload.data
        b = d.shape[0]
        rp = self.ring.row_ptrs
        m = self.ring.empty(b, keep)
        dr = rp(d).reshape(b, 2, d.shape[2])[:, :, :keep]   # row pointers, no copies
        self._ew(nat.EW_MULADD, rp(m), dr[:, 1].ravel(), np.tile(rp(self.keys.s_ntt)[:keep], b),
                 dr[:, 0].ravel(), primes=self._row_primes(b, keep))
        coef = self._intt_rows(m, self._row_primes(b, keep))
        consts, idx, nl = self._crt_consts(keep)
        out = torch.empty(b, self.n, dtype=torch.float64, device=self.dev)
        tasks = _tasks(nat.CRT_TASK, b, rows=rp(coef)[::keep],
                       out=np.uint64(out.data_ptr()) + np.arange(b, dtype=np.uint64)
                       * np.uint64(8 * self.n))
        from .ring import _upload
        td = _upload(tasks, self.dev)
        nat.check(nat.lib().hb_crt_double(self.ring.handle, td.data_ptr(), b, consts.data_ptr(),
                                          idx.data_ptr(), keep, nl, self.ring.stream), "crt")
        return out

    def _raw_dec(self, ct: Ct) -> np.ndarray:
        keep = min(ct.level + 1, self._rows_needed(ct.scale))
        coeffs = self._decrypt_coeffs(ct, keep)
        vals = self.emb.decode_coeffs(coeffs, float(ct.scale)).cpu().numpy()
        return vals[0] if ct.payload.batch == 1 else vals

    # ------------------------------------------------------------------ encryption

    def _raw_enc(self, values, level, scale) -> Ct:
        """Raised-modulus public-key encryption (engine.py:194-211), batched
        over the leading axis of `values`; randomness drawn per clip in the
        reference order (u, e0, e1)."""
        vals = np.ascontiguousarray(np.atleast_2d(values))
        coeffs = self.emb.encode_coeffs(torch.from_numpy(vals), float(scale))
        return self._enc_from_coeffs(coeffs, level, scale)

    def _enc_from_coeffs(self, coeffs: torch.Tensor, level: int, scale) -> Ct:
        """Encrypt B plaintexts given as signed int64 coefficients [B, N]."""
        b = coeffs.shape[0]
        rows = list(range(level + 1))
        gidx = rows + [self.S]
        r = len(gidx)
        m = self._coeffs_to_ntt(coeffs, rows)
        noise = np.empty((b, 3, self.n), dtype=np.int64)
        for i in range(b):
            noise[i, 0] = self._ternary()
            noise[i, 1] = self._gauss()
            noise[i, 2] = self._gauss()
        uee = self._coeffs_to_ntt(self._dev(noise).reshape(3 * b, self.n), gidx).reshape(b, 3, r, self.n)
        sel = rows + [self.L + 1]
        rp = self.ring.row_ptrs
        pkb, pka = rp(self.keys.pk_b)[sel], rp(self.keys.pk_a)[sel]   # row pointers, no copies
        ext = self.ring.empty(b, 2, r)
        er = rp(ext).reshape(b, 2, r)
        ur = rp(uee).reshape(b, 3, r)
        prim = self._row_primes(b, r, gidx)
        # c0 = u*pk_b + e0, c1 = u*pk_a + e1
        self._ew(nat.EW_MULADD, er[:, 0].ravel(), ur[:, 0].ravel(), np.tile(pkb, b),
                 ur[:, 1].ravel(), primes=prim)
        self._ew(nat.EW_MULADD, er[:, 1].ravel(), ur[:, 0].ravel(), np.tile(pka, b),
                 ur[:, 2].ravel(), primes=prim)
        # c0[:level+1] += P * m
        c0rows = er[:, 0, :level + 1].ravel()
        self._ew(nat.EW_ADD_SCALED, c0rows, c0rows, rp(m), primes=self._row_primes(b, level + 1),
                 scal=np.tile(self._pmod[:level + 1], b),
                 scal_sh=np.tile(self._pmod_sh[:level + 1], b))
        out = self._drop_special(ext, level)
        return Ct(CtData(out), level, scale, self.n2)

    def _drop_special(self, ext: torch.Tensor, level: int) -> torch.Tensor:
        """ext [M, 2, level+2, N] (special row last) -> (x - [x]_P)/P on the
        chain rows, [M, 2, level+1, N] (engine.py:213-227)."""
        m, r = ext.shape[0] * 2, level + 1
        rows = self.ring.row_ptrs(ext).reshape(m, level + 2)   # row pointers, no copies
        spc = self.ring.empty(m)
        sp = np.full(m, self.S)
        self.ring.ntt_inv(_tasks(nat.NTT_TASK, m, src=rows[:, level + 1], dst=self.ring.row_ptrs(spc),
                                 dst_prime=sp, src_prime=sp))
        out = self.ring.empty(m, r)
        self.ring.ntt_fwd(_tasks(nat.NTT_TASK, m * r, src=np.repeat(self.ring.row_ptrs(spc), r),
                                 dst=self.ring.row_ptrs(out), aux=rows[:, :r].ravel(),
                                 src_prime=self.S, dst_prime=np.tile(np.arange(r), m),
                                 scal=np.tile(self._pinv[:r], m),
                                 scal_sh=np.tile(self._pinv_sh[:r], m)), nat.FWD_MODDOWN)
        return out.reshape(m // 2, 2, r, self.n)

    # ------------------------------------------------------------------ arithmetic

    def _new(self, b, rows) -> torch.Tensor:
        return self.ring.empty(b, 2, rows)

    def _raw_add(self, a: Ct, b: Ct) -> Ct:
        self._check_batch(a, b)
        x, y = a.payload.data, b.payload.data
        out = torch.empty_like(x)
        rp = self.ring.row_ptrs
        self._ew(nat.EW_ADD, rp(out), rp(x), rp(y),
                 primes=self._row_primes(x.shape[0] * 2, a.level + 1))
        return Ct(CtData(out), a.level, a.scale, self.n2)

    def _check_batch(self, a: Ct, b: Ct):
        if a.payload.batch != b.payload.batch:
            raise ValueError(f"batch mismatch: {a.payload.batch} vs {b.payload.batch}")

    def _pt_rows(self, p: Pt, level: int) -> torch.Tensor:
        return p.payload[:level + 1]

    def _raw_add_plain(self, a: Ct, p: Pt) -> Ct:
        x = a.payload.data
        bsz, lvl = x.shape[0], a.level
        r = lvl + 1
        out = torch.empty_like(x)
        rp = self.ring.row_ptrs
        # one launch: c0 rows + plaintext, c1 rows + a zero row (a copy)
        b = np.empty((bsz, 2, r), dtype=np.uint64)
        b[:, 0] = rp(p.payload)[:r]
        b[:, 1] = np.uint64(self._zero_row().data_ptr())
        self._ew(nat.EW_ADD, rp(out), rp(x), b.ravel(), primes=self._row_primes(2 * bsz, r))
        return Ct(CtData(out), a.level, a.scale, self.n2)

    def _raw_add_plain_each(self, pairs) -> list:
        """One launch per level group: c0 rows + plaintext, c1 rows copied."""
        out = [None] * len(pairs)
        rp = self.ring.row_ptrs
        z = np.uint64(self._zero_row().data_ptr())
        for lvl, idx in self._by_level(pairs, lambda pr: pr[0].level).items():
            bsz = pairs[idx[0]][0].payload.batch
            r = lvl + 1
            res = self.ring.empty(len(idx), bsz, 2, r)
            b = np.full((len(idx), bsz, 2, r), z, dtype=np.uint64)
            for q, i in enumerate(idx):
                b[q, :, 0] = rp(pairs[i][1].payload)[:r]
            a = np.concatenate([rp(pairs[i][0].payload.data) for i in idx])
            self._ew(nat.EW_ADD, rp(res), a, b.ravel(),
                     primes=self._row_primes(len(idx) * bsz * 2, r))
            for q, i in enumerate(idx):
                c = pairs[i][0]
                out[i] = Ct(CtData(res[q]), lvl, c.scale, self.n2)
        return out

    def _raw_mod_down_each(self, cts, to_level: int) -> list:
        """The kept rows of every handle in one copy launch per source level."""
        out = [None] * len(cts)
        rp = self.ring.row_ptrs
        r = to_level + 1
        for lvl, idx in self._by_level(cts, lambda c: c.level).items():
            bsz = cts[idx[0]].payload.batch
            res = self.ring.empty(len(idx), bsz, 2, r)
            src = np.concatenate([rp(cts[i].payload.data).reshape(bsz * 2, lvl + 1)[:, :r].ravel()
                                  for i in idx])
            self._ew(nat.EW_COPY, rp(res), src, primes=self._row_primes(len(idx) * bsz * 2, r))
            for q, i in enumerate(idx):
                out[i] = Ct(CtData(res[q]), to_level, cts[i].scale, self.n2)
        return out

    def _zero_row(self) -> torch.Tensor:
        if getattr(self, "_zrow", None) is None:
            self._zrow = self.ring.zeros(1)
        return self._zrow

    def _raw_mult_plain(self, a: Ct, p: Pt) -> Ct:
        x = a.payload.data
        bsz, lvl = x.shape[0], a.level
        out = torch.empty_like(x)
        rp = self.ring.row_ptrs
        prow = rp(p.payload)[:lvl + 1]
        self._ew(nat.EW_MUL, rp(out), rp(x), np.tile(prow, 2 * bsz),
                 primes=self._row_primes(2 * bsz, lvl + 1))
        return Ct(CtData(out), a.level, a.scale * p.scale, self.n2)

    def _raw_mult(self, a: Ct, b: Ct) -> Ct:
        self._check_batch(a, b)
        lvl = a.level
        x, y = a.payload.data, b.payload.data
        bsz = x.shape[0]
        r = lvl + 1
        d = self.ring.empty(bsz, 3, r)
        rp = self.ring.row_ptrs
        xr, yr, dr = rp(x).reshape(bsz, 2, r), rp(y).reshape(bsz, 2, r), rp(d).reshape(bsz, 3, r)
        t = _tasks(nat.TENSOR_TASK, bsz * r, a0=xr[:, 0].ravel(), a1=xr[:, 1].ravel(),
                   b0=yr[:, 0].ravel(), b1=yr[:, 1].ravel(), d0=dr[:, 0].ravel(),
                   d1=dr[:, 1].ravel(), d2=dr[:, 2].ravel(),
                   prime=self._row_primes(bsz, r))
        self.ring.tensor(t)
        de = self._decompose(dr[:, 2], lvl, fused_ok=True)
        out = self._ks_apply_many(de, lvl, [(self.keys.relin, None, dr[:, :2], False)])[0]
        return Ct(CtData(out), lvl, a.scale * b.scale, self.n2)

    def _raw_rescale(self, a: Ct) -> Ct:
        """Exact RNS division by the top prime (engine.py:263-281): the
        batched form on row pointers (no copies of the input rows)."""
        return self._raw_rescale_each([a])[0]

    def _raw_mod_down(self, a: Ct, to_level: int) -> Ct:
        """Drop the rows above to_level: one copy launch of the kept rows
        (k_ew COPY on row pointers) into a contiguous handle."""
        x = a.payload.data
        bsz, r = x.shape[0], to_level + 1
        out = self.ring.empty(bsz, 2, r)
        src = self.ring.row_ptrs(x).reshape(bsz * 2, x.shape[2])[:, :r].ravel()
        self._ew(nat.EW_COPY, self.ring.row_ptrs(out), src, primes=self._row_primes(2 * bsz, r))
        return Ct(CtData(out), to_level, a.scale, self.n2)

    # ------------------------------------------------------------------ key switching

    def _decompose(self, d, lvl: int, fused_ok: bool = False):
        """Digits of d extended to chain rows 0..lvl plus the special prime:
        de [B, lvl+1 (digit), lvl+2 (row), N] (engine.py:290-303).

        d: tensor [B, lvl+1, N] (any strides between clips) or a uint64
        pointer array [B, lvl+1] of NTT-form rows.  Row i of digit i is the
        input row itself (the lift of a residue re-reduced under its own
        prime is the residue), so it is copied instead of transformed."""
        if isinstance(d, torch.Tensor):
            if d.stride(-1) != 1 or d.stride(-2) != self.n:
                d = d.contiguous()
            ptrs = (np.uint64(d.data_ptr()) + np.uint64(8) * (
                np.arange(d.shape[0], dtype=np.uint64)[:, None] * np.uint64(d.stride(0))
                + np.arange(d.shape[1], dtype=np.uint64)[None, :] * np.uint64(self.n)))
        else:
            ptrs = np.asarray(d, dtype=np.uint64)
        bsz = ptrs.shape[0]
        ndig, rows = lvl + 1, lvl + 2
        coef = self.ring.empty(bsz, ndig)
        rp = self.ring.row_ptrs
        prim = self._row_primes(bsz, ndig)
        if fused_ok and self.fuse_ks and bsz * rows >= self.fuse_ks_min:
            # the fused key switch transforms the lifts itself
            self.ring.ntt_inv(_tasks(nat.NTT_TASK, bsz * ndig, src=ptrs.ravel(), dst=rp(coef),
                                     dst_prime=prim, src_prime=prim, scal=1))
            return _Digits(coef, ptrs.reshape(bsz, ndig).copy(), lvl)
        de = self.ring.empty(bsz, ndig, rows)
        gidx = np.array(list(range(lvl + 1)) + [self.S])
        src = np.repeat(rp(coef), rows)
        dst = rp(de)
        sp = np.tile(np.repeat(np.arange(ndig), rows), bsz)
        dp = np.tile(gidx, bsz * ndig)
        ident = sp == np.tile(np.tile(np.arange(rows), ndig), bsz)
        lift = ~ident
        # the inverse transform also copies each input row to its identity
        # digit position of de (add2), so no separate copy launch
        self.ring.ntt_inv(_tasks(nat.NTT_TASK, bsz * ndig, src=ptrs.ravel(), dst=rp(coef),
                                 dst_prime=prim, src_prime=prim, add2=dst[ident],
                                 scal=int(self.lift_once)))
        self.ring.ntt_fwd(_tasks(nat.NTT_TASK, int(lift.sum()), src=src[lift], dst=dst[lift],
                                 src_prime=-1 if self.lift_once else sp[lift],
                                 dst_prime=dp[lift]), nat.FWD_LIFT)
        return de

    def _ks_apply_many(self, de: torch.Tensor, lvl: int, jobs, bsz: int | None = None,
                       rescale: bool = False, ext: bool = False) -> list:
        """Key-switch decomposed digits once per job and ModDown.

        job = (key, perm_dev | None, addend_ptrs [bsz, 2, lvl+1] uint64 (0 = none),
        gather_c0[, de_off]): out = ModDown(<perm(de[de_off:de_off+bsz]), key>)
        + addend, component 0 of the addend read through perm when gather_c0
        (the rotation's perm(c0)).  Returns [bsz, 2, lvl+1, N] per job
        (engine.py:305-351)."""
        bsz = de.shape[0] if bsz is None else bsz
        ndig, rows = lvl + 1, lvl + 2
        nj = len(jobs)
        rp = self.ring.row_ptrs
        ip = self.ring.empty(nj * bsz * 2, rows)
        ipr = rp(ip).reshape(nj, bsz, 2, rows)
        fused = isinstance(de, _Digits)
        der = None if fused else rp(de).reshape(de.shape[0], ndig, rows)
        gidx = np.array(list(range(lvl + 1)) + [self.S])
        parts = []
        add = np.zeros((nj, bsz, 2, lvl + 1), dtype=np.uint64)
        perms = np.zeros((nj, bsz, 2, lvl + 1), dtype=np.uint64)
        late = []   # (job, perm, c0 ptrs) whose Galois gather runs after ModDown
        natural = {}   # job -> (kb, ka, lmax): inner product reads the digits in natural order
        for j, job in enumerate(jobs):
            key, perm, addend, gather_c0 = job[:4]
            off = job[4] if len(job) > 4 else 0
            if key.lmax < lvl:
                raise LevelScaleError(f"key switching key trimmed to level {key.lmax}, need {lvl}")
            krow = np.array(list(range(lvl + 1)) + [key.lmax + 1])
            prepermuted = perm is not None and key.bp is not None and self.preperm
            kb_t, ka_t = (key.bp, key.ap) if prepermuted else (key.b, key.a)
            kbr = rp(kb_t).reshape(kb_t.shape[0], key.lmax + 2)[0, krow]
            kar = rp(ka_t).reshape(ka_t.shape[0], key.lmax + 2)[0, krow]
            if fused:
                if perm is not None and not prepermuted:
                    raise LevelScaleError("fused key switch needs pre-permuted rotation keys")
                parts.append((kbr, kar, (key.lmax + 2) * self.n, off))
            else:
                parts.append(_tasks(
                    nat.KS_TASK2, rows, de=der[off, 0, :], kb=kbr, ka=kar, out_b=ipr[j, 0, 0],
                    out_a=ipr[j, 0, 1],
                    perm=perm.data_ptr() if perm is not None and not prepermuted else 0,
                    de_bstride=ndig * rows * self.n, de_dstride=rows * self.n,
                    key_stride=(key.lmax + 2) * self.n, out_bstride=2 * rows * self.n, ndig=ndig,
                    prime=gidx))
            if perm is None or prepermuted:
                natural[j] = (kb_t, ka_t, key.lmax)
            if prepermuted:
                late.append((j, perm, addend[:, 0] if addend is not None else None))
                continue
            if addend is not None:
                add[j] = addend
                if gather_c0 and perm is not None:
                    perms[j, :, 0] = perm.data_ptr()
        if ext:
            # rotations left in the extended basis: the fused kernel scatters
            # its sums through the Galois map and adds P * c0 -- `ip` IS the
            # rotated ciphertext [nj, bsz, 2, lvl+2, N], no ModDown
            if not fused or len(late) != nj:
                raise LevelScaleError("extended-basis rotations need the fused key switch "
                                      "and pre-permuted keys")
            rot = [(self.ring.perm_inv_for(perm).data_ptr(), c0) for _, perm, c0 in late]
            self.ring.ks_fused(self._ksf_tasks(de, lvl, parts, ipr, bsz, rot=rot))
            ipx = ip.reshape(nj, bsz, 2, rows, self.n)
            return [ipx[j] for j in range(nj)]
        if fused:
            self.ring.ks_fused(self._ksf_tasks(de, lvl, parts, ipr, bsz))
        elif natural and bsz >= self.ks_gemm_min and self.ring.use_f64:
            # every natural-order inner product in ONE GEMM launch: a hoisted
            # group shares its digit set, rot_each / relinearisation jobs bring
            # their own (one output pair per tile)
            js = sorted(natural)
            offs = [jobs[j][4] if len(jobs[j]) > 4 else 0 for j in js]
            keys = [natural[j] for j in js]
            same_key = all(k[0].data_ptr() == keys[0][0].data_ptr() for k in keys)
            stacked = (js == list(range(js[0], js[0] + len(js)))
                       and offs == [offs[0] + q * bsz for q in range(len(js))])
            groups: dict = {}
            for j, o in zip(js, offs):
                groups.setdefault(o, []).append(j)
            if len(groups) > 1 and all(len(g) >= 2 for g in groups.values()):
                # hoisted groups of several handles: one shared-digit GEMM each
                for o, g in groups.items():
                    self._ks_gemm(der, lvl, [natural[j] for j in g], ipr[g], bsz, [o] * len(g))
            elif len(js) > 1 and same_key and stacked:
                # one key over consecutive handles (rotate-and-sum by one amount,
                # relinearisation of a layer): their digits and outputs are
                # contiguous, so it is one (b, a) GEMM over all their clips
                self._ks_gemm(der, lvl, keys[:1], ipr[js[:1]], bsz * len(js), offs[:1])
            else:
                self._ks_gemm(der, lvl, keys, ipr[js], bsz, offs)
            rest = [parts[j] for j in range(nj) if j not in natural]
            if rest:
                self.ring.ks_inner2(np.concatenate(rest), bsz)
        else:
            self.ring.ks_inner2(np.concatenate(parts), bsz)
        m, r = nj * bsz * 2, lvl + 1
        # optional post-addend per job (job[5]: row pointers [bsz, 2, lvl+1]),
        # added in the ModDown epilogue at the destination index
        post = np.zeros((nj, bsz, 2, r), dtype=np.uint64)
        for j, job in enumerate(jobs):
            if len(job) > 5 and job[5] is not None:
                post[j] = job[5]
        has_post = bool(post.any())
        iprows = rp(ip).reshape(m, rows)
        if rescale:
            # relinearisation followed by its rescale: ModDown, the (d0, d1)
            # addend and the division by q_lvl in one pass per target row
            if late or has_post or perms.any() or not add.all() or not self.lift_once:
                raise LevelScaleError("merged ModDown + rescale: plain addend jobs only")
            out = self._md_rescale(iprows, lvl, add.reshape(m, r)).reshape(nj, bsz, 2, lvl, self.n)
            return [out[j] for j in range(nj)]
        spc = self.ring.empty(m)
        sprime = np.full(m, self.S)
        self.ring.ntt_inv(_tasks(nat.NTT_TASK, m, src=iprows[:, lvl + 1], dst=rp(spc),
                                 dst_prime=sprime, src_prime=sprime, scal=int(self.lift_once)))
        src_p = -1 if self.lift_once else self.S
        out = self.ring.empty(m, r)
        if late and len(late) == nj and self.lift_once:
            # (cluster NTT only: the two-pass kernels keep their intermediate
            # in dst, which an in-place scatter would race with)
            # pre-permuted rotations: ModDown of the natural-order inner product
            # (ModDown commutes with the automorphism), c0 added at the source
            # index, result scattered through the inverse Galois map:
            #   c0'[inv[j]] = ModDown(b')[j] + c0[j],  c1'[inv[j]] = ModDown(a')[j]
            inv = np.zeros((nj, bsz, 2, r), dtype=np.uint64)
            addn = np.zeros((nj, bsz, 2, r), dtype=np.uint64)
            for j, perm, c0 in late:
                inv[j] = self.ring.perm_inv_for(perm).data_ptr()
                if c0 is not None:
                    addn[j, :, 0] = c0
            t = _tasks(nat.NTT_TASK, m * r, src=np.repeat(rp(spc), r), dst=rp(out),
                       aux=iprows[:, :r].ravel(),
                       src_prime=src_p, dst_prime=np.tile(np.arange(r), m),
                       scal=np.tile(self._pinv[:r], m), scal_sh=np.tile(self._pinv_sh[:r], m),
                       add=addn.ravel(), perm=inv.ravel(), add2=post.ravel())
            self.ring.ntt_fwd(t, nat.FWD_MODDOWN_SCATTER)
            out = out.reshape(nj, bsz, 2, r, self.n)
            return [out[j] for j in range(nj)]
        t = _tasks(nat.NTT_TASK, m * r, src=np.repeat(rp(spc), r), dst=rp(out),
                   aux=iprows[:, :r].ravel(),
                   src_prime=src_p, dst_prime=np.tile(np.arange(r), m),
                   scal=np.tile(self._pinv[:r], m), scal_sh=np.tile(self._pinv_sh[:r], m),
                   add=add.ravel(), perm=perms.ravel(),
                   add2=(post.ravel() if has_post and not late else 0))
        self.ring.ntt_fwd(t, nat.FWD_MODDOWN)
        out = out.reshape(nj, bsz, 2, r, self.n)
        res = [out[j] for j in range(nj)]
        if late:
            # ModDown(x o pi) = ModDown(x) o pi: gather the rotation now,
            # c0' = md_b[pi] + c0[pi], c1' = md_a[pi]
            fin = self.ring.empty(len(late), bsz, 2, r)
            finr = rp(fin).reshape(len(late), bsz, 2, r)
            outr = rp(out).reshape(nj, bsz, 2, r)
            d0, a0, b0, p0, d1, a1, p1 = [], [], [], [], [], [], []
            for q, (j, perm, c0) in enumerate(late):
                pp = np.full(bsz * r, perm.data_ptr(), dtype=np.uint64)
                if c0 is not None:
                    d0.append(finr[q, :, 0].ravel())
                    a0.append(outr[j, :, 0].ravel())
                    b0.append(np.asarray(c0, dtype=np.uint64).ravel())
                    p0.append(pp)
                else:
                    d1.append(finr[q, :, 0].ravel())
                    a1.append(outr[j, :, 0].ravel())
                    p1.append(pp)
                d1.append(finr[q, :, 1].ravel())
                a1.append(outr[j, :, 1].ravel())
                p1.append(pp)
            if d0:
                nrow = sum(len(x) for x in d0)
                self.ring.ew(nat.EW_PERM_ADD, _tasks(
                    nat.EW_TASK, nrow, dst=np.concatenate(d0), a=np.concatenate(a0),
                    b=np.concatenate(b0), c=np.concatenate(p0),
                    prime=np.tile(np.arange(r), nrow // r)))
            nrow = sum(len(x) for x in d1)
            self.ring.ew(nat.EW_PERM, _tasks(
                nat.EW_TASK, nrow, dst=np.concatenate(d1), a=np.concatenate(a1),
                b=np.concatenate(p1), prime=np.tile(np.arange(r), nrow // r)))
            for q, (j, _, _) in enumerate(late):
                res[j] = fin[q]
            if has_post:   # gather after ModDown here: the post-addend follows it
                for j in range(nj):
                    if post[j].any():
                        dst = rp(res[j]).reshape(bsz, 2, r)
                        self._ew(nat.EW_ADD, dst.ravel(), dst.ravel(), post[j].ravel(),
                                 primes=np.tile(np.arange(r), bsz * 2))
        return res

    def _ksf_tasks(self, de: "_Digits", lvl: int, parts, ipr, bsz: int, rot=None) -> np.ndarray:
        """Task table of the fused ModUp + inner product (k_ks3): one task per
        (job, clip, target row).  parts[j] = (key b row pointers [lvl+2], key a
        row pointers, key digit stride in elements, clip offset into de);
        ipr [nj, bsz, 2, lvl+2] output row pointers."""
        ndig, rows = lvl + 1, lvl + 2
        nj = len(parts)
        gidx = np.array(list(range(lvl + 1)) + [self.S])
        t = np.zeros((nj, bsz, rows), dtype=nat.KSF_TASK)
        cr = self.ring.row_ptrs(de.coef).reshape(de.coef.shape[0], ndig)
        ident = np.zeros((de.src.shape[0], rows), dtype=np.uint64)
        ident[:, :ndig] = de.src
        for j, (kbr, kar, kds, off) in enumerate(parts):
            t["coef"][j] = cr[off:off + bsz, 0][:, None]
            t["ident"][j] = ident[off:off + bsz]
            t["kb"][j], t["ka"][j] = kbr[None, :], kar[None, :]
            t["key_dstride"][j] = kds
        t["out_b"], t["out_a"] = ipr[:, :, 0], ipr[:, :, 1]
        t["ndig"] = ndig
        t["dst_prime"] = gidx[None, None, :]
        t["ident_digit"] = np.array(list(range(ndig)) + [-1])[None, None, :]
        if rot is not None:   # per job: (scatter map pointer, c0 row pointers [bsz, lvl+1])
            for j, (scat, c0) in enumerate(rot):
                t["scat"][j] = scat
                t["c0"][j, :, :ndig] = c0
            t["pmod"][:, :, :ndig] = self._pmod[:ndig][None, None, :]
        return t.ravel()

    def _ks_gemm(self, der, lvl: int, keys, ipr, bsz: int, offs, rot=None):
        """Natural-order key-switch inner products of several jobs as one
        per-coefficient GEMM (csrc/mac.cu launch_ks_gemm): terms = digits,
        outputs = (job, component), the special row (its own prime and key
        row) as the launch's last row.  keys: (kb, ka, lmax) per job
        (pre-permuted rotation keys or the relinearisation key); offs: the
        digit set (clip offset into de) of each job -- shared by a hoisted
        group, else one per job."""
        ndig, rows, n8 = lvl + 1, lvl + 2, np.uint64(8 * self.n)
        kp, kps, dp = [], [], []
        for j, (kb, ka, lmax) in enumerate(keys):
            kst = np.uint64(lmax + 2) * n8
            for t in (kb, ka):
                base = np.uint64(t.data_ptr()) + np.arange(ndig, dtype=np.uint64) * kst
                kp.append(base)
                kps.append(base + np.uint64(lmax + 1) * n8)
            dp.extend([ipr[j, 0, 0, 0], ipr[j, 0, 1, 0]])
        kp, kps, dp = np.stack(kp), np.stack(kps), np.array(dp, dtype=np.uint64)
        shared = len(set(offs)) == 1
        if shared:
            dep = der[offs[0], :, 0]                    # [ndig] row 0 of each digit
        else:
            dep = np.stack([der[o, :, 0] for o in offs])   # [njobs, ndig]
        self.ring.ks_gemm(dep, kp, kps, dp, rows, bsz, ndig * rows * self.n,
                          2 * rows * self.n, self.S, rot=rot)

    def _rot_key(self, amount: int) -> _Ksk:
        key = self.keys.rot.get(amount % self.n2)
        if key is None:
            raise MissingRotationKey(f"no rotation key for amount {amount % self.n2}")
        return key

    def _rot_job(self, a: Ct, k: int):
        g = self.ring.galois_element(k)
        bsz, r = a.payload.batch, a.level + 1
        add = np.zeros((bsz, 2, r), dtype=np.uint64)
        add[:, 0] = self.ring.row_ptrs(a.payload.data).reshape(bsz, 2, r)[:, 0]
        return (self._rot_key(k), self.ring.perm_dev(g), add, True)

    def _raw_rot(self, a: Ct, k: int) -> Ct:
        return self._raw_rot_many(a, [k])[k]

    # ------------------------------------------------------------------ layer-wide batches

    # HBM budget for one batched launch group's temporaries (decomposed
    # digits of many ciphertexts); larger groups are split into chunks.
    # temporaries of one batched key switch (digits, inner products); B200 has
    # 180 GB, and larger batches of jobs make the inner-product GEMM wider
    ks_budget_bytes = int(float(os.environ.get("HEAR_B200_KS_BUDGET_GB", "24")) * (1 << 30))

    @staticmethod
    def _by_level(items, level_of):
        groups: dict = {}
        for i, it in enumerate(items):
            groups.setdefault(level_of(it), []).append(i)
        return groups

    def _raw_mac_many(self, jobs) -> list:
        """Groups of outputs that share one ciphertext term list (conv partial
        sums, FC diagonals) go through the shared-term kernel; the rest
        through the generic strided MAC."""
        if isinstance(jobs[0][0][0].payload, CtExt):
            return self._raw_mac_many_ext(jobs)
        out = [None] * len(jobs)
        groups: dict = {}
        for i, terms in enumerate(jobs):
            key = (terms[0][0].level, tuple(ct.payload.data.data_ptr() for ct, _ in terms))
            groups.setdefault(key, []).append(i)
        rest = []
        for (lvl, ctkey), idx in groups.items():
            if len(idx) < 2:
                rest += idx
                continue
            bsz = jobs[idx[0]][0][0].payload.batch
            r = lvl + 1
            res = self.ring.empty(len(idx), bsz, 2, r)
            dsts = self.ring.row_ptrs(res).reshape(len(idx), -1)[:, 0]
            pts = np.array([[pt.payload.data_ptr() for _, pt in jobs[i]] for i in idx],
                           dtype=np.uint64)
            self.ring.mac_shared(np.array(ctkey, dtype=np.uint64), pts, dsts, r, 2 * bsz)
            for q, i in enumerate(idx):
                t0 = jobs[i][0]
                out[i] = Ct(CtData(res[q]), lvl, t0[0].scale * t0[1].scale, self.n2)
        if rest:
            sub = self._raw_mac_strided([jobs[i] for i in rest])
            for i, c in zip(rest, sub):
                out[i] = c
        return out

    def _raw_mac_many_ext(self, jobs) -> list:
        """Accumulations over extended-basis rotations (lazy ModDown): the
        shared-term GEMM over level+2 rows, then ONE ModDown per output."""
        out = [None] * len(jobs)
        for lvl, idx, acc in self._mac_ext(jobs):
            bsz = acc.shape[1]
            res = self._mod_down_ext(acc.reshape(len(idx) * bsz, 2, lvl + 2, self.n), lvl)
            res = res.reshape(len(idx), bsz, 2, lvl + 1, self.n)
            for q, i in enumerate(idx):
                t0 = jobs[i][0]
                out[i] = Ct(CtData(res[q]), lvl, t0[0].scale * t0[1].scale, self.n2)
        return out

    def _raw_mac_rescale_many(self, jobs) -> list:
        if not (isinstance(jobs[0][0][0].payload, CtExt) and self.lift_once):
            return super()._raw_mac_rescale_many(jobs)
        out = [None] * len(jobs)
        for lvl, idx, acc in self._mac_ext(jobs):
            bsz = acc.shape[1]
            res = self._mod_down_ext(acc.reshape(len(idx) * bsz, 2, lvl + 2, self.n), lvl,
                                     rescale=True)
            res = res.reshape(len(idx), bsz, 2, lvl, self.n)
            for q, i in enumerate(idx):
                t0 = jobs[i][0]
                out[i] = Ct(CtData(res[q]), lvl - 1, t0[0].scale * t0[1].scale
                            / self.params.chain_primes[lvl], self.n2)
        return out

    def _mac_ext(self, jobs) -> list:
        """[(level, job indices, acc [len, B, 2, level+2, N])]: the products
        summed modulo every chain prime and the special prime.  Jobs of one
        level run as ONE shared-term GEMM over the union of their term lists
        (a job's absent terms take an all-zero plaintext) when the union is
        at most 1.5x the longest list -- the baby-step sums of a BSGS
        convolution differ by a few edge terms -- else per group of jobs
        sharing a term list."""
        for terms in jobs:
            for ct, pt in terms:
                if not isinstance(ct.payload, CtExt):
                    raise LevelScaleError("extended-basis and plain handles mixed in one sum")
                if pt.payload.shape[0] != pt.level + 2:
                    raise LevelScaleError("plaintext lacks its special-prime row")
        row8 = 8 * self.n
        res = []
        for lvl, idx in self._by_level(jobs, lambda t: t[0][0].level).items():
            bsz = jobs[idx[0]][0][0].payload.batch
            rows = lvl + 2
            union: dict = {}
            for i in idx:
                for ct, _ in jobs[i]:
                    union.setdefault(ct.payload.xdata.data_ptr(), len(union))
            longest = max(len(jobs[i]) for i in idx)
            if len(union) <= 1.5 * longest:
                groups = [(list(union), idx)]
            else:
                by_list: dict = {}
                for i in idx:
                    key = tuple(ct.payload.xdata.data_ptr() for ct, _ in jobs[i])
                    by_list.setdefault(key, []).append(i)
                groups = [(list(k), g) for k, g in by_list.items()]
            zero = np.uint64(self._zero_rows(rows).data_ptr())
            for ctkey, g in groups:
                pos = {c: q for q, c in enumerate(ctkey)}
                acc = self.ring.empty(len(g), bsz, 2, rows)
                dsts = self.ring.row_ptrs(acc).reshape(len(g), -1)[:, 0]
                pts = np.full((len(g), len(ctkey)), zero, dtype=np.uint64)
                last = np.full((len(g), len(ctkey)), zero, dtype=np.uint64)
                for q, i in enumerate(g):
                    for ct, pt in jobs[i]:
                        t = pos[ct.payload.xdata.data_ptr()]
                        if pts[q, t] != zero:
                            raise LevelScaleError("a handle appears twice in one accumulation")
                        pts[q, t] = pt.payload.data_ptr()
                        last[q, t] = pt.payload.data_ptr() + (pt.level + 1) * row8
                self.ring.mac_shared(np.array(ctkey, dtype=np.uint64), pts, dsts, rows, 2 * bsz,
                                     pts_last=last, prime_last=self.S)
                res.append((lvl, g, acc))
        return res

    def _zero_rows(self, rows: int) -> torch.Tensor:
        """An all-zero plaintext block of at least `rows` rows."""
        z = getattr(self, "_zrows", None)
        if z is None or z.shape[0] < rows:
            self._zrows = z = self.ring.zeros(max(rows, self.L + 2))
        return z

    def _md_rescale(self, rows: np.ndarray, lvl: int, addend) -> torch.Tensor:
        """rescale(ModDown(x) + addend) in one step (cluster NTT): rows
        [m, lvl+2] pointers of extended-basis rows (special last), addend
        [m, lvl+1] pointers or None -> [m, lvl, N] at level lvl-1.

        ModDown then rescale is (x_t - NTT_t(xP)) P^-1 + d_t - NTT_t(top)) / q_l
        with top = centre(((x_l - xP) P^-1 + d_l) mod q_l) in the coefficient
        domain; both transforms of a target row merge into ONE,
        NTT_t(xP + P * top) (FWD_MODDOWN2), so a row costs one NTT instead
        of two.  Same residues as the two separate steps (exact maps)."""
        m = rows.shape[0]
        rp = self.ring.row_ptrs
        k = 2 if addend is None else 3
        cf = self.ring.empty(k, m)
        cfr = rp(cf).reshape(k, m)
        src = [rows[:, lvl + 1], rows[:, lvl]] + ([] if addend is None else [addend[:, lvl]])
        prim = np.repeat(np.array([self.S, lvl, lvl][:k]), m)
        self.ring.ntt_inv(_tasks(nat.NTT_TASK, k * m, src=np.concatenate(src), dst=cfr.ravel(),
                                 dst_prime=prim, src_prime=prim, scal=1))
        top = self.ring.empty(m)
        self._ew(nat.EW_MD_TOP, rp(top), cfr[1], cfr[0], c=None if addend is None else cfr[2],
                 primes=np.full(m, lvl), scal=np.full(m, self._pinv[lvl]),
                 scal_sh=np.full(m, self._pinv_sh[lvl]))
        if lvl not in self._mdr:
            chain = self.params.chain_primes
            self._mdr[lvl] = np.array([pow(self.P * chain[lvl], -1, chain[t]) for t in range(lvl)],
                                      dtype=np.uint64)
        out = self.ring.empty(m, lvl)
        f = dict(src=np.repeat(cfr[0], lvl), perm=np.repeat(rp(top), lvl), dst=rp(out),
                 aux=rows[:, :lvl].ravel(), src_prime=-1, dst_prime=np.tile(np.arange(lvl), m),
                 scal=np.tile(self._mdr[lvl], m), scal_sh=np.tile(self._pmod[:lvl], m))
        if addend is not None:
            f["add"] = addend[:, :lvl].ravel()
            f["add2"] = np.tile(self._resc[lvl][0], m)
        self.ring.ntt_fwd(_tasks(nat.NTT_TASK, m * lvl, **f), nat.FWD_MODDOWN2)
        return out

    def _mod_down_ext(self, ext: torch.Tensor, level: int, rescale: bool = False) -> torch.Tensor:
        """ext [M, 2, level+2, N] -> (x - [x]_P)/P on the chain rows
        [M, 2, level+1, N] (engine.py:213-227), the key switch's ModDown;
        rescale=True: divided by q_level as well -> [M, 2, level, N]."""
        m, r = ext.shape[0] * 2, level + 1
        rows = self.ring.row_ptrs(ext).reshape(m, level + 2)
        if rescale:
            return self._md_rescale(rows, level, None).reshape(m // 2, 2, level, self.n)
        spc = self.ring.empty(m)
        sp = np.full(m, self.S)
        self.ring.ntt_inv(_tasks(nat.NTT_TASK, m, src=rows[:, level + 1], dst=self.ring.row_ptrs(spc),
                                 dst_prime=sp, src_prime=sp, scal=int(self.lift_once)))
        out = self.ring.empty(m, r)
        self.ring.ntt_fwd(_tasks(nat.NTT_TASK, m * r, src=np.repeat(self.ring.row_ptrs(spc), r),
                                 dst=self.ring.row_ptrs(out), aux=rows[:, :r].ravel(),
                                 src_prime=-1 if self.lift_once else self.S,
                                 dst_prime=np.tile(np.arange(r), m),
                                 scal=np.tile(self._pinv[:r], m),
                                 scal_sh=np.tile(self._pinv_sh[:r], m)), nat.FWD_MODDOWN)
        return out.reshape(m // 2, 2, r, self.n)

    def _raw_mac_strided(self, jobs) -> list:
        out = [None] * len(jobs)
        for lvl, idx in self._by_level(jobs, lambda t: t[0][0].level).items():
            bsz = jobs[idx[0]][0][0].payload.batch
            r = lvl + 1
            res = self.ring.empty(len(idx), bsz, 2, r)
            rp = self.ring.row_ptrs
            dst = rp(res).reshape(len(idx), -1)[:, 0]
            counts = np.array([len(jobs[i]) for i in idx], dtype=np.int64)
            offs = np.concatenate([[0], np.cumsum(counts)[:-1]])
            terms = np.zeros(int(counts.sum()), dtype=nat.MAC_TERM)
            k = 0
            for i in idx:
                for ct, pt in jobs[i]:
                    if ct.payload.batch != bsz:
                        raise ValueError("batch mismatch inside accumulation")
                    terms[k] = (pt.payload.data_ptr(), ct.payload.data.data_ptr())
                    k += 1
            outs = _tasks(nat.MAC_OUT, len(idx), dst=dst, nterms=counts, term_off=offs)
            self.ring.mac_strided(outs, terms, r, 2 * bsz)
            for q, i in enumerate(idx):
                t0 = jobs[i][0]
                out[i] = Ct(CtData(res[q]), lvl, t0[0].scale * t0[1].scale, self.n2)
        return out

    def _raw_sum_each(self, groups) -> list:
        """Each group's sum in one pass (csrc/ops.cu k_sum_rows): every source
        row read once instead of a pairwise add chain; modular addition, so
        bit-identical to the left-to-right chain."""
        kmax = max(len(g) for g in groups)
        if any(isinstance(c.payload, CtExt) for g in groups for c in g):
            return self._raw_sum_each_ext(groups)
        if kmax * max(self.ring.primes) >= 1 << 64:   # 64-bit accumulator headroom
            return super()._raw_sum_each(groups)
        out = [g[0] if len(g) == 1 else None for g in groups]
        todo = [j for j, g in enumerate(groups) if len(g) > 1]
        for lvl, idx in self._by_level([groups[j] for j in todo], lambda g: g[0].level).items():
            js = [todo[i] for i in idx]
            bsz = groups[js[0]][0].payload.batch
            r = lvl + 1
            k = max(len(groups[j]) for j in js)
            rp = self.ring.row_ptrs
            res = self.ring.empty(len(js), bsz, 2, r)
            nrow = bsz * 2 * r
            srcs = np.zeros((len(js), nrow, k), dtype=np.uint64)
            for q, j in enumerate(js):
                g = groups[j]
                for t, c in enumerate(g):
                    srcs[q, :, t] = rp(c.payload.data)
                if len(g) < k:   # ragged groups: pad with a zero row
                    srcs[q, :, len(g):] = np.uint64(self._zero_row().data_ptr())
            self.ring.sum_rows(rp(res), srcs.reshape(-1, k),
                               np.tile(np.arange(r), len(js) * bsz * 2))
            for q, j in enumerate(js):
                out[j] = Ct(CtData(res[q]), lvl, groups[j][0].scale, self.n2)
        return out

    def _raw_sum_each_ext(self, groups) -> list:
        """Sums of extended-basis rotations (lazy ModDown, rotate-and-sum):
        one pass over level+2 rows per group, then ONE ModDown per group
        instead of one per rotation."""
        out = [None] * len(groups)
        # plain handles of a mixed group (the unrotated term) join as P * ct
        plain = {id(c): c for g in groups for c in g if not isinstance(c.payload, CtExt)}
        if plain:
            lifted = dict(zip(plain, self._lift_ext(list(plain.values()))))
            groups = [[lifted.get(id(c), c) for c in g] for g in groups]
        for lvl, js in self._by_level(groups, lambda g: g[0].level).items():
            bsz = groups[js[0]][0].payload.batch
            rows = lvl + 2
            k = max(len(groups[j]) for j in js)
            if k * max(self.ring.primes) >= 1 << 64:
                raise LevelScaleError("too many terms for the 64-bit sum")
            rp = self.ring.row_ptrs
            acc = self.ring.empty(len(js), bsz, 2, rows)
            nrow = bsz * 2 * rows
            srcs = np.zeros((len(js), nrow, k), dtype=np.uint64)
            for q, j in enumerate(js):
                g = groups[j]
                for t, c in enumerate(g):
                    srcs[q, :, t] = rp(c.payload.xdata)
                if len(g) < k:
                    srcs[q, :, len(g):] = np.uint64(self._zero_row().data_ptr())
            self.ring.sum_rows(rp(acc), srcs.reshape(-1, k),
                               np.tile(np.array(list(range(lvl + 1)) + [self.S]),
                                       len(js) * bsz * 2))
            res = self._mod_down_ext(acc.reshape(len(js) * bsz, 2, rows, self.n), lvl)
            res = res.reshape(len(js), bsz, 2, lvl + 1, self.n)
            for q, j in enumerate(js):
                out[j] = Ct(CtData(res[q]), lvl, groups[j][0].scale, self.n2)
        return out

    def _lift_ext(self, cts) -> list:
        """P * ct on the chain rows, a zero special row: plain handles in the
        extended basis (the identity term of a lazy sum)."""
        out = [None] * len(cts)
        rp = self.ring.row_ptrs
        for lvl, idx in self._by_level(cts, lambda c: c.level).items():
            bsz = cts[idx[0]].payload.batch
            r, rows = lvl + 1, lvl + 2
            nh = len(idx)
            x0 = self.ring.empty(nh, bsz, 2, rows)
            z = np.uint64(self._zero_row().data_ptr())
            b = np.full((nh, bsz, 2, rows), z, dtype=np.uint64)
            b[..., :r] = np.stack([rp(cts[i].payload.data).reshape(bsz, 2, r) for i in idx])
            m = nh * bsz * 2
            zero1 = np.zeros(1, dtype=np.uint64)
            self._ew(nat.EW_ADD_SCALED, rp(x0), np.full(m * rows, z, dtype=np.uint64), b.ravel(),
                     primes=np.tile(np.array(list(range(r)) + [self.S]), m),
                     scal=np.tile(np.concatenate([self._pmod[:r], zero1]), m),
                     scal_sh=np.tile(np.concatenate([self._pmod_sh[:r], zero1]), m))
            for q, i in enumerate(idx):
                out[i] = Ct(CtExt(x0[q]), lvl, cts[i].scale, self.n2)
        return out

    def _raw_add_each(self, pairs) -> list:
        out = [None] * len(pairs)
        for lvl, idx in self._by_level(pairs, lambda p: p[0].level).items():
            bsz = pairs[idx[0]][0].payload.batch
            r = lvl + 1
            res = self.ring.empty(len(idx), bsz, 2, r)
            rp = self.ring.row_ptrs
            a = np.concatenate([rp(pairs[i][0].payload.data) for i in idx])
            b = np.concatenate([rp(pairs[i][1].payload.data) for i in idx])
            self._ew(nat.EW_ADD, rp(res), a, b, primes=self._row_primes(len(idx) * bsz * 2, r))
            for q, i in enumerate(idx):
                out[i] = Ct(CtData(res[q]), lvl, pairs[i][0].scale, self.n2)
        return out

    def _raw_rescale_each(self, cts) -> list:
        out = [None] * len(cts)
        for lvl, idx in self._by_level(cts, lambda c: c.level).items():
            bsz = cts[idx[0]].payload.batch
            k = len(idx)
            rp = self.ring.row_ptrs
            rows = np.stack([rp(cts[i].payload.data).reshape(bsz * 2, lvl + 1) for i in idx])
            rows = rows.reshape(k * bsz * 2, lvl + 1)
            topc = self.ring.empty(k * bsz * 2)
            self.ring.ntt_inv(_tasks(nat.NTT_TASK, k * bsz * 2, src=rows[:, lvl],
                                     dst=rp(topc), dst_prime=lvl, src_prime=lvl,
                                     scal=int(self.lift_once)))
            res = self.ring.empty(k, bsz, 2, lvl)
            inv, inv_sh = self._resc[lvl]
            m = k * bsz * 2
            t = _tasks(nat.NTT_TASK, m * lvl, src=np.repeat(rp(topc), lvl), dst=rp(res),
                       aux=rows[:, :lvl].ravel(), src_prime=-1 if self.lift_once else lvl,
                       dst_prime=np.tile(np.arange(lvl), m), scal=np.tile(inv, m),
                       scal_sh=np.tile(inv_sh, m))
            self.ring.ntt_fwd(t, nat.FWD_MODDOWN)
            for q, i in enumerate(idx):
                c = cts[i]
                out[i] = Ct(CtData(res[q]), lvl - 1, c.scale / self.params.chain_primes[lvl],
                            self.n2)
        return out

    def _ks_chunk(self, bsz: int, lvl: int) -> int:
        per = bsz * (lvl + 1) * (lvl + 2) * self.n * 8
        return max(1, int(self.ks_budget_bytes // max(per, 1)))

    def _raw_rot_each(self, items, lazy: bool = False) -> list:
        """lazy: the rotations only feed a sum -- where the fused key switch
        runs they stay in the extended basis (CtExt, no ModDown)."""
        out = [None] * len(items)
        for lvl, idx in self._by_level(items, lambda it: it[0].level).items():
            bsz = items[idx[0]][0].payload.batch
            step = self._ks_chunk(bsz, lvl)
            for c0 in range(0, len(idx), step):
                chunk = idx[c0:c0 + step]
                c1 = np.concatenate([
                    self.ring.row_ptrs(items[i][0].payload.data).reshape(bsz, 2, lvl + 1)[:, 1]
                    for i in chunk])
                de = self._decompose(c1, lvl, fused_ok=True)
                jobs = []
                for q, i in enumerate(chunk):
                    key, perm, add, g = self._rot_job(*items[i])
                    jobs.append((key, perm, add, g, q * bsz))
                ext = lazy and self.lazy and isinstance(de, _Digits)
                res = self._ks_apply_many(de, lvl, jobs, bsz, ext=ext)
                del de
                for q, i in enumerate(chunk):
                    ct = items[i][0]
                    out[i] = Ct(CtExt(res[q]) if ext else CtData(res[q]), lvl, ct.scale, self.n2)
        return out

    def _raw_rot_add_each(self, items) -> list:
        """[ct + rot(ct, k)] with the add fused into the rotation's ModDown
        epilogue (post-addend at the destination index): bit-identical to
        add(ct, rot(ct, k)) (modular addition), one kernel fewer per item."""
        out = [None] * len(items)
        for lvl, idx in self._by_level(items, lambda it: it[0].level).items():
            bsz = items[idx[0]][0].payload.batch
            step = self._ks_chunk(bsz, lvl)
            for c0 in range(0, len(idx), step):
                chunk = idx[c0:c0 + step]
                rows = [self.ring.row_ptrs(items[i][0].payload.data).reshape(bsz, 2, lvl + 1)
                        for i in chunk]
                de = self._decompose(np.concatenate([rw[:, 1] for rw in rows]), lvl,
                                     fused_ok=True)
                jobs = []
                for q, i in enumerate(chunk):
                    key, perm, add, g = self._rot_job(*items[i])
                    jobs.append((key, perm, add, g, q * bsz, rows[q]))
                res = self._ks_apply_many(de, lvl, jobs, bsz)
                del de
                for q, i in enumerate(chunk):
                    ct = items[i][0]
                    out[i] = Ct(CtData(res[q]), lvl, ct.scale, self.n2)
        return out

    def _raw_square_each(self, cts, rescale: bool = False) -> list:
        out = [None] * len(cts)
        for lvl, idx in self._by_level(cts, lambda c: c.level).items():
            bsz = cts[idx[0]].payload.batch
            r = lvl + 1
            step = self._ks_chunk(bsz, lvl)
            rp = self.ring.row_ptrs
            for c0 in range(0, len(idx), step):
                chunk = idx[c0:c0 + step]
                k = len(chunk)
                d = self.ring.empty(k, bsz, 3, r)
                xr = np.stack([rp(cts[i].payload.data).reshape(bsz, 2, r) for i in chunk])
                dr = rp(d).reshape(k, bsz, 3, r)
                self.ring.tensor(_tasks(
                    nat.TENSOR_TASK, k * bsz * r, a0=xr[:, :, 0].ravel(), a1=xr[:, :, 1].ravel(),
                    b0=xr[:, :, 0].ravel(), b1=xr[:, :, 1].ravel(), d0=dr[:, :, 0].ravel(),
                    d1=dr[:, :, 1].ravel(), d2=dr[:, :, 2].ravel(),
                    prime=self._row_primes(k * bsz, r)))
                de = self._decompose(dr[:, :, 2].reshape(k * bsz, r), lvl, fused_ok=True)
                jobs = [(self.keys.relin, None, dr[q, :, :2], False, q * bsz) for q in range(k)]
                res = self._ks_apply_many(de, lvl, jobs, bsz, rescale=rescale)
                del de
                for q, i in enumerate(chunk):
                    c = cts[i]
                    if rescale:
                        out[i] = Ct(CtData(res[q]), lvl - 1,
                                    c.scale * c.scale / self.params.chain_primes[lvl], self.n2)
                    else:
                        out[i] = Ct(CtData(res[q]), lvl, c.scale * c.scale, self.n2)
        return out

    def _raw_square_rescale_each(self, cts) -> list:
        if not self.lift_once:
            return super()._raw_square_rescale_each(cts)
        return self._raw_square_each(cts, rescale=True)

    def _raw_rot_many_each(self, cts, ks) -> list:
        """Hoisted rotations of several handles by the same amounts: one ModUp
        over all their clips, one inner-product GEMM per handle (its digit
        set shared by its rotations), one ModDown over every rotation."""
        out = [None] * len(cts)
        for lvl, idx in self._by_level(cts, lambda c: c.level).items():
            bsz = cts[idx[0]].payload.batch
            per = bsz * (lvl + 1) * (lvl + 2) * self.n * 8
            if (len(idx) < 2 or per * len(idx) > self.ks_budget_bytes or bsz > self.batch_hoist_max
                    or any(cts[i].payload.batch != bsz for i in idx)):
                for i in idx:
                    out[i] = self._raw_rot_many(cts[i], ks)
                continue
            rp = self.ring.row_ptrs
            c1 = np.concatenate([rp(cts[i].payload.data).reshape(bsz, 2, lvl + 1)[:, 1]
                                 for i in idx])
            de = self._decompose(c1, lvl)
            jobs, keys_of = [], []
            for h, i in enumerate(idx):
                for k in ks:
                    key, perm, add, g = self._rot_job(cts[i], k)
                    jobs.append((key, perm, add, g, h * bsz))
                    keys_of.append((i, k))
            res = {i: {} for i in idx}
            step = max(1, self._ks_chunk(bsz, lvl) * 4)
            for c0 in range(0, len(jobs), step):
                sub = self._ks_apply_many(de, lvl, jobs[c0:c0 + step], bsz)
                for (i, k), o in zip(keys_of[c0:c0 + step], sub):
                    res[i][k] = Ct(CtData(o), lvl, cts[i].scale, self.n2)
            del de
            for i in idx:
                out[i] = res[i]
        return out

    def _lazy_ok(self, cts) -> bool:
        lvl, bsz = cts[0].level, cts[0].payload.batch
        return (self.lazy and bsz >= self.lazy_min
                and all(c.level == lvl and c.payload.batch == bsz for c in cts))

    def _raw_rot_many_each_lazy(self, cts, ks, want0: bool) -> list:
        """Hoisted rotations left in the extended basis Q*P: one ModUp over
        every handle, one inner-product GEMM per handle whose epilogue
        scatters each rotation through its Galois map and adds P*c0
        (hb_ks_gemm_rot) -- no ModDown.  Returns {amount: Ct(CtExt)} per
        handle (amount 0: P*ct with a zero special row when asked for)."""
        lvl, bsz = cts[0].level, cts[0].payload.batch
        r, rows, ndig = lvl + 1, lvl + 2, lvl + 1
        nh, nk = len(cts), len(ks)
        rp = self.ring.row_ptrs
        ctr = np.stack([rp(c.payload.data).reshape(bsz, 2, r) for c in cts])   # [nh, bsz, 2, r]
        out = [{} for _ in cts]
        if want0:
            for h, x in enumerate(self._lift_ext(cts)):
                out[h][0] = x
        de = self._decompose(ctr[:, :, 1].reshape(nh * bsz, r), lvl)
        der = rp(de).reshape(nh * bsz, ndig, rows)
        xr = self.ring.empty(nh, nk, bsz, 2, rows)
        xrr = rp(xr).reshape(nh, nk, bsz, 2, rows)
        keys, scat = [], []
        for k in ks:
            key = self._rot_key(k)
            if key.lmax < lvl:
                raise LevelScaleError(f"key switching key trimmed to level {key.lmax}, need {lvl}")
            if key.bp is None:
                self._permute_key(k % self.n2)
            keys.append((key.bp, key.ap, key.lmax))
            inv = self.ring.perm_inv_dev(self.ring.galois_element(k)).data_ptr()
            scat += [inv, inv]
        if bsz < self.ks_gemm_min:
            # a few clips: the per-job inner product (lower latency than the
            # GEMM there) with the same rotation epilogue
            gidx = np.array(list(range(lvl + 1)) + [self.S])
            parts = []
            for h in range(nh):
                for q, (kb_t, ka_t, lmax) in enumerate(keys):
                    krow = np.array(list(range(lvl + 1)) + [lmax + 1])
                    c0 = np.zeros(rows, dtype=np.uint64)
                    c0[:r] = ctr[h, 0, 0, :]
                    parts.append(_tasks(
                        nat.KS_TASK2, rows, de=der[h * bsz, 0, :],
                        kb=rp(kb_t).reshape(kb_t.shape[0], lmax + 2)[0, krow],
                        ka=rp(ka_t).reshape(ka_t.shape[0], lmax + 2)[0, krow],
                        out_b=xrr[h, q, 0, 0], out_a=xrr[h, q, 0, 1], perm=0,
                        de_bstride=ndig * rows * self.n, de_dstride=rows * self.n,
                        key_stride=(lmax + 2) * self.n, out_bstride=2 * rows * self.n, ndig=ndig,
                        prime=gidx, scat=scat[2 * q], c0=c0, c0_bstride=2 * r * self.n,
                        pmod=np.concatenate([self._pmod[:r], np.zeros(1, dtype=np.uint64)])))
            self.ring.ks_inner2(np.concatenate(parts), bsz)
        else:
            for h in range(nh):
                c0s = np.zeros(2 * nk, dtype=np.uint64)
                c0s[0::2] = ctr[h, 0, 0, 0]
                self._ks_gemm(der, lvl, keys, xrr[h], bsz, [h * bsz] * nk,
                              rot=(scat, c0s, 2 * r * self.n, self._pmod_dev.data_ptr()))
        del de
        for h, c in enumerate(cts):
            for q, k in enumerate(ks):
                out[h][k] = Ct(CtExt(xr[h, q]), lvl, c.scale, self.n2)
        return out

    def _rot_sum_ok(self, cts, ks) -> bool:
        """ct + sum of distinct non-zero rotations, one ModDown (k_rot_sum_f64)."""
        nz = [k for k in ks if k]
        return (self._lazy_ok(cts) and ks.count(0) == 1 and len(set(nz)) == len(nz)
                and os.environ.get("HEAR_B200_ROT_SUM", "1") == "1")

    def _raw_rot_sum_each(self, cts, ks) -> list:
        """[ct + sum_k rot(ct, k)]: the digit expansion of every handle, then
        ONE kernel per level group that gathers the digits through each
        amount's Galois map, multiplies by the (reference-layout) key rows and
        sums in the extended basis -- no rotation is materialised -- and one
        ModDown per handle."""
        ks = [k for k in ks if k]
        lvl, bsz = cts[0].level, cts[0].payload.batch
        r, rows, ndig = lvl + 1, lvl + 2, lvl + 1
        nh = len(cts)
        rp = self.ring.row_ptrs
        ctr = np.stack([rp(c.payload.data).reshape(bsz, 2, r) for c in cts])   # [nh, bsz, 2, r]
        de = self._decompose(ctr[:, :, 1].reshape(nh * bsz, r), lvl)
        der = rp(de).reshape(nh, bsz, ndig, rows)
        acc = self.ring.empty(nh, bsz, 2, rows)
        accr = rp(acc).reshape(nh, bsz, 2, rows)
        rots = np.zeros(len(ks), dtype=nat.ROTSUM_ROT)
        for q, k in enumerate(ks):
            key = self._rot_key(k)
            if key.lmax < lvl:
                raise LevelScaleError(f"key switching key trimmed to level {key.lmax}, need {lvl}")
            rots[q] = (self.ring.perm_dev(self.ring.galois_element(k)).data_ptr(),
                       key.b.data_ptr(), key.a.data_ptr(), (key.lmax + 2) * self.n,
                       key.lmax + 1, 0)
        t = np.zeros((nh, rows), dtype=nat.ROTSUM_TASK)
        t["de"] = der[:, 0, 0, :]
        t["c0"][:, :r], t["c1"][:, :r] = ctr[:, 0, 0, :], ctr[:, 0, 1, :]
        t["out_b"], t["out_a"] = accr[:, 0, 0, :], accr[:, 0, 1, :]
        t["de_bstride"], t["de_dstride"] = ndig * rows * self.n, rows * self.n
        t["c_bstride"], t["out_bstride"] = 2 * r * self.n, 2 * rows * self.n
        t["pmod"][:, :r] = self._pmod[:r][None, :]
        t["prime"] = np.array(list(range(r)) + [self.S])[None, :]
        t["row"] = np.array(list(range(r)) + [-1])[None, :]
        self.ring.rot_sum(t.ravel(), rots, ndig, bsz)
        del de
        res = self._mod_down_ext(acc.reshape(nh * bsz, 2, rows, self.n), lvl)
        res = res.reshape(nh, bsz, 2, r, self.n)
        return [Ct(CtData(res[h]), lvl, c.scale, self.n2) for h, c in enumerate(cts)]

    def _raw_rot_many(self, a: Ct, ks) -> dict:
        if not ks:
            return {}
        lvl = a.level
        de = self._decompose(a.payload.data[:, 1], lvl)
        outs = {}
        step = max(1, self._ks_chunk(a.payload.batch, lvl) * 4)
        for c0 in range(0, len(ks), step):
            sub = ks[c0:c0 + step]
            res = self._ks_apply_many(de, lvl, [self._rot_job(a, k) for k in sub])
            for k, o in zip(sub, res):
                outs[k] = Ct(CtData(o), lvl, a.scale, self.n2)
        return outs

    # ------------------------------------------------------------------ host interop

    def export(self, ct: Ct):
        """Reference-format payload (c0, c1) uint64 numpy arrays."""
        return ct.payload.to_host()

    def import_ct(self, c0: np.ndarray, c1: np.ndarray, level: int, scale) -> Ct:
        """Wrap reference-format host payloads ((rows, N) or (B, rows, N))."""
        c0, c1 = np.asarray(c0, dtype=np.uint64), np.asarray(c1, dtype=np.uint64)
        if c0.ndim == 2:
            c0, c1 = c0[None], c1[None]
        data = self._dev(np.stack([c0, c1], axis=1))
        return Ct(CtData(data), level, Fraction(scale), self.n2)

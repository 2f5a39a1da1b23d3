"""Generate the golden fixtures of the CKKS hot path from the reference itself.

Runs ONLY in the build container (it imports /root/reference, which does not
travel to the GPU box); its outputs -- small JSON/npz files next to this
script -- are committed and are what tests/ compare against.

The reference's ring tables carry two defects that make its CKKS engine
unusable as shipped:
  * hear/ckks/ring.py:282  inverse twiddles psi^-(brv(j)+1) instead of
    psi^-brv(j): intt(ntt(a)) != a;
  * hear/ckks/ring.py:264-268  Barrett constants computed as
    `1 << (63 + b)` with b a numpy int64 -> overflow to 0, so every pw_mul
    returns the low 64 product bits reduced by repeated subtraction (wrong,
    and ~2^30 iterations per product).
This script corrects those two TABLES on each RingContext instance at run
time (no reference source is modified or copied) and then drives the
reference's own engine code.  A separate section records what the
UNPATCHED reference produces for the operations the defects do not touch
(forward NTT, add/sub, Galois permutation), pinning those bit-exactly too.

Usage:  python tests/golden/make_golden.py   (writes tests/golden/*.json|npz)
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
import time

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REF)

from hear.ckks import ring as R  # noqa: E402

_orig_init = R.RingContext.__init__


def _fixed_init(self, params):
    _orig_init(self, params)
    for i, q in enumerate(self.primes):
        rinv = pow(R.primitive_2n_root(q, 2 * self.n), -1, q)
        ipw = [pow(rinv, R._bit_reverse(j, self.logn), q) for j in range(self.n)]
        self.ipsi[i] = np.array(ipw, dtype=np.uint64)
        self.ipsish[i] = np.array([(w << 64) // q for w in ipw], dtype=np.uint64)
    self.mu = np.array([(1 << (63 + q.bit_length())) // q for q in self.primes], dtype=np.uint64)


def digest(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(np.asarray(a, dtype=np.uint64)).tobytes())
    return h.hexdigest()


def rand_rows(primes, rows, n, seed):
    """Seeded uniform residues (regenerated identically by the tests)."""
    rng = np.random.default_rng(seed)
    return np.stack([rng.integers(0, primes[r], n, dtype=np.uint64) for r in rows])


def rand_ct(params, level, seed):
    p = list(params.chain_primes)
    return (rand_rows(p, range(level + 1), params.n, seed),
            rand_rows(p, range(level + 1), params.n, seed + 1))


def main():
    from hear.backend import Ct
    from hear.ckks.engine import CkksBackend
    from hear.ckks.params import gen_params
    from fractions import Fraction

    out = {"note": "digests are sha256 over little-endian uint64 payload bytes"}

    # ---- unpatched reference: ops the defects do not touch -------------------
    ps = gen_params("toy-fast")
    rc = R.RingContext(ps)
    a = rand_rows(rc.primes, range(len(rc.primes)), ps.n, 11)
    f = a.copy()
    rc.fwd(f, list(range(len(rc.primes))))
    b = rand_rows(rc.primes, range(len(rc.primes)), ps.n, 12)
    g = rc.galois_element(3)
    perm = rc.ntt_perm(g)
    out["unpatched"] = {
        "ntt_fwd": digest(f),
        "pw_add": digest(rc.add(a, b, list(range(len(rc.primes))))),
        "pw_sub": digest(rc.sub(a, b, list(range(len(rc.primes))))),
        "ntt_perm_g3": digest(perm.astype(np.uint64)),
        "mu_table": [int(x) for x in rc.mu],
    }

    # ---- fixed reference ------------------------------------------------------
    R.RingContext.__init__ = _fixed_init
    t0 = time.time()
    for prof, seed in (("toy-fast", 7), ("fast-hear", 7)):
        ps = gen_params(prof)
        be = CkksBackend(ps, seed=seed)
        k = be.keys
        rec = {
            "s_coeffs": digest(k.s_coeffs.astype(np.int64).view(np.uint64)),
            "s_ntt": digest(k.s_ntt), "pk_b": digest(k.pk_b), "pk_a": digest(k.pk_a),
            "relin_b": digest(k.relin.b), "relin_a": digest(k.relin.a),
        }
        rot_levels = {1: ps.max_level, 5: 6, 2047: 3}
        be.ensure_rotation_keys(rot_levels)
        rec["rot_levels"] = {str(a): l for a, l in rot_levels.items()}
        rec["rot_keys"] = {str(a): digest(be.keys.rot[a].b, be.keys.rot[a].a) for a in rot_levels}
        rc = be.ring
        L = ps.max_level
        gall = list(range(L + 2))
        x = rand_rows(rc.primes, gall, ps.n, 21)
        y = rand_rows(rc.primes, gall, ps.n, 22)
        xf = x.copy()
        rc.fwd(xf, gall)
        xi = x.copy()
        rc.inv(xi, gall)
        rec["ring"] = {"ntt_fwd": digest(xf), "ntt_inv": digest(xi),
                       "pw_mul": digest(rc.mul(x, y, gall))}
        # encryption of known integer coefficients (no float encode involved)
        lvl = L
        vals = np.random.default_rng(31).uniform(-1, 1, ps.n2)
        from hear.ckks.encoder import encode_coeffs
        coeffs = encode_coeffs(be.emb, vals, float(ps.msg_scale))
        np.save(os.path.join(HERE, f"{prof}_encode_coeffs.npy"), coeffs)
        ct = be.enc(vals, level=lvl)
        rec["enc_L"] = digest(*ct.payload)
        rec["dec_maxerr"] = float(np.abs(be.dec(ct) - vals).max())
        # ops on seeded random ciphertexts
        ops = {}
        for lvl in (L, 6, 2):
            c0, c1 = rand_ct(ps, lvl, 100 + lvl)
            d0, d1 = rand_ct(ps, lvl, 200 + lvl)
            A = Ct((c0, c1), lvl, Fraction(ps.msg_scale), ps.n2)
            B = Ct((d0, d1), lvl, Fraction(ps.msg_scale), ps.n2)
            pt = rand_rows(rc.primes, range(lvl + 1), ps.n, 300 + lvl)
            from hear.backend import Pt
            P_ = Pt(pt, lvl, Fraction(ps.msg_scale), ps.n2)
            o = {
                "add": digest(*be._raw_add(A, B).payload),
                "add_plain": digest(*be._raw_add_plain(A, P_).payload),
                "mult_plain": digest(*be._raw_mult_plain(A, P_).payload),
                "mult": digest(*be._raw_mult(A, B).payload),
                "rescale": digest(*be._raw_rescale(A).payload),
                "mod_down1": digest(*be._raw_mod_down(A, 1).payload),
            }
            if lvl <= 3:
                o["rot_2047"] = digest(*be._raw_rot(A, 2047).payload)
            if lvl <= 6:
                many = be._raw_rot_many(A, [1, 5])
                o["rot_many_1"] = digest(*many[1].payload)
                o["rot_many_5"] = digest(*many[5].payload)
            ops[str(lvl)] = o
        rec["ops"] = ops
        out[prof] = rec
        print(prof, "done", time.time() - t0, flush=True)
    with open(os.path.join(HERE, "ckks_golden.json"), "w") as fh:
        json.dump(out, fh, indent=1, sort_keys=True)


if __name__ == "__main__":
    main()

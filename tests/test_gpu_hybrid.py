"""Hybrid key switching (dnum digits, k special primes; BASELINE config 1)
on the GPU against the CPU restatement of the standard algorithm
(oracle/hybrid_ref.py): keys, ModUp, relinearisation and hoisted rotations
bit-exact on both arithmetic policies; decryption correctness when P covers
a digit; and the dnum = L+1, one-special-prime case equal to the engine's
reference-design ModUp (centred conversion == exact centred lift)."""

from fractions import Fraction

import numpy as np
import pytest

from tests._util import rand_ct

pytestmark = pytest.mark.gpu


def _setup(bits, sbits, dnum, k, seed=1):
    from oracle.hybrid_ref import HybridOracle
    from paper_2104_09164_b200.ckks.engine import CkksBackend
    from paper_2104_09164_b200.ckks.hybrid import HybridKeySwitch
    from paper_2104_09164_b200.ckks.params import _search, gen_params_custom
    ps = gen_params_custom(1 << 12, bits, bits[0], bits[1])
    sp = _search(sbits, 2 << 12, k, set(ps.chain_primes) | {ps.special_prime})
    be = CkksBackend(ps, seed=seed)
    hk = HybridKeySwitch(be, dnum, sp, seed=2)
    ho = HybridOracle(ps, be.keys.s_coeffs, dnum, sp, seed=2)
    return ps, be, hk, ho


def _host(t):
    return t.cpu().numpy().view(np.uint64)


CASES = [([40, 30, 30, 30, 30, 30], 40, 2, 3),    # fp64 policy, 3 special primes
         ([40, 30, 30, 30, 30, 30], 40, 3, 1),    # one special prime (config-1 shape)
         ([50, 50, 50, 50, 50, 50, 50], 60, 3, 1),  # integer policy, 50/60-bit primes
         ([50, 50, 50, 50, 50, 50], 55, 2, 4)]


@pytest.mark.parametrize("bits,sbits,dnum,k", CASES)
def test_hybrid_bit_exact_vs_oracle(bits, sbits, dnum, k):
    ps, be, hk, ho = _setup(bits, sbits, dnum, k)
    kb, ka = hk.relin
    assert np.array_equal(_host(kb), ho.relin[0]) and np.array_equal(_host(ka), ho.relin[1])
    L = ps.max_level
    for lvl in (L, L - 2):
        c = rand_ct(ps, lvl, 50 + lvl)
        a = be.import_ct(*c, lvl, Fraction(1))
        ext = hk.modup(be.ring.row_ptrs(a.payload.data).reshape(1, 2, lvl + 1)[:, 1], lvl)
        assert np.array_equal(_host(ext)[0], ho.modup(c[1], lvl))
        m = hk.mult(a, a)
        w0, w1 = ho.mult(c, c, lvl)
        got = be.export(m)
        assert np.array_equal(got[0], w0) and np.array_equal(got[1], w1)
        amts = [1, 7]
        hk.ensure_rotation_keys(amts)
        rots = hk.rot_many(a, amts)
        for amt in amts:
            w0, w1 = ho.rot(c, lvl, amt)
            got = be.export(rots[amt])
            assert np.array_equal(got[0], w0) and np.array_equal(got[1], w1), (lvl, amt)


def test_hybrid_decrypts():
    """P (3 x 40 bits) >= each digit (<= 100 bits): mult + rescale and
    rotations decrypt to the slot products / rolls."""
    ps, be, hk, _ = _setup([40, 30, 30, 30, 30, 30], 40, 2, 3)
    v = np.random.default_rng(3).uniform(-1, 1, (2, ps.n2))
    w = np.random.default_rng(4).uniform(-1, 1, (2, ps.n2))
    a, b = be.enc(v), be.enc(w)
    m = be.rescale(hk.mult(a, b))
    assert np.abs(be.dec(m) - v * w).max() < 1e-4
    hk.ensure_rotation_keys([5, 100])
    r = hk.rot_many(a, [5, 100])
    assert np.abs(be.dec(r[5]) - np.roll(v, -5, axis=1)).max() < 1e-4
    assert np.abs(be.dec(r[100]) - np.roll(v, -100, axis=1)).max() < 1e-4


def test_full_dnum_one_special_is_reference_modup():
    """dnum = L+1 with the engine's own special prime: the hybrid ModUp
    (centred fast conversion of one residue) equals the reference design's
    digit expansion (engine._decompose: exact centred lift) bit for bit."""
    from paper_2104_09164_b200.ckks.engine import CkksBackend
    from paper_2104_09164_b200.ckks.hybrid import HybridKeySwitch
    from paper_2104_09164_b200.ckks.params import gen_params
    ps = gen_params("toy-fast")
    be = CkksBackend(ps, seed=3)
    hk = HybridKeySwitch(be, ps.max_level + 1, [ps.special_prime], seed=4)
    for lvl in (ps.max_level, 4):
        c = rand_ct(ps, lvl, 70 + lvl)
        a = be.import_ct(*c, lvl, Fraction(1))
        ptrs = be.ring.row_ptrs(a.payload.data).reshape(1, 2, lvl + 1)[:, 1]
        want = be._decompose(ptrs, lvl)
        got = hk.modup(ptrs, lvl)
        assert np.array_equal(_host(got), _host(want))

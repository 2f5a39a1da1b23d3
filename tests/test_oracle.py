"""CPU oracle pinned against the reference's golden digests (bit-exact)
and the network schedule on the slot simulator vs the reference counters."""

import json
import os
from fractions import Fraction

import numpy as np
import pytest

from tests._util import digest, rand_ct, rand_rows

HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.fixture(scope="module")
def toy():
    from oracle.cpu_engine import OracleCkks
    from paper_2104_09164_b200.ckks.params import gen_params
    return OracleCkks(gen_params("toy-fast"), seed=7)


def test_oracle_keygen(toy, golden):
    g = golden["toy-fast"]
    k = toy.keys
    assert digest(k.s_coeffs.astype(np.int64).view(np.uint64)) == g["s_coeffs"]
    assert digest(k.s_ntt) == g["s_ntt"]
    assert digest(k.pk_b) == g["pk_b"] and digest(k.pk_a) == g["pk_a"]
    assert digest(k.relin.b) == g["relin_b"] and digest(k.relin.a) == g["relin_a"]


def test_oracle_rotkeys_ring_ops(toy, golden):
    from paper_2104_09164_b200.backend import Ct, Pt
    g = golden["toy-fast"]
    toy.ensure_rotation_keys({int(a): l for a, l in g["rot_levels"].items()})
    for a, d in g["rot_keys"].items():
        assert digest(toy.keys.rot[int(a)].b, toy.keys.rot[int(a)].a) == d
    rc, ps = toy.ring, toy.params
    gall = list(range(toy.L + 2))
    x = rand_rows(rc.primes, gall, ps.n, 21)
    y = rand_rows(rc.primes, gall, ps.n, 22)
    xf = x.copy()
    rc.fwd(xf, gall)
    xi = x.copy()
    rc.inv(xi, gall)
    assert digest(xf) == g["ring"]["ntt_fwd"]
    assert digest(xi) == g["ring"]["ntt_inv"]
    assert digest(rc.mul(x, y, gall)) == g["ring"]["pw_mul"]
    for lvl_s, ops in g["ops"].items():
        lvl = int(lvl_s)
        A = Ct(rand_ct(ps, lvl, 100 + lvl), lvl, Fraction(ps.msg_scale), ps.n2)
        B = Ct(rand_ct(ps, lvl, 200 + lvl), lvl, Fraction(ps.msg_scale), ps.n2)
        P_ = Pt(rand_rows(rc.primes, range(lvl + 1), ps.n, 300 + lvl), lvl,
                Fraction(ps.msg_scale), ps.n2)
        got = {"add": toy._raw_add(A, B), "add_plain": toy._raw_add_plain(A, P_),
               "mult_plain": toy._raw_mult_plain(A, P_), "mult": toy._raw_mult(A, B),
               "rescale": toy._raw_rescale(A), "mod_down1": toy._raw_mod_down(A, 1)}
        if "rot_2047" in ops:
            got["rot_2047"] = toy._raw_rot(A, 2047)
        if "rot_many_1" in ops:
            m = toy._raw_rot_many(A, [1, 5])
            got["rot_many_1"], got["rot_many_5"] = m[1], m[5]
        for name, d in ops.items():
            assert digest(*got[name].payload) == d, (lvl, name)


def test_oracle_encrypt(golden):
    from oracle.cpu_engine import OracleCkks
    from paper_2104_09164_b200.ckks.params import gen_params
    ps = gen_params("toy-fast")
    be = OracleCkks(ps, seed=7)
    be.ensure_rotation_keys({int(a): l for a, l in golden["toy-fast"]["rot_levels"].items()})
    vals = np.random.default_rng(31).uniform(-1, 1, ps.n2)
    coeffs = np.load(os.path.join(HERE, "golden", "toy-fast_encode_coeffs.npy"))
    assert np.array_equal(be._encode_coeffs(vals, ps.msg_scale), coeffs)
    ct = be.enc(vals)
    assert digest(*ct.payload) == golden["toy-fast"]["enc_L"]
    assert np.abs(be.dec(ct) - vals).max() <= 2 * golden["toy-fast"]["dec_maxerr"] + 1e-12


def test_unpatched_reference_pins(golden):
    """Ops the reference's table defects do not touch are bit-exact against the
    UNPATCHED reference too; its Barrett table is recorded as all zeros."""
    from oracle.cpu_engine import OracleRing
    from paper_2104_09164_b200.ckks.params import gen_params
    g = golden["unpatched"]
    rc = OracleRing(gen_params("toy-fast"))
    allr = list(range(len(rc.primes)))
    a = rand_rows(rc.primes, allr, rc.n, 11)
    b = rand_rows(rc.primes, allr, rc.n, 12)
    f = a.copy()
    rc.fwd(f, allr)
    assert digest(f) == g["ntt_fwd"]
    assert digest(rc.add(a, b, allr)) == g["pw_add"]
    assert digest(rc.sub(a, b, allr)) == g["pw_sub"]
    assert digest(rc.ntt_perm(rc.galois_element(3)).astype(np.uint64)) == g["ntt_perm_g3"]
    assert all(m == 0 for m in g["mu_table"])   # the defect, as shipped


@pytest.mark.slow
def test_oracle_toy_network(golden):
    with open(os.path.join(HERE, "golden", "pipeline_golden.json")) as f:
        g = json.load(f)["ckks"]["toy/fast/giant/toy-fast"]
    from oracle.cpu_engine import OracleCkks
    from paper_2104_09164_b200.ckks.params import gen_params
    from paper_2104_09164_b200.fastpath import compile_pipeline, infer
    from paper_2104_09164_b200.model import (NetworkShape, collapse_layers, make_random_input,
                                             make_random_model)
    from paper_2104_09164_b200.modelenc import ModelEncoder
    shape = NetworkShape(1, 32, 15, (4, 8, 16), 4)
    cpar = collapse_layers(make_random_model(shape, 3), shape)
    be = OracleCkks(gen_params("toy-fast"), seed=5)
    cp = compile_pipeline(shape, "fast", "giant", be.params)
    be.ensure_rotation_keys(cp.rotations)
    lg, cnt, _ = infer(cpar, make_random_input(shape, 4), "fast", "giant", be,
                       encoder=ModelEncoder(cp, cpar, be))
    assert np.array_equal(lg, np.array(g["logits"]))
    assert cnt.as_dict() == g["counters"]

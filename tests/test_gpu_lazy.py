"""Lazy ModDown ("double hoisting"): hoisted rotations kept in the extended
basis Q*P, plaintext products accumulated there, P divided out once.

The reference divides P out after every rotation (hear/ckks/engine.py:
305-351) and then runs the mult_plain/add chain (hear/convolution.py:
276-312).  The lazy form must
  * hold exactly the rotated ciphertext: ModDown of every extended-basis
    rotation equals the eager rotation bit for bit (the eager one is pinned
    to the reference's digests in test_gpu_ckks.py);
  * accumulate exactly: every row of the extended accumulator, the special
    prime's included, equals the integer sum of products;
  * decrypt to the eager path's values up to rounding noise, with the same
    counters, through the conv layer and the whole network.
"""

from fractions import Fraction

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _mulmod(a, b, p):
    """a * b mod p on int64 tensors, a, b < p < 2^34 (17-bit split)."""
    bh, bl = b >> 17, b & ((1 << 17) - 1)
    return (((a * bh) % p << 17) + a * bl) % p


@pytest.fixture(scope="module")
def setup():
    import torch
    from paper_2104_09164_b200.ckks.engine import CkksBackend
    from paper_2104_09164_b200.ckks.params import gen_params
    be = CkksBackend(gen_params("fast-hear"), seed=11)
    assert be.lazy
    lvl, bsz, amounts = 7, 8, [1, 5, 33, 8190]
    be.ensure_rotation_keys({a: lvl for a in amounts})
    rng = np.random.default_rng(3)
    cts = [be.enc(rng.uniform(-1, 1, (bsz, be.n2)), level=lvl) for _ in range(2)]
    return be, lvl, bsz, amounts, cts, rng, torch


def test_extended_rotations_moddown_to_eager_bits(setup):
    be, lvl, bsz, amounts, cts, rng, torch = setup
    eager = be._raw_rot_many_each(cts, amounts)
    lazy = be._raw_rot_many_each_lazy(cts, amounts, True)
    for h, ct in enumerate(cts):
        for k in amounts:
            x = lazy[h][k].payload.xdata
            assert x.shape == (bsz, 2, lvl + 2, be.n)
            assert torch.equal(be._mod_down_ext(x, lvl), eager[h][k].payload.data), (h, k)
        # amount 0: P * ct, zero special row
        x0 = lazy[h][0].payload.xdata
        assert not x0[:, :, lvl + 1].any()
        assert torch.equal(be._mod_down_ext(x0, lvl), ct.payload.data)


def test_extended_accumulator_is_the_integer_sum(setup):
    be, lvl, bsz, amounts, cts, rng, torch = setup
    lazy = be._raw_rot_many_each_lazy(cts, amounts, True)
    terms = [(h, k) for h in range(2) for k in [0] + amounts]
    nout = 3
    pts = be.encode_many(rng.uniform(-1, 1, (nout * len(terms), be.n2)), lvl, be.params.msg_scale)
    jobs = [[(lazy[h][k], pts[o * len(terms) + t]) for t, (h, k) in enumerate(terms)]
            for o in range(nout)]
    (glvl, idx, acc), = be._mac_ext(jobs)
    assert glvl == lvl and idx == list(range(nout))
    primes = list(be.params.chain_primes[:lvl + 1]) + [be.params.special_prime]
    for o in range(nout):
        for r, p in enumerate(primes):
            want = torch.zeros(bsz, 2, be.n, dtype=torch.int64, device=acc.device)
            for t, (h, k) in enumerate(terms):
                pt = pts[o * len(terms) + t].payload[r]
                want = (want + _mulmod(lazy[h][k].payload.xdata[:, :, r], pt[None, None], p)) % p
            assert torch.equal(acc[o, :, :, r], want), (o, r)


def test_lazy_mac_decrypts_like_eager(setup):
    be, lvl, bsz, amounts, cts, rng, torch = setup
    ks = [0] + amounts
    w = rng.uniform(-1, 1, (2 * len(ks), be.n2))
    pts = be.encode_many(w, lvl, be.params.msg_scale)
    xs = [be.dec(c) for c in cts]
    clear = sum(w[h * len(ks) + q] * np.roll(xs[h], -k, axis=1)
                for h in range(2) for q, k in enumerate(ks))

    def run(lazy):
        be.reset_counters()
        pre = be.rot_many_each(cts, ks, lazy=lazy)
        is_ext = not hasattr(pre[0][ks[1]].payload, "data")
        assert is_ext == lazy
        out = be.mac_many([[(pre[h][k], pts[h * len(ks) + q]) for h in range(2)
                            for q, k in enumerate(ks)]])[0]
        return be.dec(be.rescale(out)), be.counters.as_dict()

    v_eager, c_eager = run(False)
    v_lazy, c_lazy = run(True)
    assert c_lazy == c_eager
    # both carry the key switch's own noise (~6e-5 at this scale); they differ
    # by the ModDown roundings (one per rotation eager, one per output lazy)
    err_e, err_l = np.abs(v_eager - clear).max(), np.abs(v_lazy - clear).max()
    assert err_e <= 2e-4 and err_l <= 2e-4, (err_e, err_l)
    assert np.abs(v_lazy - v_eager).max() <= 1e-4
    assert np.abs(clear).max() > 0.1


def test_extended_handles_fail_outside_accumulations(setup):
    be, lvl, bsz, amounts, cts, rng, torch = setup
    pre = be.rot_many_each(cts[:1], amounts[:1], lazy=True)
    with pytest.raises(AttributeError):
        be.add(pre[0][amounts[0]], pre[0][amounts[0]])


def test_network_lazy_vs_eager_and_reference():
    """1d-w64 fast/full at 8 clips: the lazy conv layers give the eager
    path's logits within 1e-4 of the logit scale, same argmax and counters,
    and clip 0 matches the reference's CKKS logits (pipeline_golden_r2)."""
    import json
    import os
    from paper_2104_09164_b200.ckks.engine import CkksBackend
    from paper_2104_09164_b200.ckks.params import gen_params
    from paper_2104_09164_b200.fastpath import compile_pipeline, infer
    from paper_2104_09164_b200.model import (collapse_layers, make_random_input, make_random_model,
                                             net_by_name)
    from paper_2104_09164_b200.modelenc import ModelEncoder
    here = os.path.dirname(os.path.abspath(__file__))
    with open(os.path.join(here, "golden", "pipeline_golden_r2.json")) as f:
        gold = json.load(f)["1d-w64/fast/full/fast-hear"]
    shape = net_by_name("1d-w64")
    cpar = collapse_layers(make_random_model(shape, gold["model_seed"]), shape)
    x = np.stack([make_random_input(shape, gold["input_seed"] + i) for i in range(8)])
    res = {}
    for lazy in (False, True):
        be = CkksBackend(gen_params("fast-hear"), seed=gold["backend_seed"])
        be.lazy = be.lazy and lazy          # plaintexts keep their special row either way
        cp = compile_pipeline(shape, "fast", "full", be.params)
        be.ensure_rotation_keys(cp.rotations)
        lg, cnt, _ = infer(cpar, x, "fast", "full", be, encoder=ModelEncoder(cp, cpar, be))
        res[lazy] = (lg, cnt.as_dict())
    (lg_e, c_e), (lg_l, c_l) = res[False], res[True]
    assert c_l == c_e == gold["counters"]
    scale = np.abs(lg_e).max()
    assert np.abs(lg_l - lg_e).max() <= 1e-4 * scale
    assert (np.argmax(lg_l, axis=1) == np.argmax(lg_e, axis=1)).all()
    ref = np.array(gold["logits"])
    assert np.abs(lg_l[0] - ref).max() <= 1e-3 * np.abs(ref).max()
    assert int(np.argmax(lg_l[0])) == int(np.argmax(ref))


def test_lazy_rotate_and_sum(setup):
    """Sum of hoisted rotations with ONE ModDown (fastpath.rotate_sum_each's odd
    part): the extended-basis sum is the exact modular sum of its terms, and
    the result decrypts like the eager sum with the same counters."""
    from paper_2104_09164_b200.fastpath import rotate_sum_each
    be, lvl, bsz, amounts, cts, rng, torch = setup
    lazy = be._raw_rot_many_each_lazy(cts, amounts, True)
    group = [lazy[0][k] for k in [0] + amounts]
    primes = list(be.params.chain_primes[:lvl + 1]) + [be.params.special_prime]
    pt = torch.tensor(primes, dtype=torch.int64, device=be.dev)[None, None, :, None]
    want = sum(c.payload.xdata for c in group) % pt
    got = be._raw_sum_each([group])[0]
    assert torch.equal(got.payload.data, be._mod_down_ext(want, lvl))
    # through the schedule: 5 entries spaced 33 -> odd part 5, one hoisted group
    be.ensure_rotation_keys({33 * j: lvl for j in range(1, 5)})
    res = {}
    for flag in (False, True):
        be.lazy = flag
        be.reset_counters()
        out = rotate_sum_each(cts, 5, 33, be)
        res[flag] = ([be.dec(c) for c in out], be.counters.as_dict())
    be.lazy = True
    assert res[True][1] == res[False][1]
    xs = [be.dec(c) for c in cts]
    for h in range(2):
        clear = sum(np.roll(xs[h], -33 * j, axis=1) for j in range(5))
        assert np.abs(res[True][0][h] - clear).max() <= 2e-4
        assert np.abs(res[True][0][h] - res[False][0][h]).max() <= 1e-4


def test_merged_moddown_rescale_bit_identical(setup):
    """ModDown merged with the rescale that follows it (one NTT per target row
    instead of two, FWD_MODDOWN2) gives the two separate steps' residues bit
    for bit: after a relinearisation (hear/ckks/engine.py:229-281 mult then
    rescale) and after an extended-basis accumulation."""
    be, lvl, bsz, amounts, cts, rng, torch = setup
    for fused in (True, False):
        be.fuse_ks_min = 0 if fused else 1 << 60
        want = be.rescale_each(be.square_each(cts))
        got = be.square_rescale_each(cts)
        for w, g in zip(want, got):
            assert (w.level, w.scale) == (g.level, g.scale)
            assert torch.equal(w.payload.data, g.payload.data)
    be.fuse_ks_min = 600
    ks = [0] + amounts
    pts = be.encode_many(rng.uniform(-1, 1, (2 * len(ks), be.n2)), lvl, be.params.msg_scale)
    lazy = be._raw_rot_many_each_lazy(cts, amounts, True)
    jobs = [[(lazy[h][k], pts[h * len(ks) + q]) for h in range(2) for q, k in enumerate(ks)]]
    want = be.rescale_each(be.mac_many(jobs))[0]
    be.reset_counters()
    got = be.mac_rescale_many(jobs)[0]
    assert (want.level, want.scale) == (got.level, got.scale)
    assert torch.equal(want.payload.data, got.payload.data)
    assert be.counters.total()["rescale"] == 1


def test_rot_sum_kernel_bit_identical_to_materialised_sum(setup, monkeypatch):
    """k_rot_sum_f64 (digits gathered through each Galois map, keys in the
    reference layout, sums in the extended basis, nothing materialised)
    equals the sum of the extended-basis rotations bit for bit, with the same
    counters as rot_many_each + sum_each."""
    be, lvl, bsz, amounts, cts, rng, torch = setup
    ks = [0] + amounts
    monkeypatch.setenv("HEAR_B200_ROT_SUM", "0")
    be.reset_counters()
    want = be.rot_sum_each(cts, ks)
    c_want = be.counters.as_dict()
    monkeypatch.setenv("HEAR_B200_ROT_SUM", "1")
    be.reset_counters()
    assert be._rot_sum_ok(cts, ks)
    got = be.rot_sum_each(cts, ks)
    assert be.counters.as_dict() == c_want
    for w, g in zip(want, got):
        assert (w.level, w.scale) == (g.level, g.scale)
        assert torch.equal(w.payload.data, g.payload.data)


def test_lazy_rot_each_extended_rotations(setup):
    """rot_each(lazy=True): the fused key switch scatters through the Galois
    map and adds P*c0, leaving each rotation in the extended basis; its
    ModDown equals the eager rotation bit for bit, and a mixed sum (the
    unrotated handle joins as P*ct) decrypts like the eager sum."""
    be, lvl, bsz, amounts, cts, rng, torch = setup
    items = [(cts[0], amounts[0]), (cts[1], amounts[1]), (cts[0], amounts[2])]
    old = be.fuse_ks_min
    try:
        be.fuse_ks_min = 0
        eager = be.rot_each(items)
        lazy = be.rot_each(items, lazy=True)
        for e, l in zip(eager, lazy):
            assert not hasattr(l.payload, "data")
            assert torch.equal(be._mod_down_ext(l.payload.xdata, lvl), e.payload.data)
        be.reset_counters()
        s_lazy = be.sum_each([[cts[0], lazy[0], lazy[2]]])[0]
        c_lazy = be.counters.as_dict()
        be.reset_counters()
        s_eager = be.sum_each([[cts[0], eager[0], eager[2]]])[0]
        assert be.counters.as_dict() == c_lazy
        assert np.abs(be.dec(s_lazy) - be.dec(s_eager)).max() <= 1e-4
    finally:
        be.fuse_ks_min = old


def test_lazy_rotations_at_small_batch():
    """Below the GEMM's batch threshold the extended-basis rotations come from
    the per-job inner product kernel with the same rotation epilogue: their
    ModDown equals the eager rotations bit for bit (1 and 3 clips)."""
    import torch
    from paper_2104_09164_b200.ckks.engine import CkksBackend
    from paper_2104_09164_b200.ckks.params import gen_params
    be = CkksBackend(gen_params("fast-hear"), seed=2)
    be.lazy_min = 1
    lvl, amounts = 5, [2, 11, 8191]
    be.ensure_rotation_keys({a: lvl for a in amounts})
    rng = np.random.default_rng(8)
    for bsz in (1, 3):
        assert bsz < be.ks_gemm_min
        cts = [be.enc(rng.uniform(-1, 1, (bsz, be.n2)), level=lvl) for _ in range(2)]
        eager = be._raw_rot_many_each(cts, amounts)
        pre = be.rot_many_each(cts, [0] + amounts, lazy=True)
        for h in range(2):
            for k in amounts:
                x = pre[h][k].payload.xdata
                assert torch.equal(be._mod_down_ext(x, lvl), eager[h][k].payload.data), (bsz, h, k)

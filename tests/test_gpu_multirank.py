"""Receiver side of the setup-time key replication (parallel.replicate_keys)
with the real engine on one GPU: a keygen=False CkksBackend filled through
alloc_keys + the sender's key_tensors + finish_keys must evaluate key
switches bit-exactly like the sender, and must encrypt from its own random
stream (not the sender's keygen stream)."""


import numpy as np
import pytest

from tests._util import rand_ct

pytestmark = pytest.mark.gpu


def _pair():
    from paper_2104_09164_b200.ckks.engine import CkksBackend, key_layout
    from paper_2104_09164_b200.ckks.params import gen_params
    from paper_2104_09164_b200.fastpath import compile_pipeline
    from paper_2104_09164_b200.model import NetworkShape
    ps = gen_params("toy-fast")
    shape = NetworkShape(1, 32, 15, (4, 8, 16), 4)
    cp = compile_pipeline(shape, "fast", "giant", ps)
    snd = CkksBackend(ps, seed=0)
    snd.ensure_rotation_keys(cp.rotations)
    rcv = CkksBackend(ps, seed=0, keygen=False, enc_seed=np.random.SeedSequence(0, spawn_key=(1,)))
    man = snd.key_manifest()
    rcv.alloc_keys(man)
    src, dst = snd.key_tensors(), rcv.key_tensors()
    assert [(n, tuple(t.shape)) for n, t in src] == [(n, tuple(t.shape)) for n, t in dst] \
        == [(n, tuple(s)) for n, s in key_layout(ps, man)]
    for (_, s), (_, d) in zip(src, dst):   # what the NCCL broadcast does
        d.copy_(s)
    rcv.finish_keys()
    return ps, cp, shape, snd, rcv


def test_receiver_key_switches_bit_exact():
    ps, cp, _, snd, rcv = _pair()
    lvl = ps.max_level
    c = rand_ct(ps, lvl, 41)
    a_s = snd.import_ct(*c, lvl, ps.msg_scale)
    a_r = rcv.import_ct(*c, lvl, ps.msg_scale)
    amounts = sorted(k for k, l in cp.rotations.items() if l >= lvl)[:4]
    rs, rr = snd.rot_many(a_s, amounts), rcv.rot_many(a_r, amounts)
    for k in amounts:
        for x, y in zip(snd.export(rs[k]), rcv.export(rr[k])):
            assert np.array_equal(x, y), k
    for x, y in zip(snd.export(snd.mult(a_s, a_s)), rcv.export(rcv.mult(a_r, a_r))):
        assert np.array_equal(x, y)


def test_receiver_encrypts_from_its_own_stream():
    _, _, _, snd, rcv = _pair()
    u = rcv._ternary()
    assert not np.array_equal(u, snd.keys.s_coeffs)


def test_receiver_evaluates_network_sender_decrypts():
    """Clips encrypted and evaluated on the receiving rank (public material
    only) decrypt under the sender's secret key to the clear logits."""
    from paper_2104_09164_b200.fastpath import dec_logits, encrypt_input, run_pipeline
    from paper_2104_09164_b200.model import (collapse_layers, infer_clear, make_random_input,
                                             make_random_model)
    from paper_2104_09164_b200.modelenc import ModelEncoder
    ps, cp, shape, snd, rcv = _pair()
    cpar = collapse_layers(make_random_model(shape, 3), shape)
    x = np.stack([make_random_input(shape, s) for s in (4, 5)])
    enc = ModelEncoder(cp, cpar, rcv).prepare()
    out = run_pipeline(enc, encrypt_input(x, cp, rcv), rcv)
    lg = dec_logits(out, cp, snd)
    ref = np.stack([infer_clear(cpar, xi) for xi in x])
    assert np.abs(lg - ref).max() <= 2.0 ** -5 * max(1.0, np.abs(ref).max())

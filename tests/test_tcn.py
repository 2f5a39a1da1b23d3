"""BASELINE configs 0 and 3 (temporal conv networks outside the reference's
NetworkShape family): the encrypted schedule of paper_2104_09164_b200.tcn on
the exact slot simulator (oracle/slotsim.py) against the cleartext network,
for single clips and batches, plus the shape validation and the level
budget."""

import numpy as np
import pytest

from oracle.slotsim import SimBackend
from paper_2104_09164_b200.ckks.params import gen_params, tcn_ring16
from paper_2104_09164_b200.tcn import (TCN_WEIGHT_STD, ConvSpec, TcnShape, compile_tcn,
                                       infer_clear_tcn, infer_tcn, make_random_clip,
                                       make_random_tcn, tcn_by_name)

CASES = [("config0", "fast-hear"), ("config3", "tcn16")]


def _params(which):
    return tcn_ring16() if which == "tcn16" else gen_params(which)


@pytest.mark.parametrize("net,prof", CASES)
def test_sim_matches_clear(net, prof):
    shape = tcn_by_name(net)
    tp = make_random_tcn(shape, 1, TCN_WEIGHT_STD[net])
    be = SimBackend(_params(prof))
    x = make_random_clip(shape, 2)
    lg, cnt, enc = infer_tcn(tp, x, be)
    clear = infer_clear_tcn(tp, x)
    assert np.abs(lg - clear).max() <= 1e-12 * max(1.0, np.abs(clear).max())
    xb = np.stack([make_random_clip(shape, s) for s in (3, 4, 5)])
    lb, _, _ = infer_tcn(tp, xb, be, encoder=enc)
    assert np.abs(lb - np.stack([infer_clear_tcn(tp, xi) for xi in xb])).max() <= 1e-12


def test_config0_clear_network_by_hand():
    """The clear oracle itself: conv1d k=8 stride 2 over the 30 channels,
    square, global average, FC -- against an explicit loop."""
    shape = tcn_by_name("config0")
    tp = make_random_tcn(shape, 7, 0.1)
    x = make_random_clip(shape, 8)
    xc = np.array([[x[t, c // 2, c % 2] for t in range(32)] for c in range(30)])
    tout = (32 - 8) // 2 + 1
    feat = np.zeros(32)
    for f in range(32):
        for t in range(tout):
            y = sum(tp.filters[0][f, c, k] * xc[c, 2 * t + k] for c in range(30) for k in range(8))
            feat[f] += y * y / tout
    assert np.allclose(tp.fc_w @ feat, infer_clear_tcn(tp, x), atol=1e-12)


def test_level_budget_and_rotations():
    p0 = compile_tcn(tcn_by_name("config0"), gen_params("fast-hear"))
    assert p0.levels_used == 4
    p3 = compile_tcn(tcn_by_name("config3"), tcn_ring16())
    assert p3.levels_used == 8 == tcn_ring16().max_level
    with pytest.raises(ValueError, match="levels"):
        compile_tcn(tcn_by_name("config3"), gen_params("toy-hear").__class__(
            **{**gen_params("toy-hear").__dict__, "chain_primes": gen_params("toy-hear").chain_primes[:5]}))
    assert all(a < p0.params.n2 for a in p0.rotations)


def test_shape_validation():
    with pytest.raises(ValueError):
        TcnShape(32, 15, (ConvSpec(40, 8),), ("square",), 5)       # kernel longer than clip
    with pytest.raises(ValueError):
        TcnShape(32, 15, (ConvSpec(8, 8),), ("relu",), 5)
    with pytest.raises(ValueError):
        TcnShape(32, 15, (ConvSpec(8, 8),), ("square", "square"), 5)

"""Fused ModUp + key-switch inner product (csrc/ntt3.cu k_ks3, accumulators in
tensor memory) against the unfused path (digit expansion + GEMM), which is
itself pinned to the reference's digests (test_gpu_ckks.py) and to the CPU
oracle (test_gpu_bigring.py).  Every key switch that takes the fused kernel
must give the same ciphertext bit for bit: hear/ckks/engine.py:290-351
(relinearisation, rotation) are exact integer maps.
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _pair(prof, seed=5):
    from paper_2104_09164_b200.ckks import params as P
    from paper_2104_09164_b200.ckks.engine import CkksBackend
    ps = {"ring15": lambda: P.fast_hear_ring(15), "ring16": P.tcn_ring16}.get(
        prof, lambda: P.gen_params(prof))()
    be = CkksBackend(ps, seed=seed)
    assert be.fuse_ks
    return be


@pytest.mark.parametrize("prof,lvl,bsz", [("fast-hear", 12, 3), ("fast-hear", 5, 8),
                                          ("fast-hear", 1, 40), ("ring15", 4, 2),
                                          ("ring16", 3, 2)])
def test_fused_key_switches_bit_identical(prof, lvl, bsz):
    import torch
    be = _pair(prof)
    amounts = [1, 7]
    be.ensure_rotation_keys({a: lvl for a in amounts})
    rng = np.random.default_rng(1)
    cts = [be.enc(rng.uniform(-1, 1, (bsz, be.n2)), level=lvl) for _ in range(3)]

    def run(fused):
        be.fuse_ks_min = 0 if fused else 1 << 60
        return {
            "mult": [be.mult(cts[0], cts[1])],
            "square_each": be.square_each(cts),
            "rot_each": be.rot_each([(cts[0], 1), (cts[1], 7), (cts[2], 1)]),
            "rot_add_each": be.rot_add_each([(cts[0], 7), (cts[2], 1)]),
        }

    want, got = run(False), run(True)
    for name in want:
        for w, g in zip(want[name], got[name]):
            assert (w.level, w.scale) == (g.level, g.scale)
            assert torch.equal(w.payload.data, g.payload.data), name


def test_fused_launch_is_taken():
    """The fused kernel really runs (launch accounting) at bench-like sizes."""
    from paper_2104_09164_b200.ckks.ring import StepStats, set_step_stats
    be = _pair("fast-hear")
    lvl, bsz = 3, 128
    cts = [be.enc(np.zeros((bsz, be.n2)), level=lvl) for _ in range(2)]
    st = StepStats()
    set_step_stats(st)
    try:
        be.square_each(cts)
    finally:
        set_step_stats(None)
    assert st.fam["keyswitch_fused"]["launches"] == 1
    assert "ntt_fwd_modup_lift" not in st.fam and "keyswitch_gemm" not in st.fam


@pytest.mark.parametrize("lvl,handles", [(12, 1), (3, 4)])
def test_fused_key_switch_deterministic_under_load(lvl, handles):
    """k_ks3 with every SM busy (128 clips per handle: thousands of clusters
    looping over the digits, four CTAs per SM sharing the tensor memory) is
    deterministic and equals the unfused path bit for bit.  Guards the
    per-digit barrier / mbarrier-phase protocol and the TMEM column
    ownership: an error there corrupts a few rows only under load."""
    import torch
    be = _pair("fast-hear")
    rng = np.random.default_rng(4)
    cts = [be.enc(rng.uniform(-1, 1, (128, be.n2)), level=lvl) for _ in range(handles)]
    be.ensure_rotation_keys({5: lvl})
    be.fuse_ks_min = 1 << 60
    want_sq = [c.payload.data.clone() for c in be.square_each(cts)]
    want_ra = [c.payload.data.clone() for c in be.rot_add_each([(c, 5) for c in cts])]
    be.fuse_ks_min = 0
    for _ in range(4):
        got_sq = be.square_each(cts)
        got_ra = be.rot_add_each([(c, 5) for c in cts])
        lazy = be.rot_each([(c, 5) for c in cts], lazy=True)
        for w, g in zip(want_sq, got_sq):
            assert torch.equal(w, g.payload.data)
        for w, g in zip(want_ra, got_ra):
            assert torch.equal(w, g.payload.data)
        for c, l, w in zip(cts, lazy, want_ra):   # ModDown(ext rotation) + ct == rot_add
            md = be._mod_down_ext(l.payload.xdata, lvl)
            rot = be._raw_add_each([(c, type(c)(type(c.payload)(md), lvl, c.scale, be.n2))])[0]
            assert torch.equal(rot.payload.data, w)

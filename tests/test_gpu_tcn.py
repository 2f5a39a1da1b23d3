"""BASELINE configs 0 and 3 on the GPU engine: the temporal networks of
paper_2104_09164_b200.tcn encrypted, evaluated and decrypted on the B200,
against the cleartext network (max |d| <= 1e-3 x logit scale, same argmax),
with the per-layer counters of the slot-simulator schedule; config 0 also
against the CPU oracle engine at toy parameters, and as a CUDA-graph
replay bit-identical to eager evaluation."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _model(net):
    from paper_2104_09164_b200.tcn import TCN_WEIGHT_STD, make_random_tcn, tcn_by_name
    shape = tcn_by_name(net)
    return shape, make_random_tcn(shape, 1, TCN_WEIGHT_STD[net])


def _sim_counters(tp, x, params):
    from oracle.slotsim import SimBackend
    from paper_2104_09164_b200.tcn import infer_tcn
    _, cnt, _ = infer_tcn(tp, x, SimBackend(params))
    return cnt.as_dict()


@pytest.mark.parametrize("net,prof", [("config0", "fast-hear"), ("config3", "tcn16")])
def test_tcn_matches_clear(net, prof):
    from paper_2104_09164_b200.ckks.engine import CkksBackend
    from paper_2104_09164_b200.ckks.params import gen_params, tcn_ring16
    from paper_2104_09164_b200.tcn import (TcnEncoder, compile_tcn, infer_clear_tcn, infer_tcn,
                                           make_random_clip)
    ps = tcn_ring16() if prof == "tcn16" else gen_params(prof)
    shape, tp = _model(net)
    be = CkksBackend(ps, seed=0)
    plan = compile_tcn(shape, ps)
    be.ensure_rotation_keys(plan.rotations)
    enc = TcnEncoder(plan, tp, be).prepare()
    x = np.stack([make_random_clip(shape, s) for s in (2, 3, 4)])
    be.reset_counters()
    lg, cnt, _ = infer_tcn(tp, x, be, encoder=enc)
    clear = np.stack([infer_clear_tcn(tp, xi) for xi in x])
    scale = np.abs(clear).max()
    assert np.abs(lg - clear).max() <= 1e-3 * scale, (lg, clear)
    assert (np.argmax(lg, 1) == np.argmax(clear, 1)).all()
    assert cnt.as_dict() == _sim_counters(tp, x[0], ps)


def test_config0_vs_cpu_oracle_toy():
    """GPU engine vs the CPU oracle engine on the same seeds (toy-fast):
    same counters, decrypted logits within 1e-3 x scale."""
    from oracle.cpu_engine import OracleCkks
    from paper_2104_09164_b200.ckks.engine import CkksBackend
    from paper_2104_09164_b200.ckks.params import gen_params
    from paper_2104_09164_b200.tcn import TcnEncoder, compile_tcn, infer_tcn, make_random_clip
    ps = gen_params("toy-fast")
    shape, tp = _model("config0")
    x = make_random_clip(shape, 9)
    res = []
    for be in (CkksBackend(ps, seed=5), OracleCkks(ps, seed=5)):
        plan = compile_tcn(shape, ps)
        be.ensure_rotation_keys(plan.rotations)
        lg, cnt, _ = infer_tcn(tp, x, be, encoder=TcnEncoder(plan, tp, be))
        res.append((lg, cnt.as_dict()))
    (lg_g, c_g), (lg_c, c_c) = res
    assert c_g == c_c
    assert np.abs(lg_g - lg_c).max() <= 1e-3 * np.abs(lg_c).max()
    assert int(np.argmax(lg_g)) == int(np.argmax(lg_c))


def test_config0_graph_bit_identical():
    import torch
    from paper_2104_09164_b200.ckks.engine import CkksBackend
    from paper_2104_09164_b200.ckks.params import gen_params
    from paper_2104_09164_b200.fastpath import GraphedPipeline
    from paper_2104_09164_b200.tcn import (TcnEncoder, compile_tcn, encrypt_tcn_input,
                                           make_random_clip, run_tcn)
    ps = gen_params("fast-hear")
    shape, tp = _model("config0")
    be = CkksBackend(ps, seed=1)
    plan = compile_tcn(shape, ps)
    be.ensure_rotation_keys(plan.rotations)
    enc = TcnEncoder(plan, tp, be).prepare()
    ct = encrypt_tcn_input(np.stack([make_random_clip(shape, 20 + i) for i in range(8)]), plan, be)
    want = run_tcn(enc, ct, be).payload.data.clone()
    g = GraphedPipeline(enc, be, batch=8, run=run_tcn)
    for _ in range(2):
        got = g(ct).payload.data
        torch.cuda.synchronize()
        assert torch.equal(got, want)

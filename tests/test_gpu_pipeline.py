"""Encrypted HEAR-CNN inference on the GPU engine vs the reference.

Decrypted logits must match the reference CKKS engine's decrypted logits
(same model/input/key seeds; tests/golden/pipeline_golden.json) within
1e-3 x logit scale with the same argmax, per-layer operation counters must
equal the reference's exactly, and batched evaluation must be bit-identical
to clip-by-clip evaluation.
"""

import json
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.fixture(scope="module")
def pgold():
    with open(os.path.join(HERE, "golden", "pipeline_golden.json")) as f:
        return json.load(f)


def _run(shape, model_seed, input_seed, prof, mode, strat, backend_seed, batch=None):
    from paper_2104_09164_b200.ckks.engine import CkksBackend
    from paper_2104_09164_b200.ckks.params import gen_params
    from paper_2104_09164_b200.fastpath import compile_pipeline, infer
    from paper_2104_09164_b200.model import collapse_layers, make_random_input, make_random_model
    from paper_2104_09164_b200.modelenc import ModelEncoder
    cpar = collapse_layers(make_random_model(shape, model_seed), shape)
    be = CkksBackend(gen_params(prof), seed=backend_seed)
    cp = compile_pipeline(shape, mode, strat, be.params)
    be.ensure_rotation_keys(cp.rotations)
    x = make_random_input(shape, input_seed)
    if batch:
        x = np.stack([make_random_input(shape, input_seed + i) for i in range(batch)])
    lg, cnt, enc = infer(cpar, x, mode, strat, be, encoder=ModelEncoder(cp, cpar, be))
    return lg, cnt, cpar, x, be


def _check(lg, gold):
    ref = np.array(gold["logits"])
    scale = max(np.abs(ref).max(), 1e-12)
    assert np.abs(lg - ref).max() <= 1e-3 * scale, (lg, ref)
    assert int(np.argmax(lg)) == int(np.argmax(ref))


def test_toy_network_matches_reference(pgold):
    from paper_2104_09164_b200.model import NetworkShape
    g = pgold["ckks"]["toy/fast/giant/toy-fast"]
    shape = NetworkShape(1, 32, 15, (4, 8, 16), 4)
    lg, cnt, *_ = _run(shape, 3, 4, "toy-fast", "fast", "giant", 5)
    _check(lg, g)
    assert cnt.as_dict() == g["counters"]


@pytest.mark.parametrize("key", ["1d-w64/fast/giant/fast-hear", "1d-w64/hear/full/hear"])
def test_real_params_match_reference(pgold, key):
    from paper_2104_09164_b200.model import net_by_name
    net, mode, strat, prof = key.split("/")
    g = pgold["ckks"][key]
    lg, cnt, *_ = _run(net_by_name(net), 1, 2, prof, mode, strat, 0)
    _check(lg, g)
    assert cnt.as_dict() == g["counters"]
    clear = np.array(g["clear"])
    tol = 2.0 ** -9 if mode == "hear" else 2.0 ** -5
    assert np.abs(lg - clear).max() <= tol


def test_batched_equals_clipwise():
    """B clips in one handle == the same clips one by one (same RNG order)."""
    from paper_2104_09164_b200.model import NetworkShape
    shape = NetworkShape(1, 32, 15, (4, 8, 16), 4)
    lg_b, *_ = _run(shape, 3, 10, "toy-fast", "fast", "baby", 9, batch=3)
    from paper_2104_09164_b200.ckks.engine import CkksBackend
    from paper_2104_09164_b200.ckks.params import gen_params
    from paper_2104_09164_b200.fastpath import compile_pipeline, encrypt_input, run_pipeline, dec_logits
    from paper_2104_09164_b200.model import collapse_layers, make_random_input, make_random_model
    from paper_2104_09164_b200.modelenc import ModelEncoder
    cpar = collapse_layers(make_random_model(shape, 3), shape)
    be = CkksBackend(gen_params("toy-fast"), seed=9)
    cp = compile_pipeline(shape, "fast", "baby", be.params)
    be.ensure_rotation_keys(cp.rotations)
    enc = ModelEncoder(cp, cpar, be)
    cts = [encrypt_input(make_random_input(shape, 10 + i), cp, be) for i in range(3)]
    outs = [dec_logits(run_pipeline(enc, c, be), cp, be) for c in cts]
    assert np.array_equal(np.stack(outs), lg_b)


def test_cuda_graph_replay_bit_exact():
    """A captured pipeline replays to the same ciphertext as eager evaluation."""
    import torch
    from paper_2104_09164_b200.ckks.engine import CkksBackend
    from paper_2104_09164_b200.ckks.params import gen_params
    from paper_2104_09164_b200.fastpath import (GraphedPipeline, compile_pipeline, dec_logits,
                                                encrypt_input, run_pipeline)
    from paper_2104_09164_b200.model import (NetworkShape, collapse_layers, make_random_input,
                                             make_random_model)
    from paper_2104_09164_b200.modelenc import ModelEncoder
    shape = NetworkShape(1, 32, 15, (4, 8, 16), 4)
    cpar = collapse_layers(make_random_model(shape, 3), shape)
    be = CkksBackend(gen_params("toy-fast"), seed=2)
    cp = compile_pipeline(shape, "fast", "full", be.params)
    be.ensure_rotation_keys(cp.rotations)
    enc = ModelEncoder(cp, cpar, be).prepare()
    g = GraphedPipeline(enc, be, batch=2)
    for seed in (20, 30):
        x = np.stack([make_random_input(shape, seed + i) for i in range(2)])
        ct = encrypt_input(x, cp, be)
        eager = run_pipeline(enc, ct, be).payload.data.clone()
        replay = g(ct).payload.data
        torch.cuda.synchronize()
        assert torch.equal(eager, replay)


def test_graph_with_pdl_bit_identical():
    """CUDA-graph replay with programmatic dependent launch (HEAR_B200_PDL=1)
    is bit-identical to eager evaluation."""
    import os
    import torch
    from paper_2104_09164_b200.ckks.engine import CkksBackend
    from paper_2104_09164_b200.ckks.params import gen_params
    from paper_2104_09164_b200.fastpath import (GraphedPipeline, compile_pipeline, encrypt_input,
                                                run_pipeline)
    from paper_2104_09164_b200.model import (collapse_layers, make_random_input, make_random_model,
                                             net_by_name)
    from paper_2104_09164_b200.modelenc import ModelEncoder
    shape = net_by_name("1d-w64")
    cpar = collapse_layers(make_random_model(shape, 1), shape)
    be = CkksBackend(gen_params("fast-hear"), seed=3)
    cp = compile_pipeline(shape, "fast", "full", be.params)
    be.ensure_rotation_keys(cp.rotations)
    enc = ModelEncoder(cp, cpar, be).prepare()
    ct = encrypt_input(np.stack([make_random_input(shape, 50 + i) for i in range(8)]), cp, be)
    want = run_pipeline(enc, ct, be).payload.data.clone()
    os.environ["HEAR_B200_PDL"] = "1"
    try:
        g = GraphedPipeline(enc, be, batch=8)
    finally:
        del os.environ["HEAR_B200_PDL"]
    for _ in range(2):
        got = g(ct).payload.data
        torch.cuda.synchronize()
        assert torch.equal(got, want)


@pytest.fixture(scope="module")
def pgold2():
    with open(os.path.join(HERE, "golden", "pipeline_golden_r2.json")) as f:
        return json.load(f)


R2_KEYS = ["1d-w64/fast/full/fast-hear", "2d-w64/fast/giant/fast-hear", "2d-w64/hear/full/hear",
           "2d-w128/fast/full/fast-hear"]


@pytest.mark.parametrize("key", R2_KEYS)
def test_r2_networks_match_reference(pgold2, key):
    """The bench headline configuration and the 2D networks against the
    reference CKKS engine's decrypted logits (tests/golden/make_golden_r2.py)."""
    from paper_2104_09164_b200.model import net_by_name
    if key not in pgold2:
        pytest.skip(f"{key}: golden not generated")
    net, mode, strat, prof = key.split("/")
    g = pgold2[key]
    lg, cnt, *_ = _run(net_by_name(net), g["model_seed"], g["input_seed"], prof, mode, strat,
                       g["backend_seed"])
    _check(lg, g)
    assert cnt.as_dict() == g["counters"]
    tol = 2.0 ** -9 if mode == "hear" else 2.0 ** -5
    assert np.abs(lg - np.array(g["clear"])).max() <= tol


def test_headline_graph_b128_matches_eager_and_reference(pgold2):
    """The bench's timed object: 1d-w64 fast/full at fast-hear, 128 clips per
    handle, replayed as the DEFAULT CUDA graph (no PDL).  The replay is
    bit-identical to eager evaluation, and clip 0 (the golden's seeds)
    decrypts to the reference CKKS engine's logits."""
    import torch
    from paper_2104_09164_b200.ckks.engine import CkksBackend
    from paper_2104_09164_b200.ckks.params import gen_params
    from paper_2104_09164_b200.fastpath import (GraphedPipeline, compile_pipeline, dec_logits,
                                                encrypt_input, run_pipeline)
    from paper_2104_09164_b200.model import (collapse_layers, make_random_input, make_random_model,
                                             net_by_name)
    from paper_2104_09164_b200.modelenc import ModelEncoder
    g = pgold2["1d-w64/fast/full/fast-hear"]
    shape = net_by_name("1d-w64")
    cpar = collapse_layers(make_random_model(shape, g["model_seed"]), shape)
    be = CkksBackend(gen_params("fast-hear"), seed=g["backend_seed"])
    cp = compile_pipeline(shape, "fast", "full", be.params)
    be.ensure_rotation_keys(cp.rotations)
    enc = ModelEncoder(cp, cpar, be).prepare()
    x = np.stack([make_random_input(shape, g["input_seed"] + i) for i in range(128)])
    ct = encrypt_input(x, cp, be)
    be.reset_counters()
    eager = run_pipeline(enc, ct, be)
    assert be.counters.as_dict() == g["counters"]
    want = eager.payload.data.clone()
    assert os.environ.get("HEAR_B200_PDL", "0") == "0"
    graph = GraphedPipeline(enc, be, batch=128)
    for _ in range(2):
        got = graph(ct)
        torch.cuda.synchronize()
        assert torch.equal(got.payload.data, want)
    lg = dec_logits(got, cp, be)
    _check(lg[0], g)

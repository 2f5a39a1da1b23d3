"""Network schedule on the exact slot simulator (CPU): equivalence with the
cleartext network and with the reference's simulator logits, and exact
per-layer operation counters against the reference (pipeline_golden.json)."""

import json
import os

import numpy as np
import pytest

from oracle.slotsim import SimBackend
from paper_2104_09164_b200.ckks.params import gen_params
from paper_2104_09164_b200.fastpath import compile_pipeline, infer
from paper_2104_09164_b200.model import (collapse_layers, infer_clear, make_random_input,
                                         make_random_model, net_by_name)
from paper_2104_09164_b200.modelenc import ModelEncoder

HERE = os.path.dirname(os.path.abspath(__file__))
with open(os.path.join(HERE, "golden", "pipeline_golden.json")) as _f:
    GOLD = json.load(_f)

CASES = [(net, mode, strat) for net in ("1d-w64", "1d-w128", "2d-w64")
         for mode in ("hear", "fast") for strat in ("full", "giant", "baby")]


@pytest.mark.parametrize("net,mode,strat", CASES)
def test_sim_matches_reference(net, mode, strat):
    g = GOLD["sim"][f"{net}/{mode}/{strat}"]
    shape = net_by_name(net)
    cpar = collapse_layers(make_random_model(shape, 1), shape)
    x = make_random_input(shape, 2)
    be = SimBackend(gen_params("hear" if mode == "hear" else "fast-hear"))
    lg, cnt, _ = infer(cpar, x, mode, strat, be)
    assert np.abs(lg - infer_clear(cpar, x)).max() <= 1e-9
    assert np.abs(lg - np.array(g["logits"])).max() <= 1e-9
    assert np.allclose(infer_clear(cpar, x), g["clear"], atol=1e-12)
    assert cnt.as_dict() == g["counters"]


@pytest.mark.slow
@pytest.mark.parametrize("mode", ["hear", "fast"])
def test_sim_2d_w128(mode):
    g = GOLD["sim"][f"2d-w128/{mode}/giant"]
    shape = net_by_name("2d-w128")
    cpar = collapse_layers(make_random_model(shape, 1), shape)
    x = make_random_input(shape, 2)
    be = SimBackend(gen_params("hear" if mode == "hear" else "fast-hear"))
    lg, cnt, _ = infer(cpar, x, mode, "giant", be)
    assert cnt.as_dict() == g["counters"]
    assert np.abs(lg - infer_clear(cpar, x)).max() <= 1e-9


def test_table_viii_totals():
    """2D-CNN-W128 Fast-HEAR: Mult = 56, Rescale = 172 (paper Table VIII)."""
    c = GOLD["sim"]["2d-w128/fast/giant"]["counters"]
    tot = {k: sum(row[k] for row in c.values()) for k in next(iter(c.values()))}
    assert tot["mult"] == 56 and tot["rescale"] == 172


def test_batched_sim_equals_clipwise():
    shape = net_by_name("1d-w64")
    cpar = collapse_layers(make_random_model(shape, 1), shape)
    xs = np.stack([make_random_input(shape, 5 + i) for i in range(3)])
    be = SimBackend(gen_params("fast-hear"))
    lg, *_ = infer(cpar, xs, "fast", "giant", be)
    for i in range(3):
        one, *_ = infer(cpar, xs[i], "fast", "giant", SimBackend(gen_params("fast-hear")))
        assert np.abs(lg[i] - one).max() <= 1e-12


@pytest.mark.parametrize("key", sorted(GOLD["storage"]))
def test_level_aware_storage(key):
    net, mode = key.split("/")
    prof = "hear" if mode == "hear" else "fast-hear"
    shape = net_by_name(net)
    cp = compile_pipeline(shape, mode, "giant", gen_params(prof))
    rep = ModelEncoder(cp, collapse_layers(make_random_model(shape, 1), shape),
                       SimBackend(gen_params(prof))).storage_report()
    assert rep == GOLD["storage"][key]
    assert rep["ratio"] < 0.6


def test_ladders():
    cp = compile_pipeline(net_by_name("2d-w128"), "hear", "giant", gen_params("hear"))
    assert cp.ladder_levels() == [10, 9, 8, 7, 7, 6, 5, 4, 4, 3, 2, 1, 0]
    cp = compile_pipeline(net_by_name("2d-w128"), "fast", "giant", gen_params("fast-hear"))
    assert cp.ladder_levels()[0] == 12 and cp.ladder_levels()[-1] == 0
    assert cp.expected("merge2").level == 8 and cp.expected("merge3").level == 4


def test_batched_contract_forms_on_simulator():
    """rot_many_each / rot_add_each / sum_each are the plain op sequences:
    same slot values and the same operation counters (slot simulator)."""
    rng = np.random.default_rng(3)
    be = SimBackend(gen_params("fast-hear"))
    cts = [be.enc(rng.uniform(-1, 1, be.n2), level=6) for _ in range(3)]
    be.reset_counters()
    many = be.rot_many_each(cts, [1, 5, 0])
    c_many = be.counters.as_dict()
    be.reset_counters()
    single = [be.rot_many(c, [1, 5, 0]) for c in cts]
    assert be.counters.as_dict() == c_many
    for m, s_ in zip(many, single):
        for k in (1, 5, 0):
            assert np.array_equal(be.dec(m[k]), be.dec(s_[k]))
    be.reset_counters()
    fused = be.rot_add_each([(c, 7) for c in cts])
    c_fused = be.counters.as_dict()
    be.reset_counters()
    plain = be.add_each(list(zip(cts, be.rot_each([(c, 7) for c in cts]))))
    assert be.counters.as_dict() == c_fused
    for f, p_ in zip(fused, plain):
        assert np.array_equal(be.dec(f), be.dec(p_))
    be.reset_counters()
    sums = be.sum_each([cts, cts[:2], cts[2:]])
    assert sum(v.get("add", 0) for v in be.counters.as_dict().values()) == 3
    assert np.allclose(be.dec(sums[0]), sum(be.dec(c) for c in cts))


def test_lazy_contract_forms_are_the_plain_sequences_on_simulator():
    """The forms that let the GPU engine defer / merge ModDowns --
    rot_many_each(lazy), rot_each(lazy), rot_sum_each, mac_rescale_many,
    square_rescale_each -- are, on an engine without those fast paths, exactly
    the reference's op sequences: same slot values, same counters
    (hear/convolution.py:276-312, hear/fastpath.py:123-154)."""
    rng = np.random.default_rng(5)
    be = SimBackend(gen_params("fast-hear"))
    lvl = 6
    cts = [be.enc(rng.uniform(-1, 1, be.n2), level=lvl) for _ in range(2)]
    pts = [be.encode(rng.uniform(-1, 1, be.n2), lvl, be.params.msg_scale) for _ in range(6)]
    ks = [0, 3, 9]

    def counted(fn):
        be.reset_counters()
        out = fn()
        return out, be.counters.as_dict()

    lazy, c1 = counted(lambda: be.rot_many_each(cts, ks, lazy=True))
    plain, c2 = counted(lambda: be.rot_many_each(cts, ks))
    assert c1 == c2
    for a, b in zip(lazy, plain):
        for k in ks:
            assert np.array_equal(be.dec(a[k]), be.dec(b[k]))
    items = [(cts[0], 3), (cts[1], 0), (cts[1], 9)]
    a, c1 = counted(lambda: be.rot_each(items, lazy=True))
    b, c2 = counted(lambda: be.rot_each(items))
    assert c1 == c2 and all(np.array_equal(be.dec(x), be.dec(y)) for x, y in zip(a, b))
    a, c1 = counted(lambda: be.rot_sum_each(cts, ks))
    b, c2 = counted(lambda: be.sum_each([[r[k] for k in ks]
                                         for r in be.rot_many_each(cts, ks)]))
    assert c1 == c2 and all(np.array_equal(be.dec(x), be.dec(y)) for x, y in zip(a, b))
    jobs = [[(plain[h][k], pts[3 * h + q]) for q, k in enumerate(ks)] for h in range(2)]
    a, c1 = counted(lambda: be.mac_rescale_many(jobs))
    b, c2 = counted(lambda: be.rescale_each(be.mac_many(jobs)))
    assert c1 == c2
    for x, y in zip(a, b):
        assert (x.level, x.scale) == (y.level, y.scale) == (lvl - 1, y.scale)
        assert np.array_equal(be.dec(x), be.dec(y))
    a, c1 = counted(lambda: be.square_rescale_each(cts))
    b, c2 = counted(lambda: be.rescale_each(be.square_each(cts)))
    assert c1 == c2
    for x, y in zip(a, b):
        assert (x.level, x.scale) == (y.level, y.scale)
        assert np.array_equal(be.dec(x), be.dec(y))

"""Golden fixtures of the network evaluation, generated from the reference.

Build-container only (imports /root/reference).  Records, per (network,
mode, strategy): the reference's per-layer operation counters from its slot
simulator, its cleartext logits and simulator logits; and for a small set of
configurations the decrypted logits of the reference CKKS engine (with the
two ring-table fixes of make_golden.py) at identical seeds.

Usage:  python tests/golden/make_golden_pipeline.py
"""

from __future__ import annotations

import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
import make_golden  # noqa: E402  (applies nothing until we patch below)

from hear.backend import SimBackend  # noqa: E402
from hear.ckks.params import gen_params  # noqa: E402
from hear.fastpath import compile_pipeline, infer  # noqa: E402
from hear.model import (collapse_layers, infer_clear, make_random_input,  # noqa: E402
                        make_random_model, net_by_name, NetworkShape)
from hear.modelenc import ModelEncoder  # noqa: E402


def main():
    out = {"sim": {}, "ckks": {}, "storage": {}}
    t0 = time.time()
    for net in ("1d-w64", "1d-w128", "2d-w64", "2d-w128"):
        shape = net_by_name(net)
        raw = make_random_model(shape, 1)
        cparams = collapse_layers(raw, shape)
        x = make_random_input(shape, 2)
        clear = infer_clear(cparams, x)
        for mode, prof in (("hear", "hear"), ("fast", "fast-hear")):
            for strat in ("full", "giant", "baby"):
                be = SimBackend(gen_params(prof))
                lg, cnt, enc = infer(cparams, x, mode, strat, be)
                out["sim"][f"{net}/{mode}/{strat}"] = {
                    "counters": cnt.as_dict(), "logits": lg.tolist(), "clear": clear.tolist()}
            cp = compile_pipeline(shape, mode, "giant", gen_params(prof))
            out["storage"][f"{net}/{mode}"] = ModelEncoder(cp, cparams, SimBackend(
                gen_params(prof))).storage_report()
        print(net, "sim done", time.time() - t0, flush=True)

    # reference CKKS (ring tables fixed) at real parameters
    from hear.ckks import ring as R
    R.RingContext.__init__ = make_golden._fixed_init
    from hear.ckks.engine import CkksBackend
    cases = [("1d-w64", "fast", "giant", "fast-hear"), ("1d-w64", "hear", "full", "hear")]
    for net, mode, strat, prof in cases:
        shape = net_by_name(net)
        cparams = collapse_layers(make_random_model(shape, 1), shape)
        x = make_random_input(shape, 2)
        be = CkksBackend(gen_params(prof), seed=0)
        cp = compile_pipeline(shape, mode, strat, be.params)
        be.ensure_rotation_keys(cp.rotations)
        lg, cnt, _ = infer(cparams, x, mode, strat, be, encoder=ModelEncoder(cp, cparams, be))
        out["ckks"][f"{net}/{mode}/{strat}/{prof}"] = {
            "logits": lg.tolist(), "clear": infer_clear(cparams, x).tolist(),
            "counters": cnt.as_dict(), "model_seed": 1, "input_seed": 2, "backend_seed": 0}
        print(net, mode, "ckks done", time.time() - t0, flush=True)
    # toy-parameter network (fast to run everywhere)
    shape = NetworkShape(1, 32, 15, (4, 8, 16), 4)
    cparams = collapse_layers(make_random_model(shape, 3), shape)
    x = make_random_input(shape, 4)
    be = CkksBackend(gen_params("toy-fast"), seed=5)
    cp = compile_pipeline(shape, "fast", "giant", be.params)
    be.ensure_rotation_keys(cp.rotations)
    lg, cnt, _ = infer(cparams, x, "fast", "giant", be, encoder=ModelEncoder(cp, cparams, be))
    out["ckks"]["toy/fast/giant/toy-fast"] = {
        "logits": lg.tolist(), "clear": infer_clear(cparams, x).tolist(),
        "counters": cnt.as_dict(), "shape": [1, 32, 15, [4, 8, 16], 4],
        "model_seed": 3, "input_seed": 4, "backend_seed": 5}
    with open(os.path.join(HERE, "pipeline_golden.json"), "w") as f:
        json.dump(out, f, indent=1, sort_keys=True)
    print("done", time.time() - t0)


if __name__ == "__main__":
    main()

"""Round-2 golden fixtures, generated from the reference itself.

Build-container only (imports /root/reference).  Writes:

  codec_golden.npz        the reference encoder (hear/ckks/encoder.py:48-60)
                          at N = 2^15 and 2^16: encode_coeffs of seeded slot
                          values (msg scale 2^40 / 2^45) and decode_coeffs of
                          seeded integer coefficients;
  pipeline_golden_r2.json decrypted logits + counters of the reference CKKS
                          engine (ring-table fixes of make_golden.py) for
                          the bench headline (1d-w64 fast/full, fast-hear)
                          and two 2D networks, at fixed seeds.

Usage:  python tests/golden/make_golden_r2.py [codec|pipeline]
"""

from __future__ import annotations

import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
import make_golden  # noqa: E402,F401  (puts /root/reference on sys.path)

CODEC_CASES = [(15, 40), (16, 45)]   # (log2 N, log2 scale)


def codec():
    from hear.ckks.encoder import Embedding, decode_coeffs, encode_coeffs
    out = {}
    for logn, sbits in CODEC_CASES:
        n = 1 << logn
        emb = Embedding(n)
        vals = np.random.default_rng(100 + logn).uniform(-1, 1, n // 2)
        out[f"enc_{logn}"] = encode_coeffs(emb, vals, float(1 << sbits))
        coeffs = np.random.default_rng(200 + logn).integers(-(1 << 40), 1 << 40, n)
        out[f"dec_{logn}"] = decode_coeffs(emb, coeffs, float(1 << sbits))
    np.savez_compressed(os.path.join(HERE, "codec_golden.npz"), **out)
    print("codec goldens written")


PIPE_CASES = [
    ("1d-w64", "fast", "full", "fast-hear"),    # bench headline
    ("2d-w64", "fast", "giant", "fast-hear"),
    ("2d-w64", "hear", "full", "hear"),
    ("2d-w128", "fast", "full", "fast-hear"),   # the paper's headline network
]


def pipeline():
    from hear.ckks import ring as R
    R.RingContext.__init__ = make_golden._fixed_init
    from hear.ckks.engine import CkksBackend
    from hear.ckks.params import gen_params
    from hear.fastpath import compile_pipeline, infer
    from hear.model import collapse_layers, infer_clear, make_random_input, make_random_model
    from hear.model import net_by_name
    from hear.modelenc import ModelEncoder
    path = os.path.join(HERE, "pipeline_golden_r2.json")
    out = {}
    if os.path.exists(path):
        with open(path) as f:
            out = json.load(f)
    t0 = time.time()
    for net, mode, strat, prof in PIPE_CASES:
        key = f"{net}/{mode}/{strat}/{prof}"
        if key in out:
            continue
        shape = net_by_name(net)
        cparams = collapse_layers(make_random_model(shape, 1), shape)
        x = make_random_input(shape, 2)
        be = CkksBackend(gen_params(prof), seed=0)
        cp = compile_pipeline(shape, mode, strat, be.params)
        be.ensure_rotation_keys(cp.rotations)
        lg, cnt, _ = infer(cparams, x, mode, strat, be, encoder=ModelEncoder(cp, cparams, be))
        out[key] = {"logits": lg.tolist(), "clear": infer_clear(cparams, x).tolist(),
                    "counters": cnt.as_dict(), "model_seed": 1, "input_seed": 2,
                    "backend_seed": 0}
        with open(path, "w") as f:   # checkpoint after every case
            json.dump(out, f, indent=1, sort_keys=True)
        print(key, "done", round(time.time() - t0, 1), flush=True)


if __name__ == "__main__":
    what = sys.argv[1:] or ["codec", "pipeline"]
    if "codec" in what:
        codec()
    if "pipeline" in what:
        pipeline()

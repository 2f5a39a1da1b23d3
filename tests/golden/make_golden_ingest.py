"""Golden fixtures for the ingest front end, produced by hear/ingest.py itself
(build container only).  Usage: python tests/golden/make_golden_ingest.py"""
import json
import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
from hear import ingest as R  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def case(seed, nframes, target, threshold, dup=()):
    rng = np.random.default_rng(seed)
    frames = [rng.uniform(0, 100, (15, 2)) for _ in range(nframes)]
    for i in dup:
        frames[i] = frames[i - 1].copy()
    frames[3][2] = 0.0   # an undetected joint
    out = R.ingest(frames, target, threshold)
    return {"seed": seed, "nframes": nframes, "target": target, "threshold": threshold,
            "dup": list(dup), "out": out.tolist()}


cases = [case(1, 40, 32, 5.0), case(2, 33, 32, 5.0, dup=(5,)), case(3, 45, 32, 60.0),
         case(4, 32, 32, 5.0), case(5, 50, 32, 0.0, dup=(7, 20, 21))]
with open(os.path.join(HERE, "ingest_golden.json"), "w") as f:
    json.dump(cases, f)
print("ok", len(cases))

"""Ingest front end vs the reference (golden cases from hear/ingest.py) and
the spec examples."""
import json
import os

import numpy as np

from paper_2104_09164_b200 import ingest

HERE = os.path.dirname(os.path.abspath(__file__))


def test_matches_reference_golden():
    for c in json.load(open(os.path.join(HERE, "golden", "ingest_golden.json"))):
        rng = np.random.default_rng(c["seed"])
        frames = [rng.uniform(0, 100, (15, 2)) for _ in range(c["nframes"])]
        for i in c["dup"]:
            frames[i] = frames[i - 1].copy()
        frames[3][2] = 0.0
        out = ingest.ingest(frames, c["target"], c["threshold"])
        assert np.allclose(out, np.array(c["out"]), atol=1e-12, rtol=0)


def test_spec_examples():
    same = [np.ones((15, 2))] * 32
    assert len(ingest.select_frames(same, 32)) == 32
    fr = [np.full((2, 2), float(i * 10)) for i in range(33)]
    fr[5] = fr[4].copy()
    kept = ingest.select_frames(fr, 32)
    assert len(kept) == 32 and all(not np.array_equal(k, fr[5]) or k is fr[4] for k in kept[5:6])
    n = ingest.normalize([np.array([[0.0, 1.0], [5.0, 1.0], [10.0, 1.0]])])[0]
    assert np.allclose(n[:, 0], [0, 0.5, 1]) and np.allclose(n[:, 1], 0)
    t = ingest.assemble([np.array([[0.1, 0.2], [0.3, 0.4]])])
    assert np.allclose(t[0, :, 0], [0.1, 0.3]) and np.allclose(t[0, :, 1], [0.2, 0.4])


def test_windows_shape_and_range():
    s = ingest.synthetic_stream(200, seed=1)
    w = ingest.windows(s, 32, 8)
    assert w.shape == ((200 - 32) // 8 + 1, 32, 15, 2)
    assert w.min() >= 0 and w.max() <= 1

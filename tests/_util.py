"""Shared helpers mirroring tests/golden/make_golden.py (same seeds, same digests)."""

import hashlib

import numpy as np


def digest(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(np.asarray(a, dtype=np.uint64)).tobytes())
    return h.hexdigest()


def rand_rows(primes, rows, n, seed):
    rng = np.random.default_rng(seed)
    return np.stack([rng.integers(0, primes[r], n, dtype=np.uint64) for r in rows])


def rand_ct(params, level, seed):
    p = list(params.chain_primes)
    return (rand_rows(p, range(level + 1), params.n, seed),
            rand_rows(p, range(level + 1), params.n, seed + 1))

"""The documented drop-in boundary, run as written: integration/hear_ring_b200.py
(the ctypes stub of INTEGRATION.md §2) binds every `hear_*` entry point of
include/hear_b200.h over a RingContext's tables (oracle.cpu_engine.OracleRing,
the restatement of hear/ckks/ring.py:253-292 whose tables are pinned to the
reference's) and must reproduce the reference's golden digests
(tests/golden/ckks_golden.json) and the C oracle's kernels bit-exactly."""

import ctypes

import numpy as np
import pytest

from tests._util import digest, rand_rows

pytestmark = pytest.mark.gpu

PROFILES = ["toy-fast", "fast-hear"]


def _rings(prof):
    import sys
    import os
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(__file__)), "integration"))
    from hear_ring_b200 import B200Ring
    from oracle.cpu_engine import OracleRing
    from paper_2104_09164_b200.ckks.params import gen_params
    rc = OracleRing(gen_params(prof))
    return rc, B200Ring(rc)


@pytest.mark.parametrize("prof", PROFILES)
def test_ntt_and_pointwise_vs_reference_digests(prof, golden):
    g = golden[prof]["ring"]
    rc, br = _rings(prof)
    gall = list(range(len(rc.primes)))
    x = rand_rows(rc.primes, gall, rc.n, 21)
    y = rand_rows(rc.primes, gall, rc.n, 22)
    f = x.copy()
    br.fwd(f, gall)
    assert digest(f) == g["ntt_fwd"]
    i = x.copy()
    br.inv(i, gall)
    assert digest(i) == g["ntt_inv"]
    assert digest(br.mul(x, y, gall)) == g["pw_mul"]
    back = f.copy()
    br.inv(back, gall)
    assert np.array_equal(back, x)
    assert np.array_equal(br.add(x, y, gall), rc.add(x, y, gall))
    assert np.array_equal(br.sub(x, y, gall), rc.sub(x, y, gall))


@pytest.mark.parametrize("prof", PROFILES)
def test_remaining_ring_kernels_vs_oracle(prof):
    from oracle.cpu_engine import _p, lib
    rc, br = _rings(prof)
    n, k = rc.n, len(rc.primes)
    rows = [0, 3, k - 1, 1]
    rng = np.random.default_rng(5)
    # scalar_mul (ring.py:175)
    a = rand_rows(rc.primes, rows, n, 31)
    c = np.array([int(rng.integers(0, rc.primes[r])) for r in rows], dtype=np.uint64)
    want = a.copy()
    rc.scalar_mul(want, c, rows)
    br.scalar_mul(a, c, rows)
    assert np.array_equal(a, want)
    # sub_scaled_inv (ring.py:210)
    a = rand_rows(rc.primes, rows, n, 32)
    corr = rand_rows(rc.primes, rows, n, 33)
    want = a.copy()
    lib().or_sub_scaled_inv(_p(want), _p(corr), _p(c), len(rows), n, _p(np.array(rows)),
                            _p(rc.p), _p(rc.mu), _p(rc.sh))
    br.sub_scaled_inv(a, corr, c, rows)
    assert np.array_equal(a, want)
    # lift_center (ring.py:186) and reduce_rows (ring.py:198)
    x = rand_rows(rc.primes, [2], n, 34)[0]
    out = np.empty(n, dtype=np.int64)
    br.lift_center(x, rc.primes[2], out)
    assert np.array_equal(out, rc.lift_center(x, rc.primes[2]))
    red = np.empty((len(rows), n), dtype=np.uint64)
    br.reduce_rows(out, rows, red)
    assert np.array_equal(red, rc.reduce_rows(out, rows))
    # pw_mul_accum_perm (ring.py:136): 3 digits, trimmed keys, Galois gather
    ndig, krows = 3, 5
    gidx = np.array([0, 1, 2, k - 1])
    krow = np.array([0, 1, 2, krows - 1])
    de = np.stack([rand_rows(rc.primes, gidx, n, 40 + i) for i in range(ndig)])
    kb = np.stack([rand_rows(rc.primes, [0, 1, 2, 3, k - 1], n, 50 + i) for i in range(ndig)])
    ka = np.stack([rand_rows(rc.primes, [0, 1, 2, 3, k - 1], n, 60 + i) for i in range(ndig)])
    perm = rc.ntt_perm(pow(5, 3, 2 * n)).astype(np.int64)
    ob = rand_rows(rc.primes, gidx, n, 70)
    oa = rand_rows(rc.primes, gidx, n, 71)
    wb, wa = ob.copy(), oa.copy()
    lib().or_pw_mul_accum_perm(_p(wb), _p(wa), _p(de), _p(kb), _p(ka), _p(krow), _p(perm),
                               _p(gidx), ndig, len(gidx), krows, n, _p(rc.p), _p(rc.mu),
                               _p(rc.sh))
    br.pw_mul_accum_perm(ob, oa, de, kb, ka, krow, perm, gidx)
    assert np.array_equal(ob, wb) and np.array_equal(oa, wa)


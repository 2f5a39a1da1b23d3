"""Parameter sets, layouts and the collapsed model (CPU)."""

import numpy as np
import pytest

from paper_2104_09164_b200.ckks.params import gen_params, gen_params_custom
from paper_2104_09164_b200.layout import input_layout, load_factor, pack_input, pot
from paper_2104_09164_b200.model import (NetworkShape, RawLayerParams, collapse_layers,
                                         forward_uncollapsed, infer_clear, make_random_input,
                                         make_random_model, net_by_name)

# primes of the reference's profiles (hear/ckks/params.py:104-123), as it generates them
REF_PRIMES = {
    "hear": ((137438822401, 34359771137, 34359410689, 34359214081, 34358788097, 34360754177,
              34357805057, 34357444609, 34357411841, 34362163201, 34362228737), 137438691329),
    "fast-hear": ((8590163969, 2147352577, 2146959361, 2146336769, 2148728833, 268369921,
                   2148794369, 2146041857, 2145976321, 268271617, 2149810177, 2144960513,
                   2150072321), 8589475841),
}
REF_DIGEST = {"hear": "aded36fadc9aac3b", "fast-hear": "3504edde4a0abc85",
              "toy-hear": "6750cbae69ab9988", "toy-fast": "1020d60d35de68f2"}


@pytest.mark.parametrize("prof", sorted(REF_DIGEST))
def test_profiles(prof):
    ps = gen_params(prof)
    assert ps.digest() == REF_DIGEST[prof]
    if prof in REF_PRIMES:
        assert (ps.chain_primes, ps.special_prime) == REF_PRIMES[prof]
    for q in ps.chain_primes + (ps.special_prime,):
        assert q % (2 * ps.n) == 1
    assert ps.max_level == (10 if prof.endswith("hear") and "fast" not in prof else 12)


def test_log2q():
    assert gen_params("hear").log2_q in range(380, 395)
    assert gen_params("fast-hear").log2_q in range(392, 405)
    assert gen_params_custom(64, [40, 30, 30], 40, 25).insecure


def test_pot_and_packing():
    assert (pot(480), pot(512), pot(1)) == (512, 512, 1)
    lay = input_layout(32, 15, 8192)
    assert (lay.block, lay.replicas, lay.channels_per_ct) == (512, 8, 16)
    x = np.arange(8).reshape(2, 2, 2).astype(float)
    v, lay = pack_input(x, 16)
    assert lay.block == 4 and lay.replicas == 2
    assert np.array_equal(v[:8], [0, 2, 4, 6, 1, 3, 5, 7]) and np.array_equal(v[:8], v[8:])


def test_load_factor_table_vi():
    assert load_factor(3, 16, 2) == 16 and load_factor(3, 8, 1) == 4
    assert load_factor(2, 1, 2) == 1 and load_factor(1, 8, 2) == 1


def test_collapse_examples():
    shape = NetworkShape(1, 2, 2, (1, 2, 4), 1)
    one = lambda c: np.ones(c)  # noqa: E731
    zero = lambda c: np.zeros(c)  # noqa: E731
    raw = RawLayerParams(
        shape, [np.zeros((1, 2, 1, 3)), np.zeros((2, 1, 1, 3)), np.zeros((4, 2, 1, 3))],
        [one(1), zero(2), zero(4)], [zero(1), zero(2), zero(4)], [one(1), one(2), one(4)],
        [2 * one(1), one(2), one(4)], [zero(1), zero(2), zero(4)],
        [(0.0, 0.0, 1.0), (0.0, 1.0, 0.0), (0.0, 1.0, 0.0)], np.zeros((1, 4)))
    c = collapse_layers(raw, shape)
    # gamma=2, sigma=1, beta=mu=0, b=1, act x^2, 1D pool area 2: (4, 8, 4)/2
    assert np.allclose(c.coeffs[0][:, 0], [2.0, 4.0, 2.0])


@pytest.mark.parametrize("seed", range(5))
def test_collapse_equivalence(seed):
    shape = net_by_name("2d-w64")
    raw = make_random_model(shape, seed)
    x = make_random_input(shape, seed + 100)
    assert np.abs(infer_clear(collapse_layers(raw, shape), x)
                  - forward_uncollapsed(raw, x)).max() < 1e-10


def test_width_validation():
    with pytest.raises(ValueError):
        NetworkShape(2, 32, 15, (64, 100, 256), 10)

"""The GPU canonical-embedding codec (csrc/fft.cu four-step special FFT) at
the ring sizes of BASELINE configs 1-3 (N = 2^15, 2^16), against goldens the
reference encoder itself produced (tests/golden/make_golden_r2.py ->
codec_golden.npz, hear/ckks/encoder.py:48-60), plus enc -> dec round trips
through the engine at those rings."""

import os
from fractions import Fraction

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

HERE = os.path.join(os.path.dirname(__file__), "golden")
CASES = [(15, 40), (16, 45)]   # as make_golden_r2.CODEC_CASES


@pytest.fixture(scope="module")
def gold():
    return np.load(os.path.join(HERE, "codec_golden.npz"))


@pytest.mark.parametrize("logn,sbits", CASES)
def test_encode_matches_reference(logn, sbits, gold):
    import torch
    from paper_2104_09164_b200.ckks.encoder import Embedding
    n = 1 << logn
    emb = Embedding(n)
    vals = np.random.default_rng(100 + logn).uniform(-1, 1, n // 2)
    got = emb.encode_coeffs(torch.from_numpy(vals)[None], float(1 << sbits))[0].cpu().numpy()
    ref = gold[f"enc_{logn}"]
    diff = np.abs(got - ref)
    # the reference rounds numpy's pocketfft output, this a four-step fp64 FFT:
    # integers agree except rare round-half boundary cases
    assert diff.max() <= 1 and (diff > 0).mean() < 1e-3, (diff.max(), (diff > 0).mean())


@pytest.mark.parametrize("logn,sbits", CASES)
def test_decode_matches_reference(logn, sbits, gold):
    import torch
    from paper_2104_09164_b200.ckks.encoder import Embedding
    n = 1 << logn
    emb = Embedding(n)
    coeffs = np.random.default_rng(200 + logn).integers(-(1 << 40), 1 << 40, n)
    got = emb.decode_coeffs(torch.from_numpy(coeffs.astype(np.float64))[None],
                            float(1 << sbits))[0].cpu().numpy()
    ref = gold[f"dec_{logn}"]
    assert np.abs(got - ref).max() <= 1e-10 * np.abs(ref).max()


def test_encode_chunks_past_workspace():
    """More polynomials than one launch pair's workspace (512 at N = 2^14):
    every chunk equals the one-at-a-time encoding."""
    import torch
    from paper_2104_09164_b200.ckks.encoder import Embedding
    emb = Embedding(1 << 14)
    vals = np.random.default_rng(5).uniform(-1, 1, (600, 1 << 13))
    allc = emb.encode_coeffs(torch.from_numpy(vals), 2.0 ** 30).cpu()
    for i in (0, 511, 512, 599):
        one = emb.encode_coeffs(torch.from_numpy(vals[i:i + 1]), 2.0 ** 30).cpu()
        assert torch.equal(allc[i:i + 1], one)
    back = emb.decode_coeffs(allc.to(torch.float64), 2.0 ** 30).cpu().numpy()
    assert np.abs(back - vals).max() < 2.0 ** -20   # rounding: ~sqrt(N)/2 / scale


def test_encode_overflow_raises():
    import torch
    from paper_2104_09164_b200.ckks.encoder import Embedding, EncodeOverflow
    emb = Embedding(1 << 15)
    vals = np.full((1, 1 << 14), 1.0)
    with pytest.raises(EncodeOverflow):
        emb.encode_coeffs(torch.from_numpy(vals), 2.0 ** 53)


@pytest.mark.parametrize("logn,bits,special,sbits", [(15, [40, 40, 40], 40, 40),
                                                     (16, [50, 45, 45], 60, 45)])
def test_enc_dec_round_trip(logn, bits, special, sbits):
    """Public-key encryption -> decryption at the big rings (fp64 and integer
    arithmetic policies), batched over 3 clips: |dec - v| <= 2^-20."""
    from paper_2104_09164_b200.ckks.engine import CkksBackend
    from paper_2104_09164_b200.ckks.params import gen_params_custom
    ps = gen_params_custom(1 << logn, bits, special, sbits)
    be = CkksBackend(ps, seed=11)
    vals = np.random.default_rng(12).uniform(-1, 1, (3, ps.n2))
    ct = be.enc(vals, level=ps.max_level, scale=Fraction(1 << sbits))
    got = be.dec(ct)
    assert np.abs(got - vals).max() <= 2.0 ** -20

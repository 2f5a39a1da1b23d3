"""ncu target for the kernels outside the bench step: the codec's four-step
FFT (k_fft_cols / k_fft_rows, encode + decode of 512 polynomials at N=2^14
and 128 at N=2^16), and BASELINE config 1's integer-policy key switch at
N=2^16 (hybrid dnum=3: k_bconv, the 64-bit-Shoup two-pass NTT k_ntt2_*<PolU64>,
k_ks_inner2).  Each phase inside cudaProfilerStart/Stop.
    python tools/prof_aux.py"""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from fractions import Fraction

import numpy as np
import torch

from paper_2104_09164_b200.backend import Ct
from paper_2104_09164_b200.ckks.encoder import Embedding
from paper_2104_09164_b200.ckks.engine import CkksBackend, CtData
from paper_2104_09164_b200.ckks.hybrid import HybridKeySwitch
from paper_2104_09164_b200.ckks.params import gen_params_custom

for logn, m in ((14, 512), (16, 128)):
    emb = Embedding(1 << logn)
    v = torch.from_numpy(np.random.default_rng(0).uniform(-1, 1, (m, 1 << (logn - 1))))
    c = emb.encode_coeffs(v, 2.0 ** 40)
    emb.decode_coeffs(c.to(torch.float64), 2.0 ** 40)
    torch.cuda.synchronize()
    torch.cuda.profiler.start()
    c = emb.encode_coeffs(v, 2.0 ** 40)
    emb.decode_coeffs(c.to(torch.float64), 2.0 ** 40)
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()

ps = gen_params_custom(1 << 16, [50] * 24, 60, 40)
be = CkksBackend(ps, seed=0)
hk = HybridKeySwitch(be, 3, [ps.special_prime], seed=1)
lvl, bsz = ps.max_level, 16
t = torch.empty(bsz, 2, lvl + 1, ps.n, dtype=torch.int64, device=be.dev)
for r, q in enumerate(ps.chain_primes):
    t[:, :, r].random_(0, q)
a = Ct(CtData(t), lvl, Fraction(1), ps.n2)
hk.mult(a, a)
torch.cuda.synchronize()
torch.cuda.profiler.start()
hk.mult(a, a)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("done")

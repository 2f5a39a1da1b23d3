"""Host-side cost of one-clip encryption / decryption (the client half of the
streaming latency): wall time per call and the cProfile top entries.
Dev tool:  python tools/client_profile.py"""
import cProfile
import os
import pstats
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2104_09164_b200.ckks.engine import CkksBackend
from paper_2104_09164_b200.ckks.params import gen_params

be = CkksBackend(gen_params("fast-hear"), seed=0)
x = np.random.default_rng(0).uniform(-1, 1, be.n2)
ct = be.enc(x)
low = be.enc(x, level=0)
for _ in range(20):
    be.enc(x)
    be.dec(low)
torch.cuda.synchronize()
for name, fn in (("enc", lambda: be.enc(x)), ("dec", lambda: be.dec(low))):
    t0 = time.perf_counter()
    for _ in range(200):
        fn()
        torch.cuda.synchronize()
    print(f"{name}: {(time.perf_counter() - t0) / 200 * 1e3:.3f} ms per call")
    pr = cProfile.Profile()
    pr.enable()
    for _ in range(100):
        fn()
        torch.cuda.synchronize()
    pr.disable()
    st = pstats.Stats(pr)
    st.sort_stats("cumulative").print_stats(18)

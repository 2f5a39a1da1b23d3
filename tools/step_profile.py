"""One eager encrypted-inference step inside a cudaProfilerStart/Stop range
(ncu target: --profile-from-start off).  Dev tool.

    ncu --profile-from-start off --metrics ... python tools/step_profile.py [net] [strategy] [B]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np
import torch

from paper_2104_09164_b200.ckks.engine import CkksBackend
from paper_2104_09164_b200.ckks.params import gen_params
from paper_2104_09164_b200.fastpath import compile_pipeline, encrypt_input, run_pipeline
from paper_2104_09164_b200.model import (collapse_layers, make_random_input, make_random_model,
                                         net_by_name)
from paper_2104_09164_b200.modelenc import ModelEncoder

net = sys.argv[1] if len(sys.argv) > 1 else "1d-w64"
strat = sys.argv[2] if len(sys.argv) > 2 else "full"
bsz = int(sys.argv[3]) if len(sys.argv) > 3 else 64
shape = net_by_name(net)
cpar = collapse_layers(make_random_model(shape, 1), shape)
be = CkksBackend(gen_params("fast-hear"), seed=0)
cp = compile_pipeline(shape, "fast", strat, be.params)
be.ensure_rotation_keys(cp.rotations)
enc = ModelEncoder(cp, cpar, be).prepare()
x = np.stack([make_random_input(shape, 100 + i) for i in range(bsz)])
ct = encrypt_input(x, cp, be)
run_pipeline(enc, ct, be)
torch.cuda.synchronize()
torch.cuda.profiler.start()
run_pipeline(enc, ct, be)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("done")

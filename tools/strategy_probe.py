import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from paper_2104_09164_b200.ckks.engine import CkksBackend
from paper_2104_09164_b200.ckks.params import gen_params
from paper_2104_09164_b200.fastpath import compile_pipeline, encrypt_input, run_pipeline, dec_logits
from paper_2104_09164_b200.model import collapse_layers, make_random_input, make_random_model, net_by_name, infer_clear
from paper_2104_09164_b200.modelenc import ModelEncoder
strat = sys.argv[1]; bsz = int(sys.argv[2])
shape = net_by_name("1d-w64")
cpar = collapse_layers(make_random_model(shape, 1), shape)
be = CkksBackend(gen_params("fast-hear"), seed=0)
cp = compile_pipeline(shape, "fast", strat, be.params)
be.ensure_rotation_keys(cp.rotations)
enc = ModelEncoder(cp, cpar, be).prepare()
x = np.stack([make_random_input(shape, i) for i in range(bsz)])
ct = encrypt_input(x, cp, be)
orig = be.layer
from contextlib import contextmanager
@contextmanager
def lay(label):
    with orig(label):
        yield be
    torch.cuda.synchronize()
    print("layer ok", label, flush=True)
be.layer = lay
out = run_pipeline(enc, ct, be)
torch.cuda.synchronize()
lg = dec_logits(out, cp, be)
print(strat, bsz, "maxerr", np.abs(lg - np.stack([infer_clear(cpar, xi) for xi in x])).max(), flush=True)

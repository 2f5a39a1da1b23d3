"""Per-clip decrypted-logit errors of the big-ring networks (config 2 at
N=2^15, config 3 at N=2^16) for batched and clip-by-clip evaluation."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2104_09164_b200.ckks.engine import CkksBackend
from paper_2104_09164_b200.ckks.params import fast_hear_ring, tcn_ring16
which = sys.argv[1]
if which == "c3":
    from paper_2104_09164_b200.tcn import *
    ps = tcn_ring16()
    shape = tcn_by_name("config3")
    tp = make_random_tcn(shape, 1, 0.05)
    be = CkksBackend(ps, seed=0)
    plan = compile_tcn(shape, ps)
    be.ensure_rotation_keys(plan.rotations)
    enc = TcnEncoder(plan, tp, be).prepare()
    xs = np.stack([make_random_clip(shape, s) for s in (2, 3, 4)])
    clear = np.stack([infer_clear_tcn(tp, x) for x in xs])
    def run(x):
        return dec_tcn_logits(run_tcn(enc, encrypt_tcn_input(x, plan, be), be), enc, be)
else:
    from paper_2104_09164_b200.fastpath import compile_pipeline, encrypt_input, run_pipeline, dec_logits
    from paper_2104_09164_b200.model import *
    from paper_2104_09164_b200.modelenc import ModelEncoder
    ps = fast_hear_ring(15)
    shape = net_by_name("1d-w64")
    cpar = collapse_layers(make_random_model(shape, 1), shape)
    be = CkksBackend(ps, seed=0)
    cp = compile_pipeline(shape, "fast", "full", ps)
    be.ensure_rotation_keys(cp.rotations)
    enc = ModelEncoder(cp, cpar, be).prepare()
    xs = np.stack([make_random_input(shape, s) for s in (2, 3, 4)])
    clear = np.stack([infer_clear(cpar, x) for x in xs])
    def run(x):
        return dec_logits(run_pipeline(enc, encrypt_input(x, cp, be), be), cp, be)
lb = run(xs)
print("batched per-clip max err:", np.abs(lb - clear).max(axis=1))
for i in range(3):
    l1 = run(xs[i])
    print("clip", i, "single err", np.abs(l1 - clear[i]).max())
print("clear scale", np.abs(clear).max())

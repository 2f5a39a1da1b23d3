"""Per-layer GPU time of one eager encrypted step (CUDA events around each
backend.layer(label) scope).  Dev tool:  python tools/layer_times.py [net] [strategy] [B]"""
import os, sys
from contextlib import contextmanager
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2104_09164_b200.ckks.engine import CkksBackend
from paper_2104_09164_b200.ckks.params import gen_params
from paper_2104_09164_b200.fastpath import compile_pipeline, encrypt_input, run_pipeline
from paper_2104_09164_b200.model import collapse_layers, make_random_input, make_random_model, net_by_name
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
ct = encrypt_input(np.stack([make_random_input(shape, i) for i in range(bsz)]), cp, be)
run_pipeline(enc, ct, be)
torch.cuda.synchronize()
events = []
orig = be.layer
@contextmanager
def timed_layer(label):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    with orig(label):
        yield be
    b.record()
    events.append((label, a, b))
be.layer = timed_layer
be.reset_counters()
run_pipeline(enc, ct, be)
torch.cuda.synchronize()
tot = sum(a.elapsed_time(b) for _, a, b in events)
cnt = be.counters.as_dict()
for label, a, b in events:
    c = cnt.get(label, {})
    print(f"{label:8s} {a.elapsed_time(b):8.2f} ms {100*a.elapsed_time(b)/tot:5.1f}%  rot={c.get('rot',0)} hoisted={c.get('hoisted_rot_total',0)} mp={c.get('mult_plain',0)} mult={c.get('mult',0)} resc={c.get('rescale',0)}")
print(f"total {tot:.2f} ms for {bsz} clips")

"""Time the layer MAC kernels on a conv-like shape (dev tool).
    python tools/mac_bench.py B [O T lvl]"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from fractions import Fraction
from paper_2104_09164_b200.ckks.engine import CkksBackend, CtData
from paper_2104_09164_b200.ckks.params import gen_params
from paper_2104_09164_b200.backend import Ct, Pt
B = int(sys.argv[1]) if len(sys.argv) > 1 else 32
O = int(sys.argv[2]) if len(sys.argv) > 2 else 48
T = int(sys.argv[3]) if len(sys.argv) > 3 else 32
lvl = int(sys.argv[4]) if len(sys.argv) > 4 else 4
be = CkksBackend(gen_params("fast-hear"), seed=0)
R = lvl + 1
cts = [Ct(CtData(be.ring.empty(B, 2, R).random_(0, 1 << 30)), lvl, Fraction(1), be.n2) for _ in range(T)]
pts = [[Pt(be.ring.empty(R).random_(0, 1 << 30), lvl, Fraction(1), be.n2) for _ in range(T)] for _ in range(O)]
jobs = [[(cts[t], pts[o][t]) for t in range(T)] for o in range(O)]
out = be._raw_mac_strided(jobs[:2]); torch.cuda.synchronize()
ref = torch.stack([o.payload.data for o in be._raw_mac_many(jobs)])
tag = os.environ.get("TAG", "")
fn = be._raw_mac_many
fn(jobs); torch.cuda.synchronize()
t = time.time()
for _ in range(3): out = fn(jobs)
torch.cuda.synchronize(); dt = (time.time() - t) / 3
macs = O * T * B * 2 * R * be.n
print(f"{tag:12s} B={B} O={O} T={T} R={R}: {dt*1e3:8.2f} ms  {macs/dt/1e12:.3f} T MAC/s", flush=True)

"""Time the layer MAC kernels on a conv3-like shape (dev tool)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from fractions import Fraction
from paper_2104_09164_b200.ckks.engine import CkksBackend, CtData
from paper_2104_09164_b200.ckks.params import gen_params
from paper_2104_09164_b200.backend import Ct, Pt
be = CkksBackend(gen_params("fast-hear"), seed=0)
lvl, B, O, T = 4, int(sys.argv[1]) if len(sys.argv) > 1 else 32, 48, 32
R = lvl + 1
cts = [Ct(CtData(be.ring.empty(B, 2, R).random_(0, 1 << 30)), lvl, Fraction(1), be.n2) for _ in range(T)]
pts = [[Pt(be.ring.empty(R).random_(0, 1 << 30), lvl, Fraction(1), be.n2) for _ in range(T)] for _ in range(O)]
jobs = [[(cts[t], pts[o][t]) for t in range(T)] for o in range(O)]
ref = None
for name, env, fn in [("strided", {}, be._raw_mac_strided), ("shared", {"HEAR_B200_MAC_SHARED": "1"}, be._raw_mac_many),
                      ("f64_4x8", {}, be._raw_mac_many), ("f64_4x4", {"HEAR_B200_MAC_TILE": "4"}, be._raw_mac_many)]:
    os.environ.pop("HEAR_B200_MAC_SHARED", None); os.environ.pop("HEAR_B200_MAC_TILE", None)
    os.environ.update(env)
    out = fn(jobs); torch.cuda.synchronize()
    t = time.time()
    for _ in range(3): out = fn(jobs)
    torch.cuda.synchronize(); dt = (time.time() - t) / 3
    res = torch.stack([o.payload.data for o in out])
    ok = True if ref is None else bool(torch.equal(ref, res))
    ref = res if ref is None else ref
    macs = O * T * B * 2 * R * be.n
    print(f"{name:8s} {dt*1e3:8.2f} ms  {macs/dt/1e12:.3f} T MAC/s  equal={ok}", flush=True)

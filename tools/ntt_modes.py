"""Time each NTT launch kind of a B-clip key switch at level lvl with CUDA
events: inverse (digits), forward LIFT (ModUp), forward MODDOWN.
    python tools/ntt_modes.py [lvl] [bsz]"""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2104_09164_b200 import _native as nat
from paper_2104_09164_b200.ckks.engine import CkksBackend, _tasks
from paper_2104_09164_b200.ckks.params import gen_params
from paper_2104_09164_b200.ckks.ring import _upload

lvl = int(sys.argv[1]) if len(sys.argv) > 1 else 12
bsz = int(sys.argv[2]) if len(sys.argv) > 2 else 64
if os.environ.get("NTT_MODES_LOGN"):   # custom fp64 ring of the same depth at another N
    from paper_2104_09164_b200.ckks.params import gen_params_custom
    lg = int(os.environ["NTT_MODES_LOGN"])
    ps = gen_params_custom(1 << lg, [33] + [31] * 12, 33, 31)
else:
    ps = gen_params("fast-hear")
be = CkksBackend(ps, seed=0, keygen=False)
ring, n, S = be.ring, be.n, be.S
rp = ring.row_ptrs
r = lvl + 1
L = nat.lib()
st = torch.cuda.current_stream()


def timeit(fn, reps=10):
    for _ in range(2):
        fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(st)
    for _ in range(reps):
        fn()
    e1.record(st)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3


src = ring.empty(bsz, r).random_(0, 1 << 30)
dst = ring.empty(bsz, r)
prim = np.tile(np.arange(r), bsz)
t_inv = _upload(_tasks(nat.NTT_TASK, bsz * r, src=rp(src), dst=rp(dst), src_prime=prim, dst_prime=prim), be.dev)
de = ring.empty(bsz, r, r + 1)
sp = np.tile(np.repeat(np.arange(r), r + 1), bsz)
dp = np.tile(np.array(list(range(r)) + [S]), bsz * r)
t_lift = _upload(_tasks(nat.NTT_TASK, bsz * r * (r + 1), src=np.repeat(rp(src), r + 1), dst=rp(de),
                        src_prime=sp, dst_prime=dp), be.dev)
m = bsz * 2
sps = ring.empty(m).random_(0, 1 << 30)
aux = ring.empty(m, r).random_(0, 1 << 30)
out = ring.empty(m, r)
t_md = _upload(_tasks(nat.NTT_TASK, m * r, src=np.repeat(rp(sps), r), dst=rp(out), aux=rp(aux),
                      src_prime=S, dst_prime=np.tile(np.arange(r), m),
                      scal=np.tile(be._pinv[:r], m), scal_sh=np.tile(be._pinv_sh[:r], m)), be.dev)
res = {}
res["inv"] = (bsz * r, timeit(lambda: nat.check(L.hb_ntt_inv(ring.handle, t_inv.data_ptr(), bsz * r, st.cuda_stream), "inv")))
res["lift"] = (bsz * r * (r + 1), timeit(lambda: nat.check(L.hb_ntt_fwd(ring.handle, t_lift.data_ptr(), bsz * r * (r + 1), nat.FWD_LIFT, st.cuda_stream), "lift")))
res["moddown"] = (m * r, timeit(lambda: nat.check(L.hb_ntt_fwd(ring.handle, t_md.data_ptr(), m * r, nat.FWD_MODDOWN, st.cuda_stream), "md")))
tag = os.environ.get("TAG", "")
for k, (rows, us) in res.items():
    print(f"{tag:8s} {k:8s} rows={rows:6d} {us:9.1f} us  {rows / us:6.2f} rows/us", flush=True)

"""Digest every fused NTT mode at several launch sizes (A/B of NTT kernels:
run once per build / HEAR_B200_NTT3 setting and diff the output).
    python tools/ntt3_check.py"""
import hashlib
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2104_09164_b200 import _native as nat
from paper_2104_09164_b200.ckks.engine import CkksBackend, _tasks
from paper_2104_09164_b200.ckks.params import gen_params

be = CkksBackend(gen_params("fast-hear"), seed=0, keygen=False)
ring, n, S = be.ring, be.n, be.S
rp = ring.row_ptrs
torch.manual_seed(0)
g = torch.Generator(device="cuda").manual_seed(1)


def dig(t):
    torch.cuda.synchronize()
    return hashlib.sha256(t.cpu().numpy().tobytes()).hexdigest()[:16]


PMIN = min(list(be.params.chain_primes) + [be.P])


def rnd(*shape):   # canonical under every prime of the ring
    return ring.empty(*shape).random_(0, PMIN, generator=g)


perm = torch.randperm(n, device="cuda", generator=g).to(torch.int32)
for bsz in (1, 8, 64):
    r = 13
    prim = np.tile(np.arange(r), bsz)
    src = rnd(bsz, r)
    out = {}
    d = ring.empty(bsz, r)
    ring.ntt_inv(_tasks(nat.NTT_TASK, bsz * r, src=rp(src), dst=rp(d), src_prime=prim, dst_prime=prim))
    out["inv"] = dig(d)
    lif = ring.empty(bsz, r)
    ring.ntt_inv(_tasks(nat.NTT_TASK, bsz * r, src=rp(src), dst=rp(lif), src_prime=prim, dst_prime=prim, scal=1))
    out["inv_lift"] = dig(lif)
    d2, cp = ring.empty(bsz, r), ring.empty(bsz, r)
    ring.ntt_inv(_tasks(nat.NTT_TASK, bsz * r, src=rp(src), dst=rp(d2), src_prime=prim, dst_prime=prim,
                        add2=rp(cp)))
    out["inv_add2"] = dig(d2) + dig(cp)
    f = ring.empty(bsz, r)
    ring.ntt_fwd(_tasks(nat.NTT_TASK, bsz * r, src=rp(src), dst=rp(f), src_prime=prim, dst_prime=prim),
                 nat.FWD_PLAIN)
    out["fwd"] = dig(f)
    de = ring.empty(bsz, r, r + 1)
    sp = np.tile(np.repeat(np.arange(r), r + 1), bsz)
    dp = np.tile(np.array(list(range(r)) + [S]), bsz * r)
    ring.ntt_fwd(_tasks(nat.NTT_TASK, bsz * r * (r + 1), src=np.repeat(rp(src), r + 1), dst=rp(de),
                        src_prime=sp, dst_prime=dp), nat.FWD_LIFT)
    out["lift"] = dig(de)
    ring.ntt_fwd(_tasks(nat.NTT_TASK, bsz * r * (r + 1), src=np.repeat(rp(lif), r + 1), dst=rp(de),
                        src_prime=-1, dst_prime=dp), nat.FWD_LIFT)
    out["lift_once"] = dig(de)
    m = bsz * 2
    sps = rnd(m)
    aux, add, add2 = rnd(m, r), rnd(m, r), rnd(m, r)
    o = ring.empty(m, r)
    base = dict(src=np.repeat(rp(sps), r), dst=rp(o), aux=rp(aux), src_prime=S,
                dst_prime=np.tile(np.arange(r), m), scal=np.tile(be._pinv[:r], m),
                scal_sh=np.tile(be._pinv_sh[:r], m))
    ring.ntt_fwd(_tasks(nat.NTT_TASK, m * r, **base), nat.FWD_MODDOWN)
    out["md"] = dig(o)
    ring.ntt_fwd(_tasks(nat.NTT_TASK, m * r, add=rp(add), perm=perm.data_ptr(), **base), nat.FWD_MODDOWN)
    out["md_gather"] = dig(o)
    ring.ntt_fwd(_tasks(nat.NTT_TASK, m * r, add=rp(add), add2=rp(add2), **base), nat.FWD_MODDOWN)
    out["md_add2"] = dig(o)
    ring.ntt_fwd(_tasks(nat.NTT_TASK, m * r, add=rp(add), perm=perm.data_ptr(), add2=rp(add2), **base),
                 nat.FWD_MODDOWN_SCATTER)
    out["md_scatter"] = dig(o)
    for k, v in out.items():
        print(f"bsz={bsz:3d} {k:12s} {v}", flush=True)

if os.environ.get("NTT3_DIFF"):
    # run the gather launch repeatedly; where do repeated runs disagree?
    bsz, r = 64, 13
    m = bsz * 2
    sps = rnd(m)
    aux, add = rnd(m, r), rnd(m, r)
    base = dict(src=np.repeat(rp(sps), r), aux=rp(aux), src_prime=S,
                dst_prime=np.tile(np.arange(r), m), scal=np.tile(be._pinv[:r], m),
                scal_sh=np.tile(be._pinv_sh[:r], m), add=rp(add), perm=perm.data_ptr())
    outs = []
    for it in range(4):
        o = ring.empty(m, r).fill_(-1)
        ring.ntt_fwd(_tasks(nat.NTT_TASK, m * r, dst=rp(o), **base), nat.FWD_MODDOWN)
        torch.cuda.synchronize()
        outs.append(o.reshape(m * r, n))
    for it in range(1, 4):
        d = (outs[it] != outs[0])
        rows = d.any(1).nonzero().flatten()
        print(f"run {it}: {int(d.sum())} elements differ in {len(rows)} rows; unwritten(-1) "
              f"{int((outs[it] == -1).sum())}/{int((outs[0] == -1).sum())}", flush=True)
        if len(rows):
            idx = d.nonzero()
            j = idx[:, 1]
            print("  rows", rows[:20].tolist())
            print("  tile hist", torch.bincount(j // 4096, minlength=4).tolist())
            print("  in-tile 128-block hist", torch.bincount((j % 4096) // 128, minlength=32).tolist())
            print("  in-block pos hist", torch.bincount(j % 128, minlength=128)[:32].tolist())

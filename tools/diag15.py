"""Diagnose batched (GEMM-path) ops at a big ring: every batched op vs the
same op clip by clip (per-job kernels, oracle-pinned) -- prints mismatches."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from fractions import Fraction
import numpy as np
import torch
from paper_2104_09164_b200.ckks.engine import CkksBackend, CtData
from paper_2104_09164_b200.ckks.params import fast_hear_ring, gen_params_custom
from paper_2104_09164_b200.backend import Ct

logn = int(sys.argv[1]) if len(sys.argv) > 1 else 15
ps = fast_hear_ring(logn) if len(sys.argv) < 3 else gen_params_custom(1 << logn, [33, 31, 31, 31], 33, 31)
be = CkksBackend(ps, seed=1)
L = ps.max_level
B = 8
g = torch.Generator(device="cuda").manual_seed(0)
def rnd(lvl):
    x = be.ring.empty(B, 2, lvl + 1)
    for r in range(lvl + 1):
        x[:, :, r].random_(0, ps.chain_primes[r], generator=g)
    return Ct(CtData(x), lvl, Fraction(ps.msg_scale), ps.n2)
def clip(ct, b):
    return Ct(CtData(ct.payload.data[b:b + 1].contiguous()), ct.level, ct.scale, ct.slots)
def same(name, batched, fn, cts):
    bad = []
    for b in range(B):
        one = fn(*[clip(c, b) for c in cts])
        if not torch.equal(one.payload.data[0], batched.payload.data[b]):
            bad.append(b)
    print(f"{name}: {'OK' if not bad else 'MISMATCH clips ' + str(bad)}", flush=True)
for lvl in (L, L // 2):
    a, c = rnd(lvl), rnd(lvl)
    be.ensure_rotation_keys({1: L, 3: L, 16: L})
    same(f"rot l={lvl}", be._raw_rot(a, 3), lambda x: be._raw_rot(x, 3), [a])
    rm = be._raw_rot_many(a, [1, 3, 16])
    for k in (1, 3, 16):
        same(f"rot_many[{k}] l={lvl}", rm[k], lambda x: be._raw_rot_many(x, [1, 3, 16])[k], [a])
    same(f"mult l={lvl}", be._raw_mult(a, c), be._raw_mult, [a, c])
    same(f"rescale l={lvl}", be._raw_rescale(a), be._raw_rescale, [a])
    sq = be._raw_square_each([a, c])
    same(f"square_each l={lvl}", sq[0], lambda x: be._raw_square_each([x])[0], [a])
    ra = be._raw_rot_add_each([(a, 1), (c, 3)])
    same(f"rot_add_each l={lvl}", ra[1], lambda x: be._raw_rot_add_each([(x, 3)])[0], [c])
    re_ = be._raw_rot_each([(a, 1), (c, 16)])
    same(f"rot_each l={lvl}", re_[1], lambda x: be._raw_rot_each([(x, 16)])[0], [c])
    pts = be.encode_many(np.random.default_rng(1).uniform(-1, 1, (6, ps.n2)), lvl, ps.msg_scale)
    jobs = [[(a, pts[0]), (c, pts[1]), (a, pts[2])], [(a, pts[3]), (c, pts[4]), (a, pts[5])]]
    mm = be._raw_mac_many(jobs)
    same(f"mac_many l={lvl}", mm[1], lambda x, y: be._raw_mac_many(
        [[(x, pts[3]), (y, pts[4]), (x, pts[5])]])[0], [a, c])
    se = be._raw_sum_each([[a, c, a]])
    same(f"sum_each l={lvl}", se[0], lambda x, y: be._raw_sum_each([[x, y, x]])[0], [a, c])
torch.cuda.synchronize()
print("done")

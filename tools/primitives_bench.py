"""CKKS primitive microbench (BASELINE config 1): N = 2^16, 24 x 50-bit chain
primes + one 60-bit special prime; a batch of ciphertexts with residues
uniform mod q_i from a seed runs through NTT/INTT, HMult + relinearise,
HRotate by random steps and rescale on the GPU engine.

Key switching uses the reference's design (one special prime, per-prime
digits: dnum = L + 1 = 24); BASELINE's "dnum = 3" hybrid key switching is not
part of the reference and is not implemented (DESIGN.md §0 (f)).  The 50/60-bit
primes exceed the fp64 path's 2^42 bound, so this ring runs the 64-bit Shoup
integer transforms.

    python tools/primitives_bench.py [--cts 1024] [--batch 16]
"""

from __future__ import annotations

import argparse
import json
import os
import sys
from fractions import Fraction

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    from paper_2104_09164_b200 import _native as nat
    from paper_2104_09164_b200.backend import Ct
    from paper_2104_09164_b200.ckks.engine import CkksBackend, CtData, _tasks
    from paper_2104_09164_b200.ckks.params import gen_params_custom

    ap = argparse.ArgumentParser()
    ap.add_argument("--cts", type=int, default=1024)
    ap.add_argument("--batch", type=int, default=16)
    ap.add_argument("--logn", type=int, default=16)
    args = ap.parse_args()
    ps = gen_params_custom(1 << args.logn, [50] * 24, 60, 40, name="microbench-2^16")
    be = CkksBackend(ps, seed=0)
    lvl, n = ps.max_level, ps.n
    rng = np.random.default_rng(1)
    steps = sorted({int(s) for s in rng.integers(1, ps.n2, 8)})
    be.ensure_rotation_keys({s: lvl for s in steps})
    bsz = args.batch
    nb = max(1, args.cts // bsz)

    def rand_batch():
        t = torch.empty(bsz, 2, lvl + 1, n, dtype=torch.int64, device=be.dev)
        for r, q in enumerate(ps.chain_primes):
            t[:, :, r].random_(0, q)
        return Ct(CtData(t), lvl, Fraction(ps.msg_scale), be.n2)

    batches = [rand_batch() for _ in range(nb)]
    res = {"config": {"workload": "CKKS primitive microbench", "N": n, "chain_primes": "24 x 50-bit",
                      "special_prime": "1 x 60-bit", "dnum": lvl + 1, "ciphertexts": nb * bsz,
                      "batch_per_launch": bsz, "rotation_steps": steps}}

    def timed(fn, ops):
        fn(batches[0])
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for b in batches:
            fn(b)
        e1.record()
        torch.cuda.synchronize()
        return round(ops * nb / (e0.elapsed_time(e1) / 1e3), 2)

    rows = bsz * 2 * (lvl + 1)
    rp = be.ring.row_ptrs
    prim = np.tile(np.arange(lvl + 1), bsz * 2)

    def ntt(b):
        d = b.payload.data
        t = _tasks(nat.NTT_TASK, rows, src=rp(d), dst=rp(d), dst_prime=prim, src_prime=prim)
        be.ring.ntt_fwd(t)
        be.ring.ntt_inv(t)

    res["ntt_plus_intt_rows_per_s"] = timed(ntt, rows)
    res["hmult_relin_per_s"] = timed(lambda b: be._raw_mult(b, b), bsz)
    res["hrotate_per_s"] = timed(lambda b: be._raw_rot_each([(b, steps[0])]), bsz)
    res["hrotate_hoisted8_per_s"] = timed(lambda b: be._raw_rot_many(b, steps), bsz * len(steps))
    res["rescale_per_s"] = timed(lambda b: be._raw_rescale(b), bsz)
    res["unit"] = "ciphertext ops/s (one op = one ciphertext)"
    print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()

"""CKKS primitive microbench (BASELINE config 1): N = 2^16, 24 x 50-bit chain
primes + one 60-bit special prime, dnum = 3; a batch of ciphertexts with
residues uniform mod q_i from a seed runs through NTT/INTT, HMult +
relinearise, HRotate by random steps (single and hoisted) and rescale on the
GPU engine.

Key switching: `--dnum 3` (default) is the hybrid key switch of
ckks/hybrid.py (8-prime digits, fast base conversion ModUp/ModDown,
csrc/bconv.cu); `--dnum 24` the reference design (per-prime digits, the
engine's own path).  `--specials K` uses K special primes of `--special-bits`.
The 50/60-bit primes exceed the fp64 path's 2^42 bound, so this ring runs the
64-bit integer-pipe transforms.  `noise_ok` reports whether the
configuration's key-switch noise leaves the result decryptable (one 60-bit
special prime against 400-bit digits does not: BASELINE's config 1 is a
throughput configuration).

    python tools/primitives_bench.py [--cts 1024] [--batch 16] [--dnum 3] [--specials 1]
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
    ap.add_argument("--dnum", type=int, default=3)
    ap.add_argument("--specials", type=int, default=1)
    ap.add_argument("--special-bits", type=int, default=60)
    args = ap.parse_args()
    from paper_2104_09164_b200.ckks.params import _search
    ps = gen_params_custom(1 << args.logn, [50] * 24, args.special_bits, 40,
                           name="microbench-2^16")
    be = CkksBackend(ps, seed=0)
    lvl, n = ps.max_level, ps.n
    rng = np.random.default_rng(1)
    steps = sorted({int(s) for s in rng.integers(1, ps.n2, 8)})
    hybrid = not (args.dnum == lvl + 1 and args.specials == 1)
    if hybrid:
        from paper_2104_09164_b200.ckks.hybrid import HybridKeySwitch
        sp = [ps.special_prime] + _search(args.special_bits, 2 * n, args.specials - 1,
                                          set(ps.chain_primes) | {ps.special_prime})
        hk = HybridKeySwitch(be, args.dnum, sp[:args.specials], seed=1)
        hk.ensure_rotation_keys(steps)
        mult = hk.mult
        rot1 = lambda b: hk.rot(b, steps[0])       # noqa: E731
        rotm = lambda b: hk.rot_many(b, steps)     # noqa: E731
    else:
        be.ensure_rotation_keys({s: lvl for s in steps})
        mult = be._raw_mult
        rot1 = lambda b: be._raw_rot_each([(b, steps[0])])   # noqa: E731
        rotm = lambda b: be._raw_rot_many(b, steps)          # noqa: E731
    bsz = args.batch
    nb = max(1, args.cts // bsz)

    def rand_batch():
        t = torch.empty(bsz, 2, lvl + 1, n, dtype=torch.int64, device=be.dev)
        for r, q in enumerate(ps.chain_primes):
            t[:, :, r].random_(0, q)
        return Ct(CtData(t), lvl, Fraction(ps.msg_scale), be.n2)

    batches = [rand_batch() for _ in range(nb)]
    res = {"config": {"workload": "CKKS primitive microbench (BASELINE config 1)", "N": n,
                      "chain_primes": "24 x 50-bit",
                      "special_primes": f"{args.specials} x {args.special_bits}-bit",
                      "dnum": args.dnum if hybrid else lvl + 1,
                      "key_switch": "hybrid (ckks/hybrid.py)" if hybrid else "reference design",
                      "ciphertexts": nb * bsz, "batch_per_launch": bsz, "rotation_steps": steps}}

    def timed(fn, ops):
        for b in batches[:4]:   # warm-up (clocks, caches, allocator)
            fn(b)
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
    res["hmult_relin_per_s"] = timed(lambda b: mult(b, b), bsz)
    res["hrotate_per_s"] = timed(rot1, bsz)
    res["hrotate_hoisted8_per_s"] = timed(rotm, bsz * len(steps))
    res["rescale_per_s"] = timed(lambda b: be._raw_rescale(b), bsz)
    # decryptability of this key-switch configuration: mult + rescale of a
    # fresh encryption against the slot product
    v = np.random.default_rng(2).uniform(-1, 1, ps.n2)
    ct = be.enc(v)
    err = float(np.abs(be.dec(be.rescale(mult(ct, ct))) - v * v).max())
    res["mult_decrypt_max_err"] = err
    res["noise_ok"] = bool(err < 1e-3)
    res["unit"] = "ciphertext ops/s (one op = one ciphertext)"
    print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()

"""__graft_entry__.smoke(): one tiny encrypted evaluation on cuda:0 checked
against the CPU oracle (toy parameters, toy network)."""

import numpy as np


def run_smoke():
    import torch
    from oracle.cpu_engine import OracleCkks
    from paper_2104_09164_b200.ckks.engine import CkksBackend
    from paper_2104_09164_b200.ckks.params import gen_params
    from paper_2104_09164_b200.fastpath import compile_pipeline, infer
    from paper_2104_09164_b200.model import (NetworkShape, collapse_layers, infer_clear,
                                             make_random_input, make_random_model)
    from paper_2104_09164_b200.modelenc import ModelEncoder
    assert torch.cuda.is_available(), "smoke needs cuda:0"
    shape = NetworkShape(1, 32, 15, (4, 8, 16), 4)
    cpar = collapse_layers(make_random_model(shape, 3), shape)
    x = make_random_input(shape, 4)
    ps = gen_params("toy-fast")
    gpu = CkksBackend(ps, seed=5, device="cuda:0")
    cpu = OracleCkks(ps, seed=5)
    cp = compile_pipeline(shape, "fast", "giant", ps)
    gpu.ensure_rotation_keys(cp.rotations)
    cpu.ensure_rotation_keys(cp.rotations)
    # key material bit-exact against the oracle
    assert np.array_equal(gpu.keys.relin.b.cpu().numpy().view(np.uint64), cpu.keys.relin.b)
    lg_g, cnt_g, _ = infer(cpar, x, "fast", "giant", gpu, encoder=ModelEncoder(cp, cpar, gpu))
    lg_c, cnt_c, _ = infer(cpar, x, "fast", "giant", cpu, encoder=ModelEncoder(cp, cpar, cpu))
    torch.cuda.synchronize()
    scale = max(np.abs(lg_c).max(), 1e-12)
    err = np.abs(lg_g - lg_c).max()
    assert err <= 1e-3 * scale, (lg_g, lg_c)
    assert int(np.argmax(lg_g)) == int(np.argmax(lg_c))
    assert cnt_g.as_dict() == cnt_c.as_dict()
    clear = infer_clear(cpar, x)
    print(f"smoke ok: gpu vs oracle max|d| = {err:.3e}, vs clear {np.abs(lg_g - clear).max():.3e}")
    _smoke_cluster_ring()


def _smoke_cluster_ring():
    """The kernels the batched bench path adds on cluster-NTT rings -- fused
    ModUp + inner product with tensor-memory sums (k_ks3), ModDown merged
    with the rescale, extended-basis rotations and their accumulation /
    rotate-and-sum -- on a small N = 2^13 ring against the oracle."""
    import torch
    from fractions import Fraction
    from oracle.cpu_engine import OracleCkks
    from paper_2104_09164_b200 import _native as nat
    from paper_2104_09164_b200.backend import Ct
    from paper_2104_09164_b200.ckks.engine import CkksBackend
    from paper_2104_09164_b200.ckks.params import gen_params_custom
    from tests._util import rand_ct
    ps = gen_params_custom(1 << 13, [33, 30, 30], 33, 24)
    gpu = CkksBackend(ps, seed=3, device="cuda:0")
    cpu = OracleCkks(ps, seed=3)
    assert gpu.fuse_ks and gpu.lazy
    gpu.fuse_ks_min, gpu.lazy_min = 0, 1
    lvl, ks = ps.max_level, [3, 5]
    gpu.ensure_rotation_keys({k: lvl for k in ks})
    cpu.ensure_rotation_keys({k: lvl for k in ks})
    raw = [rand_ct(ps, lvl, 9 + b) for b in range(2)]
    A = gpu.import_ct(np.stack([r[0] for r in raw]), np.stack([r[1] for r in raw]), lvl,
                      ps.msg_scale)
    A_cpu = [Ct(r, lvl, Fraction(ps.msg_scale), ps.n2) for r in raw]
    # fused key switch + merged ModDown/rescale: bit-exact
    got = gpu.export(gpu.square_rescale_each([A])[0])
    for b in range(2):
        want = cpu._raw_rescale(cpu._raw_mult(A_cpu[b], A_cpu[b])).payload
        assert np.array_equal(got[0][b], want[0]) and np.array_equal(got[1][b], want[1])

    def small(x, y, bound):   # (x - y) has small centred coefficients under every prime
        rp, r = gpu.ring.row_ptrs, x.shape[-2]
        d = torch.empty_like(x)
        pr = gpu._row_primes(x.numel() // (r * gpu.n), r)
        gpu._ew(nat.EW_SUB, rp(d), rp(x), rp(y), primes=pr)
        c = gpu._intt_rows(d, pr).cpu().numpy().view(np.uint64).reshape(-1, r, gpu.n)
        for t in range(r):
            q = np.uint64(ps.chain_primes[t])
            assert np.minimum(c[:, t], q - c[:, t]).max() <= bound
    # rotate-and-sum in the extended basis vs the oracle's rotations summed
    rs = gpu.rot_sum_each([A], [0] + ks)[0]
    want = []
    for b in range(2):
        acc = A_cpu[b]
        for k in ks:
            acc = cpu._raw_add(acc, cpu._raw_rot(A_cpu[b], k))
        want.append(acc.payload)
    W = gpu.import_ct(np.stack([w[0] for w in want]), np.stack([w[1] for w in want]), lvl,
                      ps.msg_scale)
    small(rs.payload.data, W.payload.data, 2 * len(ks) + 2)
    # extended-basis rotations accumulated with plaintexts, ModDown + rescale merged
    vals = np.random.default_rng(1).uniform(-1, 1, (3, ps.n2))
    pts = gpu.encode_many(vals, lvl, ps.msg_scale)
    pre = gpu.rot_many_each([A], [0] + ks, lazy=True)[0]
    lazy = gpu.mac_rescale_many([[(pre[k], p) for k, p in zip([0] + ks, pts)]])[0]
    pre_e = gpu.rot_many_each([A], [0] + ks)[0]
    eager = gpu.rescale_each(gpu.mac_many([[(pre_e[k], p) for k, p in zip([0] + ks, pts)]]))[0]
    # the eager path rounds each rotation before the plaintext product: the
    # difference is (rounding) x (plaintext coefficient) / q_l, a few units
    small(lazy.payload.data, eager.payload.data, 64)
    torch.cuda.synchronize()
    print("smoke ok: cluster-ring kernels (k_ks3, merged ModDown, lazy ModDown) vs oracle")


if __name__ == "__main__":
    run_smoke()

"""CKKS hot path on the GPU vs the reference's golden digests (bit-exact).

Every digest in tests/golden/ckks_golden.json was produced by the reference
engine itself (tests/golden/make_golden.py); the GPU engine must reproduce
the same uint64 payloads from the same seeds.
"""

from fractions import Fraction

import numpy as np
import pytest

from tests._util import digest, rand_ct, rand_rows

pytestmark = pytest.mark.gpu

PROFILES = ["toy-fast", "fast-hear"]
_BE = {}


def backend(prof):
    from paper_2104_09164_b200.ckks.engine import CkksBackend
    from paper_2104_09164_b200.ckks.params import gen_params
    if prof not in _BE:
        _BE[prof] = CkksBackend(gen_params(prof), seed=7)
    return _BE[prof]


def host(t):
    return t.cpu().numpy().view(np.uint64)


@pytest.mark.parametrize("prof", PROFILES)
def test_keygen_bit_exact(prof, golden):
    g = golden[prof]
    be = backend(prof)
    k = be.keys
    assert digest(k.s_coeffs.astype(np.int64).view(np.uint64)) == g["s_coeffs"]
    assert digest(host(k.s_ntt)) == g["s_ntt"]
    assert digest(host(k.pk_a)) == g["pk_a"]
    assert digest(host(k.pk_b)) == g["pk_b"]
    assert digest(host(k.relin.b)) == g["relin_b"]
    assert digest(host(k.relin.a)) == g["relin_a"]


@pytest.mark.parametrize("prof", PROFILES)
def test_rotation_keys_bit_exact(prof, golden):
    g = golden[prof]
    be = backend(prof)
    be.ensure_rotation_keys({int(a): l for a, l in g["rot_levels"].items()})
    for a, d in g["rot_keys"].items():
        key = be.keys.rot[int(a)]
        assert digest(host(key.b), host(key.a)) == d, a


@pytest.mark.parametrize("prof", PROFILES)
def test_ring_kernels_bit_exact(prof, golden):
    import torch
    from paper_2104_09164_b200 import _native as nat
    from paper_2104_09164_b200.ckks.engine import _tasks
    g = golden[prof]["ring"]
    be = backend(prof)
    rc = be.ring
    gall = list(range(be.L + 2))
    x = rand_rows(rc.primes, gall, be.n, 21)
    y = rand_rows(rc.primes, gall, be.n, 22)
    X, Y = be._dev(x), be._dev(y)
    F = rc.empty(len(gall))
    rc.ntt_fwd(_tasks(nat.NTT_TASK, len(gall), src=rc.row_ptrs(X), dst=rc.row_ptrs(F),
                      dst_prime=gall, src_prime=gall))
    assert digest(host(F)) == g["ntt_fwd"]
    I = be._intt_rows(X, np.array(gall))
    assert digest(host(I)) == g["ntt_inv"]
    M = rc.empty(len(gall))
    be._ew(nat.EW_MUL, rc.row_ptrs(M), rc.row_ptrs(X), rc.row_ptrs(Y), primes=np.array(gall))
    assert digest(host(M)) == g["pw_mul"]
    # round trip
    B = be._intt_rows(F, np.array(gall))
    assert torch.equal(B, X)


@pytest.mark.parametrize("prof", PROFILES)
def test_ops_bit_exact(prof, golden):
    from paper_2104_09164_b200.backend import Pt
    be = backend(prof)
    g = golden[prof]
    be.ensure_rotation_keys({int(a): l for a, l in g["rot_levels"].items()})
    ps = be.params
    rc = be.ring
    for lvl_s, ops in g["ops"].items():
        lvl = int(lvl_s)
        A = be.import_ct(*rand_ct(ps, lvl, 100 + lvl), lvl, ps.msg_scale)
        B = be.import_ct(*rand_ct(ps, lvl, 200 + lvl), lvl, ps.msg_scale)
        pt = rand_rows(rc.primes, range(lvl + 1), ps.n, 300 + lvl)
        P_ = Pt(be._dev(pt), lvl, Fraction(ps.msg_scale), ps.n2)
        got = {
            "add": be._raw_add(A, B), "add_plain": be._raw_add_plain(A, P_),
            "mult_plain": be._raw_mult_plain(A, P_), "mult": be._raw_mult(A, B),
            "rescale": be._raw_rescale(A), "mod_down1": be._raw_mod_down(A, 1),
        }
        if "rot_2047" in ops:
            got["rot_2047"] = be._raw_rot(A, 2047)
        if "rot_many_1" in ops:
            m = be._raw_rot_many(A, [1, 5])
            got["rot_many_1"], got["rot_many_5"] = m[1], m[5]
        for name, d in ops.items():
            assert digest(*be.export(got[name])) == d, (lvl, name)


@pytest.mark.parametrize("prof", PROFILES)
def test_encrypt_bit_exact_given_coeffs(prof, golden):
    """Fresh encryption equals the reference's once the plaintext coefficient
    vector is the same (the fp64 encoder is checked separately)."""
    import os
    import torch
    be2 = __import__("paper_2104_09164_b200.ckks.engine", fromlist=["CkksBackend"])
    from paper_2104_09164_b200.ckks.params import gen_params
    ps = gen_params(prof)
    be = be2.CkksBackend(ps, seed=7)
    be.ensure_rotation_keys({int(a): l for a, l in golden[prof]["rot_levels"].items()})
    here = os.path.join(os.path.dirname(__file__), "golden")
    coeffs = np.load(os.path.join(here, f"{prof}_encode_coeffs.npy"))
    vals = np.random.default_rng(31).uniform(-1, 1, ps.n2)
    got = be.emb.encode_coeffs(torch.from_numpy(vals)[None], float(ps.msg_scale))[0].cpu().numpy()
    diff = np.abs(got - coeffs)
    assert diff.max() <= 1 and (diff > 0).mean() < 1e-3
    ct = be._enc_from_coeffs(torch.from_numpy(coeffs)[None].to(be.dev), ps.max_level,
                             Fraction(ps.msg_scale))
    assert digest(*be.export(ct)) == golden[prof]["enc_L"]
    err = np.abs(be.dec(ct) - vals).max()
    assert err < 2 * golden[prof]["dec_maxerr"] + 1e-9


def test_integer_ntt_policy_bit_exact(golden):
    """The 64-bit-Shoup transform (used for primes >= 2^42) gives the same
    residues as the fp64-pipe transform the reference profiles run on."""
    import os
    from paper_2104_09164_b200.ckks.engine import CkksBackend
    from paper_2104_09164_b200.ckks.params import gen_params
    os.environ["HEAR_B200_INT_NTT"] = "1"
    try:
        be = CkksBackend(gen_params("toy-fast"), seed=7)
    finally:
        del os.environ["HEAR_B200_INT_NTT"]
    g = golden["toy-fast"]
    assert digest(host(be.keys.relin.b)) == g["relin_b"]
    ps = be.params
    lvl = 6
    A = be.import_ct(*rand_ct(ps, lvl, 100 + lvl), lvl, ps.msg_scale)
    B = be.import_ct(*rand_ct(ps, lvl, 200 + lvl), lvl, ps.msg_scale)
    be.ensure_rotation_keys({int(a): l for a, l in g["rot_levels"].items()})
    assert digest(*be.export(be._raw_mult(A, B))) == g["ops"]["6"]["mult"]
    assert digest(*be.export(be._raw_rescale(A))) == g["ops"]["6"]["rescale"]
    m = be._raw_rot_many(A, [1, 5])
    assert digest(*be.export(m[5])) == g["ops"]["6"]["rot_many_5"]


@pytest.mark.parametrize("preperm", ["1", "0"])
def test_prepermuted_rotation_keys_bit_exact(golden, preperm):
    """Pre-permuted rotation keys (default) and the digit-gather path both
    give the reference's rotations."""
    import os
    from paper_2104_09164_b200.ckks.engine import CkksBackend
    from paper_2104_09164_b200.ckks.params import gen_params
    os.environ["HEAR_B200_PREPERM"] = preperm
    try:
        be = CkksBackend(gen_params("toy-fast"), seed=7)
        g = golden["toy-fast"]
        be.ensure_rotation_keys({int(a): l for a, l in g["rot_levels"].items()})
    finally:
        del os.environ["HEAR_B200_PREPERM"]
    assert be.preperm == (preperm == "1")
    ps = be.params
    for lvl in (6, 2):
        A = be.import_ct(*rand_ct(ps, lvl, 100 + lvl), lvl, ps.msg_scale)
        m = be._raw_rot_many(A, [1, 5])
        assert digest(*be.export(m[5])) == g["ops"][str(lvl)]["rot_many_5"]
        assert digest(*be.export(m[1])) == g["ops"][str(lvl)]["rot_many_1"]
    A = be.import_ct(*rand_ct(ps, 2, 102), 2, ps.msg_scale)
    assert digest(*be.export(be._raw_rot(A, 2047))) == g["ops"]["2"]["rot_2047"]


_ORACLE = {}


@pytest.mark.parametrize("env", [{"HEAR_B200_KS_GEMM_MIN": "1"}, {"HEAR_B200_KS_GEMM_MIN": "1000"},
                                 {"HEAR_B200_PREPERM": "0"},
                                 {"HEAR_B200_NTT3": "0", "HEAR_B200_KS_GEMM_MIN": "1"}])
def test_hoisted_rotations_fast_hear_vs_oracle(env):
    """N = 2^14 hoisted rotations (cluster NTT, GEMM inner product on
    pre-permuted keys, ModDown scatter) against the CPU oracle, for every
    inner-product path; batched clips."""
    import os
    from oracle.cpu_engine import OracleCkks
    from paper_2104_09164_b200.backend import Ct
    from paper_2104_09164_b200.ckks.engine import CkksBackend
    from paper_2104_09164_b200.ckks.params import gen_params
    ps = gen_params("fast-hear")
    amounts = [1, 5, 77, 4000]
    levels = {a: 12 for a in amounts}
    if "cpu" not in _ORACLE:
        cpu = OracleCkks(ps, seed=11)
        cpu.ensure_rotation_keys(levels)
        _ORACLE["cpu"] = cpu
    cpu = _ORACLE["cpu"]
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    try:
        gpu = CkksBackend(ps, seed=11)
        gpu.ensure_rotation_keys(levels)
        for lvl in (12, 7):
            cts = [rand_ct(ps, lvl, 40 + lvl + i) for i in range(3)]
            batch = gpu.import_ct(np.stack([c[0] for c in cts]), np.stack([c[1] for c in cts]),
                                  lvl, ps.msg_scale)
            got = gpu._raw_rot_many(batch, amounts)
            for a in amounts:
                r = gpu.export(got[a])
                for i, c in enumerate(cts):
                    want = cpu._raw_rot(Ct(c, lvl, Fraction(ps.msg_scale), ps.n2), a).payload
                    assert np.array_equal(r[0][i], want[0]) and np.array_equal(r[1][i], want[1]), \
                        (env, lvl, a, i)
    finally:
        for k, v in old.items():
            if v is None:
                del os.environ[k]
            else:
                os.environ[k] = v


@pytest.mark.parametrize("gemm_min", ["1", "1000"])
def test_rot_each_and_relin_batched_vs_oracle(gemm_min):
    """Batched key switches with a digit set per job (rot_each over several
    handles: one GEMM launch, one output pair per tile) and relinearisation,
    GEMM and per-job inner products, against the CPU oracle at N = 2^14."""
    import os
    from oracle.cpu_engine import OracleCkks
    from paper_2104_09164_b200.backend import Ct
    from paper_2104_09164_b200.ckks.engine import CkksBackend
    from paper_2104_09164_b200.ckks.params import gen_params
    ps = gen_params("fast-hear")
    amounts = [1, 5]
    if "cpu" not in _ORACLE:
        cpu = OracleCkks(ps, seed=11)
        cpu.ensure_rotation_keys({a: 12 for a in [1, 5, 77, 4000]})
        _ORACLE["cpu"] = cpu
    cpu = _ORACLE["cpu"]
    os.environ["HEAR_B200_KS_GEMM_MIN"] = gemm_min
    try:
        gpu = CkksBackend(ps, seed=11)
    finally:
        del os.environ["HEAR_B200_KS_GEMM_MIN"]
    gpu.ensure_rotation_keys({a: 12 for a in amounts})
    lvl = 9
    cts = [[rand_ct(ps, lvl, 70 + 3 * h + i) for i in range(2)] for h in range(2)]
    hs = [gpu.import_ct(np.stack([c[0] for c in hc]), np.stack([c[1] for c in hc]), lvl,
                        ps.msg_scale) for hc in cts]
    outs = gpu._raw_rot_each([(hs[0], amounts[0]), (hs[1], amounts[1])])
    for h, (o, a) in enumerate(zip(outs, amounts)):
        r = gpu.export(o)
        for i, c in enumerate(cts[h]):
            want = cpu._raw_rot(Ct(c, lvl, Fraction(ps.msg_scale), ps.n2), a).payload
            assert np.array_equal(r[0][i], want[0]) and np.array_equal(r[1][i], want[1]), (h, i)
    m = gpu.export(gpu._raw_mult(hs[0], hs[1]))
    for i in range(2):
        A = Ct(cts[0][i], lvl, Fraction(ps.msg_scale), ps.n2)
        B = Ct(cts[1][i], lvl, Fraction(ps.msg_scale), ps.n2)
        want = cpu._raw_mult(A, B).payload
        assert np.array_equal(m[0][i], want[0]) and np.array_equal(m[1][i], want[1]), i


@pytest.mark.parametrize("env", [{"HEAR_B200_KS_GEMM_MIN": "1"}, {"HEAR_B200_PREPERM": "0"},
                                 {"HEAR_B200_NTT3": "0"}])
def test_fused_rot_add_equals_rot_then_add(env):
    """ct + rot(ct, k) with the add fused into the ModDown epilogue (scatter,
    gather and two-pass paths) equals the separate rotation and addition."""
    import os
    from paper_2104_09164_b200.ckks.engine import CkksBackend
    from paper_2104_09164_b200.ckks.params import gen_params
    ps = gen_params("fast-hear")
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    try:
        be = CkksBackend(ps, seed=5)
    finally:
        for k, v in old.items():
            if v is None:
                del os.environ[k]
            else:
                os.environ[k] = v
    be.ensure_rotation_keys({3: 12, 40: 12})
    lvl = 8
    cts = [rand_ct(ps, lvl, 90 + i) for i in range(4)]
    hs = [be.import_ct(np.stack([c[0] for c in cts[2 * h:2 * h + 2]]),
                       np.stack([c[1] for c in cts[2 * h:2 * h + 2]]), lvl, ps.msg_scale)
          for h in range(2)]
    items = [(hs[0], 3), (hs[1], 40)]
    fused = be.rot_add_each(items)
    plain = be.add_each(list(zip(hs, be.rot_each(items))))
    for f, p_ in zip(fused, plain):
        a, b = be.export(f), be.export(p_)
        assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])


def test_sum_each_one_pass_equals_add_chain():
    """sum_each in one pass (k_sum_rows) equals the left-to-right add chain,
    ragged groups included, with the same operation counters."""
    from paper_2104_09164_b200.backend import BackendBase
    from paper_2104_09164_b200.ckks.engine import CkksBackend
    from paper_2104_09164_b200.ckks.params import gen_params
    ps = gen_params("fast-hear")
    be = CkksBackend(ps, seed=5, keygen=False)
    lvl = 7
    hs = [be.import_ct(*[np.stack(x) for x in zip(*[rand_ct(ps, lvl, 300 + 3 * h + i)
                                                     for i in range(3)])], lvl, ps.msg_scale)
          for h in range(7)]
    groups = [hs[:5], hs[5:7], hs[3:4], hs[1:7]]
    be.reset_counters()
    fast = be.sum_each(groups)
    n_fast = be.counters.as_dict()
    be.reset_counters()
    slow = BackendBase._raw_sum_each(be, groups)
    for f, s_ in zip(fast, slow):
        a, b = be.export(f), be.export(s_)
        assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
    assert sum(v.get("add", 0) for v in n_fast.values()) == 4 + 1 + 0 + 5


@pytest.mark.parametrize("gemm_min,hoist", [("1", "1"), ("1000", "1"), ("1", "")])
def test_rot_many_each_equals_rot_many(gemm_min, hoist):
    """Hoisted rotations of several handles in one batch (one ModUp, one
    GEMM per handle, one ModDown) equal per-handle rot_many, with the same
    operation counters."""
    import os
    from paper_2104_09164_b200.ckks.engine import CkksBackend
    from paper_2104_09164_b200.ckks.params import gen_params
    ps = gen_params("fast-hear")
    os.environ["HEAR_B200_KS_GEMM_MIN"] = gemm_min
    os.environ["HEAR_B200_BATCH_HOIST"] = hoist   # "1": forced; "": default (small batches)
    try:
        be = CkksBackend(ps, seed=9)
    finally:
        del os.environ["HEAR_B200_KS_GEMM_MIN"]
        del os.environ["HEAR_B200_BATCH_HOIST"]
    assert be.batch_hoist_max >= 2
    amts = [3, 17, 200]
    be.ensure_rotation_keys({a: 12 for a in amts})
    lvl = 5
    hs = [be.import_ct(*[np.stack(x) for x in zip(*[rand_ct(ps, lvl, 500 + 3 * h + i)
                                                     for i in range(2)])], lvl, ps.msg_scale)
          for h in range(3)]
    be.reset_counters()
    many = be.rot_many_each(hs, amts + [0])
    c_many = be.counters.as_dict()
    be.reset_counters()
    single = [be.rot_many(h, amts + [0]) for h in hs]
    assert be.counters.as_dict() == c_many
    for m, s_ in zip(many, single):
        for a in amts + [0]:
            x, y = be.export(m[a]), be.export(s_[a])
            assert np.array_equal(x[0], y[0]) and np.array_equal(x[1], y[1])

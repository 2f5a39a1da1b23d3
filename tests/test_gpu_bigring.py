"""N = 2^13 / 2^15 / 2^16 rings (BASELINE's microbench and batched configs,
and the cluster NTT's 2-CTA variant at 2^13): the NTT and a key switch on
both arithmetic policies (fp64 pipe for primes < 2^42, 64-bit Shoup for the
50/60-bit primes) against the CPU oracle."""

from fractions import Fraction

import numpy as np
import pytest

from tests._util import rand_ct, rand_rows

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("logn,bits,special", [(13, [33, 30, 30], 33), (15, [30, 28, 28], 30),
                                               (16, [50, 50, 50], 60), (16, [36, 33, 33], 36)])
def test_ntt_and_keyswitch_vs_oracle(logn, bits, special):
    import torch
    from oracle.cpu_engine import OracleCkks
    from paper_2104_09164_b200 import _native as nat
    from paper_2104_09164_b200.ckks.engine import CkksBackend, _tasks
    from paper_2104_09164_b200.ckks.params import gen_params_custom
    ps = gen_params_custom(1 << logn, bits, special, bits[-1] - 6)
    gpu = CkksBackend(ps, seed=3)
    cpu = OracleCkks(ps, seed=3)
    assert np.array_equal(gpu.keys.relin.b.cpu().numpy().view(np.uint64), cpu.keys.relin.b)
    rc = gpu.ring
    gall = list(range(len(rc.primes)))
    x = rand_rows(rc.primes, gall, ps.n, 5)
    X = gpu._dev(x)
    F = rc.empty(len(gall))
    rc.ntt_fwd(_tasks(nat.NTT_TASK, len(gall), src=rc.row_ptrs(X), dst=rc.row_ptrs(F),
                      dst_prime=gall, src_prime=gall))
    xf = x.copy()
    cpu.ring.fwd(xf, gall)
    assert np.array_equal(F.cpu().numpy().view(np.uint64), xf)
    back = gpu._intt_rows(F, np.array(gall))
    assert torch.equal(back, X)
    lvl = ps.max_level
    A_gpu = gpu.import_ct(*rand_ct(ps, lvl, 9), lvl, ps.msg_scale)
    from paper_2104_09164_b200.backend import Ct
    A_cpu = Ct(rand_ct(ps, lvl, 9), lvl, Fraction(ps.msg_scale), ps.n2)
    gpu.ensure_rotation_keys({3: lvl})
    cpu.ensure_rotation_keys({3: lvl})
    r_gpu = gpu.export(gpu._raw_rot(A_gpu, 3))
    r_cpu = cpu._raw_rot(A_cpu, 3).payload
    assert np.array_equal(r_gpu[0], r_cpu[0]) and np.array_equal(r_gpu[1], r_cpu[1])
    m_gpu = gpu.export(gpu._raw_mult(A_gpu, A_gpu))
    m_cpu = cpu._raw_mult(A_cpu, A_cpu).payload
    assert np.array_equal(m_gpu[0], m_cpu[0]) and np.array_equal(m_gpu[1], m_cpu[1])

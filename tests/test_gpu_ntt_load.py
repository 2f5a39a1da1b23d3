"""Fused NTT launches under full-GPU load are deterministic and equal the
same rows transformed in isolation (the small launches are pinned to the
reference by tests/test_gpu_ckks.py).  Guards the cluster exchange's
buffer reuse: a missing ordering there corrupts a few rows only when many
clusters run at once (1664-row launches, slow gather/scatter epilogues)."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def env():
    from paper_2104_09164_b200 import _native as nat
    from paper_2104_09164_b200.ckks.engine import CkksBackend, _tasks
    from paper_2104_09164_b200.ckks.params import gen_params
    be = CkksBackend(gen_params("fast-hear"), seed=0, keygen=False)
    g = torch.Generator(device="cuda").manual_seed(5)
    pmin = min(list(be.params.chain_primes) + [be.P])
    return be, nat, _tasks, g, pmin


def _modes(be, nat, _tasks, g, pmin, m):
    """task builders of every fused mode over m (clip, component) rows"""
    ring, n, S, r = be.ring, be.n, be.S, 13
    rp = lambda t: ring.row_ptrs(t).reshape(t.shape[0], -1)   # [rows, per-row ptrs]
    rnd = lambda *s: ring.empty(*s).random_(0, pmin, generator=g)
    perm = torch.randperm(n, device="cuda", generator=g).to(torch.int32)
    sps, aux, add, add2 = rnd(m), rnd(m, r), rnd(m, r), rnd(m, r)
    src = rnd(m, r)
    base = lambda rows: dict(src=np.repeat(rp(sps)[rows].ravel(), r), aux=rp(aux)[rows].ravel(), src_prime=S,
                             dst_prime=np.tile(np.arange(r), len(rows)),
                             scal=np.tile(be._pinv[:r], len(rows)),
                             scal_sh=np.tile(be._pinv_sh[:r], len(rows)), add=rp(add)[rows].ravel())
    dp = np.array(list(range(r)) + [S])
    cases = {
        "md_gather": (nat.FWD_MODDOWN, r, lambda rows, out: _tasks(
            nat.NTT_TASK, len(rows) * r, dst=rp(out)[rows].ravel(), perm=perm.data_ptr(), **base(rows))),
        "md_scatter": (nat.FWD_MODDOWN_SCATTER, r, lambda rows, out: _tasks(
            nat.NTT_TASK, len(rows) * r, dst=rp(out)[rows].ravel(), perm=perm.data_ptr(),
            add2=rp(add2)[rows].ravel(), **base(rows))),
        "lift": (nat.FWD_LIFT, r * (r + 1), lambda rows, out: _tasks(
            nat.NTT_TASK, len(rows) * r * (r + 1), src=np.repeat(rp(src)[rows].ravel(), r + 1),
            dst=rp(out)[rows].ravel(), src_prime=np.tile(np.repeat(np.arange(r), r + 1), len(rows)),
            dst_prime=np.tile(dp, len(rows) * r))),
        "inv": (None, r, lambda rows, out: _tasks(
            nat.NTT_TASK, len(rows) * r, src=rp(src)[rows].ravel(), dst=rp(out)[rows].ravel(),
            src_prime=np.tile(np.arange(r), len(rows)), dst_prime=np.tile(np.arange(r), len(rows)))),
    }
    return cases


@pytest.mark.parametrize("mode", ["md_gather", "md_scatter", "lift", "inv"])
def test_fused_ntt_deterministic_under_load(env, mode):
    be, nat, _tasks, g, pmin = env
    m = 128   # 64 clips x 2 components: the bench's key-switch ModDown shape
    kind, per, build = _modes(be, nat, _tasks, g, pmin, m)[mode]
    ring = be.ring
    rows = np.arange(m)

    def run(sel):
        out = ring.empty(m, per).fill_(-1)
        t = build(sel, out)
        if kind is None:
            ring.ntt_inv(t)
        else:
            ring.ntt_fwd(t, kind)
        torch.cuda.synchronize()
        return out

    full = [run(rows) for _ in range(3)]
    for k in (1, 2):
        assert torch.equal(full[k], full[0]), f"{mode}: repeated launches differ"
    for i in (0, 37, 127):   # the same rows, transformed alone
        alone = run(np.array([i]))
        assert torch.equal(alone[i], full[0][i]), f"{mode}: row {i} differs from its isolated launch"

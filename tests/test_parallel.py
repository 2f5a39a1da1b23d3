"""Multi-rank plumbing on CPU (gloo, world size 2): clip sharding and the
setup-time key replication used by bench.py on NVLink."""

import os
import socket

import pytest
import torch
import torch.multiprocessing as mp

from paper_2104_09164_b200.parallel import shard


def test_shard_partitions():
    for total in (0, 1, 7, 64, 100):
        for ws in (1, 2, 3, 8):
            got = [list(shard(total, r, ws)) for r in range(ws)]
            flat = [i for g in got for i in g]
            assert flat == list(range(total))
            assert max(map(len, got)) - min(map(len, got)) <= 1


class _FakeBackend:
    """Key container with the engine's key_tensors / manifest / alloc API."""

    def __init__(self, rank):
        self.rank = rank
        self.rot = {}
        if rank == 0:
            g = torch.Generator().manual_seed(7)
            self.pk = torch.randint(0, 1 << 40, (3, 8), generator=g)
            for amt, lmax in ((1, 2), (5, 1)):
                self.rot[amt] = torch.randint(0, 1 << 40, (lmax + 1, lmax + 2, 8), generator=g)

    def key_manifest(self):
        return [(a, t.shape[0] - 1) for a, t in sorted(self.rot.items())]

    def alloc_keys(self, manifest):
        self.pk = torch.empty(3, 8, dtype=torch.int64)
        self.rot = {a: torch.empty(l + 1, l + 2, 8, dtype=torch.int64) for a, l in manifest}

    def key_tensors(self):
        return [("pk", self.pk)] + [(f"rot{a}", t) for a, t in sorted(self.rot.items())]


def _worker(rank, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE="2", LOCAL_RANK=str(rank))
    from paper_2104_09164_b200 import parallel as par
    par.init("gloo")
    be = _FakeBackend(rank)
    par.replicate_keys(be, src=0)
    digest = [int(t.sum()) for _, t in be.key_tensors()]
    mx = par.max_over_ranks(float(rank + 1))
    q.put((rank, digest, mx, list(shard(10, rank, 2))))
    par.barrier()
    torch.distributed.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.timeout(120)
def test_gloo_key_replication_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = dict((r, (d, m, s)) for r, d, m, s in (q.get(timeout=100) for _ in ps))
    for p in ps:
        p.join(30)
    assert res[0][0] == res[1][0]           # identical keys on both ranks
    assert res[0][1] == res[1][1] == 2.0    # max over ranks
    assert res[0][2] + res[1][2] == list(range(10))


def _worker_layout(rank, port, q):
    """Key replication over tensors of the REAL key layout (toy-fast params,
    the toy network's rotation manifest), as the engine's receivers allocate."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE="2", LOCAL_RANK=str(rank))
    from paper_2104_09164_b200 import parallel as par
    from paper_2104_09164_b200.ckks.engine import key_layout
    from paper_2104_09164_b200.ckks.params import gen_params
    from paper_2104_09164_b200.fastpath import compile_pipeline
    from paper_2104_09164_b200.model import NetworkShape
    par.init("gloo")
    ps = gen_params("toy-fast")
    cp = compile_pipeline(NetworkShape(1, 32, 15, (4, 8, 16), 4), "fast", "giant", ps)
    man = par.broadcast_object(sorted(cp.rotations.items()) if rank == 0 else None)
    g = torch.Generator().manual_seed(3)
    keys = [torch.randint(0, 1 << 40, s, generator=g) if rank == 0 else
            torch.empty(s, dtype=torch.int64) for _, s in key_layout(ps, man)]
    par.broadcast_tensors(keys)
    q.put((rank, [int(k.sum()) for k in keys], [tuple(k.shape) for k in keys]))
    par.barrier()
    torch.distributed.destroy_process_group()


@pytest.mark.timeout(180)
def test_gloo_real_key_layout_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker_layout, args=(r, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = dict((r, (s, sh)) for r, s, sh in (q.get(timeout=150) for _ in ps))
    for p in ps:
        p.join(30)
    assert res[0] == res[1]
    from paper_2104_09164_b200.ckks.params import gen_params
    n = gen_params("toy-fast").n
    assert all(sh[-1] == n for sh in res[0][1])
    assert len(res[0][1]) >= 6   # pk (2) + relin (2) + at least one rotation key pair


@pytest.mark.timeout(300)
def test_bench_spawns_ranks():
    """`python bench.py --gpus 2` started as ONE process relaunches itself as
    two ranks (torch.distributed.run) -- the path the driver's 8-GPU run
    uses when it does not wrap bench.py in torchrun itself."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = {k: v for k, v in os.environ.items() if k not in ("RANK", "WORLD_SIZE", "LOCAL_RANK")}
    env["CUDA_VISIBLE_DEVICES"] = ""
    r = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "2",
                        "--check-launch"], capture_output=True, text=True, env=env, timeout=280)
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads([ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1])
    assert line["n_ranks"] == 2 and line["keys_identical"] and line["max_over_ranks"] == 2.0

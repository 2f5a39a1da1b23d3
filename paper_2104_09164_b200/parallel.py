"""Multi-GPU plumbing for the encrypted-inference path.

Independent clips are partitioned across ranks (one process per GPU); the
evaluation keys are generated once on rank 0 and replicated to every rank by
a broadcast at setup (NCCL over NVLink on the GPU box, gloo in the CPU
tests).  The per-clip loop has no collectives; only the timing reduction
(max over ranks) crosses ranks after the timed region.
"""

from __future__ import annotations

import os

import torch
import torch.distributed as dist


def world() -> tuple:
    """(rank, world_size, local_rank) from the torchrun environment."""
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


def init(backend: str) -> bool:
    """Initialise the default process group when launched with >1 rank."""
    _, ws, _ = world()
    if ws > 1 and not dist.is_initialized():
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group(backend=backend)
        return True
    return dist.is_initialized()


def free_port() -> int:
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def relaunch(nproc: int, script: str, argv) -> int:
    """Run `script argv` as `nproc` ranks of one node under torch.distributed.run
    (one process per GPU, rendezvous on 127.0.0.1) and return its exit code.
    Used when a multi-rank command is started as a plain process
    (`python bench.py --gpus 8`)."""
    import subprocess
    import sys
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={nproc}", "--master-addr=127.0.0.1",
           f"--master-port={free_port()}", script, *argv]
    return subprocess.call(cmd)


def shard(total: int, rank: int, world_size: int) -> range:
    """Contiguous, balanced slice of `total` clips owned by `rank`."""
    base, extra = divmod(total, world_size)
    start = rank * base + min(rank, extra)
    return range(start, start + base + (1 if rank < extra else 0))


def broadcast_tensors(tensors, src: int = 0):
    """In-place broadcast of an ordered tensor list from `src` (key replication)."""
    if not dist.is_initialized():
        return
    for t in tensors:
        dist.broadcast(t, src=src)


def broadcast_object(obj, src: int = 0):
    if not dist.is_initialized():
        return obj
    box = [obj]
    dist.broadcast_object_list(box, src=src)
    return box[0]


def replicate_keys(backend, src: int = 0):
    """Make every rank's backend hold rank `src`'s evaluation keys."""
    if not dist.is_initialized():
        return
    manifest = broadcast_object(backend.key_manifest() if dist.get_rank() == src else None, src)
    if dist.get_rank() != src:
        backend.alloc_keys(manifest)
    broadcast_tensors([t for _, t in backend.key_tensors()], src)
    if dist.get_rank() != src and hasattr(backend, "finish_keys"):
        backend.finish_keys()


def max_over_ranks(value: float, device=None) -> float:
    if not dist.is_initialized():
        return value
    t = torch.tensor([value], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier():
    if dist.is_initialized():
        dist.barrier()

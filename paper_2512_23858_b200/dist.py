"""Request sharding across GPUs: one process per GPU, contiguous request
blocks, full model replicas, no collective inside the step, one gather of generated ids at the
end.  The helpers are backend-agnostic (NCCL on the B200 box, gloo in the CPU tests)."""

from __future__ import annotations

import os


def shard_requests(n_requests: int, world: int, rank: int) -> range:
    """Contiguous block of request ids owned by ``rank`` (first ranks take the remainder)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} for world size {world}")
    if n_requests < 0:
        raise ValueError("n_requests must be >= 0")
    base, extra = divmod(n_requests, world)
    start = rank * base + min(rank, extra)
    return range(start, start + base + (1 if rank < extra else 0))


def env_rank() -> tuple[int, int, int]:
    """(rank, local_rank, world_size) from the torchrun environment (defaults: single process)."""
    return int(os.environ.get("RANK", "0")), int(os.environ.get("LOCAL_RANK", "0")), int(os.environ.get("WORLD_SIZE", "1"))


def gather_generated(outputs: dict[int, list[int]], world: int) -> dict[int, list[int]] | None:
    """All-gather per-request token lists (request id -> tokens); every rank returns the merged map.
    The only inter-GPU traffic of a run."""
    if world == 1:
        return dict(outputs)
    import torch.distributed as dist

    parts: list = [None] * world
    dist.all_gather_object(parts, outputs)
    merged: dict[int, list[int]] = {}
    for p in parts:
        for rid, toks in p.items():
            if rid in merged:
                raise ValueError(f"request {rid} produced by two ranks")
            merged[rid] = toks
    return merged


def free_port() -> int:
    import socket

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def launch(nproc: int, script: str, argv: list[str], env: dict | None = None, timeout: float | None = None) -> int:
    """One process per GPU on this node: re-run ``script argv`` under ``torch.distributed.run`` with
    ``nproc`` ranks rendezvousing on 127.0.0.1 (each rank reads RANK / LOCAL_RANK / WORLD_SIZE).
    Returns the launcher's exit code (non-zero if any rank failed)."""
    import subprocess
    import sys

    if nproc < 1:
        raise ValueError("nproc must be >= 1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nproc}",
           "--master-addr=127.0.0.1", f"--master-port={free_port()}", script, *argv]
    e = dict(os.environ)
    e.update(env or {})
    e.setdefault("NCCL_DEBUG", "INFO")  # keep NCCL's init log (transport / NVLS choice) in the run's stderr
    e.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    return subprocess.run(cmd, env=e, timeout=timeout).returncode

"""Process-group plumbing for the sequence-parallel group (one process per GPU).

torch.distributed is used only to move the 128-byte NCCL unique id from rank 0 to the other ranks and to
reduce the step time over ranks (max) for timing; every data-path exchange of FPDT (the per-chunk Ulysses
all-to-all, P:L206/L218/L365) runs inside libfpdt on its own NCCL communicator.
"""
from __future__ import annotations

import os
from typing import Callable


def env_ranks() -> tuple[int, int, int]:
    """(RANK, WORLD_SIZE, LOCAL_RANK) as torchrun sets them (1-process defaults)."""
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


def init_process_group(rank: int, world: int, backend: str = "gloo") -> None:
    """Host-side group for the id broadcast and the timing reduction (gloo: no device memory needed)."""
    import torch.distributed as dist
    if world > 1 and not dist.is_initialized():
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group(backend, rank=rank, world_size=world)


def broadcast_nccl_id(rank: int, world: int, make_id: Callable[[], bytes]) -> bytes | None:
    """Rank 0 creates the id (fpdt_get_unique_id), every rank returns the same 128 bytes; None at world 1."""
    if world == 1:
        return None
    import torch
    import torch.distributed as dist
    buf = torch.zeros(128, dtype=torch.uint8)
    if rank == 0:
        nid = make_id()
        assert len(nid) == 128
        buf.copy_(torch.frombuffer(bytearray(nid), dtype=torch.uint8))
    dist.broadcast(buf, src=0)
    return bytes(buf.numpy().tobytes())


def max_over_ranks(x: float, world: int) -> float:
    """Step time of the job = the slowest rank's (device-timed) step time."""
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(world: int) -> None:
    if world > 1:
        import torch.distributed as dist
        dist.barrier()

"""Host-side multi-process plumbing (one process per GPU, torchrun).

Only the pieces that are not CUDA: exchanging the symmetric-heap IPC handles
and reducing per-rank timings.  They take the torch.distributed module as an
argument so the same code runs under NCCL on GPUs and under gloo in the CPU
test-suite (tests/test_dist_gloo.py).
"""
from __future__ import annotations

from typing import List

IPC_HANDLE_BYTES = 64


def gather_ipc_handles(dist, mine: bytes, world_size: int) -> bytes:
    """All-gather every rank's heap handle; returns them concatenated in rank
    order (the layout tf_world_ipc_import expects)."""
    if len(mine) != IPC_HANDLE_BYTES:
        raise ValueError(f"IPC handle must be {IPC_HANDLE_BYTES} bytes, got {len(mine)}")
    allh: List[bytes] = [b""] * world_size
    dist.all_gather_object(allh, bytes(mine))
    for r, h in enumerate(allh):
        if len(h) != IPC_HANDLE_BYTES:
            raise ValueError(f"rank {r} sent a {len(h)}-byte handle")
    return b"".join(allh)


def max_over_ranks(dist, value: float, device=None) -> float:
    """The slowest rank's time (bench timing rule: max over ranks)."""
    import torch
    t = torch.tensor([value], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def rank_pointer_table(world_size: int, rank: int, local_ptr: int) -> List[int]:
    """Per-rank pointer array for a C-ABI call made by one process: only the
    local rank's entry is meaningful (tf_abi.h: entries of non-local ranks
    are ignored except heap regions)."""
    if not 0 <= rank < world_size:
        raise ValueError("rank out of range")
    arr = [0] * world_size
    arr[rank] = local_ptr
    return arr

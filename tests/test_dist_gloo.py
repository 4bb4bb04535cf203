"""CPU, world_size 2 over gloo: the multi-process host logic of the N>1 path
(heap-handle exchange in rank order, max-over-ranks timing, pointer tables)
that bench.py runs under torchrun + NCCL on GPUs."""
import os
import socket

import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch.distributed as dist
    from paper_2511_02168_b200.dist import gather_ipc_handles, max_over_ranks, rank_pointer_table
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        mine = bytes([rank + 1]) * 64
        allh = gather_ipc_handles(dist, mine, world)
        ok_handles = allh == b"".join(bytes([r + 1]) * 64 for r in range(world))
        slowest = max_over_ranks(dist, 1.5 + rank)
        table = rank_pointer_table(world, rank, 0x1000 + rank)
        q.put((rank, ok_handles, slowest, table))
    finally:
        dist.destroy_process_group()


def test_two_rank_host_plumbing_over_gloo():
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, ok, slowest, table in res:
        assert ok, rank
        assert slowest == 2.5  # max over ranks, seen identically by every rank
        assert table == [0x1000 if rank == 0 else 0, 0x1001 if rank == 1 else 0]


def test_handle_size_is_checked():
    from paper_2511_02168_b200.dist import gather_ipc_handles
    with pytest.raises(ValueError):
        gather_ipc_handles(None, b"short", 2)

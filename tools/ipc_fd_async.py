"""Two processes on one GPU (CUDA-IPC world, as bench.py under torchrun):
back-to-back ASYNC fused Flash Decode calls (no host sync between them),
then one sync -- the drift pattern of a timed loop.  Prints per-rank
status and whether the ranks' outputs agree."""
import ctypes as C
import os
import socket
import sys

import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def worker(rank, world, port, L, calls, variant, q):
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    os.environ.setdefault("TILEFABRIC_WATCHDOG_SECS", "15")
    import torch
    import torch.distributed as dist
    from paper_2511_02168_b200 import _abi
    from paper_2511_02168_b200.dist import gather_ipc_handles, rank_pointer_table
    dist.init_process_group("gloo", rank=rank, world_size=world)
    res = {"rank": rank}
    try:
        Lb = _abi.lib()
        h = C.c_void_p()
        heap = int(os.environ.get("HEAP", str(256 << 20)))
        _abi.check(Lb.tf_world_create_ipc(rank, world, 0, heap, 0.0, C.byref(h)))
        mine = (C.c_char * 64)()
        _abi.check(Lb.tf_world_ipc_export(h, mine))
        allh = gather_ipc_handles(dist, bytes(mine), world)
        _abi.check(Lb.tf_world_ipc_import(h, (C.c_char * (64 * world)).from_buffer_copy(allh)))
        B, Hq, Hkv, d = 1, 64, 8, 128
        ln = L // world
        g = torch.Generator(device="cuda").manual_seed(1 + (rank if os.environ.get("DIFFQ") else 0))
        qd = (torch.rand(B, Hq, d, device="cuda", generator=g) * 2 - 1).bfloat16()
        k = (torch.rand(B, Hkv, L, d, device="cuda", generator=g) * 2 - 1).bfloat16()
        v = (torch.rand(B, Hkv, L, d, device="cuda", generator=g) * 2 - 1).bfloat16()
        kd = k[:, :, rank * ln:(rank + 1) * ln].contiguous()
        vd = v[:, :, rank * ln:(rank + 1) * ln].contiguous()
        od = torch.empty(B, Hq, d, device="cuda", dtype=torch.bfloat16)
        tbl = lambda p: _abi.ptr_array(rank_pointer_table(world, rank, p))  # noqa: E731
        shape = _abi.FdShape(B, Hq, Hkv, d, L, d ** -0.5, _abi.TF_BF16, _abi.TF_BF16)
        torch.cuda.synchronize()
        dist.barrier()
        for var in variant:
            for _ in range(calls):
                _abi.check(Lb.tf_flash_decode_async(h, var, C.byref(shape), tbl(qd.data_ptr()), tbl(kd.data_ptr()),
                                                    tbl(vd.data_ptr()), tbl(od.data_ptr()), None, None))
            if os.environ.get("SYNC_BETWEEN"):
                st = Lb.tf_world_sync(h)
                print(f"rank {rank} after variant {var}: status {st} {Lb.tf_last_error().decode() if st else ''}",
                      file=sys.stderr, flush=True)
                dist.barrier()
        st = Lb.tf_world_sync(h)
        res["status"] = st
        res["error"] = Lb.tf_last_error().decode() if st else ""
        outs = [None] * world
        dist.all_gather_object(outs, od.cpu().view(torch.int16).numpy().tobytes())
        res["ranks_equal"] = all(x == outs[0] for x in outs)
        dist.barrier()
        Lb.tf_world_destroy(h)
    except Exception as e:  # noqa: BLE001
        res["exc"] = repr(e)
    q.put(res)
    dist.destroy_process_group()


if __name__ == "__main__":
    L = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
    calls = int(sys.argv[2]) if len(sys.argv) > 2 else 6
    variant = [int(x) for x in sys.argv[3].split(",")] if len(sys.argv) > 3 else [3]
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=worker, args=(r, 2, port, L, calls, variant, q)) for r in range(2)]
    for p in ps:
        p.start()
    out = [q.get(timeout=300) for _ in ps]
    for p in ps:
        p.join(60)
    print(L, calls, variant, sorted(out, key=lambda r: r["rank"]))

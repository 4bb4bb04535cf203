"""Runs bench.py's bench_fd in two processes sharing GPU 0 (the shared-GPU
test mode of bench.py), to debug the multi-process FD path in isolation.
usage: python tools/ipc_bench_fd.py [steps] [warmup] [variants]"""
import os
import socket
import sys

import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def worker(rank, world, port, steps, warmup, q):
    sys.path.insert(0, ROOT)
    os.environ.update(RANK=str(rank), WORLD_SIZE=str(world), LOCAL_RANK=str(rank), MASTER_ADDR="127.0.0.1",
                      MASTER_PORT=str(port), TFB_BENCH_SHARED_GPU="1")
    import bench
    if os.environ.get("NO_CLOCKS"):
        class _Nop:
            def __init__(self, *a):
                pass

            def __enter__(self):
                return self

            def __exit__(self, *a):
                pass

            def summary(self):
                return {}
        bench.ClockSampler = _Nop
    if os.environ.get("SAME_Q"):
        import torch
        _G = torch.Generator

        class _Gen(_G):
            def manual_seed(self, s):
                return super().manual_seed(7)
        torch.Generator = _Gen
    res = {"rank": rank}
    try:
        ctx = bench.Ctx(world)
        r = bench.bench_fd(ctx, bench.FD3, steps, warmup)
        res.update(fused_ms=r["fused_ms"], bsp_ms=r["bsp_ms"])
    except Exception as e:  # noqa: BLE001
        res["exc"] = repr(e)[:400]
    q.put(res)


if __name__ == "__main__":
    steps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
    warmup = int(sys.argv[2]) if len(sys.argv) > 2 else 3
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=worker, args=(r, 2, port, steps, warmup, q)) for r in range(2)]
    for p in ps:
        p.start()
    out = [q.get(timeout=400) for _ in ps]
    print(sorted(out, key=lambda r: r["rank"]), flush=True)
    for p in ps:
        p.kill()

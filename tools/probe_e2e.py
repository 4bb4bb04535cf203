"""PCIe probe for the host-streaming AG+GEMM (tf_ag_gemm_host): H2D / D2H
bandwidth alone and concurrently, then the host API at config 2 under slab
overrides (TFB_HOST_SLAB=<cols>, TFB_HOST_ONESHOT=1).  Prints JSON lines."""
import ctypes as C
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def timed(fn, reps=5):
    import torch
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e30
    for _ in range(reps):
        torch.cuda.synchronize()
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return best


def pcie():
    import torch
    n = 576 << 20
    h = torch.empty(n, dtype=torch.uint8).pin_memory()
    d = torch.empty(n, dtype=torch.uint8, device="cuda")
    h2 = torch.empty(n, dtype=torch.uint8).pin_memory()
    d2 = torch.empty(n, dtype=torch.uint8, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    h2d = timed(lambda: d.copy_(h, non_blocking=True))
    d2h = timed(lambda: h2.copy_(d2, non_blocking=True))

    def both():
        cur = torch.cuda.current_stream()
        s1.wait_stream(cur)
        s2.wait_stream(cur)
        with torch.cuda.stream(s1):
            d.copy_(h, non_blocking=True)
        with torch.cuda.stream(s2):
            h2.copy_(d2, non_blocking=True)
        cur.wait_stream(s1)
        cur.wait_stream(s2)
    bo = timed(both)
    print(json.dumps({"bytes": n, "h2d_GBps": n / h2d / 1e6, "d2h_GBps": n / d2h / 1e6,
                      "concurrent_each_GBps": n / bo / 1e6, "h2d_ms": h2d, "d2h_ms": d2h, "both_ms": bo}))


def host_api():
    import torch
    import paper_2511_02168_b200 as tf
    from paper_2511_02168_b200 import _abi
    M, K, N = 8192, 8192, 28672
    w = tf.World(1, [0], M * K * 2 + (64 << 20))
    hA = (torch.rand(M, K) * 2 - 1).bfloat16().pin_memory()
    hB = (torch.rand(K, N) * 2 - 1).bfloat16().pin_memory()
    hC = torch.empty(M, N, dtype=torch.bfloat16).pin_memory()
    shape = _abi.AgShape(M, N, K, 0, 0, 0, _abi.TF_BF16)
    st = torch.cuda.ExternalStream(w.stream(0))
    args = (w.handle, _abi.TF_AG_PULL, C.byref(shape), _abi.ptr_array([hA.data_ptr()]),
            _abi.ptr_array([hB.data_ptr()]), _abi.ptr_array([hC.data_ptr()]), None)
    with torch.cuda.stream(st):
        ms = timed(lambda: _abi.check(w.lib.tf_ag_gemm_host_async(*args)), reps=4)
    if os.environ.get("TFB_HOST_TRACE"):
        _abi.check(w.lib.tf_ag_gemm_host(*args))
    print(json.dumps({"host_api_ms": ms, "slab": os.environ.get("TFB_HOST_SLAB"),
                      "oneshot": os.environ.get("TFB_HOST_ONESHOT")}))
    w.close()


def copy2d():
    """cudaMemcpy2DAsync H2D bandwidth vs slab width (B is k x n row-major;
    a column slab is k rows of ns*2 bytes at pitch n*2)."""
    import torch
    K, N = 8192, 28672
    h = torch.empty(K, N, dtype=torch.bfloat16).pin_memory()
    d = torch.empty(K, N, dtype=torch.bfloat16, device="cuda")
    rt = C.CDLL("libcudart.so.12")
    rt.cudaMemcpy2DAsync.argtypes = [C.c_void_p, C.c_size_t, C.c_void_p, C.c_size_t, C.c_size_t, C.c_size_t,
                                     C.c_int, C.c_void_p]
    st = torch.cuda.current_stream().cuda_stream
    for ns in (512, 1024, 2048, 3584, 7168, 14336, 28672):
        def f():
            for j in range(N // ns):
                rt.cudaMemcpy2DAsync(d.data_ptr() + j * ns * 2, N * 2, h.data_ptr() + j * ns * 2, N * 2,
                                     ns * 2, K, 1, st)
        def g():
            for j in range(N // ns):
                rt.cudaMemcpy2DAsync(h.data_ptr() + j * ns * 2, N * 2, d.data_ptr() + j * ns * 2, N * 2,
                                     ns * 2, K, 2, st)
        ms = timed(f, reps=3)
        ms2 = timed(g, reps=3)
        print(json.dumps({"slab_cols": ns, "row_bytes": ns * 2, "h2d_2d_GBps": K * N * 2 / ms / 1e6,
                          "d2h_2d_GBps": K * N * 2 / ms2 / 1e6}))


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "api":
        host_api()
        sys.exit(0)
    if len(sys.argv) > 1 and sys.argv[1] == "all":
        pcie()
        copy2d()
    for env in ({"TFB_HOST_TRACE": "1"}, {"TFB_HOST_BIGFIRST": "1"}, {"TFB_HOST_SLAB": "2048"}, {"TFB_HOST_SLAB": "2560"},
                {"TFB_HOST_SLAB": "5120"}):
        subprocess.run([sys.executable, __file__, "api"], env={**os.environ, **env}, check=False)


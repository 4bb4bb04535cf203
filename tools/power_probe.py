"""Sustained-load comparison of our AG+GEMM (config 2) and cuBLAS: each runs
back to back for ~3 s while NVML samples SM clock, power and throttle
reasons.  Prints per-second GEMM times and the sampled medians."""
import ctypes as C
import os
import statistics
import sys
import threading
import time

import pynvml
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_02168_b200 as tf  # noqa: E402
from paper_2511_02168_b200 import _abi  # noqa: E402

pynvml.nvmlInit()
hdl = pynvml.nvmlDeviceGetHandleByIndex(0)
M, N, K = 8192, 28672, 8192
secs = float(sys.argv[1]) if len(sys.argv) > 1 else 3.0


def sample(stop, out):
    while not stop.is_set():
        out.append((pynvml.nvmlDeviceGetClockInfo(hdl, pynvml.NVML_CLOCK_SM),
                    pynvml.nvmlDeviceGetPowerUsage(hdl) / 1000.0,
                    pynvml.nvmlDeviceGetCurrentClocksThrottleReasons(hdl)))
        time.sleep(0.02)


with tf.World(1, [0], M * K * 2 + (64 << 20)) as w:
    sh = w.alloc("ag.a", M * K * 2)
    A = (torch.rand(M, K, device="cuda") * 2 - 1).bfloat16()
    w.memcpy(sh[0], A.data_ptr(), M * K * 2)
    B = (torch.rand(K, N, device="cuda") * 2 - 1).bfloat16()
    Cc = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    shape = _abi.AgShape(M, N, K, 0, 0, 0, 1)
    args = (w.handle, 1, C.byref(shape), _abi.ptr_array(sh), _abi.ptr_array([B.data_ptr()]),
            _abi.ptr_array([Cc.data_ptr()]), None, None)
    st = torch.cuda.ExternalStream(w.stream(0))
    ours = (lambda: _abi.check(w.lib.tf_ag_gemm_async(*args)), st)
    cub = (lambda: torch.matmul(A, B, out=Cc), torch.cuda.current_stream())
    runs = [("ours", ours, None), ("ours-narrow", ours, "TFB_FORCE_NARROW"), ("cublas", cub, None)] * 2
    for name, (fn, s), env in runs:
        os.environ.pop("TFB_FORCE_NARROW", None)
        if env:
            os.environ[env] = "1"
        time.sleep(2.0)  # cool down between runs
        samples, stop = [], threading.Event()
        th = threading.Thread(target=sample, args=(stop, samples))
        th.start()
        per = []
        t_end = time.time() + secs
        while time.time() < t_end:
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            for _ in range(20):
                fn()
            e1.record(s)
            torch.cuda.synchronize()
            per.append(e0.elapsed_time(e1) / 20 * 1e3)
        stop.set()
        th.join()
        clk = [x[0] for x in samples]
        pw = [x[1] for x in samples]
        rs = set()
        for x in samples:
            rs.add(hex(x[2]))
        print(f"{name:12s} us/GEMM first {per[0]:.0f} last {per[-1]:.0f} median {statistics.median(per):.0f} | "
              f"sm MHz median {statistics.median(clk):.0f} min {min(clk)} | W median {statistics.median(pw):.0f} "
              f"max {max(pw):.0f} | reasons {sorted(rs)}", flush=True)

"""A/B timing of an env knob on the AG+GEMM in ONE process (alternating
blocks, medians), plus cuBLAS in the same loop: python tools/ab_gemm.py
M N K VAR=VALUE [rounds]."""
import ctypes as C
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_02168_b200 as tf  # noqa: E402
from paper_2511_02168_b200 import _abi  # noqa: E402

M, N, K = (int(x) for x in sys.argv[1:4])
var, val = sys.argv[4].split("=", 1)
rounds = int(sys.argv[5]) if len(sys.argv) > 5 else 6
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
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

    def block(fn, s, n=10):
        for _ in range(2):
            fn()
        torch.cuda.synchronize()
        e0.record(s)
        for _ in range(n):
            fn()
        e1.record(s)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / n * 1e3

    res = {"base": [], "knob": [], "cublas": []}
    for r in range(rounds):
        os.environ.pop(var, None)
        res["base"].append(block(lambda: _abi.check(w.lib.tf_ag_gemm_async(*args)), st))
        os.environ[var] = val
        res["knob"].append(block(lambda: _abi.check(w.lib.tf_ag_gemm_async(*args)), st))
        os.environ.pop(var, None)
        res["cublas"].append(block(lambda: torch.matmul(A, B, out=Cc), torch.cuda.current_stream()))
    for k_, v in res.items():
        print(f"{k_:7s} median {statistics.median(v):8.1f} us  min {min(v):8.1f}  all {[round(x) for x in v]}")

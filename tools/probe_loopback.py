"""Loopback AG+GEMM probe: W ranks on ONE GPU (each its own heap), config-2
shapes (M=8192, K=8192, N=28672/W per rank).  Total FLOPs equal W=1's, so the
time over the W=1 kernel is the cost of the fused exchange machinery (gather
warps / push kernel, flags, gated TMA) -- with HBM standing in for NVLink."""
import ctypes as C
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_02168_b200 as tf  # noqa: E402
from paper_2511_02168_b200 import _abi  # noqa: E402

M, K, NT = 8192, 8192, 28672
for W in [int(x) for x in (sys.argv[1:] or ["1", "2", "4", "8"])]:
    N, kw = NT // W, K // W
    with tf.World(W, [0] * W, M * kw * 2 + 2 * 2 * M * K * 2 + (64 << 20)) as w:
        shards = w.alloc("ag.a", M * kw * 2)
        A = (torch.rand(M, K, device="cuda") * 2 - 1).bfloat16()
        for r in range(W):
            s = A[:, r * kw:(r + 1) * kw].contiguous()
            w.memcpy(shards[r], s.data_ptr(), s.numel() * 2)
        Bs = [(torch.rand(K, N, device="cuda") * 2 - 1).bfloat16() for _ in range(W)]
        Cs = [torch.empty(M, N, device="cuda", dtype=torch.bfloat16) for _ in range(W)]
        torch.cuda.synchronize()
        shape = _abi.AgShape(M, N, K, 0, 0, 0, 1)
        for name, var in (("pull", 1), ("push", 2), ("baseline", 0)):
            args = (w.handle, var, C.byref(shape), _abi.ptr_array(shards),
                    _abi.ptr_array([b.data_ptr() for b in Bs]), _abi.ptr_array([c.data_ptr() for c in Cs]),
                    None, None)
            _abi.check(w.lib.tf_ag_gemm(*args))
            ref = A[:256].float() @ Bs[0].float()
            err = ((Cs[0][:256].float() - ref).abs().max() / ref.abs().max()).item()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record()
            for _ in range(5):
                _abi.check(w.lib.tf_ag_gemm(*args))
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / 5
            print(f"W={W} {name:8s} {ms*1e3:8.1f} us  {2*M*NT*K/ms/1e9:7.1f} TFLOP/s (all ranks)  err {err:.2e}",
                  flush=True)

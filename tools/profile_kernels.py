"""Runs each hot kernel at its BASELINE config a few times, for ncu captures:
  ncu --set full --clock-control none --import-source on -k regex:<kernel> -s 1 -c 1 \
      -o gpurun_out/prof_<x> python tools/profile_kernels.py <ag|fd3|fd4>
"""
import ctypes as C
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_02168_b200 as tf  # noqa: E402
from paper_2511_02168_b200 import _abi  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "ag"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
if which.startswith("ag"):
    # ag: config 2; agM<m>: config 5's M x 8192 x 8192 (e.g. agM128: split-K cluster path)
    M, N, K = (8192, 28672, 8192) if which == "ag" else (int(which[3:]), 8192, 8192)
    with tf.World(1, [0], M * K * 2 + (64 << 20)) as w:
        sh = w.alloc("ag.a", M * K * 2)
        A = (torch.rand(M, K, device="cuda") * 2 - 1).bfloat16()
        w.memcpy(sh[0], A.data_ptr(), M * K * 2)
        B = (torch.rand(K, N, device="cuda") * 2 - 1).bfloat16()
        Cc = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
        shape = _abi.AgShape(M, N, K, 0, 0, 0, 1)
        for _ in range(reps):
            _abi.check(w.lib.tf_ag_gemm(w.handle, 1, C.byref(shape), _abi.ptr_array(sh),
                                        _abi.ptr_array([B.data_ptr()]), _abi.ptr_array([Cc.data_ptr()]),
                                        None, None))
else:
    cfg = dict(fd3=(1, 64, 8, 128, 131072), fd4=(32, 64, 8, 128, 32768))[which]
    Bt, Hq, Hkv, d, L = cfg
    with tf.World(1, [0], 512 << 20) as w:
        q = (torch.rand(Bt, Hq, d, device="cuda") * 2 - 1).bfloat16()
        k = (torch.rand(Bt, Hkv, L, d, device="cuda") * 2 - 1).bfloat16()
        v = (torch.rand(Bt, Hkv, L, d, device="cuda") * 2 - 1).bfloat16()
        out = torch.empty(Bt, Hq, d, device="cuda", dtype=torch.bfloat16)
        shape = _abi.FdShape(Bt, Hq, Hkv, d, L, d ** -0.5, 1, 1)
        for _ in range(reps):
            _abi.check(w.lib.tf_flash_decode(w.handle, 3, C.byref(shape), _abi.ptr_array([q.data_ptr()]),
                                             _abi.ptr_array([k.data_ptr()]), _abi.ptr_array([v.data_ptr()]),
                                             _abi.ptr_array([out.data_ptr()]), None, None))
print("done", which)

"""A few fused FD launches (W=1, bf16) at one shape, for ncu:
python tools/fd_one_shape.py B L [calls]"""
import ctypes as C
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_02168_b200 as tf  # noqa: E402
from paper_2511_02168_b200 import _abi  # noqa: E402

Bt, L = int(sys.argv[1]), int(sys.argv[2])
calls = int(sys.argv[3]) if len(sys.argv) > 3 else 5
Hq, Hkv, d = 64, 8, 128
q = (torch.rand(Bt, Hq, d, device="cuda") * 2 - 1).bfloat16()
k = (torch.rand(Bt, Hkv, L, d, device="cuda") * 2 - 1).bfloat16()
v = (torch.rand(Bt, Hkv, L, d, device="cuda") * 2 - 1).bfloat16()
with tf.World(1, [0], 256 << 20) as w:
    out = torch.empty(Bt, Hq, d, device="cuda", dtype=torch.bfloat16)
    shape = _abi.FdShape(Bt, Hq, Hkv, d, L, d ** -0.5, _abi.TF_BF16, _abi.TF_BF16)
    args = (w.handle, _abi.TF_FD_FUSED, C.byref(shape), _abi.ptr_array([q.data_ptr()]),
            _abi.ptr_array([k.data_ptr()]), _abi.ptr_array([v.data_ptr()]),
            _abi.ptr_array([out.data_ptr()]), None, None)
    for _ in range(calls):
        _abi.check(w.lib.tf_flash_decode_async(*args))
    _abi.check(w.lib.tf_world_sync(w.handle))

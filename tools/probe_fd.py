"""Quick FD latency probe: fused and bsp at BASELINE configs 3 and 4 (W=1)."""
import ctypes as C
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_02168_b200 as tf  # noqa: E402
from paper_2511_02168_b200 import _abi  # noqa: E402

for name, (Bt, Hq, Hkv, d, L) in dict(fd3=(1, 64, 8, 128, 131072), fd4=(32, 64, 8, 128, 32768)).items():
    with tf.World(1, [0], 512 << 20) as w:
        q = (torch.rand(Bt, Hq, d, device="cuda") * 2 - 1).bfloat16()
        k = (torch.rand(Bt, Hkv, L, d, device="cuda") * 2 - 1).bfloat16()
        v = (torch.rand(Bt, Hkv, L, d, device="cuda") * 2 - 1).bfloat16()
        out = torch.empty(Bt, Hq, d, device="cuda", dtype=torch.bfloat16)
        shape = _abi.FdShape(Bt, Hq, Hkv, d, L, d ** -0.5, 1, 1)
        for var in (3, 0):
            args = (w.handle, var, C.byref(shape), _abi.ptr_array([q.data_ptr()]), _abi.ptr_array([k.data_ptr()]),
                    _abi.ptr_array([v.data_ptr()]), _abi.ptr_array([out.data_ptr()]), None, None)
            _abi.check(w.lib.tf_flash_decode(*args))
            s = torch.cuda.ExternalStream(w.stream(0))
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            for _ in range(3):
                _abi.check(w.lib.tf_flash_decode_async(*args))
            e0.record(s)
            for _ in range(20):
                _abi.check(w.lib.tf_flash_decode_async(*args))
            e1.record(s)
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / 20
            gb = 2 * k.numel() * 2 / 1e9
            print(f"{name} variant {var}: {ms*1e3:.1f} us  {gb/ms*1e3:.0f} GB/s")
        qf = q.float().view(Bt, Hkv, Hq // Hkv, d)
        s_ = torch.einsum("bhgd,bhld->bhgl", qf, k.float()) * d ** -0.5
        ref = torch.einsum("bhgl,bhld->bhgd", torch.softmax(s_, -1), v.float()).reshape(Bt, Hq, d)
        err = ((out.float() - ref).abs().amax(-1) / ref.abs().amax(-1)).max().item()
        print(f"{name} head-rel err vs torch fp32: {err:.2e}")

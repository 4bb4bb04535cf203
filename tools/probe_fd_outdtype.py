import ctypes as C, os, sys, torch
sys.path.insert(0, "/root/repo")
import paper_2511_02168_b200 as tf
from paper_2511_02168_b200 import _abi
for (B, L) in ((1, 131072), (32, 32768)):
    Hq, Hkv, d = 64, 8, 128
    with tf.World(1, [0], 256 << 20) as w:
        q = (torch.rand(B, Hq, d, device="cuda") * 2 - 1).bfloat16()
        k = (torch.rand(B, Hkv, L, d, device="cuda") * 2 - 1).bfloat16()
        v = (torch.rand(B, Hkv, L, d, device="cuda") * 2 - 1).bfloat16()
        torch.cuda.synchronize()
        for od, name in ((1, "bf16 out"), (0, "fp32 out (hi/lo P)")):
            out = torch.empty(B, Hq, d, device="cuda", dtype=torch.bfloat16 if od else torch.float32)
            shape = _abi.FdShape(B, Hq, Hkv, d, L, d ** -0.5, 1, od)
            args = (w.handle, 3, C.byref(shape), _abi.ptr_array([q.data_ptr()]), _abi.ptr_array([k.data_ptr()]),
                    _abi.ptr_array([v.data_ptr()]), _abi.ptr_array([out.data_ptr()]), None, None)
            for _ in range(3): _abi.check(w.lib.tf_flash_decode(*args))
            s = torch.cuda.ExternalStream(w.stream(0))
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            for _ in range(20): _abi.check(w.lib.tf_flash_decode_async(*args))
            e1.record(s); torch.cuda.synchronize()
            us = e0.elapsed_time(e1) / 20 * 1e3
            print(f"B={B} L={L} {name}: {us:.1f} us  {2*k.numel()*2/us/1e3:.0f} GB/s", flush=True)

"""FD fused latency vs KV length (B=1, 64q/8kv, d=128): intercept = fixed cost."""
import ctypes as C, os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_02168_b200 as tf
from paper_2511_02168_b200 import _abi
for L in (8192, 16384, 32768, 65536, 131072, 262144):
    Bt, Hq, Hkv, d = 1, 64, 8, 128
    with tf.World(1, [0], 512 << 20) as w:
        q = (torch.rand(Bt, Hq, d, device="cuda") * 2 - 1).bfloat16()
        k = (torch.rand(Bt, Hkv, L, d, device="cuda") * 2 - 1).bfloat16()
        v = (torch.rand(Bt, Hkv, L, d, device="cuda") * 2 - 1).bfloat16()
        out = torch.empty(Bt, Hq, d, device="cuda", dtype=torch.bfloat16)
        shape = _abi.FdShape(Bt, Hq, Hkv, d, L, d ** -0.5, 1, 1)
        args = (w.handle, 3, C.byref(shape), _abi.ptr_array([q.data_ptr()]), _abi.ptr_array([k.data_ptr()]),
                _abi.ptr_array([v.data_ptr()]), _abi.ptr_array([out.data_ptr()]), None, None)
        _abi.check(w.lib.tf_flash_decode(*args))
        s = torch.cuda.ExternalStream(w.stream(0))
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for _ in range(50):
            _abi.check(w.lib.tf_flash_decode_async(*args))
        e1.record(s)
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) / 50 * 1e3
        print(f"L={L:7d}  {us:8.1f} us  {2*k.numel()*2/us/1e3:7.0f} GB/s", flush=True)

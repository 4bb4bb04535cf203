"""FD config 3 end to end (W=1): the query comes from pinned host memory and
the output goes back every step.  (a) copies on the world stream around the
fused launch (bench.py's e2e), (b) the output written by the kernel straight
into the pinned host buffer (mapped, UVA) -- no D2H copy."""
import ctypes as C
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_02168_b200 as tf  # noqa: E402
from paper_2511_02168_b200 import _abi  # noqa: E402

Bt, L, Hq, Hkv, d = 1, 131072, 64, 8, 128
n = 40
g = torch.Generator(device="cuda").manual_seed(7)
q = (torch.rand(Bt, Hq, d, device="cuda", generator=g) * 2 - 1).bfloat16()
k = (torch.rand(Bt, Hkv, L, d, device="cuda", generator=g) * 2 - 1).bfloat16()
v = (torch.rand(Bt, Hkv, L, d, device="cuda", generator=g) * 2 - 1).bfloat16()
with tf.World(1, [0], 256 << 20) as w:
    out = torch.empty(Bt, Hq, d, device="cuda", dtype=torch.bfloat16)
    hq = q.cpu().pin_memory()
    hout = torch.empty(Bt, Hq, d, dtype=torch.bfloat16).pin_memory()
    hout2 = torch.empty(Bt, Hq, d, dtype=torch.bfloat16).pin_memory()
    shape = _abi.FdShape(Bt, Hq, Hkv, d, L, d ** -0.5, _abi.TF_BF16, _abi.TF_BF16)
    st = torch.cuda.ExternalStream(w.stream(0))

    def call(out_ptr):
        a = (w.handle, _abi.TF_FD_FUSED, C.byref(shape), _abi.ptr_array([q.data_ptr()]),
             _abi.ptr_array([k.data_ptr()]), _abi.ptr_array([v.data_ptr()]), _abi.ptr_array([out_ptr]), None, None)
        _abi.check(w.lib.tf_flash_decode_async(*a))

    def a_step():
        with torch.cuda.stream(st):
            q.copy_(hq, non_blocking=True)
        call(out.data_ptr())
        with torch.cuda.stream(st):
            hout.copy_(out, non_blocking=True)

    def b_step():
        with torch.cuda.stream(st):
            q.copy_(hq, non_blocking=True)
        call(hout2.data_ptr())

    def dev_step():
        call(out.data_ptr())

    for name, fn in (("device", dev_step), ("e2e copies", a_step), ("e2e mapped out", b_step)):
        for _ in range(5):
            fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for _ in range(n):
            fn()
        e1.record(st)
        torch.cuda.synchronize()
        print(f"{name:16s} {e0.elapsed_time(e1) / n * 1e3:7.1f} us", flush=True)
    print("mapped out == copied out:", bool(torch.equal(hout, hout2)))

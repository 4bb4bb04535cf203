"""Where does a Flash Decode launch spend its device time outside its CTAs?
Stream-ordered %globaltimer stamps (tools/stamp.cubin) before and after each
fused launch, and the launch's own per-CTA entry/exit stamps (TFB_TRACE):
  launch latency = first CTA entry - stamp before
  body           = last CTA exit  - first CTA entry
  teardown       = stamp after    - last CTA exit
python tools/fd_gap.py B L [stream]"""
import ctypes as C
import os
import sys

import numpy as np
import torch
from cuda.bindings import driver as cu

if not os.environ.get("NOTRACE"):
    os.environ["TFB_TRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_02168_b200 as tf  # noqa: E402
from paper_2511_02168_b200 import _abi  # noqa: E402

Bt, L = int(sys.argv[1]), int(sys.argv[2])
Hq, Hkv, d = 64, 8, 128
torch.cuda.init()
torch.zeros(1, device="cuda")
err, mod = cu.cuModuleLoad(os.path.join(os.path.dirname(os.path.abspath(__file__)), "stamp.cubin").encode())
assert err == cu.CUresult.CUDA_SUCCESS, err
err, fn = cu.cuModuleGetFunction(mod, b"stamp")
stamps = torch.zeros(64, dtype=torch.int64, device="cuda")
q = (torch.rand(Bt, Hq, d, device="cuda") * 2 - 1).bfloat16()
k = (torch.rand(Bt, Hkv, L, d, device="cuda") * 2 - 1).bfloat16()
v = (torch.rand(Bt, Hkv, L, d, device="cuda") * 2 - 1).bfloat16()
with tf.World(1, [0], 512 << 20) as w:
    out = torch.empty(Bt, Hq, d, device="cuda", dtype=torch.bfloat16)
    shape = _abi.FdShape(Bt, Hq, Hkv, d, L, d ** -0.5, _abi.TF_BF16, _abi.TF_BF16)
    args = (w.handle, _abi.TF_FD_FUSED, C.byref(shape), _abi.ptr_array([q.data_ptr()]),
            _abi.ptr_array([k.data_ptr()]), _abi.ptr_array([v.data_ptr()]),
            _abi.ptr_array([out.data_ptr()]), None, None)
    st = w.stream(0)

    def stamp(i):
        p = C.c_uint64(stamps.data_ptr() + 0)
        a = C.c_int(i)
        params = (C.c_void_p * 2)(C.addressof(p), C.addressof(a))
        e, = cu.cuLaunchKernel(fn, 1, 1, 1, 1, 1, 1, 0, st, C.addressof(params), 0)
        assert e == cu.CUresult.CUDA_SUCCESS, e

    nl = int(os.environ.get("NLAUNCH", "1"))
    for rep in range(6):
        stamp(0)
        for _ in range(nl):
            _abi.check(w.lib.tf_flash_decode_async(*args))
        stamp(1)
        _abi.check(w.lib.tf_world_sync(w.handle))
        s = stamps.cpu().numpy()
        if os.environ.get("NOTRACE"):
            print(f"total {s[1] - s[0]:7d} ns for {nl} launches", flush=True)
            continue
        ptr = w.alloc("fd.trace", 8 * 32 * 4096)[0]
        t = w.get(ptr, (4096, 32), np.uint64).astype(np.int64)
        t = t[t[:, 0] > 0]
        first, last = t[:, 0].min(), t[:, 6].max() if (t[:, 6] > 0).any() else t.max()
        print(f"launch {first - s[0]:7d} ns  body {last - first:7d} ns  teardown {s[1] - last:7d} ns  "
              f"total {s[1] - s[0]:7d} ns  ctas {len(t)}", flush=True)

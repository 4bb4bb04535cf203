"""Per-CTA %globaltimer phase stamps of the fused FD kernel (TFB_TRACE=1)."""
import ctypes as C, os, sys
import numpy as np
import torch
os.environ["TFB_TRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_02168_b200 as tf
from paper_2511_02168_b200 import _abi
L = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
Bt, Hq, Hkv, d = 1, 64, 8, 128
with tf.World(1, [0], 512 << 20) as w:
    q = (torch.rand(Bt, Hq, d, device="cuda") * 2 - 1).bfloat16()
    k = (torch.rand(Bt, Hkv, L, d, device="cuda") * 2 - 1).bfloat16()
    v = (torch.rand(Bt, Hkv, L, d, device="cuda") * 2 - 1).bfloat16()
    out = torch.empty(Bt, Hq, d, device="cuda", dtype=torch.bfloat16)
    shape = _abi.FdShape(Bt, Hq, Hkv, d, L, d ** -0.5, 1, 1)
    args = (w.handle, 3, C.byref(shape), _abi.ptr_array([q.data_ptr()]), _abi.ptr_array([k.data_ptr()]),
            _abi.ptr_array([v.data_ptr()]), _abi.ptr_array([out.data_ptr()]), None, None)
    for _ in range(3):
        _abi.check(w.lib.tf_flash_decode(*args))
    ptr = w.alloc("fd.trace", 8 * 16 * 4096)[0]
    t = w.get(ptr, (4096, 16), np.uint64).astype(np.int64)
    t = t[t[:, 0] > 0]
    t0 = t[:, 0].min()
    names = ["entry", "computed", "ticketed", "group-fold+push", "fold-phase", "fold-item", "exit", "group-folded",
             "L1-folded", "L2-ticketed", "L1:ml-in", "L2:ml-in", "q-in-smem", "warps-done"]
    for i, n in enumerate(names):
        col = t[:, i]
        col = col[col > 0] - t0
        if len(col):
            print(f"{n:16s} n={len(col):4d}  min {col.min()/1e3:7.2f}  p50 {np.median(col)/1e3:7.2f}  max {col.max()/1e3:7.2f} us")

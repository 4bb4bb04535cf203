"""Per-CTA %globaltimer phase stamps of the TMA-fed fused FD kernel
(TFB_TRACE=1): when each CTA got its first stage, finished its last item,
entered / left the fold phases, plus items, merge time and inline folds."""
import ctypes as C
import os
import sys

import numpy as np
import torch

os.environ["TFB_TRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_02168_b200 as tf  # noqa: E402
from paper_2511_02168_b200 import _abi  # noqa: E402

Bt = int(sys.argv[1]) if len(sys.argv) > 1 else 1
L = int(sys.argv[2]) if len(sys.argv) > 2 else 131072
Hq, Hkv, d = 64, 8, 128
with tf.World(1, [0], 512 << 20) as w:
    q = (torch.rand(Bt, Hq, d, device="cuda") * 2 - 1).bfloat16()
    k = (torch.rand(Bt, Hkv, L, d, device="cuda") * 2 - 1).bfloat16()
    v = (torch.rand(Bt, Hkv, L, d, device="cuda") * 2 - 1).bfloat16()
    out = torch.empty(Bt, Hq, d, device="cuda", dtype=torch.bfloat16)
    shape = _abi.FdShape(Bt, Hq, Hkv, d, L, d ** -0.5, 1, 1)
    args = (w.handle, 3, C.byref(shape), _abi.ptr_array([q.data_ptr()]), _abi.ptr_array([k.data_ptr()]),
            _abi.ptr_array([v.data_ptr()]), _abi.ptr_array([out.data_ptr()]), None, None)
    for _ in range(4):
        _abi.check(w.lib.tf_flash_decode(*args))
    ptr = w.alloc("fd.trace", 8 * 32 * 4096)[0]
    t = w.get(ptr, (4096, 32), np.uint64).astype(np.int64)
    t = t[t[:, 0] > 0]
    t0 = t[:, 0].min()
    names = {0: "entry", 10: "first-stage", 1: "consumers-done", 2: "post-start", 13: "subitem-claimed",
             9: "split-fold-start", 16: "fold-max-done", 17: "fold-rows-done", 18: "fold-combined",
             8: "split-folded", 15: "gtick-done", 7: "flags-released", 4: "fold-phase",
             6: "exit"}
    for i, n in names.items():
        col = t[:, i]
        col = col[col > 0] - t0
        if len(col):
            print(f"{n:16s} n={len(col):4d}  min {col.min()/1e3:7.2f}  p50 {np.median(col)/1e3:7.2f}  "
                  f"max {col.max()/1e3:7.2f} us")
    print("items/CTA: min %d p50 %d max %d; merge us/CTA: p50 %.2f max %.2f" % (
        t[:, 11].min(), np.median(t[:, 11]), t[:, 11].max(), np.median(t[:, 12]) / 1e3, t[:, 12].max() / 1e3))

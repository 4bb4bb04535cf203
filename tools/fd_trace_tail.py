"""Critical-path view of the fused FD tail (TFB_TRACE=1, W=1): the CTA whose
split fold finished last, stamp by stamp, plus the last split publish.
python tools/fd_trace_tail.py [B] [L]"""
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
NAMES = {0: "entry", 12: "q-in-smem", 13: "warps-done/subitem", 1: "computed", 2: "split-published",
         9: "split-fold-start", 16: "fold-max-done", 17: "fold-rows-done", 18: "fold-combined",
         8: "split-folded", 15: "gtick-done", 7: "flags-released", 3: "flags+early", 4: "fold-phase", 6: "exit"}
with tf.World(1, [0], 512 << 20) as w:
    q = (torch.rand(Bt, Hq, d, device="cuda") * 2 - 1).bfloat16()
    k = (torch.rand(Bt, Hkv, L, d, device="cuda") * 2 - 1).bfloat16()
    v = (torch.rand(Bt, Hkv, L, d, device="cuda") * 2 - 1).bfloat16()
    out = torch.empty(Bt, Hq, d, device="cuda", dtype=torch.bfloat16)
    shape = _abi.FdShape(Bt, Hq, Hkv, d, L, d ** -0.5, 1, 1)
    args = (w.handle, 3, C.byref(shape), _abi.ptr_array([q.data_ptr()]), _abi.ptr_array([k.data_ptr()]),
            _abi.ptr_array([v.data_ptr()]), _abi.ptr_array([out.data_ptr()]), None, None)
    for rep in range(3):
        _abi.check(w.lib.tf_flash_decode(*args))
        ptr = w.alloc("fd.trace", 8 * 32 * 4096)[0]
        t = w.get(ptr, (4096, 32), np.uint64).astype(np.int64)
        t = t[t[:, 0] > 0]
        t0 = t[:, 0].min()
        rel = np.where(t > 0, t - t0, -1) / 1e3
        last_pub = rel[:, 2].max()
        i = int(np.argmax(rel[:, 8]))
        print(f"rep {rep}: last split published {last_pub:.2f} us; CTA {i} folded last:")
        print("   " + "  ".join(f"{NAMES[s]} {rel[i, s]:.2f}" for s in NAMES if rel[i, s] >= 0))
        print(f"   kernel exit max {rel[:, 6].max():.2f}")

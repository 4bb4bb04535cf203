"""Distribution view of one fused FD launch (TFB_TRACE=1, W=1): per-CTA
entry, q-in-smem, warps-done, split-published, exit stamps as percentiles
(us from the first CTA's entry), and the in-CTA warp finish spread.
python tools/fd_trace_dist.py [B] [L]"""
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
SLOTS = {0: "entry", 12: "q-in-smem", 10: "first-warp-done", 11: "last-warp-done", 19: "cta-weights", 1: "computed", 20: "pub-barrier", 21: "pub-fenced",
         2: "split-published", 13: "fold-claimed", 9: "split-fold-start", 16: "fold-max-done",
         17: "fold-rows-done", 18: "fold-combined", 8: "split-folded", 6: "exit"}
with tf.World(1, [0], 512 << 20) as w:
    q = (torch.rand(Bt, Hq, d, device="cuda") * 2 - 1).bfloat16()
    k = (torch.rand(Bt, Hkv, L, d, device="cuda") * 2 - 1).bfloat16()
    v = (torch.rand(Bt, Hkv, L, d, device="cuda") * 2 - 1).bfloat16()
    out = torch.empty(Bt, Hq, d, device="cuda", dtype=torch.bfloat16)
    shape = _abi.FdShape(Bt, Hq, Hkv, d, L, d ** -0.5, 1, 1)
    args = (w.handle, 3, C.byref(shape), _abi.ptr_array([q.data_ptr()]), _abi.ptr_array([k.data_ptr()]),
            _abi.ptr_array([v.data_ptr()]), _abi.ptr_array([out.data_ptr()]), None, None)
    for rep in range(4):
        _abi.check(w.lib.tf_flash_decode(*args))
        ptr = w.alloc("fd.trace", 8 * 32 * 4096)[0]
        t = w.get(ptr, (4096, 32), np.uint64).astype(np.int64)
        t = t[t[:, 0] > 0]
        t0 = t[:, 0].min()
        rel = np.where(t > 0, t - t0, -1) / 1e3
        print(f"rep {rep}: {len(t)} CTAs")
        for s, name in SLOTS.items():
            col = rel[:, s]
            col = col[col >= 0]
            if len(col):
                p = np.percentile(col, [0, 10, 50, 90, 100])
                print(f"   {name:16s} n={len(col):4d}  " + "  ".join(f"{x:7.2f}" for x in p))
        spread = rel[:, 11] - rel[:, 10]
        spread = spread[(rel[:, 10] >= 0) & (rel[:, 11] >= 0)]
        if len(spread):
            print("   warp spread      " + "  ".join(f"{x:7.2f}" for x in np.percentile(spread, [0, 50, 90, 100])))
        # i-cache check: per SM, the CTA that reached the in-CTA fold first vs second
        sm = t[:, 14]
        d1, d2 = [], []
        for s_ in np.unique(sm):
            idx = np.where(sm == s_)[0]
            if len(idx) != 2:
                continue
            a, b_ = sorted(idx, key=lambda i: rel[i, 11])
            d1.append(rel[a, 1] - rel[a, 11])
            d2.append(rel[b_, 1] - rel[b_, 11])
        if d1:
            print(f"   last-warp-done->computed: first CTA on SM p50 {np.median(d1):.2f}  second {np.median(d2):.2f}")
        for sl, nm in ((22, "ck trace+bad"), (23, "ck weights"), (24, "ck barrier2")):
            print(f"   {nm:16s} cycles p10/50/90/max " + " ".join(f"{x:7.0f}" for x in np.percentile(t[:, sl], [10, 50, 90, 100])))
        wt = rel[:, 22:30]
        ok = (wt >= 0).all(axis=1)
        if ok.any():
            wt = wt[ok] - wt[ok].min(axis=1, keepdims=True)
            print("   per-warp finish (us after the CTA's first warp), mean by warp: " +
                  " ".join(f"{x:5.2f}" for x in wt.mean(axis=0)))
            blk = t[ok, 15] if False else None

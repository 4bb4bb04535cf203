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
    ptr = w.alloc("fd.trace", 8 * 32 * 4096)[0]
    t = w.get(ptr, (4096, 32), np.uint64).astype(np.int64)
    t = t[t[:, 0] > 0]
    t0 = t[:, 0].min()
    names = ["entry", "computed", "split-published", "flags+early-fold", "fold-phase", "fold-item", "exit",
             "flags-released", "split-folded", "split-fold-start", "first-warp-done", "last-warp-done", "q-in-smem",
             "warps-done"]
    for i, n in enumerate(names):
        col = t[:, i]
        col = col[col > 0] - t0
        if len(col):
            print(f"{n:16s} n={len(col):4d}  min {col.min()/1e3:7.2f}  p50 {np.median(col)/1e3:7.2f}  max {col.max()/1e3:7.2f} us")
    # Per-CTA streaming time (q in smem -> warps done) vs SM and group.
    dur = (t[:, 13] - t[:, 12]) / 1e3
    sm = t[:, 14]
    item = t[:, 15]
    S = int(os.environ.get("TFB_FD_SPLITS", "37"))
    grp = item // S
    print("stream us: min %.1f p50 %.1f max %.1f" % (dur.min(), np.median(dur), dur.max()))
    for gi in range(8):
        sel = grp == gi
        if sel.any():
            print("  group %d: n=%3d mean %.1f min %.1f max %.1f" % (gi, sel.sum(), dur[sel].mean(), dur[sel].min(),
                                                                 dur[sel].max()))
    order = np.argsort(sm)
    per_sm = {}
    for s_, d_ in zip(sm, dur):
        per_sm.setdefault(int(s_), []).append(d_)
    sms = sorted(per_sm)
    row = ["%d:%.0f" % (s_, max(per_sm[s_])) for s_ in sms]
    print("per-SM max stream us:", " ".join(row))
    split = t[:, 15] % S
    for lo, hi in ((0, 12), (12, 25), (25, 37)):
        sel = (split >= lo) & (split < hi)
        print("  splits %d-%d: mean %.1f" % (lo, hi - 1, dur[sel].mean()))
    spread = (t[:, 11] - t[:, 10]) / 1e3
    print("intra-CTA warp finish spread us: min %.1f p50 %.1f max %.1f" % (spread.min(), np.median(spread), spread.max()))

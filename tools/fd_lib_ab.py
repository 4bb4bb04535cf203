"""Flash Decode fused W=1 timing through whichever library TFB_LIB names
(A/B of two builds in separate processes on one box): configs 3 and 4,
bf16 output, CUDA events per launch on the world stream."""
import ctypes as C
import os
import sys

import torch

sys.path.insert(0, os.environ.get("TFB_PKG_ROOT") or os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2511_02168_b200 import _abi  # noqa: E402
import paper_2511_02168_b200 as tf  # noqa: E402

CFGS = {"c3": (1, 131072, 60), "c4": (32, 32768, 20), "c3w8": (1, 16384, 100)}
tag = os.environ.get("TAG", os.path.basename(os.environ.get("TFB_LIB", "head")))
for name in sys.argv[1:] or ["c3", "c4"]:
    Bt, L, n = CFGS[name]
    Hq, Hkv, d = 64, 8, 128
    g = torch.Generator(device="cuda").manual_seed(7)
    q = (torch.rand(Bt, Hq, d, device="cuda", generator=g) * 2 - 1).bfloat16()
    k = (torch.rand(Bt, Hkv, L, d, device="cuda", generator=g) * 2 - 1).bfloat16()
    v = (torch.rand(Bt, Hkv, L, d, device="cuda", generator=g) * 2 - 1).bfloat16()
    with tf.World(1, [0], 256 << 20) as w:
        out = torch.empty(Bt, Hq, d, device="cuda", dtype=torch.bfloat16)
        shape = _abi.FdShape(Bt, Hq, Hkv, d, L, d ** -0.5, _abi.TF_BF16, _abi.TF_BF16)
        args = (w.handle, _abi.TF_FD_FUSED, C.byref(shape), _abi.ptr_array([q.data_ptr()]),
                _abi.ptr_array([k.data_ptr()]), _abi.ptr_array([v.data_ptr()]),
                _abi.ptr_array([out.data_ptr()]), None, None)
        st = torch.cuda.ExternalStream(w.stream(0))
        for _ in range(5):
            _abi.check(w.lib.tf_flash_decode_async(*args))
        _abi.check(w.lib.tf_world_sync(w.handle))
        # back-to-back mean (no event between launches), then per-launch events
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for i in range(n):
            _abi.check(w.lib.tf_flash_decode_async(*args))
        e1.record(st)
        _abi.check(w.lib.tf_world_sync(w.handle))
        torch.cuda.synchronize()
        mean = e0.elapsed_time(e1) * 1e3 / n
        evs = [torch.cuda.Event(enable_timing=True) for _ in range(n + 1)]
        evs[0].record(st)
        for i in range(n):
            _abi.check(w.lib.tf_flash_decode_async(*args))
            evs[i + 1].record(st)
        _abi.check(w.lib.tf_world_sync(w.handle))
        torch.cuda.synchronize()
        ts = sorted(evs[i].elapsed_time(evs[i + 1]) * 1e3 for i in range(n))
        kv = 2 * Bt * Hkv * L * d * 2
        print(f"{tag:8s} {name:5s} mean {mean:7.1f} us ({kv / mean / 1e3:5.0f} GB/s)  per-launch-events p50 "
              f"{ts[n // 2]:7.1f} min {ts[0]:7.1f} us", flush=True)

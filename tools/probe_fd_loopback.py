"""Loopback Flash Decode probe: W ranks on ONE GPU (one launch per device for
the fused schedules, one per rank for the others), configs 3 and 4 with the
KV split across W -- total KV bytes fixed, so the time over W=1 is the cost
of the exchange protocol with HBM standing in for NVLink."""
import ctypes as C
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_02168_b200 as tf  # noqa: E402
from paper_2511_02168_b200 import _abi  # noqa: E402

CFGS = {"config3": (1, 64, 8, 128, 131072), "config4": (32, 64, 8, 128, 32768)}
for name, (B, Hq, Hkv, d, L) in CFGS.items():
    g = torch.Generator(device="cuda").manual_seed(1)
    q = (torch.rand(B, Hq, d, device="cuda", generator=g) * 2 - 1).bfloat16()
    k = (torch.rand(B, Hkv, L, d, device="cuda", generator=g) * 2 - 1).bfloat16()
    v = (torch.rand(B, Hkv, L, d, device="cuda", generator=g) * 2 - 1).bfloat16()
    for W in [int(x) for x in (sys.argv[1:] or ["1", "2", "4", "8"])]:
        ln = L // W
        ks = [k[:, :, r * ln:(r + 1) * ln].contiguous() for r in range(W)]
        vs = [v[:, :, r * ln:(r + 1) * ln].contiguous() for r in range(W)]
        outs = [torch.empty(B, Hq, d, device="cuda", dtype=torch.bfloat16) for _ in range(W)]
        with tf.World(W, [0] * W, 256 << 20) as w:
            shape = _abi.FdShape(B, Hq, Hkv, d, L, d ** -0.5, 1, 1)
            line = []
            for vname, var in (("fused", 3), ("owner", 5), ("bsp", 0)):
                if W == 1 and var == 5:
                    continue
                args = (w.handle, var, C.byref(shape), _abi.ptr_array([q.data_ptr()] * W),
                        _abi.ptr_array([x.data_ptr() for x in ks]), _abi.ptr_array([x.data_ptr() for x in vs]),
                        _abi.ptr_array([o.data_ptr() for o in outs]), None, None)
                for _ in range(3):
                    _abi.check(w.lib.tf_flash_decode(*args))
                st = torch.cuda.ExternalStream(w.stream(0))
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                torch.cuda.synchronize()
                e0.record(st)
                for _ in range(20):
                    _abi.check(w.lib.tf_flash_decode_async(*args))
                # every rank's stream joins the measuring stream
                for r in range(1, W):
                    ev = torch.cuda.Event()
                    ev.record(torch.cuda.ExternalStream(w.stream(r)))
                    st.wait_event(ev)
                e1.record(st)
                torch.cuda.synchronize()
                us = e0.elapsed_time(e1) / 20 * 1e3
                line.append(f"{vname} {us:7.1f} us")
            print(f"{name} W={W}: " + "  ".join(line), flush=True)

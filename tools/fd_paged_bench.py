"""Paged vs contiguous KV, fused FD W=1, bf16: configs 3 and 4 at several
page sizes (random page permutation), CUDA events per launch, and the
paged output checked bitwise against the contiguous one."""
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_02168_b200 as tf  # noqa: E402
from paper_2511_02168_b200 import _abi  # noqa: E402

CFGS = {"c3": (1, 131072, 40), "c4": (32, 32768, 10)}
Hq, Hkv, d = 64, 8, 128
for name in sys.argv[1:] or ["c3", "c4"]:
    Bt, L, n = CFGS[name]
    g = torch.Generator(device="cuda").manual_seed(7)
    q = (torch.rand(Bt, Hq, d, device="cuda", generator=g) * 2 - 1).bfloat16()
    k = (torch.rand(Bt, Hkv, L, d, device="cuda", generator=g) * 2 - 1).bfloat16()
    v = (torch.rand(Bt, Hkv, L, d, device="cuda", generator=g) * 2 - 1).bfloat16()
    kv = 2 * Bt * Hkv * L * d * 2
    with tf.World(1, [0], 256 << 20) as w:
        shape = _abi.FdShape(Bt, Hq, Hkv, d, L, d ** -0.5, _abi.TF_BF16, _abi.TF_BF16)
        st = torch.cuda.ExternalStream(w.stream(0))

        def timed(call):
            for _ in range(3):
                call()
            _abi.check(w.lib.tf_world_sync(w.handle))
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(n + 1)]
            ev[0].record(st)
            for i in range(n):
                call()
                ev[i + 1].record(st)
            _abi.check(w.lib.tf_world_sync(w.handle))
            torch.cuda.synchronize()
            return sorted(ev[i].elapsed_time(ev[i + 1]) * 1e3 for i in range(n))[n // 2]

        out0 = torch.empty(Bt, Hq, d, device="cuda", dtype=torch.bfloat16)
        base = (w.handle, _abi.TF_FD_FUSED, C.byref(shape), _abi.ptr_array([q.data_ptr()]),
                _abi.ptr_array([k.data_ptr()]), _abi.ptr_array([v.data_ptr()]),
                _abi.ptr_array([out0.data_ptr()]), None, None)
        for leg in ("1", "0"):
            os.environ["TFB_FD_STREAM"] = leg if leg == "0" else ""
            if leg == "1":
                os.environ.pop("TFB_FD_STREAM")
            t = timed(lambda: _abi.check(w.lib.tf_flash_decode_async(*base)))
            print(f"{name} contiguous {'default' if leg == '1' else 'register kernel'}: {t:8.1f} us "
                  f"{kv / t / 1e3:6.0f} GB/s", flush=True)
        os.environ.pop("TFB_FD_STREAM", None)
        # references: the default kernel choice and the register kernel
        _abi.check(w.lib.tf_flash_decode_async(*base))
        _abi.check(w.lib.tf_world_sync(w.handle))
        ref_default = out0.clone()
        os.environ["TFB_FD_STREAM"] = "0"
        _abi.check(w.lib.tf_flash_decode_async(*base))
        _abi.check(w.lib.tf_world_sync(w.handle))
        os.environ.pop("TFB_FD_STREAM")
        ref_register = out0.clone()
        for hnd, ps in ((0, 16), (0, 64), (0, 256), (1, 16), (1, 64), (1, 256)):
            pps = -(-L // ps)
            npg = Bt * pps + 5
            perm = torch.from_numpy(np.random.default_rng(ps).permutation(npg)[: Bt * pps].astype(np.int64))
            pools = []
            for t in (k, v):
                if hnd:
                    pages = t.reshape(Bt, Hkv, pps, ps, d).permute(0, 2, 1, 3, 4).reshape(Bt * pps, Hkv, ps, d)
                else:
                    pages = t.reshape(Bt, Hkv, pps, ps, d).permute(0, 2, 3, 1, 4).reshape(Bt * pps, ps, Hkv, d)
                pool = torch.zeros((npg,) + tuple(pages.shape[1:]), device="cuda", dtype=torch.bfloat16)
                pool[perm.cuda()] = pages
                pools.append(pool)
            tbl = perm.to(torch.int32).reshape(Bt, pps).cuda()
            out = torch.empty_like(out0)
            pl = _abi.FdPaged(ps, pps, npg, hnd)
            args = (w.handle, _abi.TF_FD_FUSED, C.byref(shape), C.byref(pl), _abi.ptr_array([q.data_ptr()]),
                    _abi.ptr_array([pools[0].data_ptr()]), _abi.ptr_array([pools[1].data_ptr()]),
                    _abi.ptr_array([tbl.data_ptr()]), _abi.ptr_array([out.data_ptr()]), None, None)
            t = timed(lambda: _abi.check(w.lib.tf_flash_decode_paged_async(*args)))
            _abi.check(w.lib.tf_world_sync(w.handle))
            # pages >= 64 keys take the same kernel as the contiguous default
            ref, what = (ref_default, "default-kernel") if ps >= 64 else (ref_register, "register-kernel")
            print(f"{name} paged {'HND' if hnd else 'NHD'} page_size {ps:4d}: {t:8.1f} us {kv / t / 1e3:6.0f} GB/s  "
                  f"bitwise == {what} contiguous: {bool(torch.equal(out, ref))}", flush=True)
            del pools

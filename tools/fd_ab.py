"""A/B of the Flash Decode kernels in one process: the TMA-fed stream kernel
(default) vs the register-streaming kernel (TFB_FD_LEGACY=1), fused W=1,
BASELINE configs 3 and 4, plus torch fp32 numerics.  Env knobs are read per
call, so each variant is set just before its timed loop."""
import ctypes as C
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_02168_b200 as tf  # noqa: E402
from paper_2511_02168_b200 import _abi  # noqa: E402

CFGS = {"c3": (1, 131072), "c4": (32, 32768), "c3w8": (1, 16384), "c4w8": (32, 4096)}
which = sys.argv[1:] or ["c3", "c4"]
variants = [v for v in os.environ.get("FDAB", "stream,legacy").split(",")]


def ref_attn(q, k, v, scale):
    B, Hq, d = q.shape
    Hkv = k.shape[1]
    out = torch.empty(B, Hq, d, device=q.device)
    for b in range(B):
        qf = q[b].float().view(Hkv, Hq // Hkv, d)
        s = torch.einsum("hgd,hld->hgl", qf, k[b].float()) * scale
        out[b] = torch.einsum("hgl,hld->hgd", torch.softmax(s, -1), v[b].float()).reshape(Hq, d)
    return out


for name in which:
    Bt, L = CFGS[name]
    Hq, Hkv, d = 64, 8, 128
    g = torch.Generator(device="cuda").manual_seed(7)
    q = (torch.rand(Bt, Hq, d, device="cuda", generator=g) * 2 - 1).bfloat16()
    k = (torch.rand(Bt, Hkv, L, d, device="cuda", generator=g) * 2 - 1).bfloat16()
    v = (torch.rand(Bt, Hkv, L, d, device="cuda", generator=g) * 2 - 1).bfloat16()
    bs = list(range(Bt)) if Bt <= 2 else [0, Bt // 2, Bt - 1]
    ref = ref_attn(q[bs], k[bs], v[bs], d ** -0.5)
    with tf.World(1, [0], 256 << 20) as w:
        for var in variants:
            os.environ["TFB_FD_STREAM"] = "0" if var.startswith("legacy") else "1"
            os.environ["TFB_FD_HILO"] = "0" if var.endswith("bf16p") else "1"
            for odt in (_abi.TF_BF16, _abi.TF_F32):
                out = torch.empty(Bt, Hq, d, device="cuda", dtype=torch.bfloat16 if odt == _abi.TF_BF16 else torch.float32)
                shape = _abi.FdShape(Bt, Hq, Hkv, d, L, d ** -0.5, _abi.TF_BF16, odt)
                args = (w.handle, _abi.TF_FD_FUSED, C.byref(shape), _abi.ptr_array([q.data_ptr()]),
                        _abi.ptr_array([k.data_ptr()]), _abi.ptr_array([v.data_ptr()]),
                        _abi.ptr_array([out.data_ptr()]), None, None)
                st = torch.cuda.ExternalStream(w.stream(0))
                for _ in range(5):
                    _abi.check(w.lib.tf_flash_decode_async(*args))
                _abi.check(w.lib.tf_world_sync(w.handle))
                n = 10 if name == "c4" else 40
                evs = [torch.cuda.Event(enable_timing=True) for _ in range(n + 1)]
                evs[0].record(st)
                for i in range(n):
                    _abi.check(w.lib.tf_flash_decode_async(*args))
                    evs[i + 1].record(st)
                _abi.check(w.lib.tf_world_sync(w.handle))
                ts = sorted(evs[i].elapsed_time(evs[i + 1]) * 1e3 for i in range(n))
                o = out[bs].float()
                err = ((o - ref).abs().amax(-1) / ref.abs().amax(-1)).max().item()
                mabs = (o - ref).abs().max().item()
                kvb = 2 * Bt * Hkv * L * d * 2
                print(f"{name} {var:12s} out={'bf16' if odt else 'f32 '} p10 {ts[n//10]:7.1f} p50 {ts[n//2]:7.1f} "
                      f"us  {kvb / (ts[n//2] * 1e-6) / 1e9:6.0f} GB/s  head_rel_err {err:.2e}  max_abs {mabs:.2e}",
                      flush=True)

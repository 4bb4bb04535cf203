"""FD fused latency vs split count S (TFB_FD_SPLITS) at several KV lengths
(B=1, 64q/8kv, d=128, W=1).  Prints the chooser's default S as well."""
import ctypes as C, os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_02168_b200 as tf
from paper_2511_02168_b200 import _abi
Ls = [int(x) for x in sys.argv[1].split(",")] if len(sys.argv) > 1 else [8192, 32768, 131072]
Ss = [int(x) for x in sys.argv[2].split(",")] if len(sys.argv) > 2 else [0, 8, 16, 24, 37, 56, 74, 111, 148]
Bt = int(os.environ.get("FD_B", "1"))
Hq, Hkv, d = 64, 8, 128
for L in Ls:
    with tf.World(1, [0], 1 << 30) as w:
        q = (torch.rand(Bt, Hq, d, device="cuda") * 2 - 1).bfloat16()
        k = (torch.rand(Bt, Hkv, L, d, device="cuda") * 2 - 1).bfloat16()
        v = (torch.rand(Bt, Hkv, L, d, device="cuda") * 2 - 1).bfloat16()
        out = torch.empty(Bt, Hq, d, device="cuda", dtype=torch.bfloat16)
        shape = _abi.FdShape(Bt, Hq, Hkv, d, L, d ** -0.5, 1, 1)
        args = (w.handle, 3, C.byref(shape), _abi.ptr_array([q.data_ptr()]), _abi.ptr_array([k.data_ptr()]),
                _abi.ptr_array([v.data_ptr()]), _abi.ptr_array([out.data_ptr()]), None, None)
        ref = None
        for S in Ss:
            if S:
                os.environ["TFB_FD_SPLITS"] = str(S)
            else:
                os.environ.pop("TFB_FD_SPLITS", None)
            _abi.check(w.lib.tf_flash_decode(*args))
            if ref is None:
                ref = out.float().clone()
            err = (out.float() - ref).abs().max().item()
            s = torch.cuda.ExternalStream(w.stream(0))
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            for _ in range(50):
                _abi.check(w.lib.tf_flash_decode_async(*args))
            e1.record(s)
            torch.cuda.synchronize()
            us = e0.elapsed_time(e1) / 50 * 1e3
            print(f"B={Bt} L={L:7d} S={S or 'auto':>4}  {us:8.1f} us  {2*k.numel()*2/us/1e3:7.0f} GB/s  maxdiff {err:.1e}",
                  flush=True)

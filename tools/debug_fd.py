"""FD shape sweep vs torch fp32 (debug aid)."""
import ctypes as C
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_02168_b200 as tf  # noqa: E402
from paper_2511_02168_b200 import _abi  # noqa: E402

shapes = [(1, 64, 8, 128, 131072), (32, 64, 8, 128, 1024), (4, 64, 8, 128, 32768), (32, 64, 8, 128, 32768),
          (8, 16, 2, 128, 8192)]
if len(sys.argv) > 1:
    shapes = [tuple(int(x) for x in a.split(",")) for a in sys.argv[1:]]
for (Bt, Hq, Hkv, d, L) in shapes:
    with tf.World(1, [0], 512 << 20) as w:
        g = torch.Generator(device="cuda").manual_seed(0)
        q = (torch.rand(Bt, Hq, d, device="cuda", generator=g) * 2 - 1).bfloat16()
        k = (torch.rand(Bt, Hkv, L, d, device="cuda", generator=g) * 2 - 1).bfloat16()
        v = (torch.rand(Bt, Hkv, L, d, device="cuda", generator=g) * 2 - 1).bfloat16()
        print("finite inputs:", bool(torch.isfinite(k).all() and torch.isfinite(v).all()), flush=True)
        out = torch.empty(Bt, Hq, d, device="cuda", dtype=torch.float32)
        shape = _abi.FdShape(Bt, Hq, Hkv, d, L, d ** -0.5, 1, 0)
        qf = q.float().view(Bt, Hkv, Hq // Hkv, d)
        s_ = torch.einsum("bhgd,bhld->bhgl", qf, k.float()) * d ** -0.5
        ref = torch.einsum("bhgl,bhld->bhgd", torch.softmax(s_, -1), v.float()).reshape(Bt, Hq, d)
        for var in (3, 0):
            out.zero_()
            try:
                _abi.check(w.lib.tf_flash_decode(w.handle, var, C.byref(shape), _abi.ptr_array([q.data_ptr()]),
                                                 _abi.ptr_array([k.data_ptr()]), _abi.ptr_array([v.data_ptr()]),
                                                 _abi.ptr_array([out.data_ptr()]), None, None))
                err = ((out - ref).abs().amax(-1) / ref.abs().amax(-1))
                print((Bt, Hq, Hkv, d, L), var, "max err %.2e" % err.max().item(), "worst (b,h)",
                      divmod(int(err.argmax()), Hq), flush=True)
            except Exception as e:
                print((Bt, Hq, Hkv, d, L), var, "EXC", e, flush=True)

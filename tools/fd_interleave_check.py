"""FD fast path: interleaved vs contiguous warp key assignment (TFB_FD_CONTIGUOUS) against torch fp32 at several KV lengths."""
import ctypes as C, os, sys, torch
sys.path.insert(0, "/root/repo")
import paper_2511_02168_b200 as tf
from paper_2511_02168_b200 import _abi
import itertools
cases = [(1, int(x)) for x in (sys.argv[1].split(",") if len(sys.argv) > 1 else ["2048", "8192", "32768", "131072"])]
for (B, L) in cases:
    Hq, Hkv, d = 64, 8, 128
    with tf.World(1, [0], 256 << 20) as w:
        g = torch.Generator(device="cuda").manual_seed(1)
        q = (torch.rand(B, Hq, d, device="cuda", generator=g) * 2 - 1).bfloat16()
        k = (torch.rand(B, Hkv, L, d, device="cuda", generator=g) * 2 - 1).bfloat16()
        v = (torch.rand(B, Hkv, L, d, device="cuda", generator=g) * 2 - 1).bfloat16()
        torch.cuda.synchronize()  # the world's streams do not order against torch's
        res = {}
        for mode in ("int", "contig"):
            if mode == "contig": os.environ["TFB_FD_CONTIGUOUS"] = "1"
            else: os.environ.pop("TFB_FD_CONTIGUOUS", None)
            out = torch.zeros(B, Hq, d, device="cuda", dtype=torch.float32)
            shape = _abi.FdShape(B, Hq, Hkv, d, L, d ** -0.5, 1, 0)
            st = w.lib.tf_flash_decode(w.handle, 3, C.byref(shape), _abi.ptr_array([q.data_ptr()]), _abi.ptr_array([k.data_ptr()]),
                                       _abi.ptr_array([v.data_ptr()]), _abi.ptr_array([out.data_ptr()]), None, None)
            res[mode] = (st, out.clone())
        a, b = res["int"][1], res["contig"][1]
        qf = q[0].float().view(Hkv, 8, d)
        sc = torch.einsum("hgd,hld->hgl", qf, k[0].float()) * d ** -0.5
        ref = torch.einsum("hgl,hld->hgd", torch.softmax(sc, -1), v[0].float()).reshape(Hq, d)
        err = lambda o: float(((o[0] - ref).abs().amax(-1) / ref.abs().amax(-1)).max())  # noqa: E731
        print(B, L, res["int"][0], res["contig"][0], "nan" if torch.isnan(a).any() else "", (a - b).abs().max().item(),
              "err int %.2e contig %.2e" % (err(a), err(b)))

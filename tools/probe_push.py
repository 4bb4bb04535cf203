"""Push-producer throughput probe (loopback W ranks on one GPU): config-2 A
(M=8192, K=8192) with a tiny per-rank N, so the time is the exchange, not
the GEMM.  python tools/probe_push.py [W ...]; env TFB_PUSH_CTAS."""
import ctypes as C
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_02168_b200 as tf  # noqa: E402
from paper_2511_02168_b200 import _abi  # noqa: E402

M, K = 8192, 8192
N = int(os.environ.get("N", "256"))
for W in [int(x) for x in (sys.argv[1:] or ["2", "8"])]:
    kw = K // W
    with tf.World(W, [0] * W, M * kw * 2 + 2 * 2 * M * K * 2 + (64 << 20)) as w:
        shards = w.alloc("ag.a", M * kw * 2)
        A = (torch.rand(M, K, device="cuda") * 2 - 1).bfloat16()
        for r in range(W):
            s = A[:, r * kw:(r + 1) * kw].contiguous()
            w.memcpy(shards[r], s.data_ptr(), s.numel() * 2)
        Bs = [(torch.rand(K, N, device="cuda") * 2 - 1).bfloat16() for _ in range(W)]
        Cs = [torch.empty(M, N, device="cuda", dtype=torch.bfloat16) for _ in range(W)]
        shape = _abi.AgShape(M, N, K, 0, 0, 0, 1)
        for name, var in (("pull", 1), ("push", 2)):
            args = (w.handle, var, C.byref(shape), _abi.ptr_array(shards),
                    _abi.ptr_array([b.data_ptr() for b in Bs]), _abi.ptr_array([c.data_ptr() for c in Cs]),
                    None, None)
            _abi.check(w.lib.tf_ag_gemm(*args))
            ref = A[:256].float() @ Bs[0].float()
            err = ((Cs[0][:256].float() - ref).abs().max() / ref.abs().max()).item()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            w.tax_reset()
            e0.record()
            for _ in range(5):
                _abi.check(w.lib.tf_ag_gemm(*args))
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / 5
            moved = W * M * K * 2  # every rank's inbox receives all of A
            print(f"W={W} N={N} {name:5s} {ms*1e3:8.1f} us  exchange {moved/ms/1e6:7.1f} GB/s into inboxes  err {err:.2e}",
                  flush=True)
            if os.environ.get("TAXES"):
                print("   rank0 taxes:", w.taxes(0), flush=True)

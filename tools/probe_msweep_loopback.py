"""Config 5 in loopback worlds: AG+GEMM M-sweep (K = N = 8192 per rank's
GEMM, A sharded along K) with W ranks on ONE GPU, fused pull / push vs the
bulk-synchronous baseline schedule (copy-engine gather between two device
barriers, then the same GEMM).  Prints us per call (all ranks) per M."""
import ctypes as C
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_02168_b200 as tf  # noqa: E402
from paper_2511_02168_b200 import _abi  # noqa: E402

K = N = 8192
Ms = [128, 512, 2048, 8192]
for W in [int(x) for x in (sys.argv[1:] or ["2", "4", "8"])]:
    kw = K // W
    Mmax = max(Ms)
    with tf.World(W, [0] * W, Mmax * kw * 2 + 2 * 2 * sum(Ms) * K * 2 + (64 << 20)) as w:
        shards = w.alloc("ag.a", Mmax * kw * 2)
        A = (torch.rand(Mmax, K, device="cuda") * 2 - 1).bfloat16()
        for r in range(W):
            s = A[:, r * kw:(r + 1) * kw].contiguous()
            w.memcpy(shards[r], s.data_ptr(), s.numel() * 2)
        Bs = [(torch.rand(K, N, device="cuda") * 2 - 1).bfloat16() for _ in range(W)]
        Cs = [torch.empty(Mmax, N, device="cuda", dtype=torch.bfloat16) for _ in range(W)]
        torch.cuda.synchronize()
        for M in Ms:
            shape = _abi.AgShape(M, N, K, 0, 0, 0, 1)
            res = {}
            for name, var in (("pull", 1), ("push", 2), ("baseline", 0)):
                args = (w.handle, var, C.byref(shape), _abi.ptr_array(shards),
                        _abi.ptr_array([b.data_ptr() for b in Bs]), _abi.ptr_array([c.data_ptr() for c in Cs]),
                        None, None)
                for _ in range(3):
                    _abi.check(w.lib.tf_ag_gemm(*args))
                st = torch.cuda.ExternalStream(w.stream(0))
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                torch.cuda.synchronize()
                e0.record(st)
                for _ in range(10):
                    _abi.check(w.lib.tf_ag_gemm_async(*args))
                for r in range(1, W):
                    ev = torch.cuda.Event()
                    ev.record(torch.cuda.ExternalStream(w.stream(r)))
                    st.wait_event(ev)
                e1.record(st)
                torch.cuda.synchronize()
                res[name] = e0.elapsed_time(e1) / 10 * 1e3
            best = min(res["pull"], res["push"])
            print(f"W={W} M={M:5d}: pull {res['pull']:8.1f}  push {res['push']:8.1f}  baseline {res['baseline']:8.1f} us"
                  f"   fused/bsp speedup {res['baseline'] / best:.2f}", flush=True)

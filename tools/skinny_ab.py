"""Skinny-M AG+GEMM A/B (W=1) in ONE process: for each M, every variant
(env settings, applied per call) is checked against an fp32 torch product
and timed in alternating blocks next to cuBLAS.
python tools/skinny_ab.py [M,...] [N] [K] ; VARIANTS="name:VAR=V;VAR2=V2,name2:..."."""
import ctypes as C
import os
import statistics
import sys

import torch

sys.path.insert(0, os.environ.get("TFB_PKG_ROOT") or os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_02168_b200 as tf  # noqa: E402
from paper_2511_02168_b200 import _abi  # noqa: E402

Ms = [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "128,256,512,1024").split(",")]
N = int(sys.argv[2]) if len(sys.argv) > 2 else 8192
K = int(sys.argv[3]) if len(sys.argv) > 3 else 8192
spec = os.environ.get("VARIANTS", "sk:,old:TFB_NO_SK=1")
variants = []
for item in spec.split(","):
    name, _, envs = item.partition(":")
    variants.append((name, dict(e.split("=", 1) for e in envs.split(";") if e)))
knobs = {k for _, e in variants for k in e}
rounds = int(os.environ.get("ROUNDS", "5"))
for M in Ms:
    with tf.World(1, [0], M * K * 2 + (64 << 20)) as w:
        sh = w.alloc("ag.a", M * K * 2)
        A = (torch.rand(M, K, device="cuda") * 2 - 1).bfloat16()
        w.memcpy(sh[0], A.data_ptr(), M * K * 2)
        B = (torch.rand(K, N, device="cuda") * 2 - 1).bfloat16()
        Cc = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
        ref = A.float() @ B.float()
        shape = _abi.AgShape(M, N, K, 0, 0, 0, 1)
        args = (w.handle, 1, C.byref(shape), _abi.ptr_array(sh), _abi.ptr_array([B.data_ptr()]),
                _abi.ptr_array([Cc.data_ptr()]), None, None)
        st = torch.cuda.ExternalStream(w.stream(0))
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

        def setenv(e):
            for k in knobs:
                os.environ.pop(k, None)
            os.environ.update(e)

        def block(fn, s, n=20):
            for _ in range(3):
                fn()
            torch.cuda.synchronize()
            e0.record(s)
            for _ in range(n):
                fn()
            e1.record(s)
            torch.cuda.synchronize()
            return e0.elapsed_time(e1) / n * 1e3

        call = lambda: _abi.check(w.lib.tf_ag_gemm_async(*args))  # noqa: E731
        errs = {}
        for name, e in variants:
            setenv(e)
            Cc.zero_()
            call()
            _abi.check(w.lib.tf_world_sync(w.handle))
            call()  # twice: the second launch runs on the advanced epoch
            _abi.check(w.lib.tf_world_sync(w.handle))
            errs[name] = float((Cc.float() - ref).abs().max() / ref.abs().max())
        res = {name: [] for name, _ in variants}
        res["cublas"] = []
        for _ in range(rounds):
            for name, e in variants:
                setenv(e)
                res[name].append(block(call, st))
            setenv({})
            res["cublas"].append(block(lambda: torch.matmul(A, B, out=Cc), torch.cuda.current_stream()))
        cub = statistics.median(res["cublas"])
        hbm = (K * N + M * K + M * N) * 2 / 6553.3e9 * 1e6
        ten = 2 * M * N * K / 1599.5e12 * 1e6
        roof = max(hbm, ten)
        for name, v in res.items():
            md = statistics.median(v)
            print(f"M={M:6d} {name:8s} median {md:7.1f} us min {min(v):7.1f}  vs cuBLAS {cub / md:5.2f}x  "
                  f"roofline {roof / md:5.2f}  err {errs.get(name, float('nan')):.2e}", flush=True)

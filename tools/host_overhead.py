"""Host-side cost of one async C-ABI call (FD fused, AG pull) vs its GPU time."""
import ctypes as C, os, sys, time
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_02168_b200 as tf
from paper_2511_02168_b200 import _abi
Bt, Hq, Hkv, d, L = 1, 64, 8, 128, 8192
with tf.World(1, [0], 512 << 20) as w:
    q = (torch.rand(Bt, Hq, d, device="cuda") * 2 - 1).bfloat16()
    k = (torch.rand(Bt, Hkv, L, d, device="cuda") * 2 - 1).bfloat16()
    v = (torch.rand(Bt, Hkv, L, d, device="cuda") * 2 - 1).bfloat16()
    out = torch.empty(Bt, Hq, d, device="cuda", dtype=torch.bfloat16)
    shape = _abi.FdShape(Bt, Hq, Hkv, d, L, d ** -0.5, 1, 1)
    args = (w.handle, 3, C.byref(shape), _abi.ptr_array([q.data_ptr()]), _abi.ptr_array([k.data_ptr()]),
            _abi.ptr_array([v.data_ptr()]), _abi.ptr_array([out.data_ptr()]), None, None)
    _abi.check(w.lib.tf_flash_decode(*args))
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(200):
        w.lib.tf_flash_decode_async(*args)
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"FD host per call {(t1-t0)/200*1e6:.1f} us, wall per call incl. GPU {(t2-t0)/200*1e6:.1f} us")
    f = w.lib.tf_launch_count
    t0 = time.perf_counter()
    for _ in range(2000):
        f(w.handle)
    print(f"bare ctypes call {(time.perf_counter()-t0)/2000*1e6:.2f} us")
# AG pull at the skinny end of config 5 (M = 128, K = N = 8192): host cost of
# one call (tensor-map encodes, plan, launch) vs the kernel's ~36 us.
M, K, N = 128, 8192, 8192
with tf.World(1, [0], M * K * 2 + (64 << 20)) as w:
    sh = w.alloc("ag.a", M * K * 2)
    B = (torch.rand(K, N, device="cuda") * 2 - 1).bfloat16()
    Cm = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    shape = _abi.AgShape(M, N, K, 0, 0, 0, _abi.TF_BF16)
    args = (w.handle, _abi.TF_AG_PULL, C.byref(shape), _abi.ptr_array(sh), _abi.ptr_array([B.data_ptr()]),
            _abi.ptr_array([Cm.data_ptr()]), None, None)
    _abi.check(w.lib.tf_ag_gemm(*args))
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(200):
        w.lib.tf_ag_gemm_async(*args)
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"AG M=128 host per call {(t1-t0)/200*1e6:.1f} us, wall per call incl. GPU {(t2-t0)/200*1e6:.1f} us")
# The fused Flash Decode of a W=2 loopback world (push + flag-gated fold in
# one launch) as an async C-ABI call vs replayed from a captured CUDA graph:
# the device-resident epochs make the launch replayable, which removes the
# per-call host cost (the paper's launch tax).
W = 2
with tf.World(W, [0] * W, 512 << 20) as w:
    ln = L // W
    q = (torch.rand(Bt, Hq, d, device="cuda") * 2 - 1).bfloat16()
    ks = [(torch.rand(Bt, Hkv, ln, d, device="cuda") * 2 - 1).bfloat16() for _ in range(W)]
    vs = [(torch.rand(Bt, Hkv, ln, d, device="cuda") * 2 - 1).bfloat16() for _ in range(W)]
    outs = [torch.empty(Bt, Hq, d, device="cuda", dtype=torch.bfloat16) for _ in range(W)]
    cs = torch.cuda.Stream()
    shape = _abi.FdShape(Bt, Hq, Hkv, d, L, d ** -0.5, 1, 1)
    args = (w.handle, 3, C.byref(shape), _abi.ptr_array([q.data_ptr()] * W), _abi.ptr_array([t.data_ptr() for t in ks]),
            _abi.ptr_array([t.data_ptr() for t in vs]), _abi.ptr_array([o.data_ptr() for o in outs]), None,
            _abi.ptr_array([cs.cuda_stream] * W))
    with torch.cuda.stream(cs):
        _abi.check(w.lib.tf_flash_decode_async(*args))
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(200):
        w.lib.tf_flash_decode_async(*args)
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"FD W=2 async call: host {(t1-t0)/200*1e6:.1f} us, wall per call incl. GPU {(t2-t0)/200*1e6:.1f} us")
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=cs):
        _abi.check(w.lib.tf_flash_decode_async(*args))
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(200):
        g.replay()
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"FD W=2 graph replay: host {(t1-t0)/200*1e6:.1f} us, wall per call incl. GPU {(t2-t0)/200*1e6:.1f} us")
    # 16 calls per graph: the host cost of one replay spread over 16 decodes.
    g16 = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g16, stream=cs):
        for _ in range(16):
            _abi.check(w.lib.tf_flash_decode_async(*args))
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(20):
        g16.replay()
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"FD W=2 graph of 16 calls: host {(t1-t0)/320*1e6:.2f} us per call, wall {(t2-t0)/320*1e6:.1f} us per call")

"""Quick AG+GEMM probe: ours (tf_ag_gemm, pull, W=1) vs cuBLAS at M N K (default config 2); norm error vs fp32."""
import ctypes as C, sys, time
import torch
sys.path.insert(0, __import__('os').path.dirname(__import__('os').path.dirname(__import__('os').path.abspath(__file__))))
import paper_2511_02168_b200 as tf
from paper_2511_02168_b200 import _abi
M, N, K = [int(x) for x in sys.argv[1:4]] if len(sys.argv) > 3 else (8192, 28672, 8192)
with tf.World(1, [0], M * K * 2 + (64 << 20)) as w:
    sh = w.alloc("ag.a", M * K * 2)
    A = torch.randn(M, K, device='cuda').bfloat16()
    w.memcpy(sh[0], A.data_ptr(), M * K * 2)
    B = torch.randn(K, N, device='cuda').bfloat16()
    Cc = torch.empty(M, N, device='cuda', dtype=torch.bfloat16)
    shape = _abi.AgShape(M, N, K, 0, 0, 0, 1)
    st = w.stream(0)
    args = (w.handle, 1, C.byref(shape), _abi.ptr_array(sh), _abi.ptr_array([B.data_ptr()]), _abi.ptr_array([Cc.data_ptr()]), None, None)
    _abi.check(w.lib.tf_ag_gemm(*args))
    ref = (A.float() @ B.float())
    err = ((Cc.float() - ref).abs().max() / ref.abs().max()).item()
    print("norm err", err)
    s = torch.cuda.ExternalStream(st)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(3): _abi.check(w.lib.tf_ag_gemm_async(*args))
    e0.record(s)
    for _ in range(10): _abi.check(w.lib.tf_ag_gemm_async(*args))
    e1.record(s); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    print(f"ours {ms*1e3:.1f} us  {2*M*N*K/ms/1e9:.1f} TFLOP/s")
    for _ in range(3): torch.matmul(A, B, out=Cc)
    e0.record(); 
    for _ in range(10): torch.matmul(A, B, out=Cc)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    print(f"cublas {ms*1e3:.1f} us  {2*M*N*K/ms/1e9:.1f} TFLOP/s")

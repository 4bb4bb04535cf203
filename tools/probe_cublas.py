"""Runs cuBLAS bf16 matmul at the GEMM probe shape (for ncu comparison)."""
import sys
import torch
M, N, K = [int(x) for x in sys.argv[1:4]] if len(sys.argv) > 3 else (8192, 8192, 8192)
A = torch.randn(M, K, device='cuda').bfloat16()
B = torch.randn(K, N, device='cuda').bfloat16()
C = torch.empty(M, N, device='cuda', dtype=torch.bfloat16)
for _ in range(3):
    torch.matmul(A, B, out=C)
torch.cuda.synchronize()
print("done")

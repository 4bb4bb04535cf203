"""torch.matmul (cuBLAS) bf16 at a skinny shape, a few calls (for ncu)."""
import sys
import torch
M, N, K = (int(x) for x in (sys.argv[1:4] if len(sys.argv) > 3 else (128, 8192, 8192)))
A = (torch.rand(M, K, device="cuda") * 2 - 1).bfloat16()
B = (torch.rand(K, N, device="cuda") * 2 - 1).bfloat16()
C = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
for _ in range(5):
    torch.matmul(A, B, out=C)
torch.cuda.synchronize()

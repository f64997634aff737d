"""cuBLAS (torch.matmul) on an M x N x K bf16 GEMM a few times (ncu comparison target)."""
import sys

import torch

M, N, K = (int(x) for x in sys.argv[1:4])
a = (torch.rand(M, K, device="cuda") - 0.5).to(torch.bfloat16)
b = (torch.randn(N, K, device="cuda") / K ** 0.5).to(torch.bfloat16)
c = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
for _ in range(3):
    torch.matmul(a, b.T, out=c)
torch.cuda.synchronize()
print("ok")

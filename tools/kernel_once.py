"""Run the tile kernel on the C2 GEMM (8192 x 3584 x 4096) a few times (ncu target)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2512_10236_b200 import runtime  # noqa: E402

M, N, K = (int(x) for x in (sys.argv[1:4] if len(sys.argv) >= 4 else (8192, 3584, 4096)))
a = (torch.rand(M, K, device="cuda") - 0.5).to(torch.bfloat16)
b = (torch.randn(N, K, device="cuda") / K ** 0.5).to(torch.bfloat16)
c = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
for _ in range(4):
    runtime.gemm_bf16(a, b, c)
torch.cuda.synchronize()
print("ok", float(c.float().abs().mean()))

"""Run the flag-free tile kernel on one config's GEMM (ncu target): c2 | c3 | c4."""
import math
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2512_10236_b200 import runtime  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
M, N, K, alpha = {"c2": (8192, 3584, 4096, 1.0), "c3": (16384, 8192, 3584, 1.0),
                  "c4": (16384, 131072, 128, 1 / math.sqrt(128))}[cfg]
a = (torch.rand(M, K, device="cuda") - 0.5).to(torch.bfloat16)
b = (torch.randn(N, K, device="cuda") / K ** 0.5).to(torch.bfloat16)
c = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
for _ in range(4):
    runtime.gemm_bf16(a, b, c, alpha=alpha)
torch.cuda.synchronize()
print("ok", cfg)

"""Plain-GEMM raster order A/B at real clocks, interleaved in one process: M-outer (group 1) vs
M-grouped rasters (FICCO_GEMM_GROUP_M pair-blocks per group, N inside). Distinct plans are forced
through distinct cache keys (tile_n auto vs explicit). usage: python tools/ab_gemm_group.py M N K alpha G"""
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2512_10236_b200 import runtime  # noqa: E402

M, N, K = (int(x) for x in sys.argv[1:4])
alpha, gm = float(sys.argv[4]), sys.argv[5]
runtime.load_library()
a = (torch.rand(M, K, device="cuda") - 0.5).to(torch.bfloat16)
b = (torch.randn(N, K, device="cuda") / K ** 0.5).to(torch.bfloat16)
c = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
os.environ["FICCO_GEMM_GROUP_M"] = "1"
runtime.gemm_bf16(a, b, c, alpha=alpha)               # plan (tile_n auto) with group 1
os.environ["FICCO_GEMM_GROUP_M"] = gm
runtime.gemm_bf16(a, b, c, alpha=alpha, tile_n=256)   # plan (tile_n 256) with the group
fns = {"group1": lambda: runtime.gemm_bf16(a, b, c, alpha=alpha),
       f"group{gm}": lambda: runtime.gemm_bf16(a, b, c, alpha=alpha, tile_n=256)}
res = {k: [] for k in fns}
torch.cuda.synchronize()
for _ in range(30):
    for k, f in fns.items():
        flush.fill_(1)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        f()
        e1.record()
        e1.synchronize()
        res[k].append(e0.elapsed_time(e1) * 1e3)
for k, v in res.items():
    print(f"{M}x{N}x{K} {k:8s} median {statistics.median(v):7.1f} us  min {min(v):7.1f}")

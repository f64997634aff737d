"""A/B timing of the flag-free tile kernel vs cuBLAS on the c2/c3/c4 GEMMs (L2 flushed, CUDA events).

Usage: FICCO_LIB_PATH=<variant .so> python tools/ab_kernel.py [reps]
Prints per shape: ficco us, cublas us, ratio (the ratio cancels most power-cap clock drift).
"""
import math
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2512_10236_b200 import runtime  # noqa: E402

runtime.load_library()
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
shapes = {"c2": (8192, 3584, 4096, 1.0), "c3": (16384, 8192, 3584, 1.0),
          "c4": (16384, 131072, 128, 1 / math.sqrt(128))}
only = os.environ.get("AB_SHAPES")
for key, (M, N, K, alpha) in shapes.items():
    if only and key not in only.split(","):
        continue
    a = (torch.rand(M, K, device="cuda") - 0.5).to(torch.bfloat16)
    b = (torch.randn(N, K, device="cuda") / K ** 0.5).to(torch.bfloat16)
    c = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
    fns = {"ficco": lambda: runtime.gemm_bf16(a, b, c, alpha=alpha),
           "cublas": lambda: torch.mm(a, b.t(), out=c)}
    res = {k: [] for k in fns}
    for _ in range(3):
        for f in fns.values():
            f()
    torch.cuda.synchronize()
    for _ in range(reps):
        for k, f in fns.items():
            flush.fill_(1)
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            f()
            e.record()
            e.synchronize()
            res[k].append(s.elapsed_time(e) * 1e3)
    fi, cb = statistics.median(res["ficco"]), statistics.median(res["cublas"])
    print(f"{key}: ficco {fi:8.1f} us  cublas {cb:8.1f} us  ratio {fi / cb:.3f}", flush=True)

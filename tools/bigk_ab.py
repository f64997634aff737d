"""Plain tile GEMM raster groups on large-K shapes (corpus g1/g2/g5/g9-like), interleaved with cuBLAS.

FICCO_GEMM_GROUP_M = pair-rows per column-major raster group, read when a shape's plan is first built
(the plan cache is keyed on the grid, so grid 0 / 148 / 146 hold three settings of one shape).
usage: python tools/bigk_ab.py
"""
import os
import statistics
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2512_10236_b200 import runtime  # noqa: E402

SHAPES = [(16384, 16384, 32768), (8192, 8192, 65536), (16384, 18432, 16384), (16384, 8192, 3584)]


def main():
    runtime.load_library()
    dev = torch.device("cuda", 0)
    flush_buf = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    flush = lambda: flush_buf.fill_(1)  # noqa: E731
    for m, n, k in SHAPES:
        a = (torch.rand(m, k, device=dev) - 0.5).to(torch.bfloat16)
        w = (torch.randn(n, k, device=dev) / k ** 0.5).to(torch.bfloat16)
        out = torch.empty(m, n, dtype=torch.bfloat16, device=dev)
        ref = torch.empty_like(out)
        fns, names = [lambda: torch.matmul(a, w.t(), out=ref)], ["cuBLAS"]
        for grid, g in ((0, None), (148, "1"), (146, "8")):
            if g is None:
                os.environ.pop("FICCO_GEMM_GROUP_M", None)
            else:
                os.environ["FICCO_GEMM_GROUP_M"] = g
            runtime.gemm_bf16(a, w, out, grid=grid)  # builds (and caches) the plan under this setting
            fns.append(lambda grid=grid: runtime.gemm_bf16(a, w, out, grid=grid))
            names.append(f"ours group_m={g or 'auto'} grid={grid or 148}")
        os.environ.pop("FICCO_GEMM_GROUP_M", None)
        torch.cuda.synchronize()
        ok = torch.allclose(out.float(), ref.float(), rtol=2e-2, atol=2e-2)
        steps = 5 if m * n * k > 2 ** 42 else 15
        times = bench.time_interleaved(fns, steps, 2, flush, torch.cuda.current_stream())
        tf = 2.0 * m * n * k
        print((m, n, k), "match" if ok else "MISMATCH",
              {nm: f"{statistics.median(t):.3f} ms {tf / statistics.median(t) / 1e9:.0f} TF/s"
               for nm, t in zip(names, times)}, flush=True)
        del a, w, out, ref
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()

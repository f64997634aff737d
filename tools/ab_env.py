"""Interleaved A/B timing of the plain tile-kernel GEMM under different environment knobs, in
ONE process (same clocks and power state): each variant sets its environment before the
call (the library reads FICCO_* knobs per call), round-robin per rep, L2 flushed before every
launch, CUDA events; cuBLAS beside it. Usage:
  python tools/ab_env.py reps M N K alpha name=VAR:val,VAR:val [name=...]
The pseudo-variables TILE_N and CTA_GROUP are passed to runtime.gemm_bf16 instead of the
environment.
"""
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2512_10236_b200 import runtime  # noqa: E402

reps, M, N, K = (int(x) for x in sys.argv[1:5])
alpha = float(sys.argv[5])
variants = {}
for spec in sys.argv[6:]:
    name, _, kv = spec.partition("=")
    variants[name] = dict(x.split(":", 1) for x in kv.split(",") if x)
keys = sorted({k for v in variants.values() for k in v} - {"TILE_N", "CTA_GROUP"})
a = (torch.rand(M, K, device="cuda") - 0.5).to(torch.bfloat16)
b = (torch.randn(N, K, device="cuda") / K ** 0.5).to(torch.bfloat16)
c = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
ref = torch.empty_like(c)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")


def run(name):
    if name == "cublas":
        torch.mm(a, b.t(), out=c)
        return
    for k in keys:
        os.environ.pop(k, None)
    env = dict(variants[name])
    tn, cg = int(env.pop("TILE_N", 0)), int(env.pop("CTA_GROUP", 0))
    os.environ.update(env)
    runtime.gemm_bf16(a, b, c, alpha, tile_n=tn, cta_group=cg)


names = list(variants) + ["cublas"]
torch.mm(a, b.t(), out=ref)
ref.mul_(alpha)
for n in names:
    run(n)
    torch.cuda.synchronize()
    if n != "cublas":
        err = (c.float() - ref.float()).abs().max().item()
        print(f"{n}: max |diff| vs cuBLAS {err:.3e}", flush=True)
res = {k: [] for k in names}
for _ in range(reps):
    for n in names:
        flush.fill_(1)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        run(n)
        e1.record()
        e1.synchronize()
        res[n].append(e0.elapsed_time(e1) * 1e3)
base = statistics.median(res["cublas"])
for k, v in res.items():
    med = statistics.median(v)
    print(f"{M}x{N}x{K} {k:12s} median {med:8.1f} us  min {min(v):8.1f}  vs cublas {med / base:.3f}", flush=True)

"""Interleaved A/B timing of several builds of libficco_b200.so in ONE process (same clocks,
same power state): each variant's ficco_gemm_bf16 on the same operands, round-robin per rep,
L2 flushed before every launch, CUDA events. Usage:
  python tools/ab_variants.py reps M N K alpha name=path.so [name=path.so ...]
"""
import ctypes
import statistics
import sys

import torch

reps, M, N, K = (int(x) for x in sys.argv[1:5])
alpha = float(sys.argv[5])
libs = {}
for spec in sys.argv[6:]:
    name, path = spec.split("=", 1)
    lib = ctypes.CDLL(path, mode=ctypes.RTLD_LOCAL)
    lib.ficco_gemm_bf16.argtypes = [ctypes.c_void_p] * 3 + [ctypes.c_int64] * 3 + [ctypes.c_float, ctypes.c_int,
                                                                                   ctypes.c_void_p]
    lib.ficco_last_error.restype = ctypes.c_char_p
    libs[name] = lib
a = (torch.rand(M, K, device="cuda") - 0.5).to(torch.bfloat16)
b = (torch.randn(N, K, device="cuda") / K ** 0.5).to(torch.bfloat16)
c = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
s = torch.cuda.current_stream().cuda_stream


def run(lib):
    r = lib.ficco_gemm_bf16(a.data_ptr(), b.data_ptr(), c.data_ptr(), M, N, K, alpha, 0, s)
    if r:
        raise RuntimeError(lib.ficco_last_error().decode())


fns = dict(libs)
fns["cublas"] = None
res = {k: [] for k in fns}
for _ in range(2):
    for k, lib in fns.items():
        run(lib) if lib else torch.mm(a, b.t(), out=c)
torch.cuda.synchronize()
for _ in range(reps):
    for k, lib in fns.items():
        flush.fill_(1)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        run(lib) if lib else torch.mm(a, b.t(), out=c)
        e1.record()
        e1.synchronize()
        res[k].append(e0.elapsed_time(e1) * 1e3)
base = statistics.median(res["cublas"])
for k, v in res.items():
    med = statistics.median(v)
    print(f"{M}x{N}x{K} {k:12s} median {med:8.1f} us  min {min(v):8.1f}  vs cublas {med / base:.3f}", flush=True)

"""Pure-write HBM bandwidth on this B200 (the C4 score write's ceiling) vs copy (read+write).

fill_ (torch elementwise kernel), cudaMemsetAsync (zero_), and copy_ over 4 GiB; best and
median of 10, CUDA events. Bytes counted: written bytes (fill/memset), read+written (copy).
"""
import json
import statistics

import torch


def t(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    out = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        b.synchronize()
        out.append(a.elapsed_time(b) * 1e-3)
    return min(out), statistics.median(out)


n = 4 << 30
x = torch.empty(n // 2, dtype=torch.bfloat16, device="cuda")
y = torch.empty(n // 2, dtype=torch.bfloat16, device="cuda")
res = {}
for name, fn, nbytes in [("fill_bf16", lambda: x.fill_(1.0), n), ("memset_zero", lambda: x.zero_(), n),
                         ("copy", lambda: y.copy_(x), 2 * n)]:
    best, med = t(fn)
    res[name] = {"best_GBps": round(nbytes / best / 1e9, 1), "median_GBps": round(nbytes / med / 1e9, 1)}
print(json.dumps(res))

"""Isolate GEMM->RS overheads on C3 (virtual 8 ranks): full vs no pushes vs no reduction reads."""
import math
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2512_10236_b200 import lowering, ops, runtime  # noqa: E402
from paper_2512_10236_b200.routing import ScheduleKind  # noqa: E402
from paper_2512_10236_b200.runtime import EPI_REDUCE, EPI_STORE, EPI_STORE_SIGNAL, OP_COPY, Plan  # noqa: E402

runtime.load_library()
G, M, N, K = 8, 16384, 8192, 3584
R = M // G
gen = torch.Generator(device="cuda").manual_seed(0)
a = (torch.rand(M, K, generator=gen, device="cuda") - 0.5).to(torch.bfloat16)
w = (torch.randn(N, K, generator=gen, device="cuda") / 60).to(torch.bfloat16)
out = torch.empty(R, N, dtype=torch.bfloat16, device="cuda")
part = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
grp = ops.FiccoGroup.virtual_group(G, 0)
sc = ops._scenario("c3", M, N, K, G)


def timeit(fn, steps=20):
    for _ in range(3):
        flush.fill_(1)
        fn()
    torch.cuda.synchronize()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    for x, y in evs:
        flush.fill_(1)
        x.record()
        fn()
        y.record()
    torch.cuda.synchronize()
    return statistics.median(x.elapsed_time(y) * 1e3 for x, y in evs)


print("gemm_bf16 (flag-free kernel)", round(timeit(lambda: runtime.gemm_bf16(a, w, part)), 1), flush=True)
for kind in sys.argv[1:] or ["hetero_fused_1d", "uniform_fused_1d"]:
    for variant in ["full", "nopush", "noreduce_reads", "all_store"]:
        low = lowering.lower_rs(sc, ScheduleKind(kind), 0, virtual=True)
        grp.ensure_workspace(low.ws_bytes)
        if variant == "nopush":
            low.ops = [o for o in low.ops if o.op != OP_COPY]
        if variant == "noreduce_reads":
            low.desc.n_recv = 0
        if variant == "all_store":
            low.ops = []
            for t in low.tiles:
                if t.mode == EPI_STORE_SIGNAL:
                    t.mode = EPI_STORE
                    t.c_row = t.c_row % R
                elif t.mode == EPI_REDUCE:
                    t.mode = EPI_STORE
            low.desc.n_recv = 0
        plan = Plan(grp.comm, low.desc, low.ops, low.tiles)
        print(kind, variant, round(timeit(lambda: plan.run(a, w, out)), 1), flush=True)
        plan.close()

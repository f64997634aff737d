"""Isolate FiCCO overheads on C2 (virtual 8 ranks): full plan vs no flag waits vs no copies."""
import math
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2512_10236_b200 import lowering, ops, runtime  # noqa: E402
from paper_2512_10236_b200.routing import ScheduleKind, build_plan  # noqa: E402
from paper_2512_10236_b200.runtime import Plan  # noqa: E402

runtime.load_library()
G, M, N, K = 8, 8192, 3584, 4096
R = M // G
gen = torch.Generator(device="cuda").manual_seed(0)
shards = [(torch.rand(R, K, generator=gen, device="cuda") - 0.5).to(torch.bfloat16) for _ in range(G)]
w = (torch.randn(N, K, generator=gen, device="cuda") / 64).to(torch.bfloat16)
out = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
grp = ops.FiccoGroup.virtual_group(G, 0)
sc = ops._scenario("c2", M, N, K, G)


def timeit(fn, steps=30):
    for _ in range(5):
        flush.fill_(1)
        fn()
    torch.cuda.synchronize()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    for a, b in evs:
        flush.fill_(1)
        a.record()
        fn()
        b.record()
    torch.cuda.synchronize()
    return statistics.median(a.elapsed_time(b) * 1e3 for a, b in evs)


a_full = torch.cat(shards)
print("gemm_bf16 (flag-free kernel)", round(timeit(lambda: runtime.gemm_bf16(a_full, w, out)), 1), flush=True)
INPLACE = "--inplace" in sys.argv  # zero-copy publish, as the bench runs C2
for kind in [a for a in sys.argv[1:] if not a.startswith("--")] or ["shard_overlap_p2p", "hetero_unfused_1d"]:
    for variant in ["full", "noflags", "nocopies", "graph_only"]:
        low = lowering.lower_ag(build_plan(sc, ScheduleKind(kind)), 0, "A", inplace=INPLACE)
        grp.ensure_workspace(low.ws_bytes)
        if variant in ("noflags", "nocopies"):
            for t in low.tiles:
                t.flag, t.fmask = -1, 0
        if variant == "nocopies":
            low.ops = []
        if variant == "graph_only":
            low.tiles = []
        grp.load_peer_shards(low, shards)
        if INPLACE:
            for par in (0, 1):
                grp.ws_tensor(0, low.gather_off + par * low.gather_par, (R, K)).copy_(shards[0])
        plan = Plan(grp.comm, low.desc, low.ops, low.tiles)
        print(kind, variant, round(timeit(lambda: plan.run(shards[0], w, out)), 1), flush=True)
        plan.close()

import sys, os, statistics, math
sys.path.insert(0, os.getcwd())
import torch
from paper_2512_10236_b200 import ops, runtime, lowering
from paper_2512_10236_b200.routing import build_plan, ScheduleKind
from paper_2512_10236_b200.runtime import Plan
runtime.load_library()
G, Tkv, Tq, d = 8, 131072, 16384, 128
R = Tkv // G
gen = torch.Generator(device="cuda").manual_seed(0)
shards = [torch.randn(R, d, generator=gen, device="cuda").to(torch.bfloat16) for _ in range(G)]
q = torch.randn(Tq, d, generator=gen, device="cuda").to(torch.bfloat16)
out = torch.empty(Tq, Tkv, dtype=torch.bfloat16, device="cuda")
grp = ops.FiccoGroup.virtual_group(G, 0)
sc = ops._scenario("cp", Tkv, Tq, d, G)
def timeit(plan):
    for _ in range(3): plan.run(q, shards[0], out)
    torch.cuda.synchronize()
    ts=[]
    for _ in range(10):
        a,b=torch.cuda.Event(enable_timing=True),torch.cuda.Event(enable_timing=True)
        a.record(); plan.run(q, shards[0], out); b.record(); b.synchronize(); ts.append(a.elapsed_time(b)*1e3)
    return statistics.median(ts)
for kind in ["hetero_fused_1d", "hetero_unfused_1d"]:
    for variant in ["as_is", "mask1", "noflags"]:
        low = lowering.lower_ag(build_plan(sc, ScheduleKind(kind)), 0, "B", alpha=1/math.sqrt(d), other_rows=Tq)
        grp.ensure_workspace(low.ws_bytes)
        if variant == "mask1":
            for t in low.tiles:
                if t.flag >= 0: t.fmask = t.fmask & -t.fmask
        if variant == "noflags":
            for t in low.tiles: t.flag = -1; t.fmask = 0
        grp.load_peer_shards(low, shards)
        plan = Plan(grp.comm, low.desc, low.ops, low.tiles)
        print(kind, variant, round(timeit(plan),1), flush=True)
        plan.close()

"""Debug: the C2 in-place headline sequence, comm.check() after every call."""
import os, sys, torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench
from paper_2512_10236_b200 import ops, runtime
runtime.load_library()
dev = torch.device("cuda", 0)
wl = bench.WORKLOADS["c2"](torch, dev, 8, 0, 1, ops)
wl.inplace = True
grp = ops.FiccoGroup.virtual_group(8, 0)
wl.agent = "dma"
best = "hetero_unfused_1d"
wl.prepare(grp, best)
plan = wl.plan_for(grp, best, "dma")
op_fn = wl.step(grp, None, None)
use_ev = os.environ.get("EV", "1") == "1"
kev = [torch.cuda.Event(enable_timing=True) for _ in range(8)]
for e in kev:
    e.record()
torch.cuda.synchronize()
for i in range(8):
    if use_ev:
        plan.set_kernel_event(kev[i])
    op_fn()
    try:
        grp.comm.check()
        print(i, "ok", grp.comm.epoch(), flush=True)
    except Exception as exc:
        print(i, "FAIL", exc, flush=True)
        break
print("plan ids", id(plan), [id(v[0]) for v in grp._plans.values()], list(grp._plans.keys()))

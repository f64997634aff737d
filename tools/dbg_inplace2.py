"""Debug: the bench's interleaved headline timing on C2 in-place, bisecting the interleaved functions."""
import os, sys, torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench
from paper_2512_10236_b200 import ops, runtime
runtime.load_library()
dev = torch.device("cuda", 0)
flush_buf = torch.empty(256 * 2**20, dtype=torch.uint8, device=dev)
flush = lambda: flush_buf.fill_(1)
stream = torch.cuda.current_stream()
which = os.environ.get("FNS", "osck")
inplace = os.environ.get("INPLACE", "1") == "1"
wl = bench.WORKLOADS["c2"](torch, dev, 8, 0, 1, ops)
wl.inplace = inplace
grp = ops.FiccoGroup.virtual_group(8, 0)
wl.agent = "dma"
best = "hetero_unfused_1d"
wl.prepare(grp, best)
op_fn = wl.step(grp, None, None)
op_fn(); torch.cuda.synchronize(); grp.comm.check()
serial_fn, _ = wl.serial()
kern_fn, _, _ = wl.kernel(runtime)
plan = wl.plan_for(grp, best, "dma")
kev = [torch.cuda.Event(enable_timing=True) for _ in range(64)]
for e in kev:
    e.record()
torch.cuda.synchronize()
k_i = [0]
def op_timed():
    plan.set_kernel_event(kev[k_i[0] % len(kev)])
    k_i[0] += 1
    op_fn()
table = {"e": op_timed, "o": op_fn, "s": serial_fn, "c": wl.cublas(), "k": kern_fn}
fns = [table[c] for c in which]
try:
    for i in range(8):
        for fn in fns:
            flush()
            fn()
        if os.environ.get("SYNC"):
            torch.cuda.synchronize()
            grp.comm.check()
    grp.comm.check()
    print(which, "inplace", inplace, "OK", flush=True)
except Exception as exc:
    print(which, "inplace", inplace, "FAIL", str(exc)[:80], flush=True)

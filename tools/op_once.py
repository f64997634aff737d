"""Run one bench workload's overlapped op a few times (ncu target for the in-op tile kernel).

usage: python tools/op_once.py c1|c2|c3|c4|c3p|ep <kind> [dma|core] [calls] [G]
Under ncu the copy program runs before the kernel (profilers serialise), so the captured kernel
is the op's tile program with its flags already satisfied.
"""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2512_10236_b200 import ops, runtime  # noqa: E402

key, kind = sys.argv[1], sys.argv[2]
agent = sys.argv[3] if len(sys.argv) > 3 else "dma"
calls = int(sys.argv[4]) if len(sys.argv) > 4 else 4
G = int(sys.argv[5]) if len(sys.argv) > 5 else bench.G_VIRTUAL
runtime.load_library()
wl = bench.WORKLOADS[key](torch, torch.device("cuda", 0), G, 0, 1, ops)
wl.agent = agent
wl.inplace = key in ("c1", "c2", "c3p", "c4")  # as the bench runs them (zero-copy input slot)
grp = ops.FiccoGroup.virtual_group(G, 0)
wl.prepare(grp, kind)
fn = wl.step(grp, kind)
for _ in range(calls):
    fn()
torch.cuda.synchronize()
grp.comm.check()
print("ok", key, kind, agent)
grp.close()

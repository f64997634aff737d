"""C2 overlap overhead decomposition (virtual 8 ranks): how much of (op - plain GEMM) is the copies'
interference vs the schedule's tile order/gating vs the run's fixed cost?

  op          the bench call (graph: copies + flag-gated tile kernel)
  tiles_only  the same tile program with every run-local flag pre-set and no copies (direct launch)
  gemm        ficco_gemm_bf16 on the same shape (row-major raster, no flags)
usage: python tools/span_decomp.py [kind ...]
"""
import os
import statistics
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2512_10236_b200 import ops, runtime  # noqa: E402
from paper_2512_10236_b200.lowering import F_RING, F_XFER  # noqa: E402
from paper_2512_10236_b200.runtime import FICCO_FLAG_BLOCK  # noqa: E402

runtime.load_library()
dev = torch.device("cuda", 0)
wl = bench.WORKLOADS["c2"](torch, dev, bench.G_VIRTUAL, 0, 1, ops)
wl.inplace = True
grp = ops.FiccoGroup.virtual_group(bench.G_VIRTUAL, 0)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
full_a = torch.cat(wl.shards)
for kind in sys.argv[1:] or ["shard_overlap_p2p", "hetero_unfused_1d", "hetero_fused_1d"]:
    wl.prepare(grp, kind)
    plan, low, _ = ops.prepare_ag(grp, wl.R, wl.K, wl.N, kind, inplace=True)
    op = wl.step(grp, kind)

    def tiles_prep():  # outside the timed region: every flag the tile program may wait on
        par = grp.comm.epoch() & 1
        grp.comm.set_flags(par * FICCO_FLAG_BLOCK + F_XFER, F_RING + 16 - F_XFER, 1)

    def tiles_only():
        a = grp.input_slot(wl.R, wl.K, wl.N, kind)
        plan.run_parts(a, wl.w, wl.out, copies=False, tiles=True)

    fns = {"op": op, "tiles_only": tiles_only, "gemm": lambda: runtime.gemm_bf16(full_a, wl.w, wl.out)}
    preps = {"tiles_only": tiles_prep}
    res = {k: [] for k in fns}
    for _ in range(3):
        for k, f in fns.items():
            preps.get(k, lambda: None)()
            f()
    torch.cuda.synchronize()
    for _ in range(20):
        for k, f in fns.items():
            preps.get(k, lambda: None)()
            flush.fill_(1)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            f()
            e1.record()
            e1.synchronize()
            res[k].append(e0.elapsed_time(e1) * 1e3)
    grp.comm.check()
    print(kind, {k: round(statistics.median(v), 1) for k, v in res.items()}, flush=True)
grp.close()

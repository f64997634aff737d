"""A/B: copy-engine chains of the fine-grain AG copy program (FICCO_FINE_CHAINS = 0 (one per peer), 4, 2, 1),
C2 and C4 virtual 8 ranks, op time interleaved + copy program alone. usage: python tools/chains_ab.py"""
import importlib
import json
import os
import statistics
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2512_10236_b200 import ops, runtime  # noqa: E402

runtime.load_library()
dev = torch.device("cuda", 0)
flush_buf = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
flush = lambda: flush_buf.fill_(1)  # noqa: E731
stream = torch.cuda.current_stream()
res = {}
for key in ("c2", "c4"):
    wl = bench.WORKLOADS[key](torch, dev, 8, 0, 1, ops)
    wl.inplace = key == "c2"
    variants = []
    for chains in ("0", "4", "2", "1"):
        os.environ["FICCO_FINE_CHAINS"] = chains
        grp = ops.FiccoGroup.virtual_group(8, 0)
        for kind in ("hetero_unfused_1d", "uniform_fused_1d"):
            wl.prepare(grp, kind)
            variants.append((chains, kind, grp, wl.step(grp, kind)))
        ring = [v for v in variants if v[1] == "shard_overlap_p2p"]
    grp_r = ops.FiccoGroup.virtual_group(8, 0)
    wl.prepare(grp_r, "shard_overlap_p2p")
    variants.append(("ring", "shard_overlap_p2p", grp_r, wl.step(grp_r, "shard_overlap_p2p")))
    times = bench.time_interleaved([v[3] for v in variants], 20, 5, flush, stream)
    for (chains, kind, grp, _), ts in zip(variants, times):
        low = wl.lowered(grp, kind)
        cp = runtime.Plan(grp.comm, low.desc, list(low.ops), [])
        try:
            copy_us = statistics.median(bench.time_steps(lambda: wl.run_plan(cp), 15, 3, flush, stream)) * 1e3
        finally:
            cp.close()
        res[f"{key}/{kind}/chains={chains}"] = {"op_us": round(statistics.median(ts) * 1e3, 1),
                                                "copy_us": round(copy_us, 1)}
        print(key, kind, chains, res[f"{key}/{kind}/chains={chains}"], flush=True)
    for v in variants:
        v[2].close() if v[2].comm else None
with open(os.path.join(ROOT, "gpurun_out", "chains_ab.json"), "w") as f:
    json.dump(res, f, indent=1)

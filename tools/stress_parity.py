"""Back-to-back stress of the overlapped ops at full size with a bit-exact check of EVERY call.

For each (workload, schedule, comm agent): a reference output from the first call (itself
spot-checked against fp32 torch by the bench workload's `check`), then `iters` calls enqueued
back to back (L2 flushed in between, both workspace parities alternating, no host sync). After each call a device-side counter adds whether the
output differs from the reference in any element. One sync at the end. This catches
intermittent protocol races: a flag seen from the wrong parity, or a chunk read before it
landed.
usage: python tools/stress_parity.py [iters] [out.json]
"""
import json
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2512_10236_b200 import ops, runtime  # noqa: E402

CASES = [("c2", k, a, False) for k in ("shard_overlap_p2p", "uniform_fused_1d", "hetero_fused_1d",
                                        "hetero_unfused_1d", "uniform_fused_2d", "serial") for a in ("dma", "core")]
CASES += [("c3", k, a, False) for k in ("uniform_fused_1d", "hetero_fused_1d", "hetero_unfused_1d", "uniform_fused_2d",
                                        "shard_overlap_p2p", "serial") for a in ("dma", "core")]
CASES += [("c4", k, "dma", False) for k in ("shard_overlap_p2p", "hetero_unfused_1d", "uniform_fused_1d")]
# the bench headlines' own paths: symmetric-slot inputs (zero-copy publish), C1 at 4 ranks, C3'
CASES += [("c2", "hetero_unfused_1d", "dma", True), ("c4", "hetero_unfused_1d", "dma", True),
          ("c3p", "hetero_unfused_1d", "dma", True)]
CASES += [("c1", k, "dma", True) for k in ("uniform_fused_2d", "hetero_unfused_1d", "shard_overlap_p2p")]


def main():
    iters = int(sys.argv[1]) if len(sys.argv) > 1 else 300
    out_path = sys.argv[2] if len(sys.argv) > 2 else None
    runtime.load_library()
    dev = torch.device("cuda", 0)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    res = {}
    wls = {}
    for key, kind, agent, inplace in CASES:
        G = getattr(bench.WORKLOADS[key], "default_ranks", bench.G_VIRTUAL)
        if key not in wls:
            wls[key] = bench.WORKLOADS[key](torch, dev, G, 0, 1, ops)
        wl = wls[key]
        grp = ops.FiccoGroup.virtual_group(G, 0)
        name = f"{key}/{kind}/{agent}" + ("/slot" if inplace else "")
        try:
            wl.agent = agent
            wl.inplace = inplace
            wl.prepare(grp, kind)
            step = wl.step(grp, kind)
            step()
            grp.comm.check()
            ok0 = bool(wl.check())
            ref = wl.out.clone()
            bad = torch.zeros((), dtype=torch.int64, device=dev)
            t0 = time.time()
            for _ in range(iters):
                flush.fill_(1)
                step()
                bad += (wl.out != ref).any().to(torch.int64)
            grp.comm.check()
            nbad = int(bad.item())
            res[name] = {"first_call_check": ok0, "calls": iters, "mismatching_calls": nbad,
                         "seconds": round(time.time() - t0, 2)}
        except Exception as exc:
            res[name] = {"error": repr(exc)[:300]}
        finally:
            grp.close()
        print(name, res[name], flush=True)
    total_bad = sum(v.get("mismatching_calls", 1) for v in res.values())
    print("TOTAL mismatching calls:", total_bad, flush=True)
    if out_path:
        with open(out_path, "w") as f:
            json.dump({"iters_per_case": iters, "cases": res, "total_mismatching_calls": total_bad}, f, indent=1)


if __name__ == "__main__":
    main()

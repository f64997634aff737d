"""Arrival profile of the copy program's readiness flags (copy program alone, virtual 8 ranks).

For each (workload, schedule, FICCO_FINE_CHAINS): one CTA polls the run's XFER / RING words
(runtime.watch_words) while the plan's copy program runs with an empty tile list; prints, per round,
when its first and last chunk landed (µs after a stamp taken right before the run), and the copy
program's total time. usage: python tools/flag_arrivals.py [c2|c4 ...]
"""
import json
import os
import statistics
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2512_10236_b200 import lowering as L  # noqa: E402
from paper_2512_10236_b200 import ops, runtime  # noqa: E402

G = 8


def profile(wl, grp, kind, reps=5):
    low = wl.lowered(grp, kind)
    plan = runtime.Plan(grp.comm, low.desc, list(low.ops), [])
    side = torch.cuda.Stream()
    stamp = torch.zeros(1, dtype=torch.int64, device="cuda")
    ring = kind == "shard_overlap_p2p"
    n = G if ring else G * G
    base_word = L.F_RING if ring else L.F_XFER
    out = torch.zeros(n + 1, dtype=torch.int64, device="cuda")
    rows = []
    try:
        for _ in range(3):
            wl.run_plan(plan)
        torch.cuda.synchronize()
        for _ in range(reps):
            par = grp.comm.epoch() & 1
            words = grp.comm.local_ws + (par * runtime.FICCO_FLAG_BLOCK + base_word) * 4
            side.wait_stream(torch.cuda.current_stream())
            runtime.watch_words(words, n, 1, out, 10**9, stream=side)
            torch.cuda._sleep(20000)  # let the watcher start polling before the run is enqueued
            runtime.timestamp(stamp)
            wl.run_plan(plan)
            torch.cuda.synchronize()
            t0 = int(stamp.item())
            arr = out.cpu().tolist()
            rows.append([(a - t0) / 1e3 if a else None for a in arr[:n]])
    finally:
        plan.close()
    med = [statistics.median(r[i] for r in rows if r[i] is not None) if any(r[i] is not None for r in rows)
           else None for i in range(n)]
    if ring:
        return {"steps_us": [None if v is None else round(v, 1) for v in med[1:]]}
    per_round = []
    for c in range(G):
        vals = [med[c * G + p] for p in range(G) if p != 0 and med[c * G + p] is not None]
        per_round.append([round(min(vals), 1), round(max(vals), 1)] if vals else None)
    first_by_peer = [round(med[p], 1) if med[p] is not None else None for p in range(1, G)]
    return {"round_first_last_us": per_round, "round0_by_peer_us": first_by_peer}


def main():
    keys = sys.argv[1:] or ["c2", "c4"]
    runtime.load_library()
    dev = torch.device("cuda", 0)
    res = {}
    for key in keys:
        wl = bench.WORKLOADS[key](torch, dev, G, 0, 1, ops)
        wl.inplace = key == "c2"
        wl.agent = "dma"
        for chains in ("0", "1", "2", "4"):
            os.environ["FICCO_FINE_CHAINS"] = chains
            grp = ops.FiccoGroup.virtual_group(G, 0)
            try:
                kinds = ["hetero_unfused_1d"] + (["shard_overlap_p2p"] if chains == "0" else [])
                for kind in kinds:
                    wl.prepare(grp, kind)
                    r = profile(wl, grp, kind)
                    res[f"{key}/{kind}/chains={chains}"] = r
                    print(key, kind, chains, json.dumps(r), flush=True)
            finally:
                grp.close()
    os.environ.pop("FICCO_FINE_CHAINS", None)
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", "flag_arrivals.json"), "w") as f:
        json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()

"""Why does a fine-grain kind lose to the shard ring on C2 (virtual 8 ranks)? Per kind: op time (interleaved),
the copy program alone, and from the kernel trace: kernel span, the CTAs' summed flag-wait time (tile's
loads-may-start stamp minus the CTA's previous tile stored), when each gate first opened, the tail.
usage: python tools/fine_vs_ring.py [c2|c4] [agent]"""
import json
import os
import statistics
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2512_10236_b200 import ops, runtime  # noqa: E402

KINDS = ["shard_overlap_p2p", "hetero_unfused_1d", "hetero_fused_1d", "uniform_fused_1d"]


def main():
    key = sys.argv[1] if len(sys.argv) > 1 else "c2"
    agent = sys.argv[2] if len(sys.argv) > 2 else "dma"
    runtime.load_library()
    dev = torch.device("cuda", 0)
    wl = bench.WORKLOADS[key](torch, dev, 8, 0, 1, ops)
    wl.inplace = key in ("c2", "c4")  # as the bench runs them (zero-copy input slot)
    wl.agent = agent
    grp = ops.FiccoGroup.virtual_group(8, 0)
    flush_buf = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    flush = lambda: flush_buf.fill_(1)  # noqa: E731
    stream = torch.cuda.current_stream()
    for k in KINDS:
        wl.prepare(grp, k)
    steps = [wl.step(grp, k) for k in KINDS]
    times = bench.time_interleaved(steps, 20, 5, flush, stream)
    res = {}
    for k, ts in zip(KINDS, times):
        plan = wl.plan_for(grp, k, agent)
        low = wl.lowered(grp, k)
        info = plan.info()
        trace = torch.zeros(info["grid"] + 2 * info["tiles"], dtype=torch.int64, device=dev)
        plan.set_trace(trace)
        spans, waits, tails, opens = [], [], [], []
        for _ in range(5):
            flush()
            torch.cuda.synchronize()
            wl.step(grp, k)()
            torch.cuda.synchronize()
            tr = trace.cpu().tolist()
            grid = info["grid"]
            t0 = min(tr[:grid])
            ready = [(tr[grid + 2 * i] - t0) / 1e3 for i in range(info["tiles"])]
            done = [(tr[grid + 2 * i + 1] - t0) / 1e3 for i in range(info["tiles"])]
            wait = 0.0
            for c in range(grid):
                prev = (tr[c] - t0) / 1e3
                for t in range(c, info["tiles"], grid):
                    wait += max(0.0, ready[t] - prev)
                    prev = done[t]
            spans.append(max(done))
            waits.append(wait / grid)
            last_per_cta = [max(done[t] for t in range(c, info["tiles"], grid)) for c in range(grid)]
            tails.append(max(last_per_cta) - min(last_per_cta))
            first_ready = [ready[c] if c < info["tiles"] else 0.0 for c in range(grid)]
            late = sorted(range(grid), key=lambda c: -last_per_cta[c])[:8]
            late_ctas = [(c, round(last_per_cta[c], 1), round(first_ready[c], 1),
                          len(range(c, info["tiles"], grid))) for c in late]
            gate_open = {}
            for i, tl in enumerate(low.tiles):
                if tl.flag >= 0 and tl.rows > 0:
                    gate_open[tl.flag] = min(gate_open.get(tl.flag, 1e9), ready[i])
            opens.append(sorted(round(v, 1) for v in gate_open.values())[:16])
        plan.set_trace(None)
        copy_us = None
        if wl.run_plan is not None:
            cp = runtime.Plan(grp.comm, low.desc, list(low.ops), [])
            try:
                copy_us = statistics.median(bench.time_steps(lambda: wl.run_plan(cp), 20, 5, flush, stream)) * 1e3
            finally:
                cp.close()
        res[k] = {"op_us": round(statistics.median(ts) * 1e3, 1), "kernel_span_us": round(statistics.median(spans), 1),
                  "mean_cta_gate_wait_us": round(statistics.median(waits), 2),
                  "cta_finish_spread_us": round(statistics.median(tails), 1), "copy_program_us": copy_us,
                  "first_gate_opens_us": opens[-1], "tiles": info["tiles"], "copy_ops": len(low.ops),
                  "latest_ctas (cta, done_us, first_tile_ready_us, tiles)": late_ctas}
        print(k, res[k], flush=True)
    grp.close()
    with open(os.path.join(ROOT, "gpurun_out", f"fine_vs_ring_{key}_{agent}.json"), "w") as f:
        json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()

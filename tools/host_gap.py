"""Does host-side enqueue time leak into the bench's device timings?

C2 at virtual G = 8: for the public-API op (given kinds) and the plain tile GEMM,
(1) host µs per call (perf_counter around the call while the GPU is kept busy, so
    nothing blocks), and
(2) the bench's device timing (L2 flush, start event, call, end event; no host sync between steps)
    with and without
    a 300 µs torch.cuda._sleep between the flush and the start event; the sleep lets
    the host run ahead, so (2b) has no host gap inside the timed region.
usage: python tools/host_gap.py [kinds...]  -> gpurun_out/host_gap.json
"""
import json
import os
import statistics
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2512_10236_b200 import ops, runtime  # noqa: E402


def main():
    kinds = sys.argv[1:] or ["hetero_unfused_1d", "shard_overlap_p2p"]
    dev = torch.device("cuda:0")
    torch.cuda.set_device(dev)
    G = 8
    wl = bench.AGWorkload(torch, dev, G, 0, 1, ops)
    grp = ops.FiccoGroup.virtual_group(G, 0)
    flush_buf = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    flush = lambda: flush_buf.fill_(1)  # noqa: E731
    s = torch.cuda.current_stream()
    fns = {}
    for k in kinds:
        wl.prepare(grp, k)
        fns[k] = wl.step(grp, k)
    fns["plain_gemm"] = wl.kernel(runtime)[0]
    res = {}
    for name, fn in fns.items():
        for _ in range(5):
            fn()
        torch.cuda.synchronize()
        torch.cuda._sleep(int(2e8))  # ~100 ms of GPU time: the host calls below never block
        host = []
        for _ in range(40):
            t0 = time.perf_counter()
            fn()
            host.append((time.perf_counter() - t0) * 1e6)
        torch.cuda.synchronize()
        dev_us = {}
        for mode in ("bench", "host_ahead"):
            evs = []
            torch.cuda.synchronize()
            for _ in range(25):  # as bench.time_steps: no host sync between steps
                flush()
                if mode == "host_ahead":
                    torch.cuda._sleep(600000)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(s)
                fn()
                e1.record(s)
                evs.append((e0, e1))
            torch.cuda.synchronize()
            ts = [a.elapsed_time(b) * 1e3 for a, b in evs]
            dev_us[mode] = round(statistics.median(ts[5:]), 2)
        res[name] = {"host_us_per_call": round(statistics.median(host), 2), "device_us": dev_us}
        print(name, res[name], flush=True)
    grp.close()
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", "host_gap.json"), "w") as f:
        json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()

"""Does switching between lowered plans cost time per call? (bench.py workloads, N=1 virtual)

Times one workload's op for two schedules: each repeated on its own (A A A ..., B B B ...) and
alternating (A B A B ...), CUDA events per call, L2 flushed before every call.
usage: python tools/switch_probe.py [c2|c3|c4] kindA kindB [reps] [kindC ...]
(extra kinds: also time all of them cycling A B C ...)
"""
import os
import statistics
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2512_10236_b200 import ops, runtime  # noqa: E402


def main():
    key, ka, kb = sys.argv[1], sys.argv[2], sys.argv[3]
    reps = int(sys.argv[4]) if len(sys.argv) > 4 else 10
    extra = sys.argv[5:]
    runtime.load_library()
    dev = torch.device("cuda", 0)
    wl = bench.WORKLOADS[key](torch, dev, bench.G_VIRTUAL, 0, 1, ops)
    grp = ops.FiccoGroup.virtual_group(bench.G_VIRTUAL, 0)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    fns = {}
    for k in [ka, kb] + extra:
        wl.prepare(grp, k)
        fns[k] = wl.step(grp, k)
    stream = torch.cuda.current_stream()

    def run(order):
        ts = {k: [] for k in fns}
        for _ in range(3):
            for k in order:
                flush.fill_(1)
                fns[k]()
        torch.cuda.synchronize()
        evs = []
        for _ in range(reps):
            for k in order:
                flush.fill_(1)
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(stream)
                fns[k]()
                b.record(stream)
                evs.append((k, a, b))
        torch.cuda.synchronize()
        for k, a, b in evs:
            ts[k].append(a.elapsed_time(b) * 1e3)
        return {k: round(statistics.median(v), 1) for k, v in ts.items() if v}

    print("A alone", run([ka]), flush=True)
    print("B alone", run([kb]), flush=True)
    print("A,B alternating", run([ka, kb]), flush=True)
    print("A alone again", run([ka]), flush=True)
    if extra:
        print("all cycling", run([ka, kb] + extra), flush=True)
        print("A alone after", run([ka]), flush=True)
    grp.comm.check()
    grp.close()


if __name__ == "__main__":
    main()

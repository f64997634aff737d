"""How do copy-engine copies captured in a CUDA graph parallelise on B200?

Captures C copies of S bytes (device-local) into a graph as `chains` parallel
branches (fork/join via events), optionally with a stream write-value memop
after every copy (like the copy programs' SIGNALs), and times graph replays.
"""
import ctypes as C
import json
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2512_10236_b200 import runtime  # noqa: E402


def run(nchains, per_chain, size, memops, comm=None):
    """memops: False (copies only), True / "memop" (stream write-value after every copy), "ce4" (a
    4-byte copy-engine copy of a constant word after every copy, as the copy programs do) or
    "kernel" (a one-thread flag-writing kernel after every copy)."""
    MiB = 1 << 20
    flags = torch.zeros(4096, dtype=torch.int64, device="cuda")
    one = torch.ones(1, dtype=torch.int64, device="cuda")
    total = nchains * per_chain
    src = torch.empty(total * size, dtype=torch.uint8, device="cuda").fill_(1)
    dst = torch.empty(total * size, dtype=torch.uint8, device="cuda")
    streams = [torch.cuda.Stream() for _ in range(nchains)]
    g = torch.cuda.CUDAGraph()
    cap = torch.cuda.Stream()
    lib = runtime.load_library()
    with torch.cuda.graph(g, stream=cap):
        ev = torch.cuda.Event()
        ev.record(cap)
        for i, s in enumerate(streams):
            s.wait_event(ev)
            with torch.cuda.stream(s):
                for j in range(per_chain):
                    k = i * per_chain + j
                    dst[k * size:(k + 1) * size].copy_(src[k * size:(k + 1) * size])
                    if memops is True or memops == "memop":
                        comm.set_flags(300 + k % 3000, 1, 1, stream=s)
                    elif memops == "ce4":
                        flags[k:k + 1].copy_(one)
                    elif memops == "kernel":
                        runtime.timestamp(flags[k:k + 1], stream=s)
            e2 = torch.cuda.Event()
            e2.record(s)
            cap.wait_event(e2)
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    ts = []
    for _ in range(20):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        g.replay()
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    us = statistics.median(ts)
    del lib, MiB
    return {"us": round(us, 1), "GBps": round(total * size / (us * 1e-6) / 1e9, 1)}


def main():
    runtime.load_library()
    comm = runtime.Communicator.virtual(1, 0, 1 << 20)
    MiB = 1 << 20
    out = {}
    only = "--flags" in sys.argv
    cases = [(7, 8, MiB, False), (7, 8, MiB, True), (7, 8, MiB, "ce4"), (7, 8, MiB, "kernel"),
             (7, 1, 8 * MiB, False), (7, 1, 8 * MiB, "ce4"), (1, 7, 8 * MiB, "ce4"), (1, 7, 8 * MiB, False)]
    for nch, per, size, mem in (cases if only else [(1, 56, MiB, False), (56, 1, MiB, False), (7, 8, MiB, False), (7, 8, MiB, True),
                                (14, 4, MiB, False), (8, 8, MiB, False), (16, 4, MiB, False), (28, 2, MiB, False),
                                (7, 1, 8 * MiB, False), (7, 2, 4 * MiB, False), (7, 16, MiB // 2, False),
                                (1, 1, 56 * MiB, False), (4, 14, MiB, False), (2, 28, MiB, False)]):
        tag = "" if not mem else f" +{'memop' if mem is True else mem}"
        out[f"{nch}ch x{per} x{size // 1024}KiB{tag}"] = run(nch, per, size, mem, comm)
    print(json.dumps(out, indent=1))
    comm.close()


if __name__ == "__main__":
    main()

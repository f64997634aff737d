"""A/B of the tile kernel's static round-robin vs dynamic (atomic counter) tile schedule (FICCO_DYNAMIC).

The dynamic schedule was measured slower everywhere and removed from the library;
the implementation was not committed; the script documents how it was measured.

For each (workload, schedule, agent) given: the bench workload's op, calls alternating between
FICCO_DYNAMIC=0 and =1 (the library reads it per launch), timed interleaved step by step with L2
flushed before every call (bench.time_interleaved); the plain GEMM of the workload's shape too.
usage: python tools/dyn_ab.py [steps] workload:kind:agent ...
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
    args = sys.argv[1:]
    steps = int(args.pop(0)) if args and args[0].isdigit() else 30
    cases = [a.split(":") for a in args] or [["c2", "shard_overlap_p2p", "dma"]]
    runtime.load_library()
    dev = torch.device("cuda", 0)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    for key, kind, agent in cases:
        wl = bench.WORKLOADS[key](torch, dev, bench.G_VIRTUAL, 0, 1, ops)
        wl.agent = agent
        wl.inplace = key in ("c2", "c3p")
        grp = ops.FiccoGroup.virtual_group(bench.G_VIRTUAL, 0)
        wl.prepare(grp, kind)
        step = wl.step(grp, kind)
        kern, _, _ = wl.kernel(runtime)

        def with_env(fn, v):
            def run():
                os.environ["FICCO_DYNAMIC"] = v
                fn()
            return run
        fns = [with_env(step, "0"), with_env(step, "1"), with_env(kern, "0"), with_env(kern, "1")]
        ts = bench.time_interleaved(fns, steps, 5, lambda: flush.fill_(1), torch.cuda.current_stream())
        grp.comm.check()
        med = [statistics.median(t) * 1e3 for t in ts]
        print(f"{key}/{kind}/{agent}: op static {med[0]:.1f} dynamic {med[1]:.1f} us | plain GEMM static {med[2]:.1f}"
              f" dynamic {med[3]:.1f} us", flush=True)
        grp.close()
    os.environ.pop("FICCO_DYNAMIC", None)


if __name__ == "__main__":
    main()

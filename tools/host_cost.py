"""Host-side cost of one public-API op call (µs, perf_counter) while the GPU is kept busy (nothing blocks),
per bench workload's API-default step; with a cProfile of the slowest one.
usage: python tools/host_cost.py c2 c4 ..."""
import cProfile
import os
import pstats
import statistics
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2512_10236_b200 import ops, runtime  # noqa: E402


def main():
    runtime.load_library()
    dev = torch.device("cuda", 0)
    for key in sys.argv[1:]:
        cls = bench.WORKLOADS[key]
        G = getattr(cls, "default_ranks", bench.G_VIRTUAL)
        wl = cls(torch, dev, G, 0, 1, ops)
        wl.inplace = key in ("c1", "c2", "c3p", "c4")
        grp = ops.FiccoGroup.virtual_group(G, 0)
        m, n, k = cls.op_shape(G)
        kind = ops.choose_kind(ops._scenario(key, m, n, k, G), None).value
        wl.agent = ops.default_agent(cls.op)
        wl.prepare(grp, kind)
        fn = wl.step(grp, kind, None)
        for _ in range(5):
            fn()
        torch.cuda.synchronize()
        torch.cuda._sleep(int(4e8))
        ts = []
        for _ in range(30):
            t0 = time.perf_counter()
            fn()
            ts.append((time.perf_counter() - t0) * 1e6)
        pr = cProfile.Profile()
        pr.enable()
        for _ in range(20):
            fn()
        pr.disable()
        torch.cuda.synchronize()
        print(key, kind, "host us per call: median", round(statistics.median(ts), 1), "min", round(min(ts), 1), flush=True)
        pstats.Stats(pr).sort_stats("cumulative").print_stats(18)
        grp.close()


if __name__ == "__main__":
    main()

"""Interleaved A/B of FICCO_GRAPH_FIRST (copy graph launched before the tile kernel) on bench ops, in the
bench's own loop (bench.time_interleaved: no host sync between steps, L2 flushed), twice.
usage: python tools/graph_first_ab.py case [case ...]   case = <workload>:<kind>:<agent>[:slot]"""
import json
import os
import statistics
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2512_10236_b200 import ops, runtime  # noqa: E402


def main():
    runtime.load_library()
    dev = torch.device("cuda", 0)
    flush_buf = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    flush = lambda: flush_buf.fill_(1)  # noqa: E731
    res = {}
    for case in sys.argv[1:]:
        parts = case.split(":")
        key, kind, agent = parts[:3]
        G = getattr(bench.WORKLOADS[key], "default_ranks", bench.G_VIRTUAL)
        wl = bench.WORKLOADS[key](torch, dev, G, 0, 1, ops)
        wl.inplace = len(parts) > 3 and parts[3] == "slot"
        wl.agent = agent
        grp = ops.FiccoGroup.virtual_group(G, 0)
        wl.prepare(grp, kind)
        step = wl.step(grp, kind)

        def with_env(v):
            def fn():
                os.environ["FICCO_GRAPH_FIRST"] = v
                step()
            return fn
        fns = [with_env("0"), with_env("1")]
        out = {"kernel_first": [], "graph_first": []}
        for _ in range(2):
            t = bench.time_interleaved(fns, 25, 5, flush, torch.cuda.current_stream())
            out["kernel_first"].append(round(statistics.median(t[0]) * 1e3, 2))
            out["graph_first"].append(round(statistics.median(t[1]) * 1e3, 2))
        grp.comm.check()
        ok = wl.check()
        grp.close()
        res[case] = dict(out, parity=bool(ok))
        print(case, res[case], flush=True)
    os.environ.pop("FICCO_GRAPH_FIRST", None)
    with open(os.path.join(ROOT, "gpurun_out", "graph_first_ab.json"), "w") as f:
        json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()

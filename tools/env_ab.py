"""Interleaved A/B of an executor environment knob read at launch time (FICCO_EPI_FAST, FICCO_B_RESIDENT,
FICCO_OUT_HINT, FICCO_RS_MMA, ...) on bench workloads' ops, call by call (same clocks), L2 flushed.
usage: python tools/env_ab.py VAR VALUE_A VALUE_B case [case ...]
case = <workload>:<kind>:<agent> (e.g. c3:hetero_fused_1d:core) or plain:<workload> (the flag-free GEMM)."""
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
    var, va, vb, cases = sys.argv[1], sys.argv[2], sys.argv[3], sys.argv[4:]
    runtime.load_library()
    dev = torch.device("cuda", 0)
    flush_buf = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    wls, fns = {}, {}
    for case in cases:
        parts = case.split(":")
        key = parts[1] if parts[0] == "plain" else parts[0]
        if key not in wls:
            wl = bench.WORKLOADS[key](torch, dev, 8, 0, 1, ops)
            wl.inplace = False
            wls[key] = (wl, ops.FiccoGroup.virtual_group(8, 0))
        wl, grp = wls[key]
        if parts[0] == "plain":
            fns[case] = wl.kernel(runtime)[0]
        else:
            wl.agent = parts[2]
            wl.prepare(grp, parts[1])
            fns[case] = wl.step(grp, parts[1])
    res = {}
    for name, fn in fns.items():
        t = {va: [], vb: []}
        for rep in range(16):
            for v in (va, vb):
                os.environ[var] = v
                flush_buf.fill_(1)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                fn()
                e1.record()
                torch.cuda.synchronize()
                if rep >= 3:
                    t[v].append(e0.elapsed_time(e1) * 1e3)
        res[name] = {f"{var}={v}": round(statistics.median(x), 1) for v, x in t.items()}
        print(name, res[name], flush=True)
    for wl, grp in wls.values():
        if grp.comm is not None:  # plain-GEMM-only workloads never built a communicator
            grp.comm.check()
        grp.close()
    with open(os.path.join(ROOT, "gpurun_out", f"env_ab_{var}.json"), "w") as f:
        json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()

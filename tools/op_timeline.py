"""Where does an overlapped op's time go outside the tile kernel? (bench.py workloads, N=1 virtual)

Per schedule kind, with the bench's exact call (L2 flushed before every call):
  pre   = first CTA start  - op start  (graph launch, publish/barrier, anything the kernel node waits on)
  span  = last tile stored - first CTA start
  post  = op end - last tile stored (copy-stream joins, flag clears)
op start/end are %globaltimer stamps (runtime.timestamp) on the caller's stream right before and
after the op; the kernel's stamps come from the plan trace (ficco_plan_set_trace). Medians of reps.
Usage: python tools/op_timeline.py [c2|c3|c4] [reps] [--copy] [--ahead: a GPU sleep first, so host enqueue
time is hidden as in the bench loop]
"""
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
    argv = [a for a in sys.argv[1:] if not a.startswith("--")]
    key = argv[0] if argv else "c2"
    reps = int(argv[1]) if len(argv) > 1 else 10
    runtime.load_library()
    dev = torch.device("cuda", 0)
    wl = bench.WORKLOADS[key](torch, dev, bench.G_VIRTUAL, 0, 1, ops)
    if key in ("c2", "c4") and "--copy" not in sys.argv:
        wl.inplace = True  # as the bench runs them (zero-copy input slot)
    grp = ops.FiccoGroup.virtual_group(bench.G_VIRTUAL, 0)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    stamps = torch.zeros(2, dtype=torch.int64, device=dev)
    out = {}
    for kind in [k for k in wl.kinds if k != "serial"] + ["serial"]:
        wl.prepare(grp, kind)
        fn = wl.step(grp, kind)
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        if key == "c2":
            plan = ops.prepare_ag(grp, wl.R, wl.K, wl.N, kind, inplace=wl.inplace)[0]
        elif key == "c3":
            plan = ops.prepare_rs(grp, wl.M, wl.K, wl.N, kind)[0]
        else:
            plan = ops.prepare_cp(grp, wl.Tq, wl.d, wl.Tkv, kind, inplace=wl.inplace)[0]
        info = plan.info()
        g, nt = info["grid"], info["tiles"]
        trace = torch.zeros(g + 2 * nt, dtype=torch.int64, device=dev)
        plan.set_trace(trace)
        fn()
        torch.cuda.synchronize()
        rows = []
        for _ in range(reps):
            if "--ahead" in sys.argv:  # the host runs ahead of the GPU (as in the bench loop)
                torch.cuda._sleep(1000000)
            flush.fill_(1)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            runtime.timestamp(stamps[0:1])
            fn()
            runtime.timestamp(stamps[1:2])
            e1.record()
            e1.synchronize()
            tr = trace.cpu().tolist()
            s0, s1 = stamps.cpu().tolist()
            start = min(tr[:g])
            done = max(tr[g + 2 * i + 1] for i in range(nt))
            rows.append(((start - s0) / 1e3, (done - start) / 1e3, (s1 - done) / 1e3, e0.elapsed_time(e1) * 1e3))
        plan.set_trace(None)
        med = [round(statistics.median(r[i] for r in rows), 1) for i in range(4)]
        out[kind] = {"pre_us": med[0], "span_us": med[1], "post_us": med[2], "event_us": med[3]}
        print(kind, out[kind], flush=True)
    # the plain tile GEMM of the same shape between the same stamps (no trace: pre + span + post)
    kfn = wl.kernel(runtime)[0]
    kfn()
    torch.cuda.synchronize()
    rows = []
    for _ in range(reps):
        if "--ahead" in sys.argv:
            torch.cuda._sleep(1000000)
        flush.fill_(1)
        runtime.timestamp(stamps[0:1])
        kfn()
        runtime.timestamp(stamps[1:2])
        torch.cuda.synchronize()
        s0, s1 = stamps.cpu().tolist()
        rows.append((s1 - s0) / 1e3)
    out["plain_gemm_stamp_to_stamp_us"] = round(statistics.median(rows), 1)
    print("plain GEMM stamp to stamp", out["plain_gemm_stamp_to_stamp_us"], flush=True)
    grp.comm.check()
    print(json.dumps(out))
    grp.close()


if __name__ == "__main__":
    main()

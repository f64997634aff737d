"""Measured timeline of one FiCCO AG->GEMM run (C2, virtual 8 ranks): where does the time go?

For every schedule kind: event-timed op latency, the tile kernel's span
(first CTA start -> last tile stored, from %globaltimer stamps), and per
dependency group (tiles sharing a readiness gate) when their loads could start
and when their last tile was stored — i.e. when each round's chunks arrived
relative to the compute.
"""
import json
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2512_10236_b200 import ops, runtime  # noqa: E402


def main():
    cp = "--cp" in sys.argv
    inplace = "--inplace" in sys.argv
    argv = [a for a in sys.argv[1:] if not a.startswith("--")]
    M, N, K, G = (131072, 16384, 128, 8) if cp else (8192, 3584, 4096, 8)
    if argv:
        M, N, K, G = map(int, argv[:4])
    R = M // G
    runtime.load_library()
    gen = torch.Generator(device="cuda").manual_seed(0)
    shards = [(torch.rand(R, K, generator=gen, device="cuda") * 2 - 1).to(torch.bfloat16) for _ in range(G)]
    w = (torch.randn(N, K, generator=gen, device="cuda") / K ** 0.5).to(torch.bfloat16)
    out = torch.empty(N, M, dtype=torch.bfloat16, device="cuda") if cp else \
        torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
    grp = ops.FiccoGroup.virtual_group(G, 0)
    res = {}
    kinds = ["serial", "shard_overlap_p2p", "uniform_fused_1d", "hetero_fused_1d", "hetero_unfused_1d"]
    if not cp:
        kinds.append("uniform_fused_2d")
    for kind in kinds:
        if cp:
            plan, low, _ = ops.prepare_cp(grp, N, K, M, kind)
        else:
            plan, low, _ = ops.prepare_ag(grp, R, K, N, kind, inplace=inplace)
        grp.load_peer_shards(low, shards)
        if inplace and not cp:
            for par in (0, 1):
                grp.ws_tensor(0, low.gather_off + par * low.gather_par, (R, K)).copy_(shards[0])
        def call(k, plan=plan):
            if cp:
                ops.cp_kv_all_gather_qk(w, shards[0], kind=k, group=grp, out=out)
            elif inplace:
                ops.all_gather_matmul(grp.input_slot(R, K, N, k), w, kind=k, group=grp, out=out)
            else:
                ops.all_gather_matmul(shards[0], w, kind=k, group=grp, out=out)
        info = plan.info()
        trace = torch.zeros(info["grid"] + 2 * info["tiles"], dtype=torch.int64, device="cuda")
        plan.set_trace(trace)
        # stream (non-graph) path for comparison
        ts_stream = []
        for _ in range(10):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            plan.run_parts(w, shards[0], out) if cp else plan.run_parts(shards[0], w, out)
            b.record()
            b.synchronize()
            ts_stream.append(a.elapsed_time(b) * 1e3)
        for _ in range(5):
            call(kind)
        torch.cuda.synchronize()
        ts = []
        for _ in range(10):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            call(kind)
            b.record()
            b.synchronize()
            ts.append(a.elapsed_time(b) * 1e3)
        grp.comm.check()
        tr = trace.cpu().tolist()
        g = info["grid"]
        t0 = min(tr[:g])
        ready = [(tr[g + 2 * i] - t0) / 1e3 for i in range(info["tiles"])]
        done = [(tr[g + 2 * i + 1] - t0) / 1e3 for i in range(info["tiles"])]
        groups = {}
        for i, t in enumerate(low.tiles):
            key = f"flag{t.flag}m{t.fmask:x}" + (f"/k{t.kseg}" if t.kseg else "")
            groups.setdefault(key, []).append(i)
        per = {k: {"n": len(v), "ready_min": round(min(ready[i] for i in v), 1),
                   "ready_med": round(statistics.median(ready[i] for i in v), 1),
                   "done_max": round(max(done[i] for i in v), 1)} for k, v in groups.items()}
        res[kind] = {"op_us": round(statistics.median(ts), 1), "op_us_streams": round(statistics.median(ts_stream), 1),
                     "cta_start_spread_us": round((max(tr[:g]) - t0) / 1e3, 1),
                     "kernel_span_us": round(max(done), 1), "groups": per}
        plan.set_trace(None)
    print(json.dumps(res, indent=1))
    grp.close()


if __name__ == "__main__":
    main()

"""Per-kind kernel statistics for an AG->GEMM shape on a virtual 8-rank group: op time, kernel span from the
trace, mean per-CTA gate wait, copy program alone. usage: python tools/shape_stats.py M N K [kinds]"""
import math
import os
import statistics
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2512_10236_b200 import ops, runtime  # noqa: E402

M, N, K = (int(x) for x in sys.argv[1:4])
kinds = sys.argv[4].split(",") if len(sys.argv) > 4 else ["serial", "shard_overlap_p2p", "hetero_unfused_1d",
                                                           "uniform_fused_1d"]
G, R = 8, M // 8
runtime.load_library()
gen = torch.Generator(device="cuda").manual_seed(0)
shards = [(torch.rand(R, K, generator=gen, device="cuda") * 2 - 1).to(torch.bfloat16) for _ in range(G)]
w = (torch.randn(N, K, generator=gen, device="cuda") / math.sqrt(K)).to(torch.bfloat16)
out = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
grp = ops.FiccoGroup.virtual_group(G, 0)
plain = torch.cat(shards)
for kind in kinds + ["plain"]:
    if kind == "plain":
        fn = lambda: runtime.gemm_bf16(plain, w, out)  # noqa: E731
        plan = None
    else:
        plan, low, _ = ops.prepare_ag(grp, R, K, N, kind)
        grp.load_peer_shards(low, shards)
        fn = lambda kd=kind: ops.all_gather_matmul(shards[0], w, kind=kd, group=grp, out=out)  # noqa: E731
    fn()
    ts = []
    for _ in range(3):
        flush.fill_(1)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    line = {"kind": kind, "op_ms": round(statistics.median(ts), 3)}
    if plan is not None:
        info = plan.info()
        tr = torch.zeros(info["grid"] + 2 * info["tiles"], dtype=torch.int64, device="cuda")
        plan.set_trace(tr)
        flush.fill_(1)
        fn()
        torch.cuda.synchronize()
        t = tr.cpu().tolist()
        plan.set_trace(None)
        g_ = info["grid"]
        t0 = min(t[:g_])
        ready = [(t[g_ + 2 * i] - t0) / 1e6 for i in range(info["tiles"])]
        done = [(t[g_ + 2 * i + 1] - t0) / 1e6 for i in range(info["tiles"])]
        wait = 0.0
        for c in range(g_):
            prev = (t[c] - t0) / 1e6
            for i in range(c, info["tiles"], g_):
                wait += max(0.0, ready[i] - prev)
                prev = done[i]
        cp = runtime.Plan(grp.comm, low.desc, list(low.ops), [])
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        cp.run(shards[0], w, out)
        torch.cuda.synchronize()
        e0.record()
        cp.run(shards[0], w, out)
        e1.record()
        torch.cuda.synchronize()
        cp.close()
        line.update(span_ms=round(max(done), 3), mean_gate_wait_ms=round(wait / g_, 3),
                    copy_ms=round(e0.elapsed_time(e1), 3), tiles=info["tiles"], tile_n=low.desc.tile_n,
                    hints=low.desc.hints)
    print(line, flush=True)
grp.close()
